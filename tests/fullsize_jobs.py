"""Oracle jobs for the full-size parity tests (test infrastructure): each job
generates one BASELINE.json config at full size (ietigen), optionally restricted to
a subset of its right-hand-side columns, and solves it with the CPU oracle
(oracle/dp.py) to natural stopping, plus the explicit-inverse rounding variant's
iteration counts (oracle_variants, R10). Run in worker processes so that
the oracle solves of C2..C5 proceed concurrently with each other and with the GPU
tests."""
import time

import numpy as np

# the full-size oracle jobs: config key -> right-hand-side columns (None: all)
FULLSIZE_JOBS = {"C2": None, "C3": None, "C4": None, "C5c0": [0], "C5c7": [7]}
U_SAMPLES = 8192


def u_sample_index(n, seed=20250104):
    """The u positions stored in the golden files (seeded, sorted, without repeats)."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(U_SAMPLES, n), replace=False))


def oracle_job(name, cols=None, threads=None):
    """(BLAS threads limited to `threads`: the jobs run side by side.)"""
    if threads:
        import threadpoolctl
        threadpoolctl.threadpool_limits(limits=threads)
    from ietigen.bundle import make_bundle
    from oracle import dp
    from oracle_variants import explicit_inverse, slice_columns

    t0 = time.time()
    b = make_bundle(name)
    if cols is not None:
        b = slice_columns(b, cols)
    D = dp.DualPrimal(b)
    t1 = time.time()
    lam, info = D.pcg(tol=b["tol"])
    us, _ = D.recover(lam)
    t2 = time.time()
    explicit_inverse(D)
    _, info_x = D.pcg(tol=b["tol"])
    return dict(name=name, cols=cols, lam=lam, U=np.concatenate(us), iters=np.asarray(info["iters"]),
                rel_residual=np.asarray(info["rel_residual"]), iters_expl=np.asarray(info_x["iters"]),
                seconds=dict(setup=t1 - t0, pcg_recover=t2 - t1, explicit_pcg=time.time() - t2))
