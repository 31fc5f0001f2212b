"""Full-size checks (BASELINE.json configs at their real sizes, in the launch
configuration bench.py times).

1. Against the CPU oracle (oracle/dp.py) at full size: C2, C3 and C4 on every
   column, C5 on columns 0 and 7 of its 16 (independent PCGs). The
   oracle's results are the golden files tests/golden/fullsize_*.npz written by
   tests/studies/make_fullsize_golden.py (oracle/ and ietigen/ only; lambda in full,
   u at 8192 seeded positions per column and ||u||), because the full-size oracle
   needs ~10 min of host time; IETIDP_FULLSIZE_LIVE=1 runs the oracle here instead
   (worker processes, tests/fullsize_jobs.py). Per column: N_iter (parity_checks.
   check_iters, R10), true dual residual <= 1e-10, lambda (full) and u
   (sampled, and its norm) within 1e-8 at natural stopping (C5: the 16-column GPU
   solve, columns sliced out) and iteration-matched (fixed_iters = the oracle's count).
2. The partially assembled saddle system Eq. (5), which has a
   unique solution, checked equation by equation with plain sparse
   products on the input CSR (no oracle code), on all five configs:
  (a) local equilibrium on the remaining DOFs:  K_rr u_r + K_rP u_P + B_r^T lambda = j_r
  (b) coarse equilibrium:  sum_k C_k^T (K_Pr u_r + K_PP u_P - j_P) = 0
  (c) continuity:  sum_k B_r^(k) u_r^(k) = 0   (to the PCG tolerance)
  (d) one value per global primal DOF and u = 0 on tree DOFs.
"""
import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest
import scipy.sparse as sp

from ietigen.bundle import make_bundle
from oracle_variants import slice_columns
from fullsize_jobs import FULLSIZE_JOBS, u_sample_index
from parity_checks import check_iters, col_rel, load_norms

pytestmark = pytest.mark.gpu

JOBS = FULLSIZE_JOBS
LIVE = os.environ.get("IETIDP_FULLSIZE_LIVE") == "1"
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    from paper_2501_04340_b200 import ietidp
    return ietidp


class _Done:
    def __init__(self, v):
        self.v = v

    def result(self):
        return self.v


def _golden(key):
    z = np.load(os.path.join(GOLDEN, f"fullsize_{key}.npz"))
    return dict(lam=z["lam"], u_idx=z["u_idx"], u_sample=z["u_sample"], u_norm=z["u_norm"], iters=z["iters"],
                iters_expl=z["iters_expl"], rel_residual=z["rel_residual"], seconds=z["seconds"])


@pytest.fixture(scope="module")
def oracle_results():
    """The oracle's full-size results: golden files, or (IETIDP_FULLSIZE_LIVE=1) every
    full-size oracle solve submitted at once to worker processes."""
    if not LIVE:
        yield {k: _Done(_golden(k)) for k in JOBS}
        return
    from fullsize_jobs import oracle_job
    ex = ProcessPoolExecutor(max_workers=len(JOBS), mp_context=mp.get_context("spawn"))
    threads = max(1, (os.cpu_count() or 1) // len(JOBS))
    fut = {k: ex.submit(oracle_job, k[:2], cols, threads) for k, cols in JOBS.items()}
    yield fut
    ex.shutdown(wait=False, cancel_futures=True)


def _as_sampled(ref):
    """Live results -> the golden file's sampled form."""
    if "u_idx" in ref:
        return ref
    U = ref["U"]
    idx = u_sample_index(U.shape[0])
    return dict(ref, u_idx=idx, u_sample=U[idx], u_norm=np.linalg.norm(U, axis=0))


def check_u_sampled(U, ref, tol=1e-8):
    """u (concatenated, n x ncols) against the oracle's sampled u: the relative error on
    the sample and of ||u|| per column."""
    S = U[ref["u_idx"]]
    e = np.linalg.norm(S - ref["u_sample"], axis=0) / np.linalg.norm(ref["u_sample"], axis=0)
    en = np.abs(np.linalg.norm(U, axis=0) - ref["u_norm"]) / ref["u_norm"]
    assert np.all(e <= tol) and np.all(en <= tol), (e, en)
    return e


def gpu_solve(lib, b, **kw):
    s = lib.from_bundle(b, **kw)
    s.factor()
    lam, rep = s.solve()
    u = [s.get_u(k) for k in range(b["n_sub"])]
    s.close()
    return lam, u, rep


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_fullsize_saddle_equations(lib, oracle_results, name):
    # (runs first: the full-size oracle solves proceed in the background meanwhile)
    b = make_bundle(name)
    s = lib.from_bundle(b)
    s.factor()
    lam, rep = s.solve()
    assert all(rep["converged"]) and max(rep["rel_residual"]) <= 1e-10
    nl, ng, nc = b["n_lambda"], b["n_primal"], b["nrhs"]
    jump = np.zeros((nl, nc))
    coarse = np.zeros((ng, nc))
    pvals = {}
    jn2 = 0.0
    loc_err2 = 0.0
    unorm2 = 0.0
    for k, sd in enumerate(b["subs"]):
        n = sd["n"]
        K = sp.csr_matrix((sd["K_data"], sd["K_indices"], sd["K_indptr"]), shape=(n, n))
        f = sd["f"].reshape(nc, n).T
        u = s.get_u(k)
        unorm2 += float((u * u).sum())
        jn2 += float((f * f).sum())
        assert np.all(u[sd["tree"]] == 0.0)
        BtL = np.zeros((n, nc))
        np.add.at(BtL, sd["B_dof"], sd["B_sign"][:, None] * lam[sd["B_lambda"]])
        res = K @ u + BtL - f
        mask = np.ones(n, bool)
        mask[sd["tree"]] = False
        mask[sd["prim"]] = False
        loc_err2 += float((res[mask] ** 2).sum())
        np.add.at(coarse, sd["prim_gid"], res[sd["prim"]])
        np.add.at(jump, sd["B_lambda"], sd["B_sign"][:, None] * u[sd["B_dof"]])
        for q, g in zip(sd["prim"], sd["prim_gid"]):
            v = u[q]
            if g in pvals:
                assert np.array_equal(pvals[g], v)
            pvals[g] = v
    jn, un = np.sqrt(jn2), np.sqrt(unorm2)
    assert np.sqrt(loc_err2) <= 1e-9 * jn, np.sqrt(loc_err2) / jn
    assert np.linalg.norm(coarse) <= 1e-9 * jn, np.linalg.norm(coarse) / jn
    # continuity holds to the dual residual: ||B u|| = ||d - F lambda|| <= 1e-10 ||d||
    assert np.linalg.norm(jump) <= 1e-8 * un, np.linalg.norm(jump) / un


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_fullsize_oracle_parity(lib, oracle_results, name):
    b = make_bundle(name)
    lam, u, rep = gpu_solve(lib, b)
    U = np.concatenate(u)
    for key in [k for k in JOBS if k.startswith(name)]:
        ref = _as_sampled(oracle_results[key].result())
        cols = JOBS[key] or list(range(b["nrhs"]))
        bc = slice_columns(b, cols)
        it_gpu = np.asarray(rep["iters"])[cols]
        print(f"{key}: iters gpu {list(it_gpu)} oracle {list(ref['iters'])} explicit-inverse oracle "
              f"{list(ref['iters_expl'])}")
        check_iters(it_gpu, ref["iters"], ref["iters_expl"])
        assert np.all(np.asarray(rep["rel_residual"])[cols] <= 1e-10)
        assert np.all(ref["rel_residual"] <= 1e-10)
        el = col_rel(lam[:, cols], ref["lam"], floor=load_norms(bc))
        assert np.all(el <= 1e-8), el
        eu = check_u_sampled(U[:, cols], ref)
        print(f"{key}: natural stopping rel. err. lambda {el}, u (sampled) {eu}")
        # iteration-matched: the GPU on the same columns with fixed_iters = the oracle's count
        for i, c in enumerate(cols):
            b1 = slice_columns(b, [c])
            lam1, u1, rep1 = gpu_solve(lib, b1, fixed_iters=int(ref["iters"][i]))
            assert rep1["iters"] == [int(ref["iters"][i])]
            el1 = col_rel(lam1, ref["lam"][:, [i]], floor=load_norms(b1))
            assert np.all(el1 <= 1e-8), el1
            ref1 = dict(ref, u_sample=ref["u_sample"][:, [i]], u_norm=ref["u_norm"][[i]])
            eu1 = check_u_sampled(np.concatenate(u1), ref1)
            print(f"{key} column {c}: iteration-matched rel. err. lambda {el1}, u (sampled) {eu1}")
