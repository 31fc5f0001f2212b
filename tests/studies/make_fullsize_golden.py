"""Writes tests/golden/fullsize_<key>.npz: the CPU oracle's (oracle/dp.py, through
tests/fullsize_jobs.py — oracle/ and ietigen/ only) full-size solutions of the
BASELINE.json configs C2, C3, C4 (every column) and C5 (columns 0 and 7), for the
full-size GPU parity test: lambda (all entries), u at 8192 seeded sample positions
per column plus ||u|| per column, the natural-stopping iteration counts of the
committed oracle and of its explicit-inverse variant (R10), the true
residuals and the oracle's timings on this host.

    python tests/studies/make_fullsize_golden.py [C2 C3 C4 C5c0 C5c7]
"""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = __file__.rsplit("/tests/", 1)[0]
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from fullsize_jobs import FULLSIZE_JOBS, U_SAMPLES, oracle_job, u_sample_index  # noqa: E402


def save(res):
    key = res["key"]
    U = res["U"]
    idx = u_sample_index(U.shape[0])
    out = os.path.join(ROOT, "tests", "golden", f"fullsize_{key}.npz")
    np.savez_compressed(out, lam=res["lam"], u_idx=idx, u_sample=U[idx], u_norm=np.linalg.norm(U, axis=0),
                        iters=res["iters"], iters_expl=res["iters_expl"], rel_residual=res["rel_residual"],
                        cols=np.asarray(res["cols"] if res["cols"] is not None else [-1]),
                        seconds=np.asarray([res["seconds"][k] for k in ("setup", "pcg_recover", "explicit_pcg")]))
    print(key, "iters", list(res["iters"]), "expl", list(res["iters_expl"]), res["seconds"], "->", out, flush=True)


def main():
    keys = sys.argv[1:] or list(FULLSIZE_JOBS)
    threads = max(1, (os.cpu_count() or 1) // len(keys))
    with ProcessPoolExecutor(max_workers=len(keys)) as ex:
        futs = [ex.submit(oracle_job, k[:2], FULLSIZE_JOBS[k], threads) for k in keys]
        for k, f in zip(keys, futs):
            r = f.result()
            r["key"] = k
            save(r)


if __name__ == "__main__":
    main()
