"""Study (test infrastructure, run by hand): why the oracle's and the GPU's PCG
iteration counts differ on full-size C5, measured at full size.

PAPER.md:128 defines W = B_r K_rr^-1 B_r^T; PAPER.md:143-146 the Dirichlet block
S_{r_I r_I}. Three oracle variants apply the SAME operator F_DP = W + G S_PP^-1 G^T
(identical in exact arithmetic) and differ only in rounding:

  lu       oracle/dp.py as committed: K_rr^-1 through SuperLU (the plain definition);
  expl     W_k = B_I L^-T L^-1 B_I^T with L = chol(S_II) and its triangular inverse
           (the form of S_II^-1 the GPU's default loop stores);
  refined  lu plus two steps of iterative refinement with the residual b - K_rr x
           accumulated in x87 extended precision (np.longdouble): K_rr^-1 b to ~eps
           relative, i.e. the closest to exact arithmetic of the three.

For each it records the per-column iteration count of the SURVEY §8(c) PCG (tol
1e-10, natural stopping), the true residual, and the dynamic error of one
W-application against `refined` on random vectors. Usage:

  python tests/studies/c5_iteration_gap.py C5 0,7 > profiles/r02_c5_iteration_gap.txt
"""
import sys
import time

import numpy as np
import scipy.linalg as la

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from ietigen.bundle import make_bundle  # noqa: E402
from oracle import dp  # noqa: E402


def slice_columns(b, cols):
    for sd in b["subs"]:
        sd["f"] = np.ascontiguousarray(sd["f"][cols])
    b["nrhs"] = len(cols)
    return b


def ld_matvec(A, x):
    """A x with every product and sum in np.longdouble (A CSR/CSC -> CSR)."""
    A = A.tocsr()
    data = A.data.astype(np.longdouble)
    xl = x.astype(np.longdouble)
    out = np.zeros((A.shape[0],) + x.shape[1:], np.longdouble)
    rows = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
    np.add.at(out, rows, data[:, None] * xl[A.indices] if x.ndim == 2 else data * xl[A.indices])
    return out


def make_refined(L):
    Krr = L.Krr.tocsr()

    def kinv(X):
        X = np.asarray(X, np.float64)
        x = L.lu.solve(X)
        for _ in range(2):
            r = (X.astype(np.longdouble) - ld_matvec(Krr, x)).astype(np.float64)
            x = x + L.lu.solve(r)
        return x
    return kinv


def variant(D, name):
    if name == "lu":
        return D.apply_W
    if name == "expl":
        for L in D.loc:
            if len(L.rI):
                c = la.cholesky(L.SII, lower=True)
                L.Linv = la.solve_triangular(c, np.eye(len(c)), lower=True)
                L.BI = L.BD.copy()
                L.BI.data = np.sign(L.BI.data)

        def apply_W(lam):
            out = np.zeros_like(lam)
            for L in D.loc:
                if len(L.rI):
                    out += L.BI @ (L.Linv.T @ (L.Linv @ (L.BI.T @ lam)))
            return out
        return apply_W
    if name == "refined":
        for L in D.loc:
            L.kinv_ref = make_refined(L)

        def apply_W(lam):
            out = np.zeros_like(lam)
            for L in D.loc:
                out += L.Br @ L.kinv_ref(L.Br.T @ lam)
            return out
        return apply_W
    raise ValueError(name)


def main():
    name = sys.argv[1]
    cols = [int(c) for c in sys.argv[2].split(",")]
    names = sys.argv[3].split(",") if len(sys.argv) > 3 else ["lu", "expl", "refined"]
    b = slice_columns(make_bundle(name), cols)
    t0 = time.time()
    D = dp.DualPrimal(b)
    print(f"{name} columns {cols}: oracle set-up {time.time() - t0:.1f} s, n_lambda {D.nl}, n_gp {D.ng}", flush=True)
    W = {v: variant(D, v) for v in names}
    rng = np.random.default_rng(11)
    X = rng.standard_normal((D.nl, 4))
    if "refined" in W:
        ref = W["refined"](X)
        for v in names:
            e = np.linalg.norm(W[v](X) - ref, axis=0) / np.linalg.norm(ref, axis=0)
            print(f"  W-apply dynamic error vs refined, {v:8s}: max {e.max():.2e}", flush=True)
    lams = {}
    for v in names:
        D.apply_W = W[v]
        t = time.time()
        lam, info = D.pcg(tol=b["tol"])
        lams[v] = lam
        print(f"  {v:8s} iters {list(map(int, info['iters']))} true rel. residual "
              f"{['%.2e' % x for x in info['rel_residual']]} ({time.time() - t:.0f} s)", flush=True)
    base = lams[names[0]]
    for v in names[1:]:
        e = np.linalg.norm(lams[v] - base, axis=0) / np.linalg.norm(base, axis=0)
        print(f"  lambda at natural stopping, {v} vs {names[0]}: rel. diff per column {['%.1e' % x for x in e]}")


if __name__ == "__main__":
    main()
