"""Test-side helpers around the CPU oracle (oracle/dp.py): rounding variants of the
SAME operator, used to measure how far finite-precision PCG iteration counts move
under exact-arithmetic-equivalent reformulations (reading R10).

`explicit_inverse(D)` replaces the local part W_k = B_I S_II^-1 B_I^T of F_DP
(PAPER.md:128 with S_II of Eq. (10)) — applied by the
oracle through the sparse LU of K_rr — by products with the triangular inverse of
chol(S_II): W_k x = B_I L^-T (L^-1 (B_I^T x)). In exact arithmetic both are
B_r K_rr^-1 B_r^T (the r_I block of K_rr^-1 is S_II^-1)."""
import numpy as np
import scipy.linalg as la

from oracle import dp


def explicit_inverse(D):
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
    D.apply_W = apply_W
    return D


def explicit_inverse_iters(b, tol=None):
    D = explicit_inverse(dp.DualPrimal(b))
    _, info = D.pcg(tol=b["tol"] if tol is None else tol)
    return np.asarray(info["iters"])


def slice_columns(b, cols):
    """The bundle restricted to right-hand-side columns `cols` (independent PCGs,
    SURVEY Q16): a shallow copy with f sliced."""
    out = dict(b)
    out["subs"] = [dict(sd, f=np.ascontiguousarray(sd["f"][list(cols)])) for sd in b["subs"]]
    out["nrhs"] = len(cols)
    return out
