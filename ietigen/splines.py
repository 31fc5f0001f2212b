"""1-D spline spaces of the multipatch de Rham sequence.

A direction with `npatch` patches of `e` elements each, degree p, open knots at
the ends and knot multiplicity p at patch boundaries (C^0 gluing).
0-forms: B-splines B_i of degree p, i = 0..m-1, m = npatch*(e+p-1)+1.
1-forms: Curry–Schoenberg-scaled D_j = p/(t_{j+p+1}-t_{j+1}) B_{j+1,p-1}, j = 0..m-2,
so that B_i' = D_{i-1} - D_i and the discrete gradient is the signed
incidence G1[j, j+1] = +1, G1[j, j] = -1.
"""
import numpy as np
import scipy.sparse as sp


def knot_vector(x0, x1, npatch, e, p):
    """Open knot vector on [x0, x1]; interior patch boundaries repeated p times."""
    h = (x1 - x0) / npatch
    t = [x0] * (p + 1)
    for a in range(npatch):
        for q in range(1, e):
            t.append(x0 + a * h + q * h / e)
        if a < npatch - 1:
            t += [x0 + (a + 1) * h] * p
    t += [x1] * (p + 1)
    return np.array(t, dtype=np.float64)


def bspline_values(t, p, x):
    """All degree-p B-splines on knots t at points x: array (len(x), len(t)-p-1).

    Cox–de Boor recursion, right-continuous except at the last knot."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    nb0 = len(t) - 1
    B = np.zeros((len(x), nb0))
    for j in range(nb0):
        if t[j] < t[j + 1]:
            inside = (x >= t[j]) & (x < t[j + 1])
            if t[j + 1] == t[-1]:
                inside |= (x == t[-1])
            B[:, j] = inside
    for q in range(1, p + 1):
        nb = len(t) - q - 1
        Bn = np.zeros((len(x), nb))
        for j in range(nb):
            d1 = t[j + q] - t[j]
            d2 = t[j + q + 1] - t[j + 1]
            v = np.zeros(len(x))
            if d1 > 0:
                v += (x - t[j]) / d1 * B[:, j]
            if d2 > 0:
                v += (t[j + q + 1] - x) / d2 * B[:, j + 1]
            Bn[:, j] = v
        B = Bn
    return B


def dspline_values(t, p, x):
    """Curry–Schoenberg-scaled degree-(p-1) splines D_j, j = 0..m-2."""
    B = bspline_values(t, p - 1, x)  # len(t)-p functions, index j+1 -> D_j
    m = len(t) - p - 1
    D = np.zeros((B.shape[0], m - 1))
    for j in range(m - 1):
        D[:, j] = p / (t[j + p + 1] - t[j + 1]) * B[:, j + 1]
    return D


def gradient_incidence(m):
    """G1 ((m-1) x m): coefficient of D_j in the derivative is c_{j+1} - c_j."""
    r = np.arange(m - 1)
    rows = np.concatenate([r, r])
    cols = np.concatenate([r + 1, r])
    vals = np.concatenate([np.ones(m - 1), -np.ones(m - 1)])
    return sp.csr_matrix((vals, (rows, cols)), shape=(m - 1, m))


class Space1D:
    """The 1-D pair (B, D) on a sub-interval made of `npatch` patches."""

    def __init__(self, x0, x1, npatch, e, p):
        self.x0, self.x1, self.npatch, self.e, self.p = x0, x1, npatch, e, p
        self.t = knot_vector(x0, x1, npatch, e, p)
        self.m = npatch * (e + p - 1) + 1
        assert len(self.t) - p - 1 == self.m
        h = (x1 - x0) / npatch
        self.patch_bounds = [(x0 + a * h, x0 + (a + 1) * h) for a in range(npatch)]

    def quad(self, nq, a=None):
        """Gauss–Legendre points/weights, nq per element, over patch a (or all)."""
        g, w = np.polynomial.legendre.leggauss(nq)
        pats = range(self.npatch) if a is None else [a]
        X, W = [], []
        for pa in pats:
            lo, hi = self.patch_bounds[pa]
            he = (hi - lo) / self.e
            for q in range(self.e):
                c = lo + (q + 0.5) * he
                X.append(c + 0.5 * he * g)
                W.append(0.5 * he * w)
        return np.concatenate(X), np.concatenate(W)

    def B(self, x):
        return bspline_values(self.t, self.p, x)

    def D(self, x):
        return dspline_values(self.t, self.p, x)

    def mass(self, kind, a, nq=None):
        """Gram matrix of B or D over patch a (exact with p+1 points)."""
        nq = nq or self.p + 1
        x, w = self.quad(nq, a)
        V = self.B(x) if kind == "B" else self.D(x)
        return (V * w[:, None]).T @ V

    def integrals(self, kind, f, nq):
        """Vector of int f(x) phi_i(x) dx over the whole interval."""
        x, w = self.quad(nq)
        V = self.B(x) if kind == "B" else self.D(x)
        return V.T @ (w * f(x))
