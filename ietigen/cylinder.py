"""C4 geometry: the hollow cylinder r in [0.5, 1], full theta, z in [0, 1], as
16 (theta) x 2 (r) x 4 (z) NURBS patches with exact circular arcs (BASELINE.json
configs[3]).

Parametric coordinates of the whole domain: s1 in [0, 1] around the circle
(patch a covers [a/16, (a+1)/16], periodic), s2 in [0, 1] radially
(r = 0.5 + 0.5 s2), s3 = z. Patch a maps its local xi = 16 s1 - a through the
rational quadratic arc of angle 2 pi/16 (control points (1,0), (1, tan(dth/2)),
(cos dth, sin dth), weights 1, cos(dth/2), 1), rotated by a dth.

The Jacobian columns are orthogonal: d x/d s1 = r theta_s e_theta,
d x/d s2 = 0.5 e_r, d x/d s3 = e_z, |det J| = 0.5 r theta_s (theta_s = d theta/d s1),
and det J < 0 ((e_theta, e_r, e_z) is left-handed). Hence the 2-form mass matrix
int nu (J v_f).(J v_g) / |det J| ds (PAPER.md:49-56 pulled back) is,
per patch and component, a Kronecker product of 1-D Gram matrices with weights
   normal to s1:  theta_s(s1) * 2 r(s2)
   normal to s2:  1/theta_s(s1) * 0.5/r(s2)
   normal to s3:  1/theta_s(s1) * 2/r(s2),
and the weak-curl load t_f = sign(det J) int T . J v_f ds is separable for
T = T_theta(r) e_theta + T_z(r) e_z.
"""
import numpy as np
import scipy.sparse as sp

from .splines import Space1D

NTH = 16
DTH = 2 * np.pi / NTH


def arc(xi):
    """Point C(xi) on the unit-circle arc [0, DTH] and its derivative C'(xi)."""
    xi = np.asarray(xi, dtype=np.float64)
    w1 = np.cos(DTH / 2)
    P = np.array([[1.0, 0.0], [1.0, np.tan(DTH / 2)], [np.cos(DTH), np.sin(DTH)]])
    w = np.array([1.0, w1, 1.0])
    B = np.stack([(1 - xi) ** 2, 2 * xi * (1 - xi), xi ** 2], axis=-1)
    dB = np.stack([-2 * (1 - xi), 2 - 4 * xi, 2 * xi], axis=-1)
    Wt = B @ w
    dWt = dB @ w
    N = (B * w) @ P
    dN = (dB * w) @ P
    C = N / Wt[..., None]
    dC = (dN * Wt[..., None] - N * dWt[..., None]) / (Wt ** 2)[..., None]
    return C, dC


def theta_s(s1):
    """d theta / d s1 at global parametric s1 (= 16 |C'(xi)| on the unit circle)."""
    s1 = np.asarray(s1, dtype=np.float64)
    a = np.minimum(np.floor(s1 * NTH), NTH - 1)
    xi = s1 * NTH - a
    _, dC = arc(xi)
    return NTH * np.linalg.norm(dC, axis=-1)


def radius(s2):
    return 0.5 + 0.5 * np.asarray(s2, dtype=np.float64)


def _gram_w(space, kind, patch, weight, nq):
    x, w = space.quad(nq, patch)
    V = space.B(x) if kind == "B" else space.D(x)
    return (V * (w * weight(x))[:, None]).T @ V


def _int_w(space, kind, weight, nq):
    x, w = space.quad(nq)
    V = space.B(x) if kind == "B" else space.D(x)
    return V.T @ (w * weight(x))


def cylinder_spaces(cfg, sub):
    N = cfg.npatch
    return [Space1D(sub.lo[a] / N[a], sub.hi[a] / N[a], sub.hi[a] - sub.lo[a], cfg.e, cfg.p) for a in range(3)]


# separable metric weights per 2-form component: (f(s1), g(s2)); the s3 factor is 1
_W = [
    (lambda s: theta_s(s), lambda s: 2.0 * radius(s)),
    (lambda s: 1.0 / theta_s(s), lambda s: 0.5 / radius(s)),
    (lambda s: 1.0 / theta_s(s), lambda s: 2.0 / radius(s)),
]


def cylinder_mass2(cfg, sub, spaces, nu):
    nq = cfg.p + 4
    blocks = []
    for c in range(3):
        kinds = ["D", "D", "D"]
        kinds[c] = "B"
        f, g = _W[c]
        acc = None
        for qz in range(spaces[2].npatch):
            for qy in range(spaces[1].npatch):
                for qx in range(spaces[0].npatch):
                    w = nu[sub.lo[0] + qx, sub.lo[1] + qy, sub.lo[2] + qz]
                    mx = _gram_w(spaces[0], kinds[0], qx, f, nq)
                    my = _gram_w(spaces[1], kinds[1], qy, g, nq)
                    mz = spaces[2].mass(kinds[2], qz, nq)
                    term = w * sp.kron(sp.csr_matrix(mz), sp.kron(sp.csr_matrix(my), sp.csr_matrix(mx), format="csr"),
                                       format="csr")
                    acc = term if acc is None else acc + term
        blocks.append(acc)
    return sp.block_diag(blocks, format="csr")


def source_field(cfg):
    """(T_theta(r), T_z(r)) per RHS column with J = curl T."""
    if cfg.rhs == "c4":
        # J = e_theta in r in [0.5, 0.75]: T = (0, 0, 0.5 - min(r, 0.75))
        return [(None, lambda r: 0.5 - np.minimum(r, 0.75))]
    if cfg.rhs == "c4_manufactured":
        # A* = a(r) e_z, a = sin(2 pi (r - 0.5)) (n x A* = 0 on the whole boundary);
        # T = curl A* = -a'(r) e_theta, J = curl T (nu = 1)
        return [(lambda r: -2 * np.pi * np.cos(2 * np.pi * (r - 0.5)), None)]
    raise ValueError(cfg.rhs)


def cylinder_face_loads(cfg, sub, spaces):
    """t_f = sign(det J) int T . J v_f ds, sign(det J) = -1; (n_faces, nrhs)."""
    nq = cfg.p + 4
    cols = []
    for Tth, Tz in source_field(cfg):
        parts = []
        # component normal to s1: T . J_1 = T_theta r theta_s
        dims0 = [spaces[0].m, spaces[1].m - 1, spaces[2].m - 1]
        if Tth is None:
            parts.append(np.zeros(int(np.prod(dims0))))
        else:
            v1 = _int_w(spaces[0], "B", lambda s: theta_s(s), nq)
            v2 = _int_w(spaces[1], "D", lambda s: Tth(radius(s)) * radius(s), nq)
            v3 = _int_w(spaces[2], "D", lambda s: np.ones_like(s), nq)
            parts.append(-np.einsum("i,j,k->kji", v1, v2, v3).ravel())
        # component normal to s2: T . J_2 = T_r * 0.5 = 0
        dims1 = [spaces[0].m - 1, spaces[1].m, spaces[2].m - 1]
        parts.append(np.zeros(int(np.prod(dims1))))
        # component normal to s3: T . J_3 = T_z
        dims2 = [spaces[0].m - 1, spaces[1].m - 1, spaces[2].m]
        if Tz is None:
            parts.append(np.zeros(int(np.prod(dims2))))
        else:
            v1 = _int_w(spaces[0], "D", lambda s: np.ones_like(s), nq)
            v2 = _int_w(spaces[1], "D", lambda s: Tz(radius(s)), nq)
            v3 = _int_w(spaces[2], "B", lambda s: np.ones_like(s), nq)
            parts.append(-np.einsum("i,j,k->kji", v1, v2, v3).ravel())
        cols.append(np.concatenate(parts))
    return np.stack(cols, axis=1)


def assemble_cylinder(P, sd, with_face=False):
    """K^(k) = C^T M2 C (Dirichlet rows/cols removed) and j^(k) = C^T t (n_k x nrhs)."""
    from .problem import local_curl
    cfg = P.cfg
    spaces = cylinder_spaces(cfg, sd)
    C = local_curl(sd.ml)
    M2 = cylinder_mass2(cfg, sd, spaces, P.nu)
    K = (C.T @ M2 @ C).tocsr()
    t = cylinder_face_loads(cfg, sd, spaces)
    j = C.T @ t
    m = sd.local_mask
    K = K[m][:, m].tocsr()
    K = ((K + K.T) * 0.5).tocsr()
    K.sort_indices()
    j = np.ascontiguousarray(j[m])
    if with_face:
        return K, j, C[:, m], M2, t
    return K, j
