"""Input data of the device pre-processing (include/ietidp_pre.h) for one
box subdomain of a generated Problem: knot vectors, quadrature points, quadrature weights
multiplied by the geometry's separable metric factors and by the source's 1-D factors,
reluctivities per patch, the Dirichlet mask as a DOF map, and the control graph with its
weights. Data only: no spline evaluation, no Gram matrix, no Kronecker sum, no C^T M_2 C and
no spanning tree happens here (those are the device's work, and `ietigen.problem`'s on the
reference side).
"""
import numpy as np

from . import configs as cf
from .splines import Space1D


def _spaces(cfg, sd):
    N = cfg.npatch
    return [Space1D(sd.lo[a] / N[a], sd.hi[a] / N[a], sd.hi[a] - sd.lo[a], cfg.e, cfg.p) for a in range(3)]


def subdomain_desc(P, sd):
    """dict of plain arrays for ietidp_pre_assemble (one box subdomain)."""
    cfg = P.cfg
    assert len(sd.boxes) == 1, "box subdomains only (unions of patches are summed box by box)"
    spaces = _spaces(cfg, sd)
    cyl = cfg.geometry != "cube"
    nq = cfg.p + 4 if cyl else cfg.p + 1
    lq = cfg.p + 4 if cyl else cfg.p + cfg.load_nq_extra
    qx, qw0, lx, lw0 = [], [], [], []
    for a in range(3):
        x, w = spaces[a].quad(nq)
        qx.append(x)
        qw0.append(w)
        x, w = spaces[a].quad(lq)
        lx.append(x)
        lw0.append(w)
    one = lambda s: np.ones_like(s)
    if cyl:
        from .cylinder import theta_s, radius, source_field
        metric = [
            (lambda s: theta_s(s), lambda s: 2.0 * radius(s), one),
            (lambda s: 1.0 / theta_s(s), lambda s: 0.5 / radius(s), one),
            (lambda s: 1.0 / theta_s(s), lambda s: 2.0 / radius(s), one),
        ]
    else:
        metric = [(one, one, one)] * 3
    qw = [[qw0[a] * metric[c][a](qx[a]) for a in range(3)] for c in range(3)]
    npb = [sd.hi[a] - sd.lo[a] for a in range(3)]
    nu = np.empty(npb[0] * npb[1] * npb[2])
    for qz in range(npb[2]):
        for qy in range(npb[1]):
            for qx_ in range(npb[0]):
                nu[qx_ + npb[0] * (qy + npb[1] * qz)] = P.nu[(sd.lo[0] + qx_) % cfg.npatch[0], sd.lo[1] + qy, sd.lo[2] + qz]
    dof = np.full(len(sd.local_mask), -1, np.int32)
    dof[sd.local_mask] = np.arange(sd.n, dtype=np.int32)

    # loads: distinct 1-D factors per axis as (kind, values at the load points * weights)
    fac = [dict() for _ in range(3)]     # key -> index
    fval = [[] for _ in range(3)]
    fkind = [[] for _ in range(3)]

    def factor(a, kind, key, fn):
        k = (kind, key)
        if k not in fac[a]:
            fac[a][k] = len(fval[a])
            fval[a].append(lw0[a] * fn(lx[a]))
            fkind[a].append(0 if kind == "B" else 1)
        return fac[a][k]

    tcol, tcomp, tfac, tcoef = [], [], [], []
    if cyl:
        for s_, (Tth, Tz) in enumerate(source_field(cfg)):
            # t_f = sign(det J) int T . J v_f, sign(det J) = -1 (ietigen/cylinder.py)
            if Tth is not None:
                tcol.append(s_); tcomp.append(0); tcoef.append(-1.0)
                tfac.append([factor(0, "B", "ths", lambda s: theta_s(s)),
                             factor(1, "D", "Tth_r", lambda s: Tth(radius(s)) * radius(s)),
                             factor(2, "D", "one", one)])
            if Tz is not None:
                tcol.append(s_); tcomp.append(2); tcoef.append(-1.0)
                tfac.append([factor(0, "D", "one", one),
                             factor(1, "D", "Tz", lambda s: Tz(radius(s))),
                             factor(2, "B", "one", one)])
    else:
        for s_, col in enumerate(cf.source_terms(cfg)):
            for c in range(3):
                for coef, fx, fy, fz in col[c]:
                    specs = (fx, fy, fz)
                    tcol.append(s_); tcomp.append(c); tcoef.append(float(coef))
                    tfac.append([factor(a, "B" if a == c else "D", specs[a], cf.f1d(specs[a])) for a in range(3)])
    for a in range(3):
        if not fval[a]:
            factor(a, "D", "one", one)
    return dict(
        p=cfg.p, e=cfg.e, npatch=npb, knots=[sp_.t for sp_ in spaces], nq=nq, qx=qx, qw=qw, nu=nu,
        dof_of_edge=dof, n_dof=sd.n, nrhs=cfg.nrhs, lq=lq, lx=lx,
        fac_kind=[np.array(k, np.int32) for k in fkind], fac_val=[np.array(v, np.float64) for v in fval],
        term_col=np.array(tcol, np.int32), term_comp=np.array(tcomp, np.int32),
        term_fac=np.array(tfac, np.int32).reshape(-1, 3), term_coef=np.array(tcoef, np.float64))


def gauge_desc(P):
    """The weighted control graph: endpoints and the weights 1..5."""
    g = P.grid
    u, v = g.endpoints()
    return dict(nv=g.nv, ne=g.ne, eu=u.astype(np.int32), ev=v.astype(np.int32), w=P.weight.astype(np.int8))
