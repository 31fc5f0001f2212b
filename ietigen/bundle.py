"""Pack a generated Problem into the C-ABI argument set (include/ietidp.h,
`ietidp_set_subdomain`) plus generator-side extras used only by tests.

A bundle is a plain dict:
  cfg, n_sub, n_lambda, n_primal, nrhs, scaling, tol
  subs: list of dict(n, K_indptr int64, K_indices int32, K_data f64,
                     f f64 (nrhs, n) == column-major n x nrhs,
                     B_lambda int32, B_dof int32, B_sign int8,
                     tree int32, prim int32, prim_gid int32,
                     glob int64 (DOF -> global gauged unknown, -1 for tree; tests only))
"""
import numpy as np

from . import configs as cf
from .problem import build


def make_bundle(cfg, kruskal="scipy", with_problem=False):
    if isinstance(cfg, str):
        cfg = cf.get(cfg)
    P = build(cfg, kruskal=kruskal)
    subs = []
    for sd in P.subs:
        K, j = P.assemble(sd)
        subs.append(dict(
            n=sd.n,
            K_indptr=K.indptr.astype(np.int64),
            K_indices=K.indices.astype(np.int32),
            K_data=K.data.astype(np.float64),
            f=np.ascontiguousarray(j.T.astype(np.float64)),
            B_lambda=sd.B_lambda, B_dof=sd.B_dof, B_sign=sd.B_sign,
            tree=sd.tree, prim=sd.prim, prim_gid=sd.prim_gid,
            glob=sd.glob,
        ))
    b = dict(cfg=cfg, name=cfg.name, n_sub=len(subs), n_lambda=P.n_lambda,
             n_primal=P.n_primal, nrhs=cfg.nrhs, scaling=cfg.scaling, tol=cfg.tol,
             n_gauged=len(P.gauged_edges), subs=subs)
    if with_problem:
        return b, P
    return b
