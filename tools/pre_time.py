"""Device assembly and gauge timings on a full-size config: python tools/pre_time.py C5"""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from ietigen import predesc
from ietigen.problem import build
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
P = build(name)
g = predesc.gauge_desc(P)
for _ in range(2):
    tree, prim, ms = ietidp.pre_gauge(g["nv"], g["ne"], g["eu"], g["ev"], g["w"])
print(json.dumps(dict(config=name, gauge_ms=ms, nv=g["nv"], ne=g["ne"], tree_ok=bool(np.array_equal(tree, P.tree)))))
d0 = predesc.subdomain_desc(P, P.subs[0])
for rep in range(2):
    out = ietidp.pre_assemble(d0)
nnz = len(out["K_data"])
print(json.dumps(dict(single_sub=0, n=d0["n_dof"], nnz=nnz, ms=out["ms"], ms_fill=out["ms_fill"],
                      fill_gb_s=nnz * 12 / out["ms_fill"] / 1e6)))
t0 = time.time()
descs = [predesc.subdomain_desc(P, sd) for sd in P.subs]
t_desc = time.time() - t0
for rep in range(3):
    t0 = time.time()
    _, info = ietidp.pre_assemble_batch(descs, fetch=False)
    wall = time.time() - t0
    print(json.dumps(dict(batch=len(descs), nnz=info["nnz"], ms=info["ms"], ms_fill=info["ms_fill"],
                          fill_gb_s=info["nnz"] * 12 / info["ms_fill"] / 1e6, wall_ms=wall * 1e3, desc_s=t_desc)))
