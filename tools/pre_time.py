"""Device assembly and gauge timings on a full-size config: python tools/pre_time.py C5 [n_sub]"""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from ietigen import predesc
from ietigen.problem import build
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 4
P = build(name)
g = predesc.gauge_desc(P)
for _ in range(2):
    tree, prim, ms = ietidp.pre_gauge(g["nv"], g["ne"], g["eu"], g["ev"], g["w"])
print(json.dumps(dict(config=name, gauge_ms=ms, nv=g["nv"], ne=g["ne"], tree_ok=bool(np.array_equal(tree, P.tree)))))
for k in range(min(lim, len(P.subs))):
    d = predesc.subdomain_desc(P, P.subs[k])
    for rep in range(2):
        t0 = time.time()
        out = ietidp.pre_assemble(d)
        wall = time.time() - t0
    nnz = len(out["K_data"])
    print(json.dumps(dict(sub=k, n=d["n_dof"], nnz=nnz, ms=out["ms"], ms_fill=out["ms_fill"], fill_gb_s=nnz * 12 / out["ms_fill"] / 1e6, wall_ms=wall * 1e3,
                          gb_s=nnz * 12 / out["ms"] / 1e6, entries_per_us=nnz / out["ms"] / 1e3)))
