"""Factor / recovery time of a config with its first k right-hand sides only (how much of the
several-RHS sweeps is on the critical path): python tools/nrhs_exp.py C5 1 16"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1]
b = make_bundle(name)
for k in [int(x) for x in sys.argv[2:]]:
    bb = dict(b)
    bb["subs"] = [dict(sd, f=np.ascontiguousarray(sd["f"][:k])) for sd in b["subs"]]
    bb["nrhs"] = k
    s = ietidp.from_bundle(bb)
    for _ in range(4):
        s.factor()
        lam, rep = s.solve(want_lambda=False)
    print(name, "nrhs", k, {q: round(rep[q], 3) for q in ("ms_factor", "ms_coarse", "ms_pcg", "ms_recover")}, max(rep["iters"]))
    s.close()
