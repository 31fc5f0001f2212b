"""Several-RHS L2 policy experiment (default; IETIDP_L2MULTI=0 turns it off: both symmetric
operators' tiles streamed with evict_first): bitwise comparison with the default and PCG time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
b = make_bundle(name)
out = {}
for mode in ("0", "1", "0", "1"):
    os.environ["IETIDP_L2MULTI"] = mode
    s = ietidp.from_bundle(b)
    ts = []
    for _ in range(4):
        s.factor()
        lam, rep = s.solve()
        ts.append(rep["ms_pcg"])
    out[mode] = lam
    print(name, "l2multi", mode, "iters", rep["iters"][:4], "pcg ms", [round(t, 2) for t in ts[1:]], flush=True)
    s.close()
print("lambda bitwise equal:", np.array_equal(out["0"], out["1"]))
