"""One-RHS L2 residency threshold experiment: S_II's tiles are kept (evict_last, W's
evict_first) when below IETIDP_L2KEEP x L2 size (default 0.66); PCG time per setting."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
b = make_bundle(name)
out = {}
for mode in ("0.66", "1.0", "0.66", "1.0", "1.5"):
    os.environ["IETIDP_L2KEEP"] = mode
    s = ietidp.from_bundle(b)
    ts = []
    for _ in range(4):
        s.factor()
        lam, rep = s.solve()
        ts.append(rep["ms_pcg"])
    out[mode] = lam
    print(name, "l2keep", mode, "iters", rep["iters"][:1], "pcg ms", [round(t, 3) for t in ts[1:]], flush=True)
    s.close()
print("lambda bitwise equal:", np.array_equal(out["0.66"], out["1.0"]))
