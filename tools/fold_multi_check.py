"""Several-RHS fold experiment (IETIDP_FOLD_MULTI=1): the symmetric-pass partials summed
inside the gathers instead of a separate reduction phase; compares the multipliers
bitwise with the default path on a workload and times the PCG."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C5r"
b = make_bundle(name)
out = {}
for mode in ("0", "1"):
    os.environ["IETIDP_FOLD_MULTI"] = mode
    s = ietidp.from_bundle(b)
    for _ in range(3):
        s.factor()
        lam, rep = s.solve()
    u = np.concatenate([s.get_u(k) for k in range(b["n_sub"])])
    out[mode] = (lam, u, rep["iters"], rep["ms_pcg"])
    print(name, "fold_multi", mode, "iters", rep["iters"][:4], "pcg ms", round(rep["ms_pcg"], 3), flush=True)
print("lambda bitwise equal:", np.array_equal(out["0"][0], out["1"][0]),
      "u bitwise equal:", np.array_equal(out["0"][1], out["1"][1]),
      "max |dlam|:", float(np.abs(out["0"][0] - out["1"][0]).max()))
