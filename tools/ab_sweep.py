"""A/B of two library builds on the several-RHS sweeps: phases and u agreement.
IETIDP_LIB=<lib> python tools/ab_sweep.py C5 out.npy"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp
name, out = sys.argv[1], sys.argv[2]
b = make_bundle(name)
s = ietidp.from_bundle(b)
for _ in range(4):
    s.factor()
    lam, rep = s.solve()
u = np.concatenate([s.get_u(k) for k in range(0, b["n_sub"], 7)])
np.save(out, u)
np.save(out + ".lam.npy", lam)
print(os.environ.get("IETIDP_LIB"), {q: round(rep[q], 3) for q in ("ms_factor", "ms_coarse", "ms_pcg", "ms_recover")}, rep["iters"][:4])
