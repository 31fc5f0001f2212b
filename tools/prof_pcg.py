"""Factor + one solve (for ncu captures of the PCG kernel)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
loop = sys.argv[2] if len(sys.argv) > 2 else "explicit"
b = make_bundle(name)
s = ietidp.from_bundle(b, loop=loop, fixed_iters=20)
s.factor()
lam, rep = s.solve(want_lambda=False)
torch.cuda.synchronize()
print(name, loop, rep["iters"][:2], rep["ms_pcg"])
