"""One factor + solve of a workload through the C ABI (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
b = make_bundle(name)
s = ietidp.from_bundle(b)
s.analyze()
for _ in range(reps):
    s.factor()
    lam, rep = s.solve(want_lambda=False)
torch.cuda.synchronize()
print(name, rep["iters"][:4], rep["ms_factor"], rep["ms_pcg"])
