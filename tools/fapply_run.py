"""A few F-applies of a workload through the C ABI (for ncu captures of k_sym_stream)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
b = make_bundle(name)
s = ietidp.from_bundle(b)
s.factor()
nc = b["nrhs"]
x = torch.randn(nc, b["n_lambda"], dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(4):
    s.apply_F_device(x, y, nc)
torch.cuda.synchronize()
print(name, float(y.norm()))
