"""Per-iteration cost of the PCG graph loop vs. the operator kernels alone."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
b = make_bundle(name)
res = {}
for nit in (10, 40):
    s = ietidp.from_bundle(b, fixed_iters=nit, stream=torch.cuda.current_stream().cuda_stream)
    s.factor()
    for _ in range(3):
        lam, rep = s.solve(want_lambda=False)
    ts = []
    for _ in range(5):
        lam, rep = s.solve(want_lambda=False)
        ts.append(rep["ms_pcg"])
    res[nit] = min(ts)
    s.close()
print(name, "pcg ms @10 %.3f @40 %.3f -> per iteration %.1f us" % (res[10], res[40], (res[40] - res[10]) / 30 * 1e3))
s = ietidp.from_bundle(b, stream=torch.cuda.current_stream().cuda_stream)
s.factor()
nc = b["nrhs"]
x = torch.randn(nc, b["n_lambda"], dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(5):
    s.apply_F_device(x, y, nc); s.apply_precond_device(x, y, nc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    s.apply_F_device(x, y, nc)
e1.record(); torch.cuda.synchronize(); tf = e0.elapsed_time(e1) / 100
e0.record()
for _ in range(100):
    s.apply_precond_device(x, y, nc)
e1.record(); torch.cuda.synchronize(); tm = e0.elapsed_time(e1) / 100
print("apply_F %.1f us, apply_precond %.1f us (stream launches)" % (tf * 1e3, tm * 1e3))
