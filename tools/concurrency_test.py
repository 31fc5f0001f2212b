"""Does a second, independent factorisation overlap with the first one? (two handles,
two streams, two host threads). Diagnostic for splitting one factorisation into
independent subdomain groups."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from ietigen.bundle import make_bundle
from paper_2501_04340_b200 import ietidp

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
b = make_bundle(name)
st = [torch.cuda.Stream() for _ in range(2)]
S = [ietidp.from_bundle(b, stream=st[i].cuda_stream) for i in range(2)]
for s in S:
    s.analyze()
    s.factor()
    s.factor()
torch.cuda.synchronize()
def one(s, n, out, i):
    t0 = time.perf_counter()
    for _ in range(n):
        s.factor()
    out[i] = time.perf_counter() - t0
n = 10
out = [0, 0]
one(S[0], n, out, 0)
print("one handle: %.3f ms per factor" % (out[0] / n * 1e3))
for stagger in (0.0, 0.003):
    ths = [threading.Thread(target=one, args=(S[i], n, out, i)) for i in range(2)]
    t0 = time.perf_counter()
    ths[0].start()
    time.sleep(stagger)
    ths[1].start()
    for t in ths: t.join()
    dt = time.perf_counter() - t0 - stagger
    print("two handles concurrently (stagger %.1f ms): %.3f ms per pair of factors = %.2f x one"
          % (stagger * 1e3, dt / n * 1e3, dt / n / (out[0] / n)))
