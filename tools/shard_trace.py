"""Per-launch device timeline of the sharded loop on one rank (IETIDP_TRACE):
python tools/shard_trace.py C3 -> totals per launch site of the last solve."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
raw = "/tmp/ietidp_shard_trace.raw"
if os.path.exists(raw):
    os.remove(raw)
os.environ["IETIDP_TRACE"] = raw
import numpy as np  # noqa: E402
import torch  # noqa: E402
from ietigen.bundle import make_bundle  # noqa: E402
from paper_2501_04340_b200 import ietidp  # noqa: E402

b = make_bundle(name)
owner = np.zeros(b["n_sub"], np.int32)
s = ietidp.shard_from_bundle(b, owner, 0, 1, lambda ptr, n, stream: 0)
s.analyze()
for _ in range(2):
    s.factor()
    lam, rep = s.solve(want_lambda=False)
lines = [l.split() for l in open(raw).read().split("\n") if l]
idx = [i for i, l in enumerate(lines) if l[0] == "solve"]
blk = []
for i in reversed(idx):
    if blk and i != blk[-1] - 1:
        break
    blk.append(i)
tot = collections.Counter(); cnt = collections.Counter()
for i in blk:
    tot[lines[i][1]] += float(lines[i][2]); cnt[lines[i][1]] += 1
T = sum(tot.values())
print(name, "iters", rep["iters"][:4], "ms_pcg", rep["ms_pcg"], "traced us", T)
for k, v in tot.most_common(25):
    print(f"  {k:24s} {cnt[k]:5d} x {v / cnt[k]:8.2f} us = {v:10.1f} us")
