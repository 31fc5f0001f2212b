"""Per-launch device timeline of one factor + solve (IETIDP_TRACE events between launches,
no profiler): python tools/trace_run.py C2 [out.txt]. Prints totals per launch site."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
out = sys.argv[2] if len(sys.argv) > 2 else "/tmp/ietidp_trace.txt"
if os.path.exists(out):
    os.remove(out)
os.environ["IETIDP_TRACE"] = out + ".raw"
if os.path.exists(out + ".raw"):
    os.remove(out + ".raw")
import torch  # noqa: E402
from ietigen.bundle import make_bundle  # noqa: E402
from paper_2501_04340_b200 import ietidp  # noqa: E402

b = make_bundle(name)
s = ietidp.from_bundle(b)
s.analyze()
for _ in range(3):
    s.factor()
    s.solve(want_lambda=False)
rep = s.report()
lines = open(out + ".raw").read().split("\n")
lines = [l.split() for l in lines if l]
# keep the last factor and the last solve
last = {}
for ph in ("factor", "solve"):
    idx = [i for i, l in enumerate(lines) if l[0] == ph]
    # contiguous last block
    blk = []
    for i in reversed(idx):
        if blk and i != blk[-1] - 1:
            break
        blk.append(i)
    last[ph] = [lines[i] for i in sorted(blk)]
with open(out, "w") as f:
    for ph, ls in last.items():
        tot = collections.Counter()
        cnt = collections.Counter()
        for _, site, us in ls:
            tot[site] += float(us)
            cnt[site] += 1
        f.write(f"== {ph}: {len(ls)} launches, {sum(tot.values()):.1f} us\n")
        for k, v in tot.most_common():
            f.write(f"  {k:22s} {cnt[k]:4d} x {v:9.1f} us\n")
        for _, site, us in ls:
            f.write(f"    {site:22s} {float(us):8.1f}\n")
print(open(out).read()[:3000])
print(name, "ms_factor", rep["ms_factor"], "ms_pcg", rep["ms_pcg"])
