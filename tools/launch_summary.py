"""Summarise an ncu launch list (gpu__time_duration.sum CSV) of tools/prof_run.py:
per-kernel totals of the last factor+solve pass (from the last k_scatter of a factor)."""
import csv, collections, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
K, G, V = h.index('Kernel Name'), h.index('Grid Size'), h.index('Metric Value')
seq = [(r[K].split('(')[0].replace('void ', '').replace('ieti::', ''), r[G].replace(', 1, 1)', '').replace('(', ''),
        float(r[V]) / 1000) for r in rows[hi + 1:]]
starts = [i for i, s in enumerate(seq) if s[0] == 'k_scatter' and i + 1 < len(seq) and seq[i + 1][0] != 'k_fs_assemble<1>']
st = starts[-1]
end = len(seq)
tot = collections.Counter()
cnt = collections.Counter()
for s in seq[st:end]:
    tot[s[0]] += s[2]
    cnt[s[0]] += 1
print(f"launches from index {st}: {end - st}")
for k, v in tot.most_common():
    print(f"  {k:40s} {cnt[k]:4d} x  {v:9.1f} us")
print(f"  total {sum(tot.values()):.1f} us")
if len(sys.argv) > 2:
    for s in seq[st:end]:
        print(f"{s[0][:30]:30s} {s[1]:>8s} {s[2]:8.1f}")
