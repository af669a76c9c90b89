"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into per-kernel totals and shares."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iK, iV, iG = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[1:]:
    name = r[iK].split("(")[0].replace("void ", "")
    if "<" in r[iK]:
        name = r[iK].split("(sg::")[0].replace("void ", "")
    tot[name] = tot.get(name, 0.0) + float(r[iV].replace(",", "")) / 1e6
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.3f} {v / T:7.3f}")
print(f"{'total':60s} {sum(cnt.values()):8d} {T:10.3f}")
