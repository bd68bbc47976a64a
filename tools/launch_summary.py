"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel launches, total and
share of the profiled time.  Times are cold-cache and serialised (ncu), so shares, not absolutes."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0] != "ID"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
    if r[12] == "gpu__time_duration.sum":
        v = float(r[14].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[13], 1e-6)
        tot[name] += v * scale
        cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':24s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:24s} {cnt[k]:8d} {v:10.3f} {100 * v / T:6.1f}%")
print(f"{'TOTAL':24s} {sum(cnt.values()):8d} {T:10.3f}")
