"""Sum gpu__time_duration per kernel name from an ncu --csv launch list.
python scripts/ncu_sum.py launches.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]
ki, mi, vi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[h + 1:]:
    if r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) / 1e3
        cnt[name] += 1
all_us = sum(tot.values())
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100 * v / all_us:5.1f}%  n={cnt[n]:5d}  {v / cnt[n]:8.1f} us/launch  {n}")
print(f"total {all_us:.1f} us")
