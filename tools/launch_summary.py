"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel total us and share."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
tot, cnt = {}, {}
for r in rows[start + 1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("hsg::rns::", "").replace("(anonymous namespace)::", "")
    v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0 if d["Metric Unit"] == "us" else 1e3)
    tot[k] = tot.get(k, 0) + v
    cnt[k] = cnt.get(k, 0) + 1
T = sum(tot.values())
print(f"{'kernel':48s} {'launches':>8s} {'us':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:48]:48s} {cnt[k]:8d} {v:10.1f} {v / T:6.1%}")
print(f"{'total':48s} {sum(cnt.values()):8d} {T:10.1f}")
