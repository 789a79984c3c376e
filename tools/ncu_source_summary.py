"""Summarise an ncu source page (csv) by stall samples: python tools_src.py src.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ci = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ci]), int(float(r[ie])), r[si].strip()[:110]))
    except Exception:
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot, "instructions", len(data))
for d in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{d[0] / tot * 100:5.1f}% {d[1]:8d}  {d[2]}")
