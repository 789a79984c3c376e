"""Print raw ncu metrics matching substrings for every kernel in a report:
   python tools/ncu_raw_grep.py REP substr [substr...]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for row in rows[2:]:
    print("==", row[h.index("Kernel Name")][:80])
    for i, name in enumerate(h):
        if any(s in name for s in sys.argv[2:]):
            v = row[i]
            if v not in ("", "0", "n/a"):
                print(f"  {name} = {v} {units[i]}")
