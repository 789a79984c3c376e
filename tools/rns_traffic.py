"""Per-op DRAM traffic of the Tier-R primitives (run on the GPU box; needs ncu).

  python tools/rns_traffic.py OUT.json [--batch 16] [--dnum 2 --K 13]

For each op, one eager call on `batch` ciphertexts (N=2^16, L=24, 44-bit special primes; dnum/K as
given, default the bench shape dnum=2, K=13) under ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum; the kernels of the call are summed and divided by the batch.  ncu
serialises launches and flushes caches between them, so traffic is an upper bound of what the
graph-replayed bench sees; times here are NOT bench values."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = sys.argv[1]
batch = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 16
def _arg(name, default):
    return int(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


N, l = 1 << 16, 24
K, dnum = _arg("--K", 13), _arg("--dnum", 2)
key = 2 * dnum * (l + 1 + K) * N * 8
alg = {"ntt": 2 * 2 * (l + 1) * N * 8, "mul_relin": 4 * (l + 1) * N * 8 + key + 2 * (l + 1) * N * 8,
       "mul_relin_rescale": 4 * (l + 1) * N * 8 + key + 2 * l * N * 8,
       "rescale": 2 * (l + 1) * N * 8 + 2 * l * N * 8, "rotate": 2 * (l + 1) * N * 8 + key + 2 * (l + 1) * N * 8}
res = {"shape": {"logN": 16, "L": l, "K": K, "dnum": dnum, "logp": 44, "batch": batch},
       "method": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "--clock-control none --profile-from-start off, tools/rns_prof.py OP --reps 1",
       "ops": {}}
for op in ("ntt", "mul_relin", "mul_relin_rescale", "rescale", "rotate"):
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--profile-from-start", "off", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "rns_prof.py"), op, "--batch", str(batch), "--reps", "1",
           "--K", str(K), "--dnum", str(dnum)]
    txt = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
    lines = [x for x in txt.splitlines() if x.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0, "gpu__time_duration.sum": 0.0}
    kernels = set()
    for r in rows:
        name, unit, val = r["Metric Name"], r["Metric Unit"], float(r["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
                 "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        if name in tot:
            tot[name] += val * scale
        kernels.add(r["Kernel Name"].split("(")[0][-60:])
    cts = batch  # rns_prof's ntt transforms 2 x batch polynomials = batch ciphertexts
    traffic = (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / cts
    res["ops"][op] = {"dram_bytes_per_ct": traffic, "alg_bytes_per_ct": alg[op],
                      "traffic_over_alg": traffic / alg[op], "ncu_us_per_ct": tot["gpu__time_duration.sum"] / cts,
                      "launches": len(rows) // 3, "kernels": sorted(kernels)}
    print(op, res["ops"][op]["dram_bytes_per_ct"] / 1e6, "MB/ct vs alg", alg[op] / 1e6, flush=True)
with open(out_path, "w") as f:
    json.dump(res, f, indent=1)
