"""Generate tests/golden/cli/cases.json (TEST INFRASTRUCTURE; run here, where /root/reference exists).

Runs the reference's own command-line driver (/root/reference/proj/tools/hestat_cli.cpp, compiled
unmodified against the reference headers with the CLI11 shim by oracle/Makefile into
oracle/_ref/hestat_cli_ref) on every case below and records, per case, the exit code, stdout, the
first stderr line and the JSON report without wall_seconds.  tests/test_cli.py replays the same
command lines through the same driver compiled against the drop-in headers and libhestat_gpu.so
(build/hestat_cli_gpu) on the GPU and requires identical records: report values and mre bit for bit
(nlohmann prints round-trip doubles), CostMeter counts, assumptions, messages and exit codes.

    python tests/golden/make_cli_golden.py
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "cli")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "hestat_cli_ref")

# {table} is replaced by the path of the committed CSV fixture
CASES = {
    # the determinism contract's command (tests/cli_determinism.sh)
    "bench_kurt_det": "bench --measure kurt --n 5000 --domain 0:20 --scale 20 --seed 9 --slots 1024",
    "bench_znorm_2chunks": "bench --measure znorm --n 40000 --domain 0:100 --scale 100 --slots 32768 --seed 2",
    "bench_znorm_nodebug": "bench --measure znorm --n 4096 --domain 0:100 --scale 100 --slots 4096 --no-debug",
    "bench_skew": "bench --measure skew --n 3000 --domain 0:20 --scale 20 --slots 4096 --seed 3",
    "bench_pcc": "bench --measure pcc --n 5000 --domain 0:20 --scale 20 --slots 8192 --seed 4 --rho 0.6",
    "bench_cv": "bench --measure cv --n 3000 --domain 1:20 --scale 20 --slots 4096 --seed 5",
    "bench_kurt_noquant": "bench --measure kurt --n 2000 --domain 0:20 --scale 20 --slots 2048 --no-quantize",
    "bench_znorm_scale45": "bench --measure znorm --n 2048 --domain 0:100 --scale 100 --slots 2048 --scale-bits 45",
    "bench_bad_measure": "bench --measure bogus --n 100 --slots 128",
    "bench_bad_domain": "bench --measure znorm --n 100 --slots 128 --domain 5:1",
    "approx_invsqrt_c1": "approx --fn invsqrt --n 4096 --slots 4096 --domain 0.01:1 --scale 1 --degree 15 --iters 2 --seed 11",
    "approx_invsqrt_default": "approx --fn invsqrt --n 4096 --slots 4096 --domain 0.01:1 --scale 1 --seed 11",
    "approx_invsqrt_3chunks": "approx --fn invsqrt --n 5000 --slots 2048 --domain 0.001:100 --scale 100 --seed 12",
    "approx_inv_grid": "approx --fn inv --grid --n 2048 --slots 2048 --domain 0.001:100 --scale 100",
    "approx_sqrt": "approx --fn sqrt --n 2048 --slots 2048 --domain 0.001:100 --scale 100 --seed 13",
    "approx_sign": "approx --fn sign --n 2048 --slots 2048 --domain -1:1 --seed 14",
    "approx_baseline": "approx --fn invsqrt --baseline --n 1024 --slots 1024 --domain 0.01:1 --scale 1",
    "approx_baseline_iters": "approx --fn invsqrt --baseline --iters 10 --n 1024 --slots 1024 --domain 0.01:1 --scale 1",
    "approx_domain_error": "approx --fn invsqrt --n 1024 --slots 1024 --domain 0.001:300 --scale 100",
    "approx_bad_fn": "approx --fn cube --n 128 --slots 128",
    "dataset_znorm": "dataset --file {table} --measure znorm --x charges --scale 20 --slots 1024",
    "dataset_pcc": "dataset --file {table} --measure pcc --x age --y bmi --scale 100 --slots 1024",
    "dataset_kurt": "dataset --file {table} --measure kurt --x bmi --scale 100 --slots 1024",
    "dataset_missing_column": "dataset --file {table} --measure znorm --x weight --slots 1024",
    "dataset_missing_file": "dataset --file /nonexistent/table.csv --measure znorm --x age --slots 1024",
    "dataset_bad_cell": "dataset --file tests/golden/cli/bad.csv --measure znorm --x age --slots 128",
    "no_subcommand": "",
}


def write_table(path):
    """A small seeded CSV (1500 rows, a few missing cells) for the dataset subcommand."""
    rng = np.random.default_rng(2508)
    n = 1500
    age = rng.integers(18, 65, n)
    bmi = np.round(rng.normal(30.0, 6.0, n), 2)
    charges = np.round(rng.lognormal(0.0, 0.5, n) * 2.0, 4)
    with open(path, "w") as f:
        f.write("age,bmi,charges\n")
        for i in range(n):
            b = "NA" if i % 97 == 13 else f"{bmi[i]}"
            c = "?" if i % 211 == 5 else f"{charges[i]}"
            f.write(f"{age[i]},{b},{c}\n")


def run_case(cli, args, table, tmp):
    out_path = os.path.join(tmp, "report.json")
    if os.path.exists(out_path):
        os.remove(out_path)
    argv = [cli] + (args.replace("{table}", table).split() if args else [])
    if args.startswith(("bench", "approx", "dataset")):
        argv += ["--out", out_path]
    r = subprocess.run(argv, capture_output=True, text=True, timeout=600, cwd=ROOT)
    rec = {"rc": r.returncode, "stdout": r.stdout,
           "stderr_first": (r.stderr.splitlines() or [""])[0]}
    if os.path.exists(out_path):
        rep = json.load(open(out_path))
        rep.pop("wall_seconds", None)
        rec["report"] = rep
    return rec


def main():
    if not os.path.exists(REF_CLI):
        sys.exit("oracle/_ref/hestat_cli_ref missing: run make -C oracle (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    table = os.path.join(OUT, "table.csv")
    write_table(table)
    with open(os.path.join(OUT, "bad.csv"), "w") as f:
        f.write("age,bmi\n31,22.5\n40,27.1\n4x,30.0\n")
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        recs = {name: run_case(REF_CLI, args, "tests/golden/cli/table.csv", tmp) for name, args in CASES.items()}
    json.dump({"cases": CASES, "records": recs}, open(os.path.join(OUT, "cases.json"), "w"), indent=1, sort_keys=True)
    for k, v in recs.items():
        print(f"{k:26s} rc={v['rc']} {v['stdout'].strip()[:70] or v['stderr_first'][:70]}")


if __name__ == "__main__":
    main()
