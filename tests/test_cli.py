"""The reference's command-line driver (tools/hestat_cli.cpp: approx / bench / dataset, StatReport JSON,
exit codes) compiled unmodified against the drop-in headers (build/hestat_cli_gpu, tests/dropin/Makefile)
reproduces the reference's own run of the same driver (tests/golden/cli/cases.json, written by
tests/golden/make_cli_golden.py from oracle/_ref/hestat_cli_ref): reports bit for bit except
wall_seconds, console lines, error messages and exit codes.  Also the determinism contract of
tests/cli_determinism.sh (reference): two runs with one seed differ only in wall_seconds."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "cli", "cases.json")
GPU_CLI = os.path.join(ROOT, "build", "hestat_cli_gpu")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "hestat_cli_ref")


def _gold():
    return json.load(open(GOLD))


def _run(cli, args, tmp_path):
    out = os.path.join(str(tmp_path), "report.json")
    if os.path.exists(out):
        os.remove(out)
    argv = [cli] + (args.replace("{table}", "tests/golden/cli/table.csv").split() if args else [])
    if args.startswith(("bench", "approx", "dataset")):
        argv += ["--out", out]
    r = subprocess.run(argv, capture_output=True, text=True, timeout=600, cwd=ROOT)
    rec = {"rc": r.returncode, "stdout": r.stdout, "stderr_first": (r.stderr.splitlines() or [""])[0]}
    if os.path.exists(out):
        rep = json.load(open(out))
        rep.pop("wall_seconds", None)
        rec["report"] = rep
    return rec


def test_golden_cases_cover_every_subcommand_and_exit_class():
    g = _gold()
    recs = g["records"]
    assert set(recs) == set(g["cases"])
    assert {c.split()[0] for c in g["cases"].values() if c} == {"approx", "bench", "dataset"}
    assert {r["rc"] for r in recs.values()} >= {0, 1, 2, 3}
    assert all("report" in r for r in recs.values() if r["rc"] == 0)


@pytest.mark.skipif(not os.path.exists(REF_CLI), reason="oracle/_ref/hestat_cli_ref not built (no /root/reference)")
def test_reference_cli_reproduces_golden(tmp_path):
    """Pins the fixture: the reference's driver, rebuilt here, still writes exactly the committed records."""
    g = _gold()
    for name, args in g["cases"].items():
        assert _run(REF_CLI, args, tmp_path) == g["records"][name], name


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(json.load(open(GOLD))["cases"]))
def test_cli_matches_reference(name, tmp_path):
    g = _gold()
    assert os.path.exists(GPU_CLI), "build/hestat_cli_gpu missing: run make -C tests/dropin"
    got = _run(GPU_CLI, g["cases"][name], tmp_path)
    assert got == g["records"][name]


@pytest.mark.gpu
def test_cli_determinism_contract(tmp_path):
    args = "bench --measure kurt --n 5000 --domain 0:20 --scale 20 --seed 9 --slots 1024"
    reps = []
    for i in range(2):
        out = os.path.join(str(tmp_path), f"r{i}.json")
        r = subprocess.run([GPU_CLI] + args.split() + ["--out", out], capture_output=True, text=True, cwd=ROOT,
                           timeout=600)
        assert r.returncode == 0, r.stderr
        lines = [ln for ln in open(out).read().splitlines() if '"wall_seconds"' not in ln]
        reps.append(lines)
    assert reps[0] == reps[1]
