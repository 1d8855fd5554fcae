"""The reference's benchmark suites and run driver on the GPU operators (suite.py / cli.py),
at the smallest sizes: CSV layouts of bench.cpp, the TOMOSPM1 operator cache, and the
reconstruct path's per-iteration trace."""
import csv
import json
import os
import subprocess
import sys

import pytest

from paper_1705_07497_b200 import suite as S

pytestmark = pytest.mark.gpu


def _rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def test_table1_ci(tmp_path):
    base = S.RunConfig(output_dir=str(tmp_path), cache_dir=str(tmp_path / "cache"))
    logs = []
    assert S.run_bench_suite("table1", "ci", base, logs.append)
    rows = _rows(tmp_path / "table1_ci.csv")
    assert len(rows) == 2 * 3 * 3
    assert {r["backend"] for r in rows} == {"direct", "fused", "surrogate"}
    assert all(float(r["apply_ms"]) > 0 for r in rows)
    # the operator cache is used on the second pass
    assert S.run_bench_suite("table1", "ci", base, logs.append)
    assert any(line.startswith("cached:") for line in logs)


def test_table2_and_tables345_ci(tmp_path):
    base = S.RunConfig(output_dir=str(tmp_path), cache_dir=str(tmp_path / "cache"), iters=4, cg_steps=3)
    assert S.run_bench_suite("table2", "ci", base, print)
    rows = _rows(tmp_path / "table2_ci.csv")
    assert len(rows) == 18 and all(int(r["iterations"]) == 4 for r in rows)
    assert all(0 < float(r["final_rel_l1"]) < 2 and float(r["cg_s"]) <= float(r["total_s"]) for r in rows)
    base.iters = 30
    assert S.run_bench_suite("tables345", "ci", base, print)
    rows = _rows(tmp_path / "tables345_ci.csv")
    assert len(rows) == 3 * 2 * 4
    crossed = [r for r in rows if r["threshold"] == "1e-2"]
    assert all(int(r["iterations"]) > 0 for r in crossed)


def test_cli_reconstruct(tmp_path):
    args = [sys.executable, "-m", "paper_1705_07497_b200.cli", "reconstruct", "--n", "64", "--iters", "5",
            "--backend", "surrogate", "--out", str(tmp_path), "--cache-dir", str(tmp_path / "c")]
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "built and cached" in r.stdout and "iterations=5" in r.stdout
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "cached:" in r.stdout
    lines = open(tmp_path / "runs.jsonl").read().splitlines()
    assert len(lines) == 2 and json.loads(lines[0])["final_rel_l1"] == json.loads(lines[1])["final_rel_l1"]
    assert any(f.endswith("_trace.csv") for f in os.listdir(tmp_path))
