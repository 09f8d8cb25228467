"""The mdgemm_b200 CLI (tools/mdgemm_b200_cli.cpp) keeps the reference CLI's
`bench` / `info` interface and its CSV contract
`case,m,n,k,trials,best_seconds,gflops` (bench.cpp:53-64)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "mdgemm_b200")
needs_cli = pytest.mark.skipif(not os.path.exists(CLI), reason="tools/mdgemm_b200 not built")


@needs_cli
def test_info_without_gpu_prints_config_and_case_table():
    r = subprocess.run([CLI, "info"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0
    assert "double: mc=64 nc=512 kc=128 mr=4 nr=4" in r.stdout
    assert "domain cases: 0, 1a, 1b, 1c, 2ab, 2ac, 2bc, 3" in r.stdout


@needs_cli
def test_bad_arguments_exit_2():
    assert subprocess.run([CLI, "bench", "--bogus"], capture_output=True, timeout=60).returncode == 2
    assert subprocess.run([CLI], capture_output=True, timeout=60).returncode == 2


@needs_cli
@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--host"], ["--numerics", "exact"]])
def test_bench_csv_contract(tmp_path, extra):
    out = tmp_path / "b.csv"
    r = subprocess.run([CLI, "bench", "--case", "zczd", "--case", "dssd", "--min", "64", "--max", "192", "--step", "64",
                        "--trials", "2", "--out", str(out)] + extra, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "case,m,n,k,trials,best_seconds,gflops"
    rows = [l.split(",") for l in lines[1:]]
    assert [(c, m) for c, m, *_ in rows] == [("zczd", "64"), ("zczd", "128"), ("zczd", "192"),
                                             ("dssd", "64"), ("dssd", "128"), ("dssd", "192")]
    for c, m, n, k, trials, best, gflops in rows:
        assert m == n == k and trials == "2" and float(best) > 0 and float(gflops) > 0


@needs_cli
@pytest.mark.gpu
@pytest.mark.parametrize("numerics", ["fast", "exact"])
def test_conformance_subcommand(numerics):
    # the reference CLI's `test` (tools/mdgemm.cpp:54-84): full storage and scalar sweeps on a label of
    # every case, per-element bound checked by the CLI's own brute-force product
    cases = ["dssd", "zdds", "dzds", "cdds", "szzs", "zzds", "zdzs", "zczd"]
    args = [CLI, "test", "--numerics", numerics]
    for c in cases:
        args += ["--case", c]
    r = subprocess.run(args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    # per label: 4 sizes + rectangle + 6..8 storage variants + 16 scalar points + complex alpha
    checks = int(r.stdout.split()[0])
    assert checks >= len(cases) * (4 + 1 + 6 + 17), r.stdout
    assert " 0 failures" in r.stdout


@needs_cli
def test_conformance_subcommand_rejects_bad_config():
    r = subprocess.run([CLI, "test", "--numerics", "bogus"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 1 and "gpu.numerics" in r.stderr


@needs_cli
@pytest.mark.gpu
def test_bench_roofline_columns_and_gpus(tmp_path):
    out = tmp_path / "b.csv"
    r = subprocess.run([CLI, "bench", "--case", "dssd", "--case", "cccs", "--size", "256", "--trials", "2", "--gpus",
                        "1", "--roofline", "--out", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "case,m,n,k,trials,best_seconds,gflops,gpus,peak_gflops,frac_of_peak"
    rows = [l.split(",") for l in lines[1:]]
    assert [row[0] for row in rows] == ["dssd", "cccs"]
    assert float(rows[0][8]) == 37000.0 and float(rows[1][8]) == 72000.0
    for row in rows:
        assert row[7] == "1" and abs(float(row[9]) - float(row[6]) / float(row[8])) < 1e-3
