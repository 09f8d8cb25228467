"""bench.py's output contract: one JSON line with the driver's keys, for the
B200 arm (GPU, single rank and a functional two-rank run) and the reference
arm (the reference CPU engine; runs here without a GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run(args, env=None, timeout=600):
    r = subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    pytest.importorskip("oracle.oracle")
    from oracle import oracle as O
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    d = run(["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-size", "64"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_b200_arm_line():
    d = run(["bench.py", "--sizes", "256:512:256", "--steps", "2", "--warmup", "3", "--cpu-size", "64"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["unit"] == "GFLOPS" and d["higher_is_better"] is True
    roof = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof) and roof["achieved"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    # per step: one dual-pipe launch per scheduled group of calls, the packs of a group's small
    # operands in one grouped launch (pack_group_kernel), large operands one launch each -- at
    # least a pack and a gemm launch per group, at most 2 packs + gemm + split-K reduce per call
    groups = d["step_kernels"]["dual_d"]["launches"]
    assert 2 * 2 * groups <= d["gpu_launches"] <= 2 * 256 * 4
    assert d["step_kernels"]["dual_d"]["launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.gpu
@pytest.mark.parametrize("shard,port", [("columns", 29561), ("chains", 29562)])
def test_two_rank_path_functional(shard, port):
    # two ranks on one GPU with gloo (test hook): exercises both splits (column panels with the A
    # broadcast, whole calls by C-buffer chain) and the max-over-ranks timing; rank 0 alone prints
    d = run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
             "--master-port", str(port), "bench.py", "--gpus", "2", "--size", "512", "--labels", "dddd,zzzd,cdds,ssss",
             "--steps", "1", "--warmup", "1", "--shard", shard], env={"MDGEMM_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert ("chain" in d["config"]["parallelism"]) == (shard == "chains")
