"""bench.py on the CPU: the reference arm (the oracle) prints one valid JSON line, and the
--gpus N launcher starts N ranks itself when no torchrun environment is present."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, timeout=600):
    env = dict(os.environ, OMP_NUM_THREADS="8")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                          timeout=timeout, env=env)


def test_reference_arm_json_line():
    res = _run(["--impl", "reference", "--config", "C2", "--steps", "2", "--warmup", "0"])
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "bits/s"
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["higher_is_better"] is True
    assert line["metric"].startswith("reconciled bits/sec")
    assert line["config"]["bp_schedule"] == "layered" and line["config"]["frames_timed"] >= 2


def test_launch_plan():
    import bench
    assert bench.launch_plan(1, {}) == "single"
    assert bench.launch_plan(4, {}) == "spawn"
    assert bench.launch_plan(2, {"WORLD_SIZE": "2"}) == "rank"
    assert bench.launch_plan(1, {"WORLD_SIZE": "1"}) == "rank"
    with pytest.raises(SystemExit):
        bench.launch_plan(8, {"WORLD_SIZE": "2"})
    with pytest.raises(SystemExit):
        bench.launch_plan(0, {})


def test_gpus_2_spawns_two_ranks_one_line():
    """`bench.py --gpus 2` without torchrun re-launches itself as 2 ranks (torch.distributed.run,
    127.0.0.1); rank 0 alone prints (reference arm: the others exit 0 without work)."""
    res = _run(["--impl", "reference", "--gpus", "2", "--config", "C2", "--steps", "1", "--warmup", "0"])
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["impl"] == "reference"
