"""bench.py --gpus N (the flag was ignored).  Launcher decisions, and a real
relaunch under torch.distributed.run on CPU (the reference arm needs no GPU): without
WORLD_SIZE, --gpus 2 spawns two ranks and rank 0 prints n_gpus = 2; a WORLD_SIZE that
disagrees with --gpus exits non-zero."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_launch_plan():
    assert bench.launch_plan(1, {}) == ("run", 1)
    assert bench.launch_plan(4, {}) == ("spawn", 4)
    assert bench.launch_plan(4, {"WORLD_SIZE": "4"}) == ("run", 4)
    assert bench.launch_plan(1, {"WORLD_SIZE": "1"}) == ("run", 1)
    assert bench.launch_plan(2, {"WORLD_SIZE": "8"})[0] == "error"
    assert bench.launch_plan(8, {"WORLD_SIZE": "1"})[0] == "error"
    assert bench.launch_plan(0, {})[0] == "error"


def test_spawn_cmd():
    cmd = bench.spawn_cmd(8, ["--gpus", "8", "--steps", "3"], 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert "--master-port=29511" in cmd and cmd[-4:] == ["--gpus", "8", "--steps", "3"]


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


def test_mismatched_world_size_exits_nonzero():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--impl", "reference", "--steps", "1"], env=_env(WORLD_SIZE="3"),
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr


def test_gpus_2_spawns_two_ranks_reference_arm():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       env=_env(OMP_NUM_THREADS="2"), capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2 and out["steps"] == 1
    assert out["cpu_baseline"]["cores"] >= 1 and out["e2e"]["h2d_bytes_per_step"] == 0
