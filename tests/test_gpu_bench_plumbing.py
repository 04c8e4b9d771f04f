"""bench.py's N > 1 path end to end on the one GPU (plumbing mode: both ranks
on cuda:0 with gloo, NOT a measurement): `python bench.py --gpus 2` launches
the two ranks itself, they exchange B through the p2p path (CUDA IPC within
the device) and rank 0 prints one JSON line with n_gpus = 2."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_plumbing():
    env = dict(os.environ, CASC_BENCH_PLUMBING="1")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "1", "--steps", "2",
                        "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-int8",
                        "--no-next4", "--no-small"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    assert "plumbing_test" in d
    assert "copy engines" in d["config"]["parallelism"]
    assert d["gpu_launches"] > 0
