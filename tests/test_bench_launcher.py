"""bench.py --gpus N starts N ranks itself when not under torchrun (CPU stand-in, gloo)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--selftest-cpu",
                          "--steps", "3", "--warmup", "1", *extra],
                         capture_output=True, text=True, timeout=180, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_spawned_two_ranks_report_the_whole_job():
    line = _run("--gpus", "2")
    assert line["n_gpus"] == 2
    assert line["config"]["global_units_per_step"] == 128
    assert line["config"]["units_per_gpu_per_step"] == 64
    # max over ranks: rank 1 sleeps 4 ms per step, so the step can not be faster
    assert line["ms_per_step"] >= 4.0


def test_single_rank_default():
    line = _run()
    assert line["n_gpus"] == 1 and line["config"]["global_units_per_step"] == 64


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--selftest-cpu",
                          "--gpus", "2"], capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "refusing" in out.stderr
