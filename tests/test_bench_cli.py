"""bench.py's launcher logic that needs no GPU."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_more_ranks_than_devices_fails_at_once():
    """`bench.py --gpus N` spawns one process per GPU; with fewer devices than ranks it must say so and exit instead of
    leaving rank 0 waiting in the rendezvous for a rank that died (observed on a one-GPU box before the check)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "PB200_BENCH_SAME_DEVICE")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0
    assert "needs 64 CUDA devices" in r.stderr, r.stderr
    assert r.stdout.strip() == ""


def test_rank_beyond_the_devices_fails_before_the_rendezvous():
    env = dict(os.environ, RANK="63", LOCAL_RANK="63", WORLD_SIZE="64", MASTER_ADDR="127.0.0.1", MASTER_PORT="29999")
    env.pop("PB200_BENCH_SAME_DEVICE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0
    assert "CUDA device" in r.stderr, r.stderr
