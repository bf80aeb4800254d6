"""bench.py's multi-rank launch on CPU: `python bench.py --gpus 2` (no torchrun around it)
re-runs itself as 2 ranks through torch.distributed.run (rendezvous on 127.0.0.1); --dry-run
exercises only the launch plumbing (gloo group, max over ranks, rank 0's JSON line)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_gpus_2_spawns_two_ranks():
    line = run("--gpus", "2", "--steps", "3", "--warmup", "3", "--dry-run")
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert line["max_over_ranks"] == 2.0  # the max of the ranks' values, rank 1's


def test_bench_gpus_1_runs_in_process():
    line = run("--gpus", "1", "--steps", "3", "--dry-run")
    assert line["n_gpus"] == 1 and line["max_over_ranks"] == 1.0
