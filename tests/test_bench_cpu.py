"""bench.py's launch contract without a GPU: `--gpus N` outside torchrun
spawns N ranks itself (torch.distributed.run on 127.0.0.1) and every rank
sees WORLD_SIZE == N; the dry run does the rank plumbing over gloo."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_self_spawns_ranks():
    line = _run("--gpus", "2", "--dry-run")
    assert line["world"] == 2 and line["n_gpus"] == 2 and line["max_rank_plus_1"] == 2.0


def test_bench_single_rank_default():
    line = _run("--dry-run")
    assert line["world"] == 1 and line["n_gpus"] == 1
