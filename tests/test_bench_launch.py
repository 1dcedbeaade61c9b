"""bench.py's multi-GPU launcher, exercised on CPU: `--gpus 2` outside
torchrun re-launches itself as two ranks (torch.distributed.run, 127.0.0.1);
with --plan-only the ranks rendezvous over gloo and report their shard of the
workload (c5: the 64-image batch split round-robin, strong scaling)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_bench_self_spawns_two_ranks_c5_split():
    d = _run("--gpus", "2", "--plan-only", "--workload", "c5")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    a, b = d["shards"]
    assert sorted(a + b) == list(range(64)) and not set(a) & set(b)
    assert d["max_images_per_rank"] == 32


def test_bench_single_rank_default_workload():
    d = _run("--plan-only")
    assert d["n_gpus"] == 1 and d["workload"] == "c2" and d["scaling"] == "weak"
