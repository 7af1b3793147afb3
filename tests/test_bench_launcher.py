"""bench.py --gpus N launches N ranks itself (torch.distributed.run) when no launcher did, and
rank 0 prints one JSON line aggregating all ranks: checked on CPU ranks with the gloo dry run."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                       capture_output=True, text=True, timeout=240)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_launcher_spawns_and_aggregates_two_ranks():
    out = _run(["--gpus", "2", "--dry-run-gloo", "--master-port", "29611"])
    assert out["n_gpus"] == 2
    assert out["ranks"] == [0, 1]
    assert out["value"] == 3.0          # (0 + 1) + (1 + 1): every rank contributed


def test_launcher_single_process():
    out = _run(["--dry-run-gloo", "--master-port", "29613"])
    assert out["n_gpus"] == 1 and out["ranks"] == [0]
