"""bench.py's multi-GPU launcher on CPU (gloo): ``--gpus N`` without a torchrun
environment re-launches N ranks, the view shards and the all-reduce of the
training step add up, and rank 0 prints one JSON line with n_gpus = N."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, capture_output=True,
                          text=True, env=env, cwd=REPO, timeout=240)


def _json_lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n", [1, 2])
def test_dry_run_reports_launched_world(n):
    r = _run(["--gpus", str(n), "--dry-run", "--steps", "2", "--warmup", "3", "--train-views", "8"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == n and d["allreduce_ok"] is True
    assert d["views_per_rank"] == 8 // n


@pytest.mark.timeout(120)
def test_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "3", "--dry-run", "--steps", "1"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in r.stderr
