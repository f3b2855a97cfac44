"""bench.py's multi-rank harness on CPU: ``--gpus N`` launches N ranks itself
(torch.distributed.run), and the dry run goes through the gloo rendezvous, the
barriers and the max-over-ranks timing and prints one JSON line with n_gpus = N."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=240, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.timeout(300)
def test_dry_run_two_ranks():
    line = _run("--gpus", "2", "--dry-run", "--steps", "4", "--warmup", "3")
    assert line["n_gpus"] == 2 and line["dry_run"] and line["steps"] == 4 and line["value"] > 0


@pytest.mark.timeout(300)
def test_dry_run_one_rank():
    line = _run("--dry-run", "--steps", "3")
    assert line["n_gpus"] == 1


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr
