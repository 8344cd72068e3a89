"""bench.py's launch contract on CPU: `--gpus N` re-launches itself as N
ranks (torchrun) and the sharded result is bit-identical to one rank; the GPU
arm refuses to pretend N GPUs when fewer are visible."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=240):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p.returncode, (json.loads(lines[-1]) if lines else None), p


@pytest.mark.parametrize("gpus,pop", [(2, 24), (3, 25)])
def test_dry_run_ranks_match_one_rank(gpus, pop):
    rc1, one, p1 = _run("--gpus", "1", "--dry-run", "--pop", str(pop))
    rcn, many, pn = _run("--gpus", str(gpus), "--dry-run", "--pop", str(pop))
    assert rc1 == 0 and rcn == 0, (p1.stderr[-2000:], pn.stderr[-2000:])
    assert one["n_gpus"] == 1 and many["n_gpus"] == gpus
    assert many["digest"] == one["digest"] and many["moves"] == one["moves"]


def test_gpus_beyond_visible_devices_fails_loudly():
    import torch

    want = max(2, torch.cuda.device_count() + 1)
    rc, line, p = _run("--gpus", str(want), "--steps", "1", "--warmup", "1")
    assert rc != 0
    assert line is not None and "error" in line
