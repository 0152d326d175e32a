"""bench.py host logic (no GPU needed): the multi-rank launcher refuses to time fewer ranks than
asked, and the --gpus / WORLD_SIZE consistency check."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=env, cwd=ROOT)


def test_gpus_beyond_visible_fails_cleanly():
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("this node has >= 2 GPUs: the launcher would start real ranks")
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 2
    assert "needs 2 visible GPUs" in r.stderr and r.stdout.strip() == ""


def test_world_size_mismatch_fails():
    r = _run(["--gpus", "4"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
