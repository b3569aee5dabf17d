"""bench.py's launch contract on a box without GPUs: --gpus N must launch N
ranks or fail loudly -- never time one GPU and call it N."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=600, env=env)


def test_gpus_2_without_gpus_fails_clearly():
    import torch
    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        import pytest
        pytest.skip("this box has 2 GPUs")
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
    assert "--gpus 2 needs 2 visible GPUs" in r.stderr


def test_world_size_mismatch_fails_clearly():
    r = _run(["--gpus", "2", "--steps", "1"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "--gpus 2 but the launcher started 1 ranks" in r.stderr
