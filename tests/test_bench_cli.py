"""bench.py's launcher contract on a box without enough GPUs: --gpus N either
spawns N ranks (torchrun) or fails loudly; the reference arm never maps the
product library."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch

    return torch.cuda.device_count()


@pytest.mark.skipif(_gpus() >= 2, reason="this box has 2 GPUs: --gpus 2 would run")
def test_gpus_n_without_devices_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "--gpus 2 needs 2 CUDA devices" in r.stderr


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "3", "--steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)


def test_reference_arm_does_not_load_the_product_library():
    """--impl reference imports only workloads.py (by path) and the reference
    from baseline/_ref: libgett_b200.so must not be mapped."""
    code = ("import sys; sys.argv=['bench.py']; import bench, json; "
            "maps=open('/proc/self/maps').read(); "
            "print(json.dumps({'mapped': 'libgett_b200' in maps, "
            "'pkg': any(m.startswith('paper_2410_06770_b200') for m in sys.modules)}))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d == {"mapped": False, "pkg": False}
