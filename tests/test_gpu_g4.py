"""K4 TMA tile::gather4 variant (FX_POOL_VARIANT=3, csrc/fx_pool_async.cuh
k_pool_g4): the K4 parity tests of test_gpu_core re-run in a subprocess with
the variant selected (the variant is read once per process)."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(os.environ.get("FX_POOL_VARIANT") == "3", reason="already running under the gather4 variant")
def test_k4_gather4_variant_parity():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, FX_POOL_VARIANT="3")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_core.py"), "-k",
                        "engine_pool or pool_many or partial_pool or multi_shard or empty_bags or strided or mixed"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
