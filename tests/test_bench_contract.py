"""bench.py driver contract on the CPU side: the reference arm (`--impl
reference`, the unmodified reference Ranker copied into oracle/_ref, on the
host cores) prints one JSON line with the contract's keys, the same config
as our arm, and never loads the product library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "hot-cache-32x10Mx128-cache2pct"
    assert d["config"]["cache_rows_frac"] == 0.02 and d["config"]["pushdown_threshold"] is None


def test_reference_arm_does_not_load_the_product():
    """The arm's process must not import paper_2410_12794_b200 (whose
    __init__ loads libflexemb.so): bench.py asserts it; check the maps too."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "maps = open('/proc/self/maps').read();"
            "assert 'libflexemb' not in maps, 'libflexemb.so mapped';"
            "assert not any(k.startswith('paper_2410_12794_b200') for k in sys.modules)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]


@__import__("pytest").mark.gpu
def test_gpu_arm_json_line():
    """Our arm at N=1 (short run): contract keys, roofline, clocks, e2e with
    host-copy byte counts and a kernel-launch count."""
    import pytest
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3", "--no-cpu"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["value"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["peak"] > 0 and rf["achieved"] > 0 and rf["unit"] == "GB/s"
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 20 * 40 and "sm_mhz" in d["clocks"]
    assert d["config"]["workload"] == "hot-cache-32x10Mx128-cache2pct" and 0 < d["hit_rate"] < 1
