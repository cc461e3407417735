import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libflexemb.so")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def pytest_sessionfinish(session, exitstatus):
    """Under the bounds-checked build (FX_LIB_PATH=.../libflexemb_chk.so, the
    compute-sanitizer stand-in) any out-of-range device subscript recorded
    during the session fails it."""
    if not os.environ.get("FX_LIB_PATH", "").endswith("_chk.so"):
        return
    mod = sys.modules.get("paper_2410_12794_b200._lib")
    if mod is None:
        return
    import torch
    if not torch.cuda.is_available():
        return
    rep = mod.bounds_report()
    st = mod.lib.fx_bounds_selftest()  # 1: an injected out-of-range read is caught
    line = f"FX_BOUNDS report: {rep} (selftest after the session: {st})"
    print("\n" + line)
    out = os.environ.get("FX_BOUNDS_LOG")
    if out:
        with open(out, "a") as f:
            f.write(line + "\n")
    if rep is None or rep["violations"] > 0 or st != 1:
        session.exitstatus = 1
