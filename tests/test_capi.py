"""The C-ABI library loads without a GPU and exports every entry point
declared in include/flexemb.h (no compute calls here)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "flexemb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    for n in ("fx_table_init", "fx_gather_pool", "fx_gather_rows", "fx_combine", "fx_route", "fx_bucket",
              "fx_dedup", "fx_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2410_12794_b200._lib as L
    lib = ctypes.CDLL(L.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(L.EXPORTED) == sorted(n for n in _declared() if n in L._SIGS)
    assert set(_declared()) <= set(L._SIGS), "every declared symbol has a ctypes signature"


def test_host_helpers_without_gpu():
    import paper_2410_12794_b200._lib as L
    import oracle as O
    assert L.lib.fx_version() >= 1
    for seed, t in ((0, 0), (7, 3), (2**31, 99), (2**63 + 5, 1)):
        assert L.lib.fx_table_base(seed % 2**64, t) == int(O.table_base(seed % 2**64, t))


def test_segment_struct_layout():
    import paper_2410_12794_b200._lib as L
    assert L.SEGMENT_BYTES == 8 * 8 + 4 + 4 + 2 * 8


def test_build_entry_does_not_need_the_library():
    """__graft_entry__.build() must work on a fresh checkout where
    libflexemb.so does not exist yet: loading the build module may not run
    the package __init__ (which refuses to import without the library)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, __graft_entry__ as g; m = g._build_module(); "
            "assert callable(m.build) and m.LIB.endswith('libflexemb.so'); "
            "assert 'paper_2410_12794_b200' not in sys.modules")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
