"""INTEGRATION.md §2 executed as written: the ctypes stub that replaces
ServerStore.partial_pool, run with the reference's OWN PartialResult class
(the unmodified embserve copied to oracle/_ref by build()), against the
reference's golden partial_pool vectors."""

import os
import re

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_partial_pool(golden_dir):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import ref_arm
    if not ref_arm.available():
        pytest.skip("oracle/_ref (the reference copy) is not built")
    emb = ref_arm.import_reference()
    RoutingViolationError = emb.errors.RoutingViolationError
    PartialResult = emb.pooling.PartialResult
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 2. C-ABI binding"):text.index("## 3.")]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    code = code.replace('ctypes.CDLL("paper_2410_12794_b200/libflexemb.so")',
                        f'ctypes.CDLL("{os.path.join(ROOT, "paper_2410_12794_b200", "libflexemb.so")}")')
    ns = {"PartialResult": PartialResult, "RoutingViolationError": RoutingViolationError}
    exec(compile(code, "INTEGRATION.md#2", "exec"), ns)
    z = np.load(os.path.join(golden_dir, "pool.npz"))
    for k in range(int(z["n_pp"][0])):
        seed, rows, dim = (int(v) for v in z[f"pp{k}_meta"])
        idx = [int(i) for i in z[f"pp{k}_idx"]]
        shard = torch.from_numpy(O.table_block(seed, 0, dim, 0, rows)).cuda()
        pr = ns["partial_pool"](shard, 0, rows, idx, 0)
        assert isinstance(pr, PartialResult) and pr.count == len(idx) and pr.source == 0
        assert pr.vector.tobytes() == z[f"pp{k}_vec"].tobytes(), k
    shard = torch.from_numpy(O.table_block(0, 0, 8, 0, 100)).cuda()
    with pytest.raises(RoutingViolationError):
        ns["partial_pool"](shard, 0, 100, [3, 150], 0)


def test_store_c_abi():
    """fx_store_create / fx_store_shard_view / fx_poll_error through ctypes:
    the rank's shards materialised bit-exactly, placement validated with the
    reference's rules, rows of other ranks rejected."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes
    from paper_2410_12794_b200 import _lib
    L = _lib.lib

    class Shard(ctypes.Structure):
        _fields_ = [("table", ctypes.c_int32), ("owner", ctypes.c_int32), ("start", ctypes.c_int64),
                    ("end", ctypes.c_int64)]
    rows = (ctypes.c_int64 * 2)(1000, 300)
    dims = (ctypes.c_int32 * 2)(30, 64)
    sh = (Shard * 3)(Shard(0, 0, 0, 600), Shard(0, 1, 600, 1000), Shard(1, 0, 0, 300))
    h = ctypes.c_void_p()
    torch.cuda.set_device(0)
    assert L.fx_store_create(ctypes.byref(h), 0, 2, rows, dims, 3, sh, 0, 7, None) == 0
    torch.cuda.synchronize()
    base, st, en, ld, dm = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    assert L.fx_store_shard_view(h, 0, 599, ctypes.byref(base), ctypes.byref(st), ctypes.byref(en), ctypes.byref(ld),
                                 ctypes.byref(dm)) == 0
    assert (st.value, en.value, dm.value, ld.value) == (0, 600, 30, 32)
    buf = torch.empty(600 * 32, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib.fx_memcpy_async(buf.data_ptr(), base.value, 600 * 32 * 4, None), "copy")
    got = buf.view(600, 32)[:, :30].cpu().numpy()
    assert got.tobytes() == O.table_block(7, 0, 30, 0, 600).tobytes()
    rc = L.fx_store_shard_view(h, 0, 700, ctypes.byref(base), None, None, None, None)
    assert rc == _lib.FX_E_ROUTING_VIOLATION
    L.fx_store_destroy(h)
    bad = (Shard * 2)(Shard(0, 0, 0, 600), Shard(0, 1, 500, 1000))
    rc = L.fx_store_create(ctypes.byref(h), 0, 1, rows, dims, 2, bad, 0, 7, None)
    assert rc == _lib.FX_E_CONFIG and b"overlap at row 500" in L.fx_last_error()
    st_ = _lib.Status(torch.device("cuda", 0))
    st_.code.fill_(3)
    st_.err.fill_(42)
    c, p = ctypes.c_int32(), ctypes.c_int64()
    assert L.fx_poll_error(st_.code.data_ptr(), st_.err.data_ptr(), ctypes.byref(c), ctypes.byref(p), None) == 0
    assert (c.value, p.value) == (3, 42)
