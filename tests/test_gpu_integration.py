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
    ref_arm.import_reference()
    from embserve.errors import RoutingViolationError
    from embserve.pooling import PartialResult
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
