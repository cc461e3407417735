"""Small fused-step workload for compute-sanitizer (memcheck / racecheck /
synccheck) or, where compute-sanitizer is unavailable (it is closed on the
GPU pool), for the bounds-checked build (FX_LIB_PATH=.../libflexemb_chk.so:
every cache / step array subscript checked on the device, report printed at
the end): every decision mode of csrc/fx_step.cu on tiny shapes —
parallel chain with rejections, the sequential path, pushdown threshold,
"always" admission, pipeline_depth 2 (dynamic presence), staging while the
cache fills, a rejected batch — each checked against the vectorised oracle.

    compute-sanitizer --tool memcheck python scripts/sanitize_step.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from step_harness import run_compare  # noqa: E402


def main():
    torch.cuda.set_device(0)
    import paper_2410_12794_b200 as P
    T, N, D = 4, 20_000, 32
    dep = P.init_store([P.TableMeta(t, N, D) for t in range(T)], [P.ShardSpec(t, 0, N, 0) for t in range(T)], 0)
    cases = [dict(alpha=0.6, cache_frac=0.05, batch=128), dict(alpha=1.0, cache_frac=0.002, batch=128),
             dict(alpha=1.0, cache_frac=0.02, batch=64, threshold=2),
             dict(alpha=0.9, cache_frac=0.01, batch=64, admission="always"),
             dict(alpha=0.8, cache_frac=0.01, batch=64, depth=2)]
    bad = 0
    for c in cases:
        rep, _ = run_compare(tables=T, rows=N, dim=D, pooling=(1, 12), n_batches=4, dep=dep, check_vectors=16,
                             log=lambda r: None, **c)
        nb = sum(len(r["bad"]) for r in rep)
        bad += nb
        print(c, "mismatches", nb, flush=True)
    print("sanitize_step done, mismatches", bad)
    from paper_2410_12794_b200 import _lib
    rep = _lib.bounds_report()
    if rep is not None:
        st = _lib.lib.fx_bounds_selftest()
        print("FX_BOUNDS report:", rep, "selftest (1 = an injected out-of-range read is caught):", st, flush=True)
        bad += rep["violations"] + (st != 1)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
