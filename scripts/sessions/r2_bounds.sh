#!/bin/bash
# bounds-checked build (libflexemb_chk.so, FX_BOUNDS) over the fused step
# workload and the single-GPU GPU tests: the compute-sanitizer stand-in
O=gpurun_out/s5
mkdir -p $O
export FX_LIB_PATH=$PWD/paper_2410_12794_b200/libflexemb_chk.so
export FX_BOUNDS_LOG=$PWD/$O/bounds_report.txt
timeout 900 python scripts/sanitize_step.py > $O/sanitize_step_chk.log 2>&1; echo "rc=$?" >> $O/sanitize_step_chk.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not g4" > $O/pytest_chk.log 2>&1; echo "rc=$?" >> $O/pytest_chk.log
echo done
