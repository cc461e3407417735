#!/bin/bash
# end-of-round validation on one B200: full GPU suite, smoke, default bench
# (both arms), launch list of a steady-state cfg3 batch, and the whole suite
# again under the bounds-checked build
O=gpurun_out/f2
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --graph-step 0 --steps 4 --warmup 6 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
FX_LIB_PATH=$PWD/paper_2410_12794_b200/libflexemb_chk.so FX_BOUNDS_LOG=$PWD/$O/bounds_report.txt timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not g4" > $O/pytest_chk.log 2>&1; echo "rc=$?" >> $O/pytest_chk.log
echo done
