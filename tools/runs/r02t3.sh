#!/bin/bash
# recorded-path release: tests first, then trace + A/B
OUT=gpurun_out/r02t3; mkdir -p $OUT
cp ab/libprism_relist.so paper_2605_08581_b200/libprism.so
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
cp ab/libprism_trace.so paper_2605_08581_b200/libprism.so
PRISM_TRACE_OUT=$OUT/trace_c3.json timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/bench_trace.json 2> $OUT/bench_trace.err; echo "trace rc=$?"
python tools/trace_sum.py $OUT/trace_c3.json > $OUT/trace_c3.txt; head -50 $OUT/trace_c3.txt
VARIANTS="relaux relist" ROUNDS=2 OUT=$OUT/ab bash tools/ab_run.sh
