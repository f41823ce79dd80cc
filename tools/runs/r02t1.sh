#!/bin/bash
# in-graph kernel start timeline (diagnostics build ab/libprism_trace.so)
OUT=gpurun_out/r02t1; mkdir -p $OUT
cp ab/libprism_trace.so paper_2605_08581_b200/libprism.so
PRISM_TRACE_OUT=$OUT/trace_c3.json timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "c3 rc=$?"
python tools/trace_sum.py $OUT/trace_c3.json > $OUT/trace_c3.txt; head -90 $OUT/trace_c3.txt
