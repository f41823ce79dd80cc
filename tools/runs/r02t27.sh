#!/bin/bash
OUT=gpurun_out/r02t27; mkdir -p $OUT
cp ab/libprism_trace.so paper_2605_08581_b200/libprism.so
PRISM_TRACE_OUT=$OUT/trace_c3.json timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/bench_trace.json 2> $OUT/bench_trace.err; echo "trace rc=$?"
python tools/trace_sum.py $OUT/trace_c3.json > $OUT/trace_c3.txt
