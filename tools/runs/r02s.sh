#!/bin/bash
OUT=gpurun_out/r02s; mkdir -p $OUT
for i in 1 2 3; do timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3_$i.json 2> $OUT/bench_c3_$i.err; done
timeout 600 python tools/diag_wave.py --steps 12 > $OUT/diag.log 2>&1
