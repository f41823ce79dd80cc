#!/bin/bash
OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 900 python bench.py --gpus 2 --same-device --backend gloo --steps 6 --warmup 3 > $OUT/c3_n2.json 2> $OUT/c3_n2.err; echo "c3 n2 rc=$?"
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"
