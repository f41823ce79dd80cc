#!/bin/bash
# ncu evidence for one timed bench step (run under gpurun on one GPU).
#   1. launch list: every kernel in the NVTX "timed" range with its duration
#   2. --set full of the top hand-written kernels of one wave (-lineinfo build)
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --profile-only --no-cpu-baseline > $OUT/ncu_bench_launch.log 2>&1
ncu --set full --import-source on --nvtx --nvtx-include "timed/" --clock-control none \
    -k regex:"${KREGEX:-k_build_keys|k_propagate|k_gather|k_prot_gather|k_wp_create|k_wp_touch|k_wp_plan|k_prematch}" -c ${NFULL:-10} \
    -o $OUT/prof_full python bench.py --steps 1 --warmup 1 --profile-only --no-cpu-baseline > $OUT/ncu_bench_full.log 2>&1
ls -la $OUT
