#!/bin/bash
# launch list only (see ncu_capture.sh)
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --profile-only --no-cpu-baseline > $OUT/ncu_bench_launch.log 2>&1
tail -2 $OUT/ncu_bench_launch.log
