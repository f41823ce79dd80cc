#!/bin/bash
OUT=gpurun_out/r02t30; mkdir -p $OUT
VARIANTS="head pt128 pt512" ROUNDS=2 OUT=$OUT/ab bash tools/ab_run.sh
VARIANTS="head pt128 pt512" ROUNDS=1 BENCH="--workload mu1m --no-cpu-baseline" OUT=$OUT/abmu bash tools/ab_run.sh
