#!/bin/bash
OUT=gpurun_out/r02c5; mkdir -p $OUT
VARIANTS="base head" ROUNDS=2 BENCH="--workload c5 --no-cpu-baseline" OUT=$OUT/ab bash tools/ab_run.sh
VARIANTS="base head" ROUNDS=1 BENCH="--workload mu1m --no-cpu-baseline" OUT=$OUT/abmu bash tools/ab_run.sh
