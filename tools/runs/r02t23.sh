#!/bin/bash
OUT=gpurun_out/r02t23; mkdir -p $OUT
cp ab/libprism_samp.so paper_2605_08581_b200/libprism.so
timeout 1200 python -m pytest tests/test_parity_at_scale.py tests/test_wave_fused.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest samp rc=$?"; tail -1 $OUT/pytest.log
VARIANTS="head samp bmax tffin" ROUNDS=2 OUT=$OUT/ab bash tools/ab_run.sh
VARIANTS="head samp" ROUNDS=1 BENCH="--workload mu1m --no-cpu-baseline" OUT=$OUT/abmu bash tools/ab_run.sh
