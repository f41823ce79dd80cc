#!/bin/bash
OUT=gpurun_out/r02t29; mkdir -p $OUT
cp ab/libprism_pm4.so paper_2605_08581_b200/libprism.so
timeout 1200 python -m pytest tests/test_wave_fused.py tests/test_parity_at_scale.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
VARIANTS="head pm1 pm2 pm4" ROUNDS=2 OUT=$OUT/ab bash tools/ab_run.sh
