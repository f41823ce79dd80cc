#!/bin/bash
OUT=gpurun_out/r02t11; mkdir -p $OUT
cp ab/libprism_qagg.so paper_2605_08581_b200/libprism.so
timeout 1200 python -m pytest tests/test_device_qas.py tests/test_wave_fused.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
VARIANTS="head qagg" ROUNDS=3 OUT=$OUT/ab bash tools/ab_run.sh
