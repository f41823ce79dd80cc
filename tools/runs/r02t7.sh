#!/bin/bash
OUT=gpurun_out/r02t7; mkdir -p $OUT
cp ab/libprism_cvec.so paper_2605_08581_b200/libprism.so
timeout 1200 python -m pytest tests/test_wave_fused.py tests/test_parity_at_scale.py tests/test_long_paths.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
cp ab/libprism_s512.so paper_2605_08581_b200/libprism.so
timeout 1200 python -m pytest tests/test_parity_at_scale.py -m gpu -x -q > $OUT/pytest2.log 2>&1; echo "pytest2 rc=$?"; tail -2 $OUT/pytest2.log
VARIANTS="runsort cvec s512" ROUNDS=3 OUT=$OUT/ab bash tools/ab_run.sh
