#!/bin/bash
OUT=gpurun_out/r02t28; mkdir -p $OUT
cp ab/libprism_pc1.so paper_2605_08581_b200/libprism.so
timeout 1500 python -m pytest tests/test_device_dart.py tests/test_wave_fused.py tests/test_parity_at_scale.py tests/test_serve.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
VARIANTS="head pc1" ROUNDS=3 OUT=$OUT/ab bash tools/ab_run.sh
VARIANTS="head pc1" ROUNDS=1 BENCH="--workload mu1m --no-cpu-baseline" OUT=$OUT/abmu bash tools/ab_run.sh
VARIANTS="head pc1" ROUNDS=1 BENCH="--workload c5 --no-cpu-baseline" OUT=$OUT/abc5 bash tools/ab_run.sh
