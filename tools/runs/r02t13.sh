#!/bin/bash
OUT=gpurun_out/r02t13; mkdir -p $OUT
cp ab/libprism_tfw.so paper_2605_08581_b200/libprism.so
timeout 1500 python -m pytest tests/test_wave_fused.py tests/test_device_dart.py tests/test_parity_at_scale.py tests/test_global_demand.py tests/test_serve.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
VARIANTS="head tfw" ROUNDS=3 OUT=$OUT/ab bash tools/ab_run.sh
cp ab/libprism_trace.so paper_2605_08581_b200/libprism.so
PRISM_TRACE_OUT=$OUT/trace_c3.json timeout 600 python bench.py --no-cpu-baseline --steps 10 > $OUT/bench_trace.json 2> $OUT/bench_trace.err; echo "trace rc=$?"
python tools/trace_sum.py $OUT/trace_c3.json > $OUT/trace_c3.txt; head -20 $OUT/trace_c3.txt
