#!/bin/bash
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_device_qas.py tests/test_wave_fused.py tests/test_serve.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
timeout 900 python bench.py --workload c2 --mode serve > $OUT/c2.json 2> $OUT/c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "c3 rc=$?"
