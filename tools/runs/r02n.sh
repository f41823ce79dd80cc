#!/bin/bash
OUT=gpurun_out/r02n; mkdir -p $OUT
timeout 900 python -m pytest tests/test_wave_fused.py tests/test_global_demand.py tests/test_kv_payload.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --workload mu1m --no-cpu-baseline > $OUT/bench_mu.json 2> $OUT/bench_mu.err; echo "bench mu rc=$?"
