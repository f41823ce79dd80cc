#!/bin/bash
# commit-chain fusions (plan+levels, conflicts in the cut verdict, label reset in alloc, finalize in the sweep)
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_wave_fused.py tests/test_parity_at_scale.py tests/test_serve.py tests/test_global_demand.py tests/test_long_paths.py tests/test_device_dart.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3_$i.json 2> $OUT/bench_c3_$i.err; echo "c3 rc=$?"; done
timeout 900 python bench.py --workload mu1m --no-cpu-baseline > $OUT/bench_mu.json 2> $OUT/bench_mu.err; echo "mu rc=$?"
