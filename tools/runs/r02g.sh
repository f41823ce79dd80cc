#!/bin/bash
OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_device_dart.py tests/test_wave_fused.py tests/test_parity_at_scale.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 600 python tools/diag_wave.py --steps 3 > $OUT/diag.log 2>&1; echo "diag rc=$?"
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?"
OUT=$OUT timeout 900 bash tools/ncu_launches.sh
