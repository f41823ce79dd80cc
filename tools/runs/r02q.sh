#!/bin/bash
OUT=gpurun_out/r02q; mkdir -p $OUT
timeout 600 python tools/diag_wave.py --steps 3 > $OUT/diag.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --workload mu1m --no-cpu-baseline > $OUT/bench_mu.json 2> $OUT/bench_mu.err; echo "bench mu rc=$?"
timeout 900 python -m pytest tests/test_wave_fused.py tests/test_parity_at_scale.py -m gpu -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
