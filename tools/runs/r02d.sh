#!/bin/bash
# round-2 session baseline: GPU tests, C3 + mu1M bench lines, C3 launch list, --set full of the QAS kernels
OUT=gpurun_out/r02d; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --workload mu1m --no-cpu-baseline > $OUT/bench_mu.json 2> $OUT/bench_mu.err; echo "bench mu rc=$?"
OUT=$OUT timeout 900 bash tools/ncu_launches.sh
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "timed/" --clock-control none \
    -k regex:"k_qas|q_" -c 8 -o $OUT/prof_full python bench.py --steps 1 --warmup 1 --profile-only --no-cpu-baseline > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
ls -la $OUT
