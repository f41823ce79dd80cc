#!/bin/bash
# one gpurun session: GPU tests, bench line, ncu launch list + one --set full capture
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
if [ -z "$NONCU" ]; then
  timeout 600 bash tools/ncu_launches.sh
  timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "timed/" --clock-control none \
    -k regex:"${KREGEX:-k_build_coop|k_protect_coop|k_propagate|k_build_keys|k_gather}" -c ${NFULL:-5} \
    -o $OUT/prof_full python bench.py --steps 1 --warmup 1 --profile-only --no-cpu-baseline > $OUT/ncu_bench_full.log 2>&1
  echo "ncu full rc=$?"
fi
ls -la $OUT
