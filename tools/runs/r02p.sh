#!/bin/bash
# round-2 evidence session: full GPU tests, the default bench line, mu1M, the ncu launch list of C3 and --set full of its top kernels
OUT=gpurun_out/r02p; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --workload mu1m --no-cpu-baseline > $OUT/bench_mu.json 2> $OUT/bench_mu.err; echo "bench mu rc=$?"
OUT=$OUT timeout 900 bash tools/ncu_launches.sh
timeout 1200 ncu --set full --import-source on --nvtx --nvtx-include "timed/" --clock-control none \
    -k regex:"k_qas_small|k_propagate|k_build_coop|k_ss_sort|k_ss_select|k_wp_create|k_prematch|k_release_par|k_tf_scan" -c 9 \
    -o $OUT/prof_full python bench.py --steps 1 --warmup 1 --profile-only --no-cpu-baseline > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
