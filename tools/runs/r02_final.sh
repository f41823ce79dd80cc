#!/bin/bash
# round-2 evidence: GPU tests, every bench line, ncu launch list + --set full of the top kernels, memcheck
OUT=gpurun_out/r02f; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --workload mu1m > $OUT/bench_mu1m.json 2> $OUT/bench_mu1m.err
timeout 900 python bench.py --workload c5 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 1200 python bench.py --workload c4 --mode serve > $OUT/serve_c4_10m.json 2> $OUT/serve_c4_10m.err
timeout 900 python bench.py --workload c2 --mode serve > $OUT/serve_c2.json 2> $OUT/serve_c2.err
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $OUT/reference.json 2> $OUT/reference.err
OUT=$OUT timeout 900 bash tools/ncu_launches.sh
timeout 1200 ncu --set full --import-source on --nvtx --nvtx-include "timed/" --clock-control none \
    -k regex:"k_qas_small|k_propagate|k_ss_select|k_ss_sort|k_ss_filter|k_wp_create|k_prematch|k_release_par|k_wp_hits" -c 9 \
    -o $OUT/prof_full python bench.py --steps 1 --warmup 1 --profile-only --no-cpu-baseline > $OUT/ncu_full.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_wave_fused.py tests/test_serve.py tests/test_kv_payload.py -m gpu -q -x -k "not sampled_selection_at_scale" > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck.log
ls -la $OUT
