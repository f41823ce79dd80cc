#!/bin/bash
# round-2 evidence at HEAD: full GPU suite, bench lines, reference arm, launch list, --set full
OUT=gpurun_out/r02zi; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --workload mu1m --no-cpu-baseline > $OUT/bench_mu.json 2> $OUT/bench_mu.err; echo "mu rc=$?"
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --kv-bytes 256 --no-cpu-baseline --steps 10 > $OUT/bench_c3_kv256.json 2> $OUT/bench_c3_kv256.err; echo "kv rc=$?"
timeout 900 python bench.py --workload c4 --mode serve --requests 1000000 --no-cpu-baseline > $OUT/serve_c4_1m.json 2> $OUT/serve_c4_1m.err; echo "serve rc=$?"
timeout 600 python bench.py --impl reference > $OUT/reference.json 2> $OUT/reference.err; echo "ref rc=$?"
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --profile-only --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --import-source on --nvtx --nvtx-include "timed/" --clock-control none \
    -k regex:"k_qas_small|k_propagate|k_ss_select|k_ss_sort|k_ss_filter|k_wp_create|k_tf_local" -c 7 \
    -o $OUT/prof_full python bench.py --steps 1 --warmup 3 --profile-only --no-cpu-baseline > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
ls -la $OUT
