#!/bin/bash
OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kv_payload.py tests/test_sglang_adapter.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
timeout 900 python bench.py --kv-bytes 256 --no-cpu-baseline --steps 10 > $OUT/c3_kv256.json 2> $OUT/c3_kv256.err; echo "c3 kv rc=$?"
timeout 900 python bench.py --workload c5 --kv-bytes 1024 --no-cpu-baseline --steps 10 > $OUT/c5_kv1k.json 2> $OUT/c5_kv1k.err; echo "c5 kv rc=$?"
