#!/bin/bash
OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_wave_fused.py -m gpu -x -q -k "inflight or step_host" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -30 $OUT/pytest.log
