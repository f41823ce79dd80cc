#!/bin/bash
OUT=gpurun_out/r02k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_global_demand.py tests/test_wave_fused.py tests/test_parity_at_scale.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -40 $OUT/pytest.log
