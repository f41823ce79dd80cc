#!/bin/bash
OUT=gpurun_out/r02i; mkdir -p $OUT
timeout 900 python -m pytest tests/test_serve.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -40 $OUT/pytest.log
