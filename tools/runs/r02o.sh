#!/bin/bash
OUT=gpurun_out/r02o; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -30 $OUT/pytest.log
python tools/dbg_global.py 1 > $OUT/dbg_g1.log 2>&1; tail -3 $OUT/dbg_g1.log
