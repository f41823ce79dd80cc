#!/bin/bash
OUT=gpurun_out/r02t9; mkdir -p $OUT
VARIANTS="cvec povl3 povl5" ROUNDS=2 OUT=$OUT/ab bash tools/ab_run.sh
