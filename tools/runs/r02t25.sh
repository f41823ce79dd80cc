#!/bin/bash
OUT=gpurun_out/r02t25; mkdir -p $OUT
VARIANTS="head prop6 ev4 tf8 ds592" ROUNDS=2 OUT=$OUT/ab bash tools/ab_run.sh
