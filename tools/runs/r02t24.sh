#!/bin/bash
OUT=gpurun_out/r02t24; mkdir -p $OUT
VARIANTS="head fin1k sl128 sl512" ROUNDS=2 OUT=$OUT/ab bash tools/ab_run.sh
