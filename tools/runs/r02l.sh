#!/bin/bash
OUT=gpurun_out/r02l; mkdir -p $OUT
timeout 900 python bench.py --workload c5 --steps 10 > $OUT/c5.json 2> $OUT/c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --workload c5 --steps 10 --gpus 2 --same-device --backend gloo > $OUT/c5_n2.json 2> $OUT/c5_n2.err; echo "c5 n2 rc=$?"
timeout 1200 python bench.py --workload c4 --mode serve > $OUT/c4serve10m.json 2> $OUT/c4serve10m.err; echo "c4 10M rc=$?"
