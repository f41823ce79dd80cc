#!/bin/bash
OUT=gpurun_out/r02j; mkdir -p $OUT
timeout 900 python bench.py --workload c4 --mode serve --requests 1000000 --parity-requests 20000 > $OUT/serve1m.json 2> $OUT/serve1m.err; echo "serve1m rc=$?"
tail -c 2500 $OUT/serve1m.json; tail -5 $OUT/serve1m.err
timeout 900 python bench.py --workload c4 --mode serve --requests 1000000 --parity-requests 10000 --gpus 2 --same-device --backend gloo > $OUT/serve1m_n2.json 2> $OUT/serve1m_n2.err; echo "n2 rc=$?"
tail -c 1500 $OUT/serve1m_n2.json; tail -5 $OUT/serve1m_n2.err
