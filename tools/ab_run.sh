#!/bin/bash
# same-box A/B: alternate the variants in ab/ under the same bench command
# usage: VARIANTS="base new" ROUNDS=3 BENCH="--no-cpu-baseline" bash tools/ab_run.sh
OUT=${OUT:-gpurun_out/ab}; mkdir -p $OUT
cp paper_2605_08581_b200/libprism.so $OUT/../libprism_orig.so 2>/dev/null
for r in $(seq 1 ${ROUNDS:-3}); do
  for v in $VARIANTS; do
    cp ab/libprism_$v.so paper_2605_08581_b200/libprism.so
    timeout 600 python bench.py ${BENCH:---no-cpu-baseline} > $OUT/${v}_$r.json 2> $OUT/${v}_$r.err
    python -c "import json,sys;d=json.load(open('$OUT/${v}_$r.json'));print('$v', $r, round(d['ms_per_step'],4), round(d['value']/1e6,3), 'e2e', round((d.get('e2e') or {}).get('value', 0)/1e6, 3), d.get('parity',{}) and d['parity'].get('identical'))"
  done
done
