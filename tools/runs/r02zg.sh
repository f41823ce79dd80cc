#!/bin/bash
# HEAD check: full GPU suite, smoke, one C3 bench line
OUT=gpurun_out/r02zg; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "c3 rc=$?"
