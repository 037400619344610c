#!/bin/bash
# validation of the per-file-compiled library: GPU tests, smoke, default bench line
O=gpurun_out/r2c26
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
tail -3 $O/pytest.log; tail -2 $O/smoke.log; tail -c 1500 $O/bench.log
