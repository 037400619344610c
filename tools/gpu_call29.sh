#!/bin/bash
# racecheck of the one-launch ALM after the loop-top barrier; the fused-path tests; the
# full-size (n = 1e7) parity tests; the G1 solve time
O=gpurun_out/r2c29
mkdir -p $O
CS="compute-sanitizer --print-limit 50 --error-exitcode 99"
timeout 1500 $CS --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $O/racecheck_smoke.log 2>&1; echo "rc=$?" >> $O/racecheck_smoke.log
timeout 900 python -m pytest tests/test_gpu_full_size.py -x -q -p no:cacheprovider --durations=5 > $O/full_size.log 2>&1; echo "rc=$?" >> $O/full_size.log
timeout 900 python -m pytest tests/test_gpu_alm_native.py tests/test_gpu_solve.py -x -q -p no:cacheprovider > $O/fused_tests.log 2>&1; echo "rc=$?" >> $O/fused_tests.log
timeout 600 python tools/g1_solve.py > $O/g1.log 2>&1
for f in $O/*.log; do echo "== $f"; tail -8 $f; done
