#!/bin/bash
# compute-sanitizer, second pass: memcheck over the native loops, the sharded path and the
# golden solves; racecheck + synccheck over the smoke solve (the one-launch kernels)
O=gpurun_out/r2c28
mkdir -p $O
CS="compute-sanitizer --print-limit 50 --error-exitcode 99"
timeout 1800 $CS --tool memcheck python -m pytest tests/test_gpu_alm_native.py tests/test_gpu_admm_native.py tests/test_gpu_shard.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > $O/memcheck_native.log 2>&1; echo "rc=$?" >> $O/memcheck_native.log
timeout 1800 $CS --tool memcheck python -m pytest tests/test_gpu_solve.py -x -q -p no:cacheprovider > $O/memcheck_solve.log 2>&1; echo "rc=$?" >> $O/memcheck_solve.log
timeout 1500 $CS --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $O/racecheck_smoke.log 2>&1; echo "rc=$?" >> $O/racecheck_smoke.log
timeout 900 $CS --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $O/synccheck_smoke.log 2>&1; echo "rc=$?" >> $O/synccheck_smoke.log
for f in $O/*.log; do echo "== $f"; tail -6 $f; done
