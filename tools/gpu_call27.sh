#!/bin/bash
# compute-sanitizer passes: memcheck over the smoke solve (every one-launch and multi-launch
# kernel it touches) and the kernel tests; racecheck + synccheck over the kernel tests
O=gpurun_out/r2c27
mkdir -p $O
CS="compute-sanitizer --print-limit 50 --error-exitcode 99"
timeout 1200 $CS --tool memcheck --leak-check no python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo "rc=$?" >> $O/memcheck_smoke.log
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ops.py -x -q -p no:cacheprovider > $O/memcheck_kernels.log 2>&1; echo "rc=$?" >> $O/memcheck_kernels.log
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > $O/racecheck_kernels.log 2>&1; echo "rc=$?" >> $O/racecheck_kernels.log
timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > $O/synccheck_kernels.log 2>&1; echo "rc=$?" >> $O/synccheck_kernels.log
for f in $O/*.log; do echo "== $f"; tail -6 $f; done
