#!/bin/bash
# compute-sanitizer, third pass: racecheck over the native/one-launch loop tests and the
# operator tests; memcheck over the scale and full-size parity tests (multi-wave grids)
O=gpurun_out/r2c30
mkdir -p $O
CS="compute-sanitizer --print-limit 50 --error-exitcode 99"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_alm_native.py tests/test_gpu_admm_native.py tests/test_gpu_ops.py -x -q -p no:cacheprovider > $O/racecheck_native.log 2>&1; echo "rc=$?" >> $O/racecheck_native.log
timeout 2400 $CS --tool memcheck python -m pytest tests/test_gpu_full_size.py tests/test_gpu_scale_parity.py -x -q -p no:cacheprovider > $O/memcheck_scale.log 2>&1; echo "rc=$?" >> $O/memcheck_scale.log
for f in $O/*.log; do echo "== $f"; grep -v "^=========     \|^=========         " $f | tail -12; done
