#!/bin/bash
# One GPU-box pass: bench line, launch list, one full ncu capture of the top kernels, smoke.
set -x
mkdir -p gpurun_out
TAG=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'spmm|constraint|diag|lincomb|sddmm|assemble|basis' -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'spmm|constraint|diag_update' -s 3 -c 3 -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; tail -3 gpurun_out/ncu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
# solver iteration kernels at n=1e7 (ALM inner iterations + ADMM steps): launch list
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'spmm|constraint|diag|lincomb|cg_|assemble' -s 30 -c 150 --csv --log-file gpurun_out/launches_solver_$TAG.csv python tools/profile_alm.py 1e7 6 12 4 > /dev/null 2>&1
timeout 600 python tools/profile_alm.py 1e7 6 20 5 2>&1 | tail -2
