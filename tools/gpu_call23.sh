#!/bin/bash
O=gpurun_out/r2c23
T=/tmp/ncu_r2c23
mkdir -p $O $T
for k in diag_cg_apply_kernel diag_cg_step_kernel diag_step_end_rows_kernel lincomb_kernel; do
  timeout 400 ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -f -o $T/$k \
    python tools/profile_alm.py 1e7 6 6 6 > $O/$k.log 2>&1
  ncu -i $T/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>&1
done
for k in basis_project_kernel basis_subtract_kernel; do
  timeout 400 ncu --set full --clock-control none -k regex:$k -s 200 -c 1 -f -o $T/$k \
    python tools/capped_solve.py 1e6 10 > $O/$k.log 2>&1
  ncu -i $T/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>&1
done
du -sh $O
