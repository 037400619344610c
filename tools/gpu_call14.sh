#!/bin/bash
O=gpurun_out/r2c14
T=/tmp/ncu_r2c14
mkdir -p $O $T
for e in 1 2; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:spmm_tiled_kernelILi32ELi2ELi${e}ELi0E" -s 1 -c 1 -f -o $T/hr_epi$e \
    python tools/profile_alm.py 1e6 10 4 2 822 > $O/hr_epi$e.log 2>&1
  ncu -i $T/hr_epi$e.ncu-rep --page raw --csv > $O/hr_epi${e}_raw.csv 2>&1
  ncu -i $T/hr_epi$e.ncu-rep --page source --csv > $O/hr_epi${e}_source.csv 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  --kernel-name-base mangled -k "regex:spmm_tiled_kernelILi32ELi2ELi0ELi0E" -s 1 -c 1 -f -o $T/hr_epi0 \
  python tools/profile_alm.py 1e6 10 4 2 822 > $O/hr_epi0.log 2>&1
ncu -i $T/hr_epi0.ncu-rep --page raw --csv > $O/hr_epi0_raw.csv 2>&1
du -sh $O
