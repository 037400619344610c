#!/bin/bash
O=gpurun_out/r2c22
T=/tmp/ncu_r2c22
mkdir -p $O $T
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lanczos_fused -c 1 -f -o $T/lz \
  python tools/g1_solve.py > $O/lz.log 2>&1
ncu -i $T/lz.ncu-rep --page raw --csv > $O/lanczos_fused_raw.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/capped_solve.py 2e5 10 > $O/capped_solve_launches.csv 2>&1
python tools/capped_solve.py 2e5 10 > $O/capped_solve_plain.txt 2>&1
du -sh $O
