#!/bin/bash
O=gpurun_out/r2c7
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.txt 2>&1
tail -3 $O/gputests.txt
timeout 300 python tools/profile_alm.py 1e7 6 20 6 > $O/alm_1e7_plain.txt 2>&1
cat $O/alm_1e7_plain.txt | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  python tools/profile_alm.py 1e7 6 12 4 > $O/alm_1e7_launches.csv 2>&1
timeout 300 python tools/profile_alm.py 1e6 10 20 6 822 > $O/highrank_plain.txt 2>&1
cat $O/highrank_plain.txt | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  python tools/profile_alm.py 1e6 10 6 3 822 > $O/highrank_launches.csv 2>&1
