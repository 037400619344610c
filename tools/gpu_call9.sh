#!/bin/bash
# round-2 measurement: tests, smoke, default bench, the bench's launch list and its top kernel under ncu
O=gpurun_out/r2c9
T=/tmp/ncu_r2c9
mkdir -p $O $T
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.txt 2>&1
tail -2 $O/gputests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
tail -c 600 $O/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python bench.py --steps 2 --warmup 1 --no-solve --no-completion --no-solver --no-cpu-baseline --no-e2e \
  > $O/bench_launches.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tiled_kernel -s 3 -c 1 -f -o $T/spmm \
  python bench.py --steps 2 --warmup 1 --no-solve --no-completion --no-solver --no-cpu-baseline --no-e2e > $O/spmm_ncu.log 2>&1
ncu -i $T/spmm.ncu-rep --page raw --csv > $O/spmm_raw.csv 2>&1
ncu -i $T/spmm.ncu-rep --page details --csv > $O/spmm_details.csv 2>&1
timeout 600 ncu --set full --clock-control none -k regex:diag_update_kernel -s 3 -c 1 -f -o $T/upd \
  python bench.py --steps 2 --warmup 1 --no-solve --no-completion --no-solver --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $T/upd.ncu-rep --page raw --csv > $O/update_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none -k regex:diag_constraint -s 3 -c 1 -f -o $T/con \
  python bench.py --steps 2 --warmup 1 --no-solve --no-completion --no-solver --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $T/con.ncu-rep --page raw --csv > $O/constraint_raw.csv 2>&1
du -sh $O
