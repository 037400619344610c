#!/bin/bash
# round-2 profiling call: gather probe, completion kernels and one-launch kernels under ncu, default bench.
# Full-set reports stay in /tmp on the box (gpurun_out is capped at 64 MiB); their raw-page
# CSV exports come back.
O=gpurun_out/r2
T=/tmp/ncu_r2
mkdir -p $O $T
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
if [ "$1" == "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.txt 2>&1
  tail -5 $O/gputests.txt
fi
./tools/micro/gather_probe > $O/gather_plain.txt 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_op_read.sum --csv \
  ./tools/micro/gather_probe > $O/gather_ncu.csv 2>&1
for k in constraint_kernel single_entry_apply_kernel assemble_kernel spmm_tiled_kernel; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f -o $T/completion_$k \
    python tools/probe_completion.py 1.25e6 1.25e6 2.5e7 > $O/completion_ncu_$k.log 2>&1
  ncu -i $T/completion_$k.ncu-rep --page raw --csv > $O/completion_${k}_raw.csv 2>&1
  ncu -i $T/completion_$k.ncu-rep --page details --csv > $O/completion_${k}_details.csv 2>&1
done
for k in alm_fused_kernel admm_step_fused_kernel lanczos_fused_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o $T/fused_$k \
    python tools/g1_solve.py > $O/fused_ncu_$k.log 2>&1
  ncu -i $T/fused_$k.ncu-rep --page raw --csv > $O/fused_${k}_raw.csv 2>&1
  ncu -i $T/fused_$k.ncu-rep --page details --csv > $O/fused_${k}_details.csv 2>&1
done
timeout 300 python tools/profile_alm.py 1e6 10 20 6 822 > $O/highrank_plain.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  python tools/profile_alm.py 1e6 10 6 3 822 > $O/highrank_launches.csv 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
tail -3 $O/bench.err
du -sh $O
