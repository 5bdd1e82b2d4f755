#!/bin/bash
# ncu evidence for profiles/ (run under gpurun on one GPU; never a multi-rank command).
#  1) launch list of librx kernels in a short bench (gpu__time_duration; cold-cache, serialised)
#  2) --set full captures of selected kernels (args: kernel names)
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-kk --no-cpu --ring-gib 0.25"
BK="python bench.py --steps 1 --warmup 3 --kk-steps 1 --no-cpu --ring-gib 0.25"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
  --log-file gpurun_out/launches_pam.csv $B > gpurun_out/ncu_launch_pam.log 2>&1
if [ -n "$KK" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
  --log-file gpurun_out/launches_all.csv $BK > gpurun_out/ncu_launch_all.log 2>&1
fi
for k in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-20} -c 1 \
    -o gpurun_out/prof_$k $B > gpurun_out/ncu_full_$k.log 2>&1
done
