#!/bin/bash
# Evidence for profiles/<tag>/ (one GPU, under gpurun):
#   bench.json        : the default bench line (with the CPU oracle baseline)
#   launches.csv      : ncu launch list (gpu__time_duration, --clock-control none) of a short bench
#   prof_<k>.ncu-rep  : ncu --set full of the dominant kernels (-> dram traffic, stalls, op mix)
TAG=${1:-r01}
mkdir -p gpurun_out/$TAG
timeout 400 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
B="python bench.py --steps 2 --warmup 3 --no-cpu --kk-steps 1 --ring-gib 0.5 --no-c5 --no-c3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
  --log-file gpurun_out/$TAG/launches.csv $B > gpurun_out/$TAG/ncu_launch.log 2>&1
BP="python bench.py --steps 2 --warmup 3 --no-cpu --no-kk --ring-gib 0.25 --no-c5 --no-c3"
for k in k_lms_seg k_pam_be k_pam_fe k_norm_stats k_norm_apply k_lms_prefix; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$k -s 3 -c 1 \
    -o gpurun_out/$TAG/prof_$k $BP > gpurun_out/$TAG/ncu_full_$k.log 2>&1
done
BK="python bench.py --steps 1 --warmup 3 --no-cpu --kk-steps 2 --ring-gib 0.25 --no-c5 --no-c3"
for k in k_kk_s1 k_kk_s2 k_cfo_spec k_cfo_fine k_kk_zprime k_lms_final; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$k -s 6 -c 1 \
    -o gpurun_out/$TAG/prof_kk_$k $BK > gpurun_out/$TAG/ncu_full_kk_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_lms_seg<.bool.1" -s 4 -c 1 -o gpurun_out/$TAG/prof_kk_k_lms_seg $BK \
  > gpurun_out/$TAG/ncu_full_kk_k_lms_seg.log 2>&1
python tools/profile_digest.py gpurun_out/$TAG
