#!/bin/bash
# Evidence for profiles/<tag>/ (one GPU, under gpurun; never a multi-rank command):
#   launches.csv      : ncu launch list (gpu__time_duration, --clock-control none) of the timed C2 + C4
#                       regions of bench.py (--timed-only: no isolated passes / e2e / quality records)
#   prof_<k>.ncu-rep  : ncu --set full of the dominant kernels (-> DRAM traffic, stalls, op mix);
#                       prof_kk_* from the C4 KK run, the others from the C2 PAM run
#   digests           : tools/profile_digest.py (text only travels back)
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
B="python bench.py --timed-only --steps 2 --warmup 3 --ring-gib 0.25"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
  --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
for k in k_pam_be k_pam_fe k_pam_theta k_norm_stats k_lms_prefix; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$k -s 3 -c 1 \
    -o $O/prof_$k $B > $O/ncu_full_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_lms_seg<.bool.0" -s 1 -c 1 -o $O/prof_k_lms_seg $B > $O/ncu_full_k_lms_seg.log 2>&1
BK="python bench.py --timed-only --no-pam --steps 2 --warmup 3 --ring-gib 0.25"
for k in k_kk_s1 k_kk_s2 k_cfo_spec k_cfo_fine k_lms_final; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$k -s 6 -c 1 \
    -o $O/prof_kk_$k $BK > $O/ncu_full_kk_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_lms_seg<.bool.1" -s 4 -c 1 -o $O/prof_kk_k_lms_seg $BK > $O/ncu_full_kk_k_lms_seg.log 2>&1
python tools/profile_digest.py $O
