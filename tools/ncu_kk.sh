#!/bin/bash
# ncu --set full of the KK (C4) kernels of the timed region only (bench.py --timed-only --no-pam),
# one launch each, then the text digest (tools/profile_digest.py). Under gpurun, one GPU.
TAG=${1:-kk}
O=gpurun_out/$TAG
mkdir -p $O
BK="python bench.py --timed-only --no-pam --steps 2 --warmup 3 --ring-gib 0.25"
for k in ${KERNELS:-k_kk_s1 k_kk_s2 k_cfo_spec}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$k -s 6 -c 1 \
    -o $O/prof_kk_$k $BK > $O/ncu_full_kk_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_lms_seg<.bool.1" -s 4 -c 1 -o $O/prof_kk_k_lms_seg $BK > $O/ncu_full_kk_k_lms_seg.log 2>&1
python tools/profile_digest.py $O
