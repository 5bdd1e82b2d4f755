#!/bin/bash
# ncu --set full of the KK equaliser kernel of the timed C4 region, kept as .ncu-rep (gpurun_out), plus
# per-CUDA-line stall digest.
TAG=${1:-lms}
O=gpurun_out/$TAG
mkdir -p $O
BK="python bench.py --timed-only --no-pam --steps 2 --warmup 3 --ring-gib 0.25"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_lms_seg<.bool.1" -s 4 -c 1 -o $O/prof_kk_k_lms_seg $BK > $O/ncu.log 2>&1
python tools/ncu_lines_cuda.py $O/prof_kk_k_lms_seg.ncu-rep 60 > $O/lines.txt 2> $O/lines.err
ncu -i $O/prof_kk_k_lms_seg.ncu-rep --page source --csv --print-source cuda,sass 2>&1 | head -5 > $O/head.csv
