#!/bin/bash
# ncu --set full of ONE kernel (regex $2) of the timed C4 region, report kept in gpurun_out/$1 (fetched back),
# plus the per-CUDA-line stall digest. Usage: bash tools/ncu_one.sh <tag> <kernel-regex> [skip]
TAG=$1; K=$2; SKIP=${3:-6}
O=gpurun_out/$TAG
mkdir -p $O
BK="python bench.py --timed-only --no-pam --steps 2 --warmup 3 --ring-gib 0.25 $BENCH_EXTRA"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$K" -s $SKIP -c 1 -o $O/prof $BK > $O/ncu.log 2>&1
python tools/ncu_lines_cuda.py $O/prof.ncu-rep 60 > $O/lines.txt 2> $O/lines.err
