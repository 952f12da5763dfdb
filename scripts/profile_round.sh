#!/bin/bash
# ncu evidence for one round (run on the GPU box via gpurun; 1 GPU, never a
# multi-rank command).  Writes into gpurun_out/; summarise into profiles/ with
# scripts/summarize_ncu.py.
#   1. launch list of the bench command (cold-cache, serialised: compare shares)
#   2. one --set full capture of each hot kernel (forward, merge copy, scan)
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --profile > $OUT/launches_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"forward|merge_copy|merge_scan" -s 9 -c 6 \
    -o $OUT/full_$TAG python bench.py --steps 2 --warmup 3 --profile > $OUT/full_$TAG.log 2>&1
tail -2 $OUT/full_$TAG.log
