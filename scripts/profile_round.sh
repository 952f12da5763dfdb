#!/bin/bash
# ncu evidence for one round (run on the GPU box via gpurun; 1 GPU, never a
# multi-rank command).  Writes into gpurun_out/; summarise into profiles/ with
# scripts/summarize_ncu.py.
#   1. launch list of the default bench command (cold-cache, serialised by
#      ncu: compare kernel shares, not absolute times)
#   2. --set full of each kernel measured alone (bench --serial: bulk-copy K1,
#      then the merge in stream order, + the scan) -> per-kernel DRAM traffic
#   3. --set full of the default pass's kernels (tile K1, follow merge); ncu
#      serialises them, so the L2 reuse of the concurrent pass is not visible
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --profile > $OUT/launches_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"forward|merge_copy|merge_scan" -s 9 -c 6 \
    -o $OUT/full_$TAG python bench.py --serial --steps 2 --warmup 3 --profile > $OUT/full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"forward_tile|merge_follow" -s 4 -c 4 \
    -o $OUT/full_${TAG}_pipe python bench.py --steps 2 --warmup 3 --profile > $OUT/full_${TAG}_pipe.log 2>&1
tail -2 $OUT/full_$TAG.log
