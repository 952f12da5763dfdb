#!/bin/bash
# ncu evidence for one round (run on the GPU box via gpurun; 1 GPU, never a
# multi-rank command under --set full).  Writes into gpurun_out/; summarise
# into profiles/ with `python scripts/summarize_ncu.py TAG` (here, no GPU).
#   1. launch list of the default bench command (cold-cache, serialised by
#      ncu: compare kernel shares, not absolute times)
#   2. --set full of one launch of every data-plane kernel on configs B and A
#      (scripts/profile_kernels.py: scan, tee, bulk K1, merge, tile K1,
#      follow merge) -> per-kernel DRAM traffic keyed by config and launch size
#   3. on a box with >= 2 GPUs: NVLink tx/rx bytes of the producer's K1 in a
#      2-rank pair run (rank 1 plain, rank 0 under ncu with a metric list only)
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --profile > $OUT/launches_$TAG.log 2>&1
for C in B A D; do
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -o $OUT/full_${TAG}_$C python scripts/profile_kernels.py $C > $OUT/full_${TAG}_$C.log 2>&1
  tail -1 $OUT/full_${TAG}_$C.log
done
NGPU=$(nvidia-smi -L | wc -l)
if [ "$NGPU" -ge 2 ]; then
  PORT=$((29500 + RANDOM % 1000))
  env RANK=1 LOCAL_RANK=1 WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$PORT \
      python bench.py --gpus 2 --steps 4 --warmup 2 --k1 tile --no-e2e > $OUT/nvl_${TAG}_rank1.log 2>&1 &
  env RANK=0 LOCAL_RANK=0 WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$PORT \
      ncu --clock-control none -k regex:forward --csv --log-file $OUT/nvl_$TAG.csv \
      --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum \
      python bench.py --gpus 2 --steps 4 --warmup 2 --k1 tile --no-e2e > $OUT/nvl_${TAG}_rank0.log 2>&1
  wait
fi
