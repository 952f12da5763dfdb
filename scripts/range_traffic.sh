#!/bin/bash
# DRAM traffic and L2 read hits of ONE whole pass (both kernels, concurrent as
# in the timed run) via ncu range replay: bench.py --profile with
# FSX_PROFILER_RANGE=1 brackets the last pass with cudaProfilerStart/Stop.
# Unlike kernel replay, range replay keeps the colocated pass's K1 and merge
# concurrent, so its counters are the pass's own.  Run on the GPU box:
#   bash scripts/range_traffic.sh TAG [extra bench args...]
# -> gpurun_out/range_TAG.csv
set -u
TAG=$1; shift
mkdir -p gpurun_out
FSX_PROFILER_RANGE=1 ncu --replay-mode ${FSX_RANGE_MODE:-range} --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_write.sum \
  --csv --log-file gpurun_out/range_$TAG.csv python bench.py --steps 3 --warmup 3 --profile "$@" \
  > gpurun_out/range_$TAG.log 2>&1
echo "$TAG rc=$?"
