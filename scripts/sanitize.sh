#!/bin/bash
# compute-sanitizer over the small GPU parity cases (memcheck /
# racecheck / synccheck on K1 and K3).  Run on the GPU box; summaries land in
# gpurun_out/sanitize_*.txt.
set -u
OUT=gpurun_out
mkdir -p $OUT
SEL='forward_single_shot and (0 or 1 or 7 or 256 or 4096) or forward_chunked_flags or unaligned or merge_edge_cases or validation or early_start or fused_digest or batch_mixed or small_put or small_lane or host_digest or tee or colocated or forward_place or graph or host_span'
# racecheck skips lane_kernel: its poller and worker warps hand descriptors
# over through shared memory with fence.cta + volatile flag release/acquire
# pairs (fsx_kernels.cu, small-message lane), a synchronisation racecheck does
# not model (it reports every such hand-over as a hazard); the lane runs under
# memcheck and synccheck like every other kernel
for tool in memcheck racecheck synccheck; do
  EXCL=""
  [ $tool = racecheck ] && EXCL="--kernel-name-exclude kns=lane_kernel"
  timeout 1500 compute-sanitizer --tool $tool $EXCL --print-limit 20 --error-exitcode 3 \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -x -q -p no:cacheprovider \
      -k "$SEL or hidden_state_stream or ring_depth" > $OUT/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a $OUT/sanitize_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_$tool.txt | tail -3 | tee -a $OUT/sanitize_summary.txt
done
# the bulk-copy K1 and the pair protocol across processes (IPC) under memcheck
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 3 --target-processes all \
    python -m pytest tests/test_gpu_pairs.py -x -q -p no:cacheprovider -k "gpucount or bulk" \
    > $OUT/sanitize_memcheck_pairs.txt 2>&1
echo "memcheck (pairs, IPC) rc=$?" | tee -a $OUT/sanitize_summary.txt
grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_memcheck_pairs.txt | tail -3 | tee -a $OUT/sanitize_summary.txt
