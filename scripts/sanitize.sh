#!/bin/bash
# compute-sanitizer over the small GPU parity cases (memcheck /
# racecheck / synccheck on K1 and K3).  Run on the GPU box; summaries land in
# gpurun_out/sanitize_*.txt.
set -u
OUT=gpurun_out
mkdir -p $OUT
SEL='forward_single_shot and (0 or 1 or 7 or 256 or 4096) or forward_chunked_flags or unaligned or merge_edge_cases or validation or early_start or fused_digest or batch_mixed or small_put or colocated or forward_place or graph_replay or host_span'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 3 \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -x -q -p no:cacheprovider \
      -k "$SEL or hidden_state_stream or ring_depth" > $OUT/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a $OUT/sanitize_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_$tool.txt | tail -3 | tee -a $OUT/sanitize_summary.txt
done
# the non-default kernel instances (persistent-warp K1 + TMA bulk-copy merge;
# bulk-copy K1 + bulk-copy run merge for early start)
for ALT in "FSX_FWD_VARIANT=0 FSX_MERGE_TMA=1" "FSX_FWD_VARIANT=5 FSX_MERGE_STREAM=2" "FSX_MERGE_STREAM=3"; do
  env $ALT timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 \
      --error-exitcode 3 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
      -k "$SEL" > $OUT/sanitize_memcheck_alt.txt 2>&1
  echo "memcheck ($ALT) rc=$?" | tee -a $OUT/sanitize_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_memcheck_alt.txt | tail -3 | tee -a $OUT/sanitize_summary.txt
done
