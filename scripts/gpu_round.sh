#!/bin/bash
# One GPU-box pass of the round's evidence (run through gpurun from the repo
# root, after `python -c "import __graft_entry__ as g; g.build()"` here):
# GPU test suite, smoke, bench lines (configs B/A/D + the reference arm),
# config-E sweeps, the drop-in and C++ pass runners, and the ncu captures.
#   bash scripts/gpu_round.sh TAG
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests_$TAG.txt 2>&1; echo "pytest rc=$?" >> $O/gpu_tests_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.txt 2>&1
timeout 600 python bench.py > $O/bench_${TAG}_full.json 2> $O/bench_${TAG}.err
timeout 600 python bench.py --impl reference > $O/bench_${TAG}_reference_arm.json 2>> $O/bench_${TAG}.err
for C in A C D; do
  timeout 600 python bench.py --config $C >> $O/bench_configs_AD_$TAG.jsonl 2>> $O/bench_${TAG}.err
  timeout 600 python bench.py --config $C --impl reference >> $O/bench_reference_arm_AD_$TAG.jsonl 2>> $O/bench_${TAG}.err
done
timeout 600 python scripts/sweep_forward.py --graph --cpu-ref > $O/k1_sweep_configE_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 600 python scripts/sweep_forward.py --graph --flush > $O/k1_sweep_flush_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 600 python scripts/sweep_forward.py --graph --flush --bulk > $O/k1_sweep_flush_bulk_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 600 python scripts/sweep_forward.py --graph --form kernel > $O/k1_sweep_graph_kernel_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 600 python scripts/sweep_forward.py --graph --form auto > $O/k1_sweep_graph_auto_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 600 build/bench_fabric 4 > $O/bench_fabric_dropin_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 120 build/probe_small_path 7168 > $O/small_path_phases_$TAG.jsonl 2>> $O/bench_${TAG}.err
[ -x build/probe_k1_floor ] && timeout 120 build/probe_k1_floor > $O/k1_floor_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 600 build/bench_pass 50 > $O/bench_pass_cpp_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 600 python scripts/bench_stream.py > $O/stream_configC_$TAG.jsonl 2>> $O/bench_${TAG}.err
timeout 1800 bash scripts/profile_round.sh $TAG
rm -f $O/sanitize_summary.txt
timeout 3000 bash scripts/sanitize.sh
