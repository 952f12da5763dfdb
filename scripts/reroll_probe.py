"""Diagnostic (profiles/colocated_bimodality_r01k.md): run bench.py's N=1
config-B measurement twice in ONE process -- the second with fresh fabric,
slab and batch allocations -- to see whether the colocated pass's slow mode
belongs to the process or to its allocations.  Prints both JSON lines."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

sys.argv = [sys.argv[0], "--no-e2e", "--no-cpu-baseline"] + sys.argv[1:]
args = bench.parse()
bench.CONFIG = args.config
bench.REQUESTS = bench.CONFIGS[bench.CONFIG]["requests"]
bench.CHUNK_ROWS = bench.CONFIGS[bench.CONFIG]["chunk_rows"]
if args.requests is None:
    args.requests = bench.REQUESTS
for _ in range(3):
    bench.run_single(args)
    args.serial = False
