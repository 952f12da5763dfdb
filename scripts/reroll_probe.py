"""Diagnostic (profiles/colocated_bimodality_r01k.md): run bench.py's N=1
config-B measurement several times in ONE process -- each with fresh fabric,
slab and batch allocations -- and log where the slab and the batch buffers
landed next to whether the colocated pass came up fast or slow."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_12118_b200 import dataplane as D  # noqa: E402

sys.argv = [sys.argv[0], "--no-e2e", "--no-cpu-baseline"] + sys.argv[1:]
args = bench.parse()
bench.CONFIG = args.config
bench.REQUESTS = bench.CONFIGS[bench.CONFIG]["requests"]
bench.CHUNK_ROWS = bench.CONFIGS[bench.CONFIG]["chunk_rows"]
if args.requests is None:
    args.requests = bench.REQUESTS
seen = []
_init = D.DataPlaneBatch.__init__


def _logged(self, fab, *a, **k):
    _init(self, fab, *a, **k)
    seen.append({"slab": hex(fab.slab_ptr(1, 0)), "src": hex(self.src_buf.data_ptr()),
                 "embeds": hex(self.embeds.data_ptr())})


D.DataPlaneBatch.__init__ = _logged
bench.DataPlaneBatch = D.DataPlaneBatch
runs = int(os.environ.get("REROLL_RUNS", "3"))
for _ in range(runs):
    n0 = len(seen)
    import io
    import contextlib
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        bench.run_single(args)
    line = json.loads([l for l in buf.getvalue().splitlines() if l.startswith("{")][-1])
    args.serial = False
    p = line["pass_schedule"]["probe"]
    print(json.dumps({"value": line["value"], "pipelined_ms": p["pipelined_ms"], "serial_ms": p["serial_ms"],
                      "buffers": seen[n0]}), flush=True)
