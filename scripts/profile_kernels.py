"""One launch of each data-plane kernel on a config's batch, bracketed by
cudaProfilerStart/Stop, for `ncu --profile-from-start off --set full`
(scripts/profile_round.sh).  Warm-up launches run before the range.  Writes
gpurun_out/profile_kernels_<config>.json: per kernel, the algorithmic bytes
of the launch as bench.py counts them, so scripts/summarize_ncu.py can key
the DRAM traffic by (config, kernel, launch size).

  python scripts/profile_kernels.py B
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_12118_b200 import _native as N  # noqa: E402
from paper_2603_12118_b200 import trace as T  # noqa: E402
from paper_2603_12118_b200.dataplane import DataPlaneBatch  # noqa: E402
from paper_2603_12118_b200.fabric import DeviceFabric  # noqa: E402

CHUNK = {"A": None, "B": 1024, "D": 1024}


def main(config: str) -> None:
    rules = T.RULES[config]
    reqs = T.config_requests(config)
    lay = T.layout(reqs, rules.row_bytes)
    P, rows = lay.payload_bytes, lay.total_item_rows
    fab = DeviceFabric({0: 0, 1: 0}, {0: 0, 1: 0})
    fab.slab_register(1, max(1 << 30, 2 * P))
    b = DataPlaneBatch(fab, reqs, rules, 0, 1, chunk_rows=CHUNK[config])
    b.synth_inputs()
    s = torch.cuda.Stream()

    def once():
        assert b.alloc()
        b.scan(s)                                    # merge_scan_kernel
        b.tee(s, mode=N.MERGE_COPY_ONLY)             # merge_tee_kernel
        b.release()
        assert b.alloc()
        b.forward(s, host_notify=False, bulk=True)   # forward_tma_kernel
        b.merge(s, mode=N.MERGE_COPY_ONLY)           # merge_copy_kernel
        b.release()
        assert b.alloc()
        b.forward(s, host_notify=False, tile=True)   # forward_tile_kernel
        b.merge(s, early_start=True, mode=N.MERGE_COPY_ONLY)  # merge_follow_kernel (flags set)
        b.release()

    with torch.cuda.stream(s):
        for _ in range(3):
            once()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        once()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    out = {"config": config, "payload": P, "placeholder_rows": rows,
           "alg_bytes": {"merge_tee_kernel": 3 * P + 4 * rows, "forward_tma_kernel": 2 * P,
                         "forward_tile_kernel": 2 * P, "merge_copy_kernel": 2 * P + 4 * rows,
                         "merge_follow_kernel": 2 * P + 4 * rows,
                         "merge_scan_kernel": 4 * lay.total_rows + 4 * rows}}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"profile_kernels_{config}.json"), "w") as fh:
        json.dump(out, fh)
    print(json.dumps(out))
    fab.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "B")
