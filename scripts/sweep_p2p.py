#!/usr/bin/env python
"""Config E (BASELINE.json configs[4]): chunk-size sweep of the P2P forward at
2 / 4 / 8 GPUs of one box -- disjoint producer->consumer pairs 0->1, 2->3, ...
running concurrently, K1 pushing into the peer's slab over NVLink/NVSwitch in
each of its three peer forms (register tiles with a system-scope count per
tile; register tiles counted at gpu scope with one system-scope publish per
chunk; bulk-copy tiles) -- next to cudaMemcpyPeerAsync of the same bytes.  One process,
one stream per pair, CUDA events per pair; reports per-pair GB/s against
900 GB/s per direction (nominal) / 770 GB/s (measured peer copy,
B200_PROFILING.md) and the aggregate.  Needs >= 2 GPUs; prints a note and
exits 0 on a 1-GPU box.

  python scripts/sweep_p2p.py [--gpus 2|4|8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = [64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]


def main():
    import torch

    from paper_2603_12118_b200.fabric import DeviceFabric

    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--chunk", type=int, default=1 << 20)
    ap.add_argument("--cpu-ref", action="store_true",
                    help="also time the reference CPU forward (oracle/_ref SidecarFabric, 1 thread) per size")
    args = ap.parse_args()
    cref = None
    if args.cpu_ref:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O  # the reference CPU path, timed beside the kernel (checker library)
        cref = O.REF
    n = min(args.gpus, torch.cuda.device_count())
    if n < 2:
        print(json.dumps({"note": "config E P2P sweep needs >= 2 GPUs", "gpus": n}))
        return
    n -= n % 2
    pairs = [(2 * k, 2 * k + 1) for k in range(n // 2)]
    fab = DeviceFabric({g: 0 for g in range(n)}, {g: g for g in range(n)})
    for _, c in pairs:
        fab.slab_register(c, (256 << 20) + (1 << 20))
    src = {p: torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{p}") for p, _ in pairs}
    dstbuf = {c: torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{c}") for _, c in pairs}
    for p, _ in pairs:
        fab.synth(p, 99 + p, src[p].data_ptr(), src[p].numel())
    streams = {p: torch.cuda.Stream(device=f"cuda:{p}") for p, _ in pairs}
    torch.cuda.synchronize()
    for size in SIZES:
        reps = max(4, (1 << 30) // size)
        chunk = min(args.chunk, size)
        offs = {c: fab.slab_alloc(c, size) for _, c in pairs}
        res = {}
        forms = {"fsx_tile": {}, "fsx_gpucount": {"peer_gpu_count": True}, "fsx_bulk": {"bulk": True}}
        for impl in list(forms) + ["memcpy_peer"]:
            ev = {}
            for p, c in pairs:
                s = streams[p]
                with torch.cuda.device(p), torch.cuda.stream(s):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    for r in range(reps + 2):
                        if r == 2:
                            e0.record(s)
                        if impl in forms:
                            nch = -(-size // chunk)
                            fab.forward(p, src[p].data_ptr(), c, offs[c], size, chunk,
                                        fab.flags_alloc(c, nch), s, host_notify=False, **forms[impl])
                        else:
                            dstbuf[c][:size].copy_(src[p][:size], non_blocking=True)
                    e1.record(s)
                    ev[p] = (e0, e1)
            torch.cuda.synchronize()
            per = [size * reps / (ev[p][0].elapsed_time(ev[p][1]) * 1e-3) / 1e9 for p, _ in pairs]
            res[impl] = {"per_pair_gbs": [round(x, 1) for x in per],
                         "aggregate_gbs": round(sum(per), 1),
                         "frac_of_900": round(min(per) / 900.0, 3),
                         "frac_of_770_measured": round(min(per) / 770.0, 3)}
        for _, c in pairs:
            fab.slab_free(c, offs[c])
        if cref is not None:
            iters = max(2, min(200, (256 << 20) // size))
            secs = cref.ref_forward_bench(size, iters, 1)
            res["cpu_reference"] = {"payload_gbs": round(size * iters / secs / 1e9, 3), "threads": 1}
        print(json.dumps({"gpus": n, "pairs": len(pairs), "bytes": size, "chunk_bytes": chunk,
                          **res}), flush=True)
    fab.close()


if __name__ == "__main__":
    main()
