#!/usr/bin/env python
"""K1 sweep on one B200 (intra-device forward, HBM-bound, 2 x payload bytes):
chunk-size sweep of BASELINE config E plus the config-B video item, timed with
CUDA events on the launching stream.  Prints one JSON line per size; compares
with cudaMemcpyAsync D2D (torch copy_) of the same bytes.

  --graph   capture the repetitions of both arms in a CUDA graph and time the
            replay: kernel throughput without the per-call host path (which
            dominates below ~16 MiB when each call goes through Python).
  --flush   (with --graph) write a 256 MiB buffer before every repetition so
            each copy reads its source from HBM, not L2; the flush-only graph
            is timed too and subtracted."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import argparse

    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--bulk", action="store_true", help="bulk-copy K1 tiles (FSX_FWD_BULK)")
    ap.add_argument("--form", choices=["auto", "kernel", "dma"], default="auto",
                    help="auto: the library's choice (copy-engine form for small local transfers); "
                         "kernel: always K1 (FSX_FWD_KERNEL); dma: always the copy-engine form")
    ap.add_argument("--flush", action="store_true", help="L2 flush before every repetition (--graph)")
    ap.add_argument("--cpu-ref", action="store_true",
                    help="also time the reference CPU forward (oracle/_ref SidecarFabric, 1 thread) per size")
    args = ap.parse_args()
    cref = None
    if args.cpu_ref:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O  # the reference CPU path, timed beside the kernel (checker library)
        cref = O.REF

    from paper_2603_12118_b200.fabric import DeviceFabric

    dma = {"auto": None, "kernel": False, "dma": True}[args.form]
    sizes = [64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]
    fab = DeviceFabric({0: 0, 1: 0}, {0: 0, 1: 0})
    fab.slab_register(1, 1 << 30)
    s = torch.cuda.Stream()
    src = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fab.synth(0, 1234, src.data_ptr(), src.numel())
    ref = torch.empty_like(src)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.flush else None
    cases = [(n, 0) for n in sizes] + [(117_440_512, 7_340_032), (256 << 20, 1 << 20),
                                       (256 << 20, 64 << 10)]
    for n, chunk in cases:
        # enough repetitions that each measurement moves >= 2 GiB
        reps = max(8, (2 << 30) // n)
        if args.graph:
            reps = min(reps, 256)
        off = fab.slab_alloc(1, n)
        nch = 1 if chunk <= 0 or chunk >= n else -(-n // chunk)
        with torch.cuda.stream(s):
            for _ in range(3):
                fab.forward(0, src.data_ptr(), 1, off, n, chunk, fab.flags_alloc(1, nch), s, dma=dma)
            torch.cuda.synchronize()
            if args.graph:
                fb = fab.flags_alloc(1, nch)
                g, gc, gf = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(reps):  # fixed flags/token: nobody waits on them here
                        if flush_buf is not None:
                            flush_buf.fill_(1)
                        fab.forward(0, src.data_ptr(), 1, off, n, chunk, fb, s, token=(1 << 40) + n,
                                    host_notify=False, bulk=args.bulk, dma=dma)
                with torch.cuda.graph(gc, stream=s):
                    for _ in range(reps):
                        if flush_buf is not None:
                            flush_buf.fill_(1)
                        ref[:n].copy_(src[:n])
                if flush_buf is not None:
                    with torch.cuda.graph(gf, stream=s):
                        for _ in range(reps):
                            flush_buf.fill_(1)
                    gf.replay()
                g.replay()
                gc.replay()
                torch.cuda.synchronize()
                fwd_run, cpy_run = g.replay, gc.replay
            else:
                def fwd_run():
                    for _ in range(reps):
                        fab.forward(0, src.data_ptr(), 1, off, n, chunk, fab.flags_alloc(1, nch), s, dma=dma)

                def cpy_run():
                    for _ in range(reps):
                        ref[:n].copy_(src[:n])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fwd_run()
            e1.record(s)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(s)
            cpy_run()
            c1.record(s)
            c1.synchronize()
            cms = c0.elapsed_time(c1) / reps
            if flush_buf is not None and args.graph:
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record(s)
                gf.replay()
                f1.record(s)
                f1.synchronize()
                fms = f0.elapsed_time(f1) / reps
                ms, cms = ms - fms, cms - fms
        cpu = {}
        if cref is not None and chunk == 0:
            iters = max(2, min(200, (256 << 20) // max(n, 1)))
            secs = cref.ref_forward_bench(n, iters, 1)
            cpu = {"cpu_ref_us": round(secs / iters * 1e6, 1),
                   "cpu_ref_payload_gbs": round(n * iters / secs / 1e9, 3), "cpu_ref_threads": 1}
        d0 = fab.stats()["dma_forwards"]
        fab.forward(0, src.data_ptr(), 1, off, n, chunk, fab.flags_alloc(1, nch), s, bulk=args.bulk, dma=dma)
        s.synchronize()
        fab.slab_free(1, off)
        # the K1 form that ran: the copy engine (counted), else bulk when asked
        # or when the library picks it (a local aligned batch above 2 MiB)
        auto_bulk = args.form == "auto" and n > (2 << 20)
        form = "dma" if fab.stats()["dma_forwards"] > d0 else ("bulk" if args.bulk or auto_bulk else "tile")
        print(json.dumps({"k1": form, "form_arg": args.form, "graph": args.graph,
                          "l2_flush": bool(args.flush and args.graph), "bytes": n, **cpu, "chunk_bytes": chunk,
                          "chunks": nch, "us": round(ms * 1e3, 2),
                          "hbm_gbs": round(2 * n / (ms * 1e-3) / 1e9, 1),
                          "memcpy_us": round(cms * 1e3, 2),
                          "memcpy_hbm_gbs": round(2 * n / (cms * 1e-3) / 1e9, 1)}), flush=True)
    fab.close()


if __name__ == "__main__":
    main()
