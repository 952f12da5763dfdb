#!/usr/bin/env python
"""Probe the host->device ceiling that bounds bench.py's e2e leg: pinned H2D
of the config-B payload (4 x 112 MiB) as one copy per item, as 7 MiB chunks on
one stream, and as chunks spread over 2 / 4 streams (copy engines)."""
import json
import time

import torch


def run(nbytes=469_762_048, chunk=7_340_032, streams=1, reps=5):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(7)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        for i, off in enumerate(range(0, nbytes, chunk)):
            n = min(chunk, nbytes - off)
            with torch.cuda.stream(ss[i % streams]):
                d[off:off + n].copy_(h[off:off + n], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
    return round(best, 2)


if __name__ == "__main__":
    out = {"single_copy": run(chunk=469_762_048)}
    for s in (1, 2, 4):
        out[f"chunks_7MiB_{s}_streams"] = run(streams=s)
    out["chunks_32MiB_2_streams"] = run(chunk=32 << 20, streams=2)
    print(json.dumps(out))
