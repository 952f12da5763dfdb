#!/usr/bin/env python
"""Sustained vs burst HBM copy on this B200, timed like bench.py times its
kernels (CUDA events around each launch inside a back-to-back loop): the
practical ceiling the forward/merge kernels are compared against.  torch
copy_ (cudaMemcpyAsync D2D) of 470 MB (config B payload per step)."""
import json

import torch


def main():
    n = 469_762_048
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    c = torch.empty_like(a)
    a.fill_(3)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(5):
            b.copy_(a)
        torch.cuda.synchronize()
        # burst: isolated launches
        burst = []
        for _ in range(10):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            b.copy_(a)
            e1.record(s)
            e1.synchronize()
            burst.append(2 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        # sustained: two copies per "step", back to back, 40 steps (like bench)
        evs = []
        for i in range(40):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            (b if i % 2 else c).copy_(a)
            e1.record(s)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        sus = [2 * n / (x.elapsed_time(y) * 1e-3) / 1e9 for x, y in evs]
    print(json.dumps({"bytes": n, "burst_gbs_best": round(max(burst), 1),
                      "burst_gbs_median": round(sorted(burst)[5], 1),
                      "sustained_gbs_median": round(sorted(sus)[20], 1),
                      "sustained_gbs_min": round(min(sus), 1)}))


if __name__ == "__main__":
    main()
