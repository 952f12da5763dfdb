"""Probe: does HBM move more bytes per second with several independent copy
streams in flight than with one?  (Range replay showed the colocated pass --
K1 || merge -- moving 1.75 GB of DRAM traffic at ~7.3 TB/s while each kernel
alone runs at ~6.1-6.6 TB/s.)  torch copy_ (cudaMemcpyAsync D2D kernels) of
the same total bytes split over 1, 2, 4 streams, and split into 2/4 regions
but issued on one stream.  Prints JSON lines; run on the GPU box."""
import json
import torch

torch.cuda.init()
TOTAL = 940 << 20
src = torch.empty(TOTAL, dtype=torch.uint8, device="cuda")
dst = torch.empty(TOTAL, dtype=torch.uint8, device="cuda")
src.fill_(1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(k, same_stream, reps=20):
    parts = TOTAL // k
    times = []
    for it in range(reps + 3):
        flush.fill_(it & 0xff)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        for i in range(k):
            s = cur if same_stream else streams[i]
            if not same_stream:
                s.wait_event(e0)
            with torch.cuda.stream(s):
                dst[i * parts:(i + 1) * parts].copy_(src[i * parts:(i + 1) * parts])
            if not same_stream:
                ev = torch.cuda.Event()
                ev.record(s)
                cur.wait_event(ev)
        e1.record(cur)
        e1.synchronize()
        if it >= 3:
            times.append(e0.elapsed_time(e1))
    times.sort()
    ms = times[len(times) // 2]
    print(json.dumps({"copies": k, "streams": 1 if same_stream else k, "bytes": TOTAL,
                      "ms_median": round(ms, 4), "gbs_rw": round(2 * TOTAL / (ms * 1e-3) / 1e9, 1)}),
          flush=True)


for k in (1, 2, 4, 8):
    run(k, True)
    if k > 1:
        run(k, False)
