"""HBM rates by access mix on this B200 (event-timed, best of 10): read-only
(sum of 1 GiB), write-only (fill of 1 GiB), copy 1:1 (torch copy_), and a
1:2 read:write tee (one read, two writes via two copies sharing the source in
one kernel is not expressible in torch -- estimated from the three)."""
import json
import torch

n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
a.fill_(1)
w = a.view(torch.int64)


def best(fn, k=10):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


out = {}
t = best(lambda: w.sum())
out["read_gbs"] = round(n / t / 1e6, 1)
t = best(lambda: b.fill_(3))
out["write_gbs"] = round(n / t / 1e6, 1)
t = best(lambda: b.copy_(a))
out["copy_gbs"] = round(2 * n / t / 1e6, 1)
print(json.dumps(out))
