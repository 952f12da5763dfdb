"""Quick timing of the N=1 pass forms on config B (event-timed, 20 passes each):
tee (fused forward + merge), K1 (bulk / tile) then merge, direct placement."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_12118_b200 import _native as N  # noqa: E402
from paper_2603_12118_b200 import trace as T  # noqa: E402
from paper_2603_12118_b200.dataplane import DataPlaneBatch  # noqa: E402
from paper_2603_12118_b200.fabric import DeviceFabric  # noqa: E402


def main(config="B", count=None, passes=20):
    rules = T.RULES[config]
    reqs = T.config_requests(config, count)
    fab = DeviceFabric({0: 0, 1: 0}, {0: 0, 1: 0})
    lay = T.layout(reqs, rules.row_bytes)
    fab.slab_register(1, max(1 << 30, 2 * lay.payload_bytes))
    b = DataPlaneBatch(fab, reqs, rules, 0, 1, chunk_rows=1024 if config != "A" else None)
    b.synth_inputs()
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    out = {"config": config, "payload": lay.payload_bytes}

    def timed(fn, n=passes):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for e0, e1 in evs:
            e0.record(s)
            fn()
            e1.record(s)
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(c) for a, c in evs)
        return round(ts[len(ts) // 2], 4)

    b.scan(s)

    def tee():
        assert b.alloc()
        b.tee(s, mode=N.MERGE_COPY_ONLY)
        b.release()

    def serial(bulk):
        def f():
            assert b.alloc()
            b.forward(s, host_notify=False, bulk=bulk)
            b.merge(s, mode=N.MERGE_COPY_ONLY)
            b.release()
        return f

    def k1(bulk):
        def f():
            assert b.alloc()
            b.forward(s, host_notify=False, bulk=bulk)
            b.release()
        return f

    def merge_only():
        b.merge(s, mode=N.MERGE_COPY_ONLY)

    def place():
        b.place(s, mode=N.MERGE_COPY_ONLY)

    with torch.cuda.stream(s):
        out["tee_ms"] = timed(tee)
        out["k1_bulk_ms"] = timed(k1(True))
        out["k1_tile_ms"] = timed(k1(False))
        out["merge_ms"] = timed(merge_only)
        out["serial_bulk_ms"] = timed(serial(True))
        out["place_ms"] = timed(place)
        out["tee2_ms"] = timed(tee)
    P = lay.payload_bytes
    out["tee_payload_gbs"] = round(P / out["tee_ms"] / 1e6, 1)
    out["tee_3x_gbs"] = round(3 * P / out["tee_ms"] / 1e6, 1)
    out["serial_payload_gbs"] = round(P / out["serial_bulk_ms"] / 1e6, 1)
    print(json.dumps(out))
    fab.close()


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["B"]))
