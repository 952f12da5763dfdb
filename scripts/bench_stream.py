#!/usr/bin/env python
"""Config C (Qwen2.5-Omni audio output path) on one B200: per decode step the
thinker forwards one hidden-state row per active request to the talker
(B = 32 x 3584-d bf16 = 7,168 B, executor_sim.hpp:556-562), and the talker
forwards one 4-byte code per request to the vocoder (16 requests,
:543-549).  Latency-bound: reported as per-step message latency (push launch
to rows landed in the consumer's input, CUDA events, p50/p99) and pipelined
msgs/s, next to the reference CPU path (oracle/_ref: SidecarFabric::send per
message + run_until_idle per step, 1 core).  Prints one JSON line per case."""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(p / 100 * (len(xs) - 1))))]


def run_case(fab, name, src_gpu, dst_gpu, batch, row_bytes, steps=2000, slots=64):
    import torch

    chs = [fab.channel_open(src_gpu, dst_gpu, row_bytes, slots) for _ in range(batch)]
    rows = torch.empty((batch, row_bytes), dtype=torch.uint8, device="cuda")
    fab.synth(src_gpu, 7, rows.data_ptr(), rows.numel())
    out = torch.empty_like(rows)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(50):  # warm-up
            fab.channel_push(chs, rows.data_ptr(), row_bytes, s)
            fab.channel_pull(chs, out.data_ptr(), row_bytes, s)
        torch.cuda.synchronize()
        # latency: one step at a time (push -> pull), device-timed
        lat = []
        for _ in range(min(steps, 500)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fab.channel_push(chs, rows.data_ptr(), row_bytes, s)
            fab.channel_pull(chs, out.data_ptr(), row_bytes, s)
            e1.record(s)
            e1.synchronize()
            lat.append(e0.elapsed_time(e1) * 1e3)
        # throughput: steps issued back to back
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(steps):
            fab.channel_push(chs, rows.data_ptr(), row_bytes, s)
            fab.channel_pull(chs, out.data_ptr(), row_bytes, s)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
    assert torch.equal(out, rows)
    # CUDA graph of one decode step (push + pull): the channel counters live
    # on the device, so the same graph replays every step without host work.
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = torch.cuda.current_stream()
        fab.channel_push(chs, rows.data_ptr(), row_bytes, cs)
        fab.channel_pull(chs, out.data_ptr(), row_bytes, cs)
    torch.cuda.synchronize()
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        for _ in range(20):
            g.replay()
        glat = []
        for _ in range(min(steps, 500)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gs)
            g.replay()
            e1.record(gs)
            e1.synchronize()
            glat.append(e0.elapsed_time(e1) * 1e3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gs)
        for _ in range(steps):
            g.replay()
        e1.record(gs)
        e1.synchronize()
        gms = e0.elapsed_time(e1)
    assert torch.equal(out, rows)
    # 64 decode steps in one graph: the per-step device cost once the push and
    # the pull live inside the models' own step graphs (no launch per step)
    k = 64
    g64 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g64):
        cs = torch.cuda.current_stream()
        for _ in range(k):
            fab.channel_push(chs, rows.data_ptr(), row_bytes, cs)
            fab.channel_pull(chs, out.data_ptr(), row_bytes, cs)
    torch.cuda.synchronize()
    with torch.cuda.stream(gs):
        for _ in range(3):
            g64.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, steps // k)
        e0.record(gs)
        for _ in range(reps):
            g64.replay()
        e1.record(gs)
        e1.synchronize()
        in_graph_us = e0.elapsed_time(e1) * 1e3 / (reps * k)
    assert torch.equal(out, rows)
    # producer and consumer as two independent chains (as on two GPUs): 64
    # pushes in one graph on one stream, 64 pulls in another on a second
    # stream, replayed concurrently; the device flags and the in-kernel ring
    # backpressure are the only coupling
    gp, gq = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gp):
        cs = torch.cuda.current_stream()
        for _ in range(k):
            fab.channel_push(chs, rows.data_ptr(), row_bytes, cs)
    with torch.cuda.graph(gq):
        cs = torch.cuda.current_stream()
        for _ in range(k):
            fab.channel_pull(chs, out.data_ptr(), row_bytes, cs)
    torch.cuda.synchronize()
    sp, sq = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        with torch.cuda.stream(sq):
            gq.replay()
        with torch.cuda.stream(sp):
            gp.replay()
        torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    done_p, done_q = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(sq)
    sp.wait_event(start)
    reps2 = max(1, steps // k)
    for _ in range(reps2):
        with torch.cuda.stream(sq):
            gq.replay()
        with torch.cuda.stream(sp):
            gp.replay()
    done_p.record(sp)
    done_q.record(sq)
    torch.cuda.synchronize()
    two_chain_us = max(start.elapsed_time(done_p), start.elapsed_time(done_q)) * 1e3 / (reps2 * k)
    assert torch.equal(out, rows)
    graph = {"step_latency_us_p50": round(pct(glat, 50), 2),
             "step_latency_us_p99": round(pct(glat, 99), 2),
             "msgs_per_s": round(batch * steps / (gms * 1e-3), 1),
             "step_us_inside_a_64_step_graph": round(in_graph_us, 2),
             "msgs_per_s_inside_a_64_step_graph": round(batch / (in_graph_us * 1e-6), 1),
             "step_us_push_and_pull_chains_concurrent": round(two_chain_us, 2),
             "msgs_per_s_push_and_pull_chains_concurrent": round(batch / (two_chain_us * 1e-6), 1)}
    for ch in chs:
        fab.channel_close(ch)
    import oracle as O

    ref = {}
    if O.REF is not None:
        n = 200
        t = O.REF.ref_stream_bench(row_bytes, batch, n)
        ref = {"msgs_per_s": round(batch * n / t, 1), "us_per_step": round(t / n * 1e6, 1),
               "cores": 1, "kind": "reference"}
    return {"case": name, "requests": batch, "row_bytes": row_bytes,
            "step_latency_us_p50": round(pct(lat, 50), 2), "step_latency_us_p99": round(pct(lat, 99), 2),
            "msgs_per_s": round(batch * steps / (ms * 1e-3), 1),
            "gbs": round(batch * steps * row_bytes / (ms * 1e-3) / 1e9, 3),
            "launches_per_step": 2, "cuda_graph": graph, "reference_cpu": ref}


def main():
    from paper_2603_12118_b200.fabric import DeviceFabric

    fab = DeviceFabric({0: 0, 1: 0, 2: 0}, {0: 0, 1: 0, 2: 0})
    fab.slab_register(1, 256 << 20)
    fab.slab_register(2, 64 << 20)
    for args in [("thinker->talker hidden 3584", 0, 1, 32, 7168),
                 ("thinker->talker hidden 1024 (reference shape_rules)", 0, 1, 32, 2048),
                 ("talker->vocoder codes", 1, 2, 16, 4)]:
        print(json.dumps(run_case(fab, *args)), flush=True)
    fab.close()


if __name__ == "__main__":
    main()
