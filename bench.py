#!/usr/bin/env python
"""Benchmark of the sidecar data plane (BASELINE.json metric: forwarded GB/s
per producer->consumer pair vs 900 GB/s NVLink; merged req/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fsx|reference]

Workload (BASELINE.json configs[1]): Qwen2.5-VL video->text,
R = 4 requests per step, each one video of 16 frames x 1024 tokens x 3584-d
bf16 (117,440,512 B) forwarded as 16 per-frame chunks of 7,340,032 B with a
completion flag each, and merged into the placeholder rows of the
[1800 + 16384, 3584] prompt embedding.  A step = one data-plane pass over the
batch: slab segments allocated, every item forwarded into its segment with
per-chunk flags, merged into the prompt rows, segments released.

  N = 1: producer and consumer are the same B200 (intra-device forward, HBM):
         the forward and the merge run as ONE kernel (fsx_forward_merge, the
         tee: each row read once, stored into the slab and into its prompt
         row), with the placeholder scan pipelined one pass ahead.
  N > 1: one process per GPU; rank 2k produces into rank 2k+1's slab over
         NVLink (CUDA IPC), rank 2k+1 merges with in-kernel early start and
         acks; pairs are independent ("scaling": "weak", no collective on the
         data path).  Without RANK/WORLD_SIZE in the environment, bench.py
         --gpus N spawns the N ranks itself (127.0.0.1 rendezvous).

Inputs are larger than L2 (470 MB payload + 521 MB prompt embeddings per
step vs 126 MB L2), so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "B"
REQUESTS = 4
CHUNK_ROWS = 1024  # one video frame = 7,340,032 B
# --config selects another BASELINE.json merge workload (parity/extra lines; the
# driver's default line is config B).
CONFIGS = {
    "A": {"requests": 64, "chunk_rows": None,
          "workload": "A: InternVL3 image->text, mllm-chat trace (seed 42), 256 x 4096-d bf16 per image"},
    "B": {"requests": 4, "chunk_rows": 1024,
          "workload": "B: Qwen2.5-VL video->text, 16 frames x 1024 tokens x 3584-d bf16 per request"},
    "D": {"requests": 32, "chunk_rows": 1024,
          "workload": "D: servegen-like mixed image/video/audio trace (seed 42), 3584-d bf16"},
    # config C: a decode step of the Qwen2.5-Omni audio path -- one 3584-d bf16
    # hidden-state row per active thinker request to the talker, one 4-byte
    # code per talker request to the vocoder (executor_sim.hpp:540-564)
    "C": {"requests": 32, "chunk_rows": None, "codes": 16, "row_bytes": 7168,
          "workload": "C: Qwen2.5-Omni decode step, 32 x 7168 B thinker->talker hidden rows + "
                      "16 x 4 B talker->vocoder codes"},
}
METRIC = "forwarded GB/s per producer\u2192consumer pair vs 900 GB/s NVLink; merged req/s"  # BASELINE.json
KERNELS = {
    "tee": "fsx::kern::merge_tee_kernel (fsx_forward_merge: forward + merge in one kernel)",
    "forward": "fsx::kern::forward_tma_kernel (K1, bulk-copy tiles, all items of the step in one launch)",
    "merge": "fsx::kern::merge_copy_kernel (K3b, warp per placeholder row, stream-ordered)",
    "follow": "fsx::kern::merge_follow_kernel (K3b early start: warp per placeholder row, chunk flag acquired per row)",
    "scan": "fsx::kern::merge_scan_kernel (K3a placeholder scan)",
}


# N>1: the K1 forms for peer (NVLink) destinations (fsx_forward_batch options)
K1_FORMS = {"tile": 64,         # register tiles (FSX_FWD_KERNEL), system-scope acq_rel count per tile
            "gpucount": 16,     # register tiles, gpu-scope count, one fence.sc.sys + flag per chunk
            "bulk": 4,          # bulk-copy (cp.async.bulk) tiles into the peer slab
            "dma": 32}          # copy engine (cudaMemcpyAsync per chunk) + one flag kernel per transfer


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["fsx", "reference"], default="fsx")
    p.add_argument("--config", choices=sorted(CONFIGS), default="B")
    p.add_argument("--requests", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--colocated", action="store_true",
                   help="also time the colocated schedule (K1 || early-start merge on one GPU, "
                        "round 1's headline): two kernels spinning on each other's progress")
    p.add_argument("--no-verify", dest="verify", action="store_false",
                   help="N>1: skip the consumers' bit-exactness check of the merged embeddings "
                        "against a local pass (on by default)")
    p.add_argument("--profile", action="store_true",
                   help="short run for ncu: no clocks, no cpu baseline, no e2e")
    p.add_argument("--k1", choices=["auto"] + sorted(K1_FORMS), default="auto",
                   help="N>1: the K1 form pushing into peer slabs (auto: probe all, time the fastest)")
    p.add_argument("--transfer", choices=["slab", "direct"], default="slab",
                   help="N>1 pairs: K1 into the consumer slab + early-start merge (slab), or the "
                        "producer placing rows straight into the consumer's prompt (direct)")
    p.add_argument("--chunk-rows", type=int, default=None,
                   help="rows per flagged chunk (default: the config's, one video frame for B/D)")
    p.add_argument("--sets", type=int, default=2,
                   help="N>1: slab segment sets per consumer (the next transfer overlaps the merge)")
    p.add_argument("--pin-device", type=int, default=None,
                   help="N>1 protocol runs on a 1-GPU box: every rank on this device, gloo for setup")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(config: str, kernel: str, alg_bytes: int):
    """DRAM bytes per launch of `kernel` on `config` from the committed
    `ncu --set full` capture (profiles/traffic_r02s.json, written by
    scripts/profile_round.sh), only when that capture is of the same kernel on
    the same launch size; else (None, reason)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_r02s.json")) as fh:
            rec = json.load(fh).get(f"{config}:{kernel}")
    except Exception:
        rec = None
    if not rec:
        return None, f"no ncu capture of {kernel} on config {config} committed"
    if int(rec.get("alg_bytes", -1)) != int(alg_bytes):
        return None, f"committed capture is of a {rec.get('alg_bytes')}-byte launch, not {alg_bytes}"
    return int(rec["dram_bytes"]), rec.get("source")


# ---------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.12)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference path on the host cores

def cpu_reference_pass(reqs, rules, merge_threads):
    """One pass of the reference data plane (oracle/_ref: SidecarFabric compiled
    unmodified + the derived merge) over `reqs`.  Returns (seconds, payload bytes,
    kind).  Inputs are synthesised before the timed call."""
    import ctypes as C

    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2603_12118_b200 import trace as T

    lay = T.layout(reqs, rules.row_bytes)
    rb = rules.row_bytes
    emb = np.concatenate([np.frombuffer(O.synth_payload(T.text_seed(q), q.total_rows * rb), np.uint8)
                          for q in reqs]).copy()
    tok = np.concatenate([T.prompt_tokens(q) for q in reqs])
    src = [np.frombuffer(O.synth_payload(T.payload_seed(it.ref_id, 0), it.rows * rb), np.uint8)
           for it in lay.items]
    status = np.zeros(len(reqs), np.int32)
    if O.REF is not None:
        # the reference fabric is single-threaded by construction; on all host
        # threads it runs as one SidecarFabric per thread over a share of the
        # requests, each thread merging its own (ref_dataplane_pass_mt)
        ptrs = (C.c_void_p * len(src))(*[s.ctypes.data for s in src])
        ids = (C.c_char_p * len(src))(*[it.ref_id.encode() for it in lay.items])
        secs = O.REF.ref_dataplane_pass_mt(len(reqs), len(src), rb, T.PLACEHOLDER_ID, emb.ctypes.data,
                                           tok.ctypes.data, lay.req_row_off.ctypes.data,
                                           lay.req_item_off.ctypes.data, ptrs,
                                           lay.item_rows.ctypes.data, ids, 0, 1, merge_threads,
                                           status.ctypes.data)
        if secs < 0:
            raise RuntimeError(O.REF.ref_last_error().decode())
        return secs, lay.payload_bytes, "reference"
    # No reference build on this host: the C restatement of the merge only
    # (forwarding cost of the reference not represented).
    t0 = time.perf_counter()
    O.merge(rb, T.PLACEHOLDER_ID, emb, tok, lay.req_row_off, lay.req_item_off, src, lay.item_rows,
            nthreads=merge_threads)
    return time.perf_counter() - t0, lay.payload_bytes, "port"


def cpu_baseline(min_seconds=12.0, max_passes=80):
    from paper_2603_12118_b200 import trace as T

    rules = T.RULES[CONFIG]
    reqs = cpu_sample(T)
    payload = T.layout(reqs, rules.row_bytes).payload_bytes
    threads = os.cpu_count() or 1
    total_s, total_b, n, kind = 0.0, 0, 0, "reference"
    while total_s < min_seconds and n < max_passes:
        s, b, kind = cpu_reference_pass(reqs, rules, threads)
        total_s += s
        total_b += b
        n += 1
    used = min(threads, len(reqs))  # one reference fabric (thread) per request at most
    return {"value": round(total_b / total_s / 1e9, 4), "unit": "GB/s", "cores": used,
            "kind": kind,
            "sample": (f"{n} passes of {len(reqs)} config-{CONFIG} request(s) ({payload:,} B of "
                       "embeddings per pass): SidecarFabric::send_payload -> run_until_idle "
                       "(reference, compiled unmodified, single-threaded by construction: one "
                       f"fabric per thread over a share of the requests) + CPU merge, {used} of "
                       f"{threads} host threads; {total_s:.1f} s of CPU work"),
            "merged_req_per_s": round(n * len(reqs) / total_s, 3)}


def cpu_sample(T, scale: int = 1):
    """Bounded CPU sample of the workload: the first requests of the batch
    whose embeddings add up to >= 100 MiB, and at least one request per host
    thread while the batch has them (config B: the whole 4-video batch).
    scale: the fsx arm at N > 1 moves N/2 pairs' (or encoders') batches per
    step, so the reference arm draws from that many requests."""
    rules = T.RULES[CONFIG]
    full = T.config_requests(CONFIG, REQUESTS * max(1, scale))
    want = min(len(full), os.cpu_count() or 1)
    out, acc = [], 0
    for q in full:
        out.append(q)
        acc += q.placeholder_rows * rules.row_bytes
        if acc >= 100 << 20 and len(out) >= want:
            break
    return out


# ---------------------------------------------------------------------------
# reference arm

def run_reference_c(args):
    """Config C on the reference CPU path: every hidden-state row of a decode
    step is a SidecarFabric::send with its own envelope, event and delivery
    (oracle/_ref, the reference compiled unmodified; single-threaded by
    construction), codes likewise."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # the reference CPU path (checker library)

    cfg = CONFIGS["C"]
    nh, row, nc = cfg["requests"], cfg["row_bytes"], cfg["codes"]
    O.REF.ref_stream_bench(row, nh, max(1, args.warmup))
    O.REF.ref_stream_bench(4, nc, max(1, args.warmup))
    t = O.REF.ref_stream_bench(row, nh, args.steps) + O.REF.ref_stream_bench(4, nc, args.steps)
    step_bytes = nh * row + nc * 4
    value = step_bytes * args.steps / t / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t / args.steps * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "us_per_step": round(t / args.steps * 1e6, 1),
        "msgs_per_s": round((nh + nc) * args.steps / t, 1),
        "config": {"workload": cfg["workload"], "parallelism": "reference CPU path, 1 process"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} decode steps: {nh} hidden rows + {nc} codes, one "
                                   "SidecarFabric::send per message + run_until_idle per step"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_reference(args, rank):
    if rank != 0:
        return
    if CONFIG == "C":
        run_reference_c(args)
        return
    from paper_2603_12118_b200 import trace as T

    rules = T.RULES[CONFIG]
    threads = os.cpu_count() or 1
    # the same per-step workload as the fsx arm at this N: N/2 pairs (A/B) or
    # N/2 encoders (D) each with a batch of REQUESTS requests
    reqs = cpu_sample(T, max(1, args.gpus // 2))
    for _ in range(args.warmup):
        cpu_reference_pass(reqs, rules, threads)
    secs, nbytes, kind = 0.0, 0, "reference"
    for _ in range(args.steps):
        s, b, kind = cpu_reference_pass(reqs, rules, threads)
        secs += s
        nbytes += b
    value = nbytes / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "merged_req_per_s": round(args.steps * len(reqs) / secs, 4),
        "config": {"workload": CONFIGS[CONFIG]["workload"],
                   "requests_per_step": len(reqs),
                   "chunk_bytes": "single shot (reference has no chunking)",
                   "parallelism": "reference CPU path, 1 process"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": min(threads, len(reqs)),
                         "kind": kind,
                         "sample": f"each step: {len(reqs)} config-{CONFIG} request(s) forwarded "
                                   "through the reference SidecarFabric (one fabric per host "
                                   "thread, each over a share of the requests) + CPU merge, all "
                                   "host threads"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# config C (streaming decode step), one GPU

def run_config_c(args):
    """A decode step of the Qwen2.5-Omni audio path on one B200: the thinker's
    32 hidden-state rows pushed through 32 streaming channels into the
    talker's input, the talker's 16 codes through 16 channels into the
    vocoder's input (fsx_channel_push / pull, seq-ordered rings in the
    consumer slabs, per-slot flags, device-resident counters), one CUDA graph
    per step.  e2e: the same messages from host memory through the
    drop-in's small-message path (fsx_put_small_alloc -> lane -> fsx_ticket_take
    back into host memory), host time per step."""
    import ctypes as C

    import torch

    from paper_2603_12118_b200 import _native as N
    from paper_2603_12118_b200.fabric import DeviceFabric

    cfg = CONFIGS["C"]
    nh, row, nc = cfg["requests"], cfg["row_bytes"], cfg["codes"]
    torch.cuda.set_device(0)
    fab = DeviceFabric({0: 0, 1: 0, 2: 0}, {0: 0, 1: 0, 2: 0})
    fab.slab_register(1, 256 << 20)
    fab.slab_register(2, 64 << 20)
    hch = [fab.channel_open(0, 1, row, 64) for _ in range(nh)]
    cch = [fab.channel_open(1, 2, 4, 64) for _ in range(nc)]
    # a step's rows and codes in one buffer (one copy each way for e2e)
    inbuf = torch.empty(nh * row + nc * 4, dtype=torch.uint8, device="cuda")
    outbuf = torch.empty_like(inbuf)
    hrows, codes = inbuf[:nh * row].view(nh, row), inbuf[nh * row:].view(nc, 4)
    hout, cout = outbuf[:nh * row].view(nh, row), outbuf[nh * row:].view(nc, 4)
    fab.synth(0, 7, hrows.data_ptr(), hrows.numel())
    fab.synth(1, 8, codes.data_ptr(), codes.numel())
    step_bytes = nh * row + nc * 4
    s = torch.cuda.Stream()

    def step(st):
        # the step's hidden rows and codes in ONE push launch and ONE pull
        # launch (fsx_channel_push_groups / _pull_groups: 48 streams, two
        # row sizes, two buffers)
        fab.channel_push_groups([(hch, hrows.data_ptr(), row), (cch, codes.data_ptr(), 4)], st)
        fab.channel_pull_groups([(hch, hout.data_ptr(), row), (cch, cout.data_ptr(), 4)], st)

    def step_per_group(st):  # round-2 r02q form: push + pull per group (4 launches)
        fab.channel_push(hch, hrows.data_ptr(), row, st)
        fab.channel_pull(hch, hout.data_ptr(), row, st)
        fab.channel_push(cch, codes.data_ptr(), 4, st)
        fab.channel_pull(cch, cout.data_ptr(), 4, st)

    def graph_of(fn):
        with torch.cuda.stream(s):
            for _ in range(max(3, args.warmup)):
                fn(s)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        l0 = fab.stats()["kernel_launches"]
        with torch.cuda.graph(gr, stream=s):
            fn(s)
        nk = fab.stats()["kernel_launches"] - l0
        with torch.cuda.stream(s):
            for _ in range(max(3, args.warmup)):
                gr.replay()
        torch.cuda.synchronize()
        return gr, nk

    def time_graph(gr):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(args.steps):
                gr.replay()
            e1.record(s)
            e1.synchronize()
        return e0.elapsed_time(e1) / args.steps

    g4, k4 = graph_of(step_per_group)
    hout.zero_()
    cout.zero_()
    ms_per_group = time_graph(g4)
    assert torch.equal(hout, hrows) and torch.equal(cout, codes), "streamed rows differ (per group)"
    hout.zero_()
    cout.zero_()
    g, kernels_per_step = graph_of(step)
    with ClockSampler(0) as clk:
        ms_step = time_graph(g)
    assert torch.equal(hout, hrows) and torch.equal(cout, codes), "streamed rows differ"
    # e2e: host rows through the drop-in's small-message path, host-timed
    hin = torch.empty(nh * row + nc * 4, dtype=torch.uint8, pin_memory=True)
    hin.copy_(inbuf.cpu())
    hh, hc = hin[:nh * row].view(nh, row), hin[nh * row:].view(nc, 4)
    back = (C.c_uint8 * row)()

    def e2e_step():
        ts = []
        for r in range(nh):
            off, t = C.c_int64(), C.c_int64()
            N.call("fsx_put_small_alloc", fab._h, 1, hh[r].data_ptr(), row, 0, C.byref(off), C.byref(t))
            ts.append((1, off.value, t.value, row))
        for r in range(nc):
            off, t = C.c_int64(), C.c_int64()
            N.call("fsx_put_small_alloc", fab._h, 2, hc[r].data_ptr(), 4, 0, C.byref(off), C.byref(t))
            ts.append((2, off.value, t.value, 4))
        for gpu, off, t, n in ts:
            sent, landed = C.c_uint64(), C.c_uint64()
            N.call("fsx_ticket_take", fab._h, t, back, n, C.byref(sent), C.byref(landed))
            assert sent.value == landed.value
            fab.slab_free(gpu, off)

    for _ in range(20):
        e2e_step()
    e_steps = max(50, args.steps)
    h0 = time.perf_counter()
    for _ in range(e_steps):
        e2e_step()
    lane_us = (time.perf_counter() - h0) / e_steps * 1e6
    assert bytes(back[:4]) == bytes(hc[nc - 1].numpy().tobytes())
    # e2e headline: the decode step from host memory -- the step's rows copied
    # in (pinned), the channel graph, the delivered rows copied out, the
    # stream synchronised, host wall time per step
    hout_pinned = torch.empty(hin.numel(), dtype=torch.uint8, pin_memory=True)

    def host_step():  # stream-ordered: step s+1's copy-in waits for step s's copy-out
        with torch.cuda.stream(s):
            inbuf.copy_(hin, non_blocking=True)
            g.replay()
            hout_pinned.copy_(outbuf, non_blocking=True)

    for _ in range(20):
        host_step()
    s.synchronize()
    h0 = time.perf_counter()
    for _ in range(e_steps):
        host_step()
    s.synchronize()
    e2e_us = (time.perf_counter() - h0) / e_steps * 1e6
    assert torch.equal(hout_pinned, hin)
    peak, peak_kind = load_peaks()
    value = step_bytes / (ms_step * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (reference synth_payload bytes, K0 on device)",
        "us_per_step": round(ms_step * 1e3, 2),
        "msgs_per_s": round((nh + nc) / (ms_step * 1e-3), 1),
        "config": {"workload": cfg["workload"],
                   "placement": "thinker, talker and vocoder slabs on one B200 (intra-device channels)",
                   "schedule": "one CUDA graph per decode step: one push launch and one pull launch "
                               "for the hidden rows and the codes together (channel groups)",
                   "parallelism": "1 GPU", "l2": "decode-step working set is L2-resident by nature"},
        "roofline": {"bound": "hbm", "kernel": "fsx::kern::chan_push_kernel + chan_pull_kernel",
                     "achieved": round(2 * step_bytes / (ms_step * 1e-3) / 1e9, 2), "peak": peak,
                     "peak_kind": f"{peak_kind} hbm_gbs (copy, burst)", "unit": "GB/s",
                     "frac": round(2 * step_bytes / (ms_step * 1e-3) / 1e9 / peak, 6), "traffic": None,
                     "traffic_note": "latency-bound: a decode step moves 229 KB; the step time is the "
                                     "two kernel nodes' launch and flag round trips, not bandwidth",
                     "algorithmic_bytes_per_launch": 2 * step_bytes},
        "schedules": {"groups": {"what": "push + pull of both groups in one launch each",
                                 "kernels_per_step": kernels_per_step, "us_per_step": round(ms_step * 1e3, 2)},
                      "per_group": {"what": "push + pull per group (hidden rows, then codes)",
                                    "kernels_per_step": k4, "us_per_step": round(ms_per_group * 1e3, 2)}},
        "gpu_launches": kernels_per_step * args.steps, "gpu_launches_per_step": kernels_per_step,
        "clocks": clk.summary(),
        "e2e": {"value": round(step_bytes / (e2e_us * 1e-6) / 1e9, 4), "unit": "GB/s",
                "h2d_bytes_per_step": step_bytes, "d2h_bytes_per_step": step_bytes,
                "us_per_step": round(e2e_us, 2),
                "path": "every step: the step's rows and codes copied in from pinned host memory "
                        "(one copy), the channel step graph, the delivered rows copied back out "
                        "(one copy), stream-ordered; host wall time over all steps, synchronised "
                        "at the end",
                "small_message_lane_us_per_step": round(lane_us, 2),
                "small_message_lane_path": "per message through ctypes: fsx_put_small_alloc -> "
                                           "fsx_ticket_take -> fsx_slab_free (Python-call bound; the "
                                           "C++ drop-in does the same in 42-46 us, "
                                           "profiles/bench_fabric_dropin_r02p.jsonl)"},
    }
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O  # the reference CPU path (checker library), timed beside the kernels

        if O.REF is not None:
            n = 400
            t = O.REF.ref_stream_bench(row, nh, n)
            line["cpu_baseline"] = {"value": round(nh * row * n / t / 1e9, 4), "unit": "GB/s", "cores": 1,
                                    "kind": "reference",
                                    "us_per_step": round(t / n * 1e6, 1),
                                    "sample": f"{n} decode steps of {nh} x {row} B hidden rows through the "
                                              "reference SidecarFabric::send + run_until_idle (one "
                                              "thread: the reference is single-threaded)"}
    for ch in hch + cch:
        fab.channel_close(ch)
    fab.close()
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# fsx arm, one GPU

def run_single(args):
    """N = 1: producer and consumer share one B200.  The timed pass is the
    tee (fsx_forward_merge); the other schedules of the same pass and each
    kernel alone are measured in the same process for the line's
    `schedules` / `kernels` objects."""
    import torch

    from paper_2603_12118_b200 import _native as N
    from paper_2603_12118_b200 import trace as T
    from paper_2603_12118_b200.dataplane import DataPlaneBatch
    from paper_2603_12118_b200.fabric import DeviceFabric

    dev = 0
    torch.cuda.set_device(dev)
    rules = T.RULES[CONFIG]
    reqs = T.config_requests(CONFIG, args.requests)
    fab = DeviceFabric({0: 0, 1: 0}, {0: dev, 1: dev})
    lay = T.layout(reqs, rules.row_bytes)
    fab.slab_register(1, max(1 << 30, 2 * lay.payload_bytes))
    stream = torch.cuda.Stream(device=dev)
    side = torch.cuda.Stream(device=dev)
    mstream = torch.cuda.Stream(device=dev, priority=torch.cuda.Stream.priority_range()[1])
    batch = DataPlaneBatch(fab, reqs, rules, src_gpu=0, dst_gpu=1, chunk_rows=CHUNK_ROWS)
    with torch.cuda.stream(stream):
        batch.synth_inputs(stream)
    torch.cuda.synchronize()
    payload = lay.payload_bytes
    n_rows = lay.total_item_rows
    # algorithmic bytes per launch: the tee reads every item row
    # once and writes it twice (slab segment + prompt row) and reads one
    # position per row; K1 reads + writes the payload; the merge reads the
    # slab + writes the prompt rows + reads the positions.
    tee_bytes = 3 * payload + 4 * n_rows
    fwd_bytes = 2 * payload
    merge_bytes = 2 * payload + 4 * n_rows
    s8d_pass_bytes = fwd_bytes + merge_bytes  # forward + merge counted separately

    # The placeholder scan only needs token ids, so every schedule runs it one
    # pass ahead on a side stream into a second scan slot: pass s copies with
    # the positions scanned during pass s-1 and scans for pass s+1.
    scanned = [torch.cuda.Event(), torch.cuda.Event()]
    merged = [torch.cuda.Event(), torch.cuda.Event()]
    fork = torch.cuda.Event()
    counter = [0]
    graph_launched = [0]
    ev = []
    ev_pool = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))
               for _ in range(max(args.steps, 20) + 1)]

    def begin(record):
        s = counter[0]
        counter[0] += 1
        cur, nxt = s % 2, (s + 1) % 2
        assert batch.alloc()
        if s > 0:
            stream.wait_event(merged[(s - 1) % 2])  # previous pass (any stream) done
        fork.record(stream)
        side.wait_event(fork)
        batch.scan(side, slot=nxt)
        scanned[nxt].record(side)
        stream.wait_event(scanned[cur])
        e = ev_pool[len(ev)] if record else (None, None, None)
        if record:
            e[0].record(stream)
        return cur, e

    def end(cur, e, record):
        merged[cur].record(stream)
        if record:
            e[2].record(stream)
            ev.append(e)
        batch.release()

    def step_tee(record=False):
        cur, e = begin(record)
        batch.tee(stream, mode=N.MERGE_COPY_ONLY, slot=cur)
        if record:
            e[1].record(stream)
        end(cur, e, record)

    def step_serial(record=False):
        cur, e = begin(record)
        batch.forward(stream, host_notify=False, bulk=True)
        if record:
            e[1].record(stream)
        batch.merge(stream, mode=N.MERGE_COPY_ONLY, slot=cur)
        end(cur, e, record)

    def step_follow(record=False):
        # K1, then the early-start merge in stream order (its flags are all
        # set): the follow kernel's own rate at full occupancy
        cur, e = begin(record)
        batch.forward(stream, host_notify=False, bulk=True)
        if record:
            e[1].record(stream)
        batch.merge(stream, early_start=True, mode=N.MERGE_COPY_ONLY, slot=cur)
        end(cur, e, record)

    def step_colocated(record=False):
        # K1 (register tiles) and the early-start merge concurrently: the merge
        # follows K1's chunk flags on a high-priority stream, one CTA per SM
        cur, e = begin(record)
        mstream.wait_event(scanned[cur])
        batch.forward(stream, host_notify=False, l2_keep=True)
        if record:
            e[1].record(stream)
        with torch.cuda.stream(mstream):
            batch.merge(mstream, early_start=True, slot=cur,
                        mode=N.MERGE_COPY_ONLY | N.MERGE_COLOCATED | N.MERGE_DISCARD)
        join = torch.cuda.Event()
        join.record(mstream)
        stream.wait_event(join)
        end(cur, e, record)

    def step_place(record=False):
        cur, e = begin(record)
        batch.place(stream, mode=N.MERGE_COPY_ONLY, slot=cur)
        if record:
            e[1].record(stream)
        end(cur, e, record)

    def step_graph(record=False):
        # the tee pass as one CUDA graph launch: the tee || the next pass's scan
        s = counter[0]
        counter[0] += 1
        assert batch.alloc()
        if s > 0:
            stream.wait_event(merged[(s - 1) % 2])
        e = ev_pool[len(ev)] if record else None
        if record:
            e[0].record(stream)
        batch.run_graph(stream)
        graph_launched[0] += batch.graph_kernels
        if record:
            e[1].record(stream)
        merged[s % 2].record(stream)
        if record:
            e[2].record(stream)
            ev.append(e)
        batch.release()

    # two-set form of the graph schedule (small passes): consecutive passes on
    # two streams over two sets of slab segments / prompt rows, so one pass's
    # tail overlaps the next one's ramp (a server keeps several batches in
    # flight the same way); filled in by the probe below
    sets2 = {"batches": None, "streams": None}
    extra_streams = []

    def step_graph2(record=False):
        s = counter[0]
        counter[0] += 1
        b, st = sets2["batches"][s % 2], sets2["streams"][s % 2]
        e = ev_pool[len(ev)] if record else None
        if record:
            e[0].record(st)
        b.run_graph(st)
        graph_launched[0] += b.graph_kernels
        if record:
            e[1].record(st)
            e[2].record(st)
            ev.append(e)

    host_issue = [0.0]  # host microseconds to issue one pass (last timed())

    def timed(step, n, record=True):
        """n passes between two events on `stream` (which waits for the last
        scan and the last pass); returns (ms per pass, per-pass events,
        fsx kernel launches).  record=False: no per-pass events in between."""
        ev.clear()
        l0 = fab.stats()["kernel_launches"] + graph_launched[0]
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record(stream)
        for s2 in extra_streams:
            s2.wait_event(start)
        h0 = time.perf_counter()
        for _ in range(n):
            step(record=record)
        host_issue[0] = (time.perf_counter() - h0) / n * 1e6
        stream.wait_event(scanned[counter[0] % 2])
        for s2 in extra_streams:
            stream.wait_stream(s2)
        stop.record(stream)
        torch.cuda.synchronize()
        return (start.elapsed_time(stop) / n, list(ev),
                fab.stats()["kernel_launches"] + graph_launched[0] - l0)

    def span(evs, a, b):
        return statistics.mean(x[a].elapsed_time(x[b]) for x in evs)

    with torch.cuda.stream(stream):
        batch.scan(side, slot=0)
        scanned[0].record(side)
        for _ in range(max(3, args.warmup)):
            step_tee()
        step = step_tee
        probe = None
        # launch-bound small passes (config A) may run faster as one CUDA
        # graph launch per pass: probed, the faster form is timed
        if payload < (128 << 20) and not args.profile:
            eager_ms = timed(step_tee, 10)[0]
            assert batch.alloc()
            # one graph per pass: the tee of this pass || the scan of the next
            batch.capture(stream, kind="tee_pipelined")
            batch.scan(stream, slot=0)
            batch.release()
            for _ in range(3):
                step_graph()
            graph_ms = timed(step_graph, 10)[0]
            probe = {"eager_ms": round(eager_ms, 4), "graph_ms": round(graph_ms, 4)}
            if graph_ms < eager_ms:
                step = step_graph
            # the two-set form: a second batch (its own inputs, slab segments,
            # prompt rows, scan slots), both held allocated, graphs on two streams
            b2 = DataPlaneBatch(fab, reqs, rules, src_gpu=0, dst_gpu=1, chunk_rows=CHUNK_ROWS)
            st2 = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(st2):
                b2.synth_inputs(st2)
            torch.cuda.synchronize()
            assert batch.alloc() and b2.alloc()
            batch.capture(stream, kind="tee_pipelined")
            b2.capture(st2, kind="tee_pipelined")
            batch.scan(stream, slot=0)
            b2.scan(st2, slot=0)
            sets2["batches"], sets2["streams"] = (batch, b2), (stream, st2)
            extra_streams.append(st2)
            for _ in range(4):
                step_graph2()
            two_ms = timed(step_graph2, 20)[0]
            probe["two_set_graph_ms"] = round(two_ms, 4)
            if two_ms < min(graph_ms, eager_ms):
                step = step_graph2
            else:  # back to one set (step_graph allocates per pass)
                extra_streams.clear()
                torch.cuda.synchronize()
                b2.release()
                batch.release()
        for _ in range(3):
            step()
        # the timed region: K passes, no per-pass events in between
        with ClockSampler(dev) as clk:
            ms_step, _, launches = timed(step, args.steps, record=False)
        host_us_step = host_issue[0]
        # the same passes again with events around each tee launch: its
        # in-pass kernel time for the roofline
        for _ in range(2):
            step()
        ms_evented, ev_main, _ = timed(step, max(5, min(args.steps, 20)))
        tee_ms = span(ev_main, 0, 1)
        if step is step_graph2:  # the other schedules run on one set
            extra_streams.clear()
            torch.cuda.synchronize()
            sets2["batches"][1].release()
            batch.release()
        schedules = {}
        kernels = {}
        if not args.profile:
            iso = max(5, min(args.steps, 20))
            for _ in range(3):
                step_serial()
            serial_ms, ev_s, _ = timed(step_serial, iso)
            kernels["forward"] = (span(ev_s, 0, 1), fwd_bytes, "forward")
            kernels["merge"] = (span(ev_s, 1, 2), merge_bytes, "merge")
            for _ in range(2):
                step_follow()
            _, ev_f, _ = timed(step_follow, iso)
            kernels["follow"] = (span(ev_f, 1, 2), merge_bytes, "follow")
            for _ in range(3):
                step_place()
            place_ms, _, _ = timed(step_place, iso)
            colo = None
            if args.colocated:
                # the colocated pass, as a long-lived server would run it: five
                # back-to-back 10-pass measurements in this one process
                for _ in range(3):
                    step_colocated()
                colo = [round(timed(step_colocated, 10)[0], 4) for _ in range(5)]
            schedules = {
                "tee": {"what": "scan one pass ahead || fsx_forward_merge (the timed pass)",
                        "ms_per_step": round(ms_step, 4)},
                "serial": {"what": "K1 (bulk-copy tiles) then the merge, stream order",
                           "ms_per_step": round(serial_ms, 4)},
                "colocated": ({"what": "K1 || early-start merge on a high-priority stream",
                               "runs_ms": colo, "first_ms": colo[0],
                               "steady_median_ms": statistics.median(colo[1:])} if colo else
                              {"what": "K1 || early-start merge on a high-priority stream (round 1's "
                                       "headline; opt-in: --colocated)",
                               "last_measured": "0.290 ms steady median, profiles/bench_r02i_full.json"}),
                "direct_placement": {"what": "fsx_forward_place: rows straight into the prompt, "
                                             "no slab segment (not the reference's semantics)",
                                     "ms_per_step": round(place_ms, 4),
                                     "payload_gbs": round(payload / (place_ms * 1e-3) / 1e9, 1)},
            }
            if probe:
                schedules["tee"]["graph_probe"] = probe
    # parity guard on the measured data: statuses all zero, and the merged
    # embeddings of the timed passes equal a plain K1-then-merge pass
    for slot in (0, 1):
        st = batch.status_host(slot)
        assert (st == 0).all(), st
    if not args.profile:
        ref_b = DataPlaneBatch(fab, reqs, rules, src_gpu=0, dst_gpu=1, chunk_rows=CHUNK_ROWS)
        ref_b.synth_inputs()
        assert ref_b.alloc()
        ref_b.forward(host_notify=False)
        ref_b.merge()
        torch.cuda.synchronize()
        assert torch.equal(ref_b.embeds, batch.embeds), "timed passes differ from a serial pass"
        if sets2["batches"] is not None:  # the second set of the two-set probe / schedule
            assert torch.equal(ref_b.embeds, sets2["batches"][1].embeds), "second set differs"
        ref_b.release()
        del ref_b

    peak, peak_kind = load_peaks()

    def kernel_obj(name, ms, nbytes):
        gbs = nbytes / (ms * 1e-3) / 1e9
        traffic, why = load_traffic(CONFIG, name, nbytes)
        o = {"kernel": KERNELS[name], "ms_per_launch": round(ms, 4),
             "algorithmic_bytes_per_launch": nbytes, "achieved_gbs": round(gbs, 1),
             "frac": round(gbs / peak, 4), "traffic": traffic}
        if traffic is None:
            o["traffic_note"] = why
        else:
            o["traffic_source"] = why
        return o

    overlapped = step is step_graph2
    # two-set schedule: consecutive passes' tee launches overlap on two
    # streams, so one launch's event span is not its share of the time; the
    # tee's rate is then its algorithmic bytes per pass over the pass time
    kern = {"tee": kernel_obj("tee", ms_step if overlapped else tee_ms, tee_bytes)}
    if overlapped:
        kern["tee"]["event_span_ms_per_launch"] = round(tee_ms, 4)
    for k, (ms, nb, name) in kernels.items():
        kern[k] = kernel_obj(name, ms, nb)
    t = kern["tee"]
    roofline = {"bound": "hbm", "kernel": t["kernel"], "achieved": t["achieved_gbs"], "peak": peak,
                "peak_kind": f"{peak_kind} hbm_gbs (copy, burst)", "unit": "GB/s", "frac": t["frac"],
                "traffic": t["traffic"],
                "algorithmic_bytes_per_launch": tee_bytes,
                "bytes_formula": "3 x payload (item rows read once, written to the slab segment and "
                                 "to the prompt row) + 4 B position per placeholder row",
                "measured": (("CUDA events around each tee launch on its stream (a second run of the "
                             "timed schedule, pass time with those events %.4f ms), mean over the passes"
                             % ms_evented) if not overlapped else
                            ("algorithmic bytes per pass / timed pass time: consecutive passes' tee "
                             "launches overlap on two streams (event span of one launch %.4f ms)" % tee_ms)),
                "frac_of_nominal_8000": round(t["achieved_gbs"] / 8000.0, 4),
                "s8d_pass_bytes": s8d_pass_bytes,
                "s8d_pass_gbs": round(s8d_pass_bytes / (ms_step * 1e-3) / 1e9, 1),
                "s8d_note": "SURVEY 8d counts the intra-device forward (2 x payload) and the merge "
                            "(2 x payload + positions) separately; the tee never reads the slab back"}
    if t["traffic"] is None:
        roofline["traffic_note"] = t["traffic_note"]
    value = payload / (ms_step * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (reference synth_payload bytes, K0 on device)",
        "merged_req_per_s": round(len(reqs) / (ms_step * 1e-3), 1),
        "config": {"workload": CONFIGS[CONFIG]["workload"],
                   "placement": "intra-device forward (producer == consumer GPU) + merge",
                   "schedule": ("scan (side stream, one pass ahead) + fsx_forward_merge" +
                                (" as one CUDA graph per pass (the tee || the next pass's scan)"
                                 if step is step_graph else "") +
                                (" as one CUDA graph per pass, consecutive passes on two streams "
                                 "over two sets of slab segments / prompt rows (held allocated)"
                                 if step is step_graph2 else "")),
                   "requests_per_step": len(reqs), "payload_bytes_per_step": payload,
                   "chunk_bytes": (CHUNK_ROWS or 0) * rules.row_bytes or "single shot",
                   "prompt_rows_per_step": lay.total_rows,
                   "parallelism": "1 GPU", "l2": "inputs larger than L2 (no flush needed)"},
        "roofline": roofline,
        "kernels": kern,
        "schedules": schedules,
        "nvlink": {"applies": False, "why": "N=1: producer and consumer share one B200"},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "host_us_per_step": round(host_us_step, 1),
        "clocks": clk.summary(),
    }
    if not args.profile and not args.no_e2e:
        line["e2e"] = run_e2e(args, fab, reqs, rules, stream)
    if not args.profile and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    fab.close()
    print(json.dumps(line), flush=True)


def run_e2e(args, fab, reqs, rules, stream):
    """Same metric through the C ABI with HOST buffers: pinned host payloads
    are copied into the consumer slab every step (fsx_forward_host), merged,
    and the per-request status is read back to the host."""
    import numpy as np
    import torch

    from paper_2603_12118_b200 import trace as T
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    # host->device copies per flagged chunk: 4 frames (28 MiB) -- every H2D copy
    # costs a fixed gap on the copy engine, and 7 MiB copies lose ~3 % of the
    # PCIe rate (profiles/e2e_chunk_sweep_r01g.jsonl)
    e2e_chunk = 4 * CHUNK_ROWS if CHUNK_ROWS else None
    batch = DataPlaneBatch(fab, reqs, rules, src_gpu=0, dst_gpu=1, chunk_rows=e2e_chunk)
    with torch.cuda.stream(stream):
        batch.synth_inputs(stream)
    torch.cuda.synchronize()
    # the producer's outputs in one pinned buffer, item i at src_off[i] (the
    # same layout as on the device); views per item
    pinned = torch.empty(batch.src_buf.numel(), dtype=torch.uint8, pin_memory=True)
    pinned.copy_(batch.src_buf)
    host = []
    for i, it in enumerate(batch.lay.items):
        nb = it.rows * batch.rb
        off = int(batch.src_off[i])
        host.append(pinned[off:off + nb].numpy())
    status_h = torch.empty(len(reqs), dtype=torch.int32, pin_memory=True)
    h2d = sum(h.nbytes for h in host)
    # the merge follows the host->device copy chunk by chunk (early start on
    # the per-chunk flags the copy publishes) on a high-priority stream, so a
    # step costs the PCIe transfer plus the last chunk's merge
    from paper_2603_12118_b200 import _native as N
    mstream = torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])

    def step():
        assert batch.alloc()
        batch.forward_host(host, stream)
        with torch.cuda.stream(mstream):
            batch.merge(mstream, early_start=True,
                        mode=N.MERGE_FULL | N.MERGE_COLOCATED | N.MERGE_DISCARD)
            status_h.copy_(batch.status[:len(reqs)], non_blocking=True)
        mstream.synchronize()
        stream.synchronize()
        batch.release()
        if int(status_h.numpy().max()) != 0:
            raise RuntimeError("merge validation failed in e2e step")

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
        steps = max(5, min(args.steps, 20))
        t0 = time.perf_counter()
        for _ in range(steps):
            step()
        dt = (time.perf_counter() - t0) / steps
        # PCIe ceiling of this box: one pinned host -> device copy of the same
        # bytes (torch copy_, cudaMemcpyAsync), timed the same way
        dev_buf = torch.empty(h2d, dtype=torch.uint8, device="cuda")
        pin = torch.empty(h2d, dtype=torch.uint8, pin_memory=True)
        dev_buf.copy_(pin, non_blocking=True)
        stream.synchronize()
        t1 = time.perf_counter()
        for _ in range(3):
            dev_buf.copy_(pin, non_blocking=True)
        stream.synchronize()
        h2d_peak = h2d / ((time.perf_counter() - t1) / 3) / 1e9
        del dev_buf, pin
    return {"value": round(h2d / dt / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 4 * len(reqs), "ms_per_step": round(dt * 1e3, 3),
            "steps": steps, "pcie_h2d_copy_gbs": round(h2d_peak, 2),
            "frac_of_pcie_h2d": round(h2d / dt / 1e9 / h2d_peak, 3),
            "path": "fsx_forward_host (pinned host -> consumer slab, per-frame chunks + flags) "
                    "-> fsx_merge (early start on the copy's chunk flags) -> status D2H, wall clock "
                    "per step",
            "boundary": "per step the payload crosses PCIe host->device and the per-request merge "
                        "status comes back; token ids, the prompt's text rows and the merge "
                        "descriptors stay on the device across steps (the on-GPU LLM consumer owns "
                        "them).  The reference executors send from pageable vectors: that path "
                        "(through the drop-in C++ API) is profiles/bench_fabric_dropin_r02.jsonl"}


# ---------------------------------------------------------------------------
# fsx arm, N GPUs: independent producer->consumer pairs

def _probe_k1(args, run_steps, red_dev, first):
    """--k1 auto: every rank runs 5 steps with each K1 form (the consumers'
    side is the same for all); the form with the lowest max-over-ranks
    device time per step is used for the timed region.  Returns (form,
    {form: ms per step}, next step number)."""
    import torch
    import torch.distributed as dist

    if args.k1 != "auto":
        return args.k1, {}, first
    probe = {}
    s = first
    for form in K1_FORMS:
        run_steps(form, s, 2)  # warm this form
        s += 2
        ms = torch.tensor([run_steps(form, s, 5)], dtype=torch.float64, device=red_dev)
        s += 5
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        probe[form] = round(ms.item() / 5, 4)
    return min(probe, key=probe.get), probe, s


def run_pairs(args, rank, world):
    """One process per GPU: rank 2k pushes its encoder outputs into rank
    2k+1's receive slab over NVLink (K1 on the producer, CUDA IPC mapping);
    rank 2k+1 merges with in-kernel early start on the chunk flags (K3) and
    acks the step into the producer's ack flag.  The consumer holds `--sets`
    sets of slab segments (and prompt batches) so step s+1's transfer never
    waits for step s's merge and ack: the producer only waits for the ack of
    step s-sets of the same set.  No collective on the data path; timing is
    the max over ranks of the device-timed region."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_12118_b200 import _native as N
    from paper_2603_12118_b200 import pairs as PR
    from paper_2603_12118_b200 import trace as T
    from paper_2603_12118_b200.dataplane import DataPlaneBatch
    from paper_2603_12118_b200.fabric import DeviceFabric, _stream_ptr

    local, pinned, red_dev = _rank_device(args, rank)
    me = PR.role(rank, world)
    P, Cg = me.producer_gpu, me.consumer_gpu
    rules = T.RULES[CONFIG]
    reqs = T.config_requests(CONFIG, args.requests)
    lay = T.layout(reqs, rules.row_bytes)
    stream = torch.cuda.Stream(device=local)
    sets = 1 if me.alone else max(1, args.sets)
    slab_bytes = max(1 << 30, sets * lay.payload_bytes + (64 << 20))
    # both logical gpus of the pair are bound to this process's device; the
    # peer's slab is imported (mapped over NVLink) under its logical id
    fab = DeviceFabric({P: 0, Cg: 0}, {P: local, Cg: local})
    if me.alone:
        fab.slab_register(Cg, slab_bytes)
        mine = None
    elif me.producer:
        fab.slab_register(P, 1 << 20)  # ack flags (one per segment set) live in this small slab
        mine = fab.slab_export(P)
    else:
        fab.slab_register(Cg, slab_bytes)
        mine = fab.slab_export(Cg)
    handles = PR.exchange(mine)
    if not me.alone:
        fab.slab_import(Cg if me.producer else P, *handles[me.peer])
    consumer = me.alone or not me.producer
    nb = sets if consumer else 1
    batches = [DataPlaneBatch(fab, reqs, rules, P, Cg, chunk_rows=CHUNK_ROWS) for _ in range(nb)]
    batch = batches[0]
    with torch.cuda.stream(stream):
        for b in batches:
            b.synth_inputs(stream)
    if consumer:
        for b in batches:
            assert b.alloc()
    torch.cuda.synchronize()
    offs = PR.exchange(None if not consumer or me.alone else [b.slab_off.tolist() for b in batches])
    set_offs = [np.array(o, dtype=np.int64) for o in offs[me.peer]] if (me.producer and not me.alone) \
        else [b.slab_off for b in batches]
    chunk_rows = CHUNK_ROWS or max(1, max((it.rows for it in lay.items), default=1))
    chunks = [max(1, -(-it.rows // chunk_rows)) for it in lay.items]
    M = len(lay.items)
    # Direct placement over NVLink (--transfer direct): the producer writes
    # each row straight into the consumer's prompt embedding and status
    # (CUDA IPC mappings of the consumer's tensors) with fsx_forward_place --
    # the forward and the merge as ONE kernel over peer memory -- and sets a
    # done flag in the consumer's ring; no slab segment, no consumer merge.
    direct = (not me.alone) and args.transfer == "direct"
    place_mb = []
    if direct:
        from torch.multiprocessing.reductions import reduce_tensor
        shared = PR.exchange([(reduce_tensor(b.embeds), reduce_tensor(b.status)) for b in batches]
                             if consumer else None)
        if me.producer:
            remote = []  # keep the mapped tensors alive for the run
            src_ptrs = torch.from_numpy(batch.src_off + batch.src_buf.data_ptr()).to(stream.device)
            for (fe, ae), (fs, as_) in shared[me.peer]:
                emb, st = fe(*ae), fs(*as_)
                remote.append((emb, st))
                mb = batch.merge_batch(False, N.MERGE_FULL)
                mb.d_embeds = emb.data_ptr()
                mb.d_status = st.data_ptr()
                mb.d_item_src = src_ptrs.data_ptr()
                place_mb.append(mb)
    xfers = (N.Transfer * max(M, 1))()
    view = np.frombuffer(xfers, dtype=N.TRANSFER_DTYPE, count=max(M, 1))[:M]
    for i, it in enumerate(lay.items):
        xfers[i] = N.Transfer(P, Cg, batch.src_buf.data_ptr() + int(batch.src_off[i]), 0,
                              it.rows * batch.rb, chunk_rows * batch.rb, 0, 0, None)
    k1_opts = [0]

    def step(s):
        if me.alone:
            batch.forward(stream, host_notify=False)
            batch.merge(stream)
            return
        k = s % sets
        sched = PR.schedule(s, chunks)
        if direct:
            done, tok = sched[0]  # this step's first flag slot carries the done token
            if me.producer:
                if s >= sets:
                    fab.stream_wait_flags(P, k, 1, PR.ack_token(s - sets), stream)
                fab.forward_place(P, Cg, place_mb[k], done_flag=done, token=tok, stream=stream)
            else:
                fab.stream_wait_flags(Cg, done, 1, tok, stream)
                fab.signal_flags(P, k, 1, PR.ack_token(s), Cg, stream)
            return
        if me.producer:
            if s >= sets:  # the consumer acked step s-sets: segment set k is free again
                fab.stream_wait_flags(P, k, 1, PR.ack_token(s - sets), stream)
            view["dst_off"] = set_offs[k]
            view["flag_base"] = [fb for fb, _ in sched]
            view["token"] = [tok for _, tok in sched]
            N.call("fsx_forward_batch", fab._h, M, xfers, k1_opts[0], _stream_ptr(stream))  # one K1 launch
        else:
            b = batches[k]
            for i in range(M):
                b.flag_base[i], b.tokens[i] = sched[i]
                b.n_chunks[i] = chunks[i]
            # waits per chunk inside K3; merged slab rows are dropped from L2
            b.merge(stream, early_start=True, mode=N.MERGE_FULL | N.MERGE_DISCARD)
            fab.signal_flags(P, k, 1, PR.ack_token(s), Cg, stream)

    def run_steps(form, first, n):
        k1_opts[0] = K1_FORMS[form]
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s in range(first, first + n):
            step(s)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    with torch.cuda.stream(stream):
        for s in range(args.warmup):
            step(s)
        nxt = args.warmup
        form, k1_probe = args.k1 if args.k1 != "auto" else "tile", {}
        if not me.alone and not direct:
            form, k1_probe, nxt = _probe_k1(args, run_steps, red_dev, nxt)
        k1_opts[0] = K1_FORMS[form]
        for s in range(nxt, nxt + 2):
            step(s)
        nxt += 2
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        l0 = fab.stats()["kernel_launches"]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            start.record(stream)
            for s in range(nxt, nxt + args.steps):
                step(s)
            end.record(stream)
            torch.cuda.synchronize()
        dist.barrier()
        launches = fab.stats()["kernel_launches"] - l0
        nxt += args.steps
    e2e = _e2e_phase(args, step, stream, red_dev, PR.pairs_in(world) * lay.payload_bytes,
                     [batch.src_buf] if (me.producer or me.alone) else [],
                     (lambda s: batches[s % sets]) if consumer else None,
                     first=nxt, n_requests=PR.pairs_in(world) * len(reqs))
    # the copy-engine comparator: the producer copies the same items into the
    # same peer slab segments with cudaMemcpyAsync (peer copy), event-timed
    ce_ms = torch.zeros(1, dtype=torch.float64, device=red_dev)
    torch.cuda.synchronize()
    dist.barrier()
    if me.producer and not me.alone and not direct:
        base = fab.slab_ptr(Cg, 0)
        with torch.cuda.stream(stream):
            def copies():
                for i, it in enumerate(lay.items):
                    N.call("fsx_copy_engine", fab._h, P, base + int(set_offs[0][i]),
                           batch.src_buf.data_ptr() + int(batch.src_off[i]), it.rows * batch.rb,
                           _stream_ptr(stream))
            copies()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(5):
                copies()
            b.record(stream)
            torch.cuda.synchronize()
            ce_ms[0] = a.elapsed_time(b) / 5
    dist.all_reduce(ce_ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    verified = None
    if consumer:
        for b in batches:
            st = b.status_host()
            assert (st == 0).all(), st
        if args.verify:
            # the pair-merged prompt embeddings must equal a local intra-device
            # forward + merge of the same requests (both bit-exact to the oracle)
            torch.cuda.synchronize()
            for b in batches:
                b.release()  # the run is over: make room in the slab for the local pass
            local_b = DataPlaneBatch(fab, reqs, rules, P, Cg, chunk_rows=CHUNK_ROWS)
            local_b.synth_inputs()
            assert local_b.alloc()
            local_b.forward(host_notify=False)
            local_b.merge()
            torch.cuda.synchronize()
            verified = all(bool(torch.equal(local_b.embeds, b.embeds)) for b in batches)
            local_b.release()
            assert verified, "pair-merged embeddings differ from the local reference pass"
    ms = torch.tensor([start.elapsed_time(end)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    tot_launch = torch.tensor([launches], dtype=torch.float64, device=red_dev)
    dist.all_reduce(tot_launch)
    # every consumer's check, reduced to rank 0 (1 = bit-exact or no check made there)
    ok = torch.tensor([0.0 if verified is False else 1.0], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    verified = bool(args.verify) and ok.item() == 1.0
    n_pairs = PR.pairs_in(world)
    payload_all = n_pairs * lay.payload_bytes * args.steps
    ms_step = ms.item() / args.steps
    if rank == 0:
        pair_gbs = lay.payload_bytes / (ms_step * 1e-3) / 1e9
        ce = ce_ms.item()
        line = {
            "metric": METRIC, "value": round(payload_all / (ms.item() * 1e-3) / 1e9, 2),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "merged_req_per_s": round(n_pairs * len(reqs) / (ms_step * 1e-3), 1),
            "config": {"workload": CONFIGS[CONFIG]["workload"],
                       "placement": "encoder GPU 2k -> LLM GPU 2k+1 over NVLink (CUDA IPC slab), "
                                    "early-start merge on the consumer",
                       "requests_per_step_per_pair": len(reqs), "pairs": n_pairs,
                       "chunk_bytes": chunk_rows * rules.row_bytes,
                       "slab_segment_sets": sets,
                       "transfer": ("direct placement: fsx_forward_place, producer rows straight "
                                    "into the consumer's prompt rows over NVLink (one kernel), "
                                    "done flag; no slab, no consumer merge") if direct else
                                   f"K1 ({form}) into the consumer slab + early-start merge",
                       "parallelism": f"{n_pairs} independent producer->consumer pairs"},
            "roofline": {"bound": "nvlink", "achieved": round(pair_gbs, 1), "peak": 770.0,
                         "unit": "GB/s", "frac": round(pair_gbs / 770.0, 4), "traffic": None,
                         "traffic_note": "NVLink bytes: scripts/profile_round.sh nvl section "
                                         "(nvltx__bytes / nvlrx__bytes, >= 2-GPU boxes)",
                         "what": "payload per pair per step / max-over-ranks step time",
                         "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                         "frac_of_nominal_900": round(pair_gbs / 900.0, 4)},
            "k1_forms": {"chosen": form, "probe_ms_per_step": k1_probe},
            "copy_engine": ({"what": "cudaMemcpyAsync peer copies (copy engine) of the same items into "
                                     "the same slab segments, no flags, event-timed on the producer",
                             "ms_per_step": round(ce, 4),
                             "pair_gbs": round(lay.payload_bytes / (ce * 1e-3) / 1e9, 1),
                             "k1_over_copy_engine": round(ce / ms_step, 4)} if ce > 0 else None),
            "gpu_launches": int(tot_launch.item()),
            "e2e": e2e,
            "verified": verified,
            "pinned_device": pinned,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    fab.close()
    dist.destroy_process_group()


def _rank_device(args, rank):
    """(device, pinned, reduction device) for one rank: LOCAL_RANK's GPU with
    NCCL for setup/timing, or every rank pinned to --pin-device with gloo (the
    protocol tests on a 1-GPU box: CUDA IPC works between processes of one
    device, NCCL does not allow that)."""
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", rank))
    pinned = args.pin_device
    if pinned is not None:
        local = pinned
    torch.cuda.set_device(local)
    if pinned is None:
        # a rank that dies must not leave the others waiting for the default
        # 10 minutes in a setup collective or barrier
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(minutes=3))
        return local, pinned, "cuda"
    dist.init_process_group("gloo", timeout=datetime.timedelta(minutes=3))
    return local, pinned, "cpu"


def run_fanout(args, rank, world):
    """Config D across the box (BASELINE.json configs[3]): encoder replicas on
    the even ranks, LLM replicas on the odd ranks; every item goes to the LLM
    replica the reference dispatcher policy assigns its request to
    (paper_2603_12118_b200/fanout.py), so encoders fan out to several LLMs and
    LLMs fan in from several encoders.  Each encoder maps the slabs of the LLMs
    it feeds (CUDA IPC) and pushes all its items of a step with one batched K1
    call over NVLink; each LLM merges with in-kernel early start and acks
    every encoder that fed it.  Every LLM holds two sets of slab segments
    (--sets), so an encoder's next transfer does not wait for the
    current merge.  No collective on the data path."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_12118_b200 import _native as N
    from paper_2603_12118_b200 import fanout as FO
    from paper_2603_12118_b200 import pairs as PR
    from paper_2603_12118_b200 import trace as T
    from paper_2603_12118_b200.dataplane import DataPlaneBatch, _align
    from paper_2603_12118_b200.fabric import DeviceFabric, _stream_ptr

    local, pinned, red_dev = _rank_device(args, rank)
    rules = T.RULES[CONFIG]
    rb = rules.row_bytes
    n_prod = len(range(0, world, 2))
    reqs = T.config_requests(CONFIG, args.requests * n_prod)  # weak scaling: per encoder
    chunk_rows = CHUNK_ROWS or max(it.rows for q in reqs for it in q.items)
    pl = FO.plan(reqs, world, chunk_rows)
    producer = rank % 2 == 0
    me = rank // 2  # encoder ordinal (even ranks) / LLM ordinal (odd ranks)
    stream = torch.cuda.Stream(device=local)
    fab = DeviceFabric({g: 0 for g in range(world)}, {g: local for g in range(world)})
    sets = max(1, args.sets)
    batch, batches = None, []
    if producer:
        fab.slab_register(rank, 1 << 20)  # ack flags: index = LLM ordinal x sets + set
        mine = fab.slab_export(rank)
    else:
        reqs_c = [reqs[k] for k in pl.consumer_requests(me)]
        batches = [DataPlaneBatch(fab, reqs_c, rules, rank, rank, chunk_rows=chunk_rows)
                   for _ in range(sets)]
        batch = batches[0]
        fab.slab_register(rank, max(1 << 30, (sets + 1) * batch.lay.payload_bytes + (64 << 20)))
        mine = fab.slab_export(rank)
    handles = PR.exchange(mine)
    peers = ([pl.consumers[c] for c in pl.consumers_of(me)] if producer
             else [pl.producers[p] for p in pl.producers_of(me)])
    for r in peers:
        fab.slab_import(r, *handles[r])
    for b in batches:
        with torch.cuda.stream(stream):
            b.synth_inputs(stream)
        assert b.alloc()
    torch.cuda.synchronize()
    offs = PR.exchange(None if producer else [b.slab_off.tolist() for b in batches])

    items = pl.producer_items(me) if producer else []
    xfers = (N.Transfer * max(len(items), 1))()
    view = np.frombuffer(xfers, dtype=N.TRANSFER_DTYPE, count=max(len(items), 1))[:len(items)]
    slots = [pl.item_slot(k, j) for k, j in items]
    my_bytes = 0
    src_buf = None
    if producer:
        sizes = [reqs[k].items[j].rows * rb for k, j in items]
        src_off = np.concatenate([[0], np.cumsum([_align(n) for n in sizes])]).astype(np.int64)
        src_buf = torch.empty(max(int(src_off[-1]), 256), dtype=torch.uint8, device=local)
        for i, (k, j) in enumerate(items):
            it = reqs[k].items[j]
            fab.synth(rank, T.payload_seed(it.ref_id, 0), src_buf.data_ptr() + int(src_off[i]),
                      sizes[i], stream)
            c, idx = slots[i]
            xfers[i] = N.Transfer(rank, pl.consumers[c], src_buf.data_ptr() + int(src_off[i]),
                                  0, sizes[i], chunk_rows * rb, 0, 0, None)
        my_bytes = int(sum(sizes))
        torch.cuda.synchronize()
    # destination offsets of every item in each segment set of its LLM
    set_offs = [np.array([int(offs[pl.consumers[c]][k][idx]) for c, idx in slots], dtype=np.int64)
                for k in range(sets)] if producer else []
    acks_from = pl.consumers_of(me) if producer else []
    acks_to = pl.producers_of(me) if not producer else []
    k1_opts = [0]

    def step(s):
        k = s % sets
        if producer:
            if s >= sets:  # every LLM this encoder fed acked step s-sets: set k is free again
                for c in acks_from:
                    fab.stream_wait_flags(rank, c * sets + k, 1, PR.ack_token(s - sets), stream)
            if items:
                sch = [pl.schedule(s, c, idx) for c, idx in slots]
                view["dst_off"] = set_offs[k]
                view["flag_base"] = [b for b, _ in sch]
                view["token"] = [t for _, t in sch]
                N.call("fsx_forward_batch", fab._h, len(items), xfers, k1_opts[0], _stream_ptr(stream))
        else:
            b = batches[k]
            for idx, (q, j) in enumerate(pl.consumer_items[me]):
                b.flag_base[idx], b.tokens[idx] = pl.schedule(s, me, idx)
                b.n_chunks[idx] = pl.chunks[q][j]
            # waits per chunk inside K3; merged slab rows are dropped from L2
            b.merge(stream, early_start=True, mode=N.MERGE_FULL | N.MERGE_DISCARD)
            for p in acks_to:
                fab.signal_flags(pl.producers[p], me * sets + k, 1, PR.ack_token(s), rank, stream)

    def run_steps(form, first, n):
        k1_opts[0] = K1_FORMS[form]
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s in range(first, first + n):
            step(s)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    with torch.cuda.stream(stream):
        for s in range(args.warmup):
            step(s)
        form, k1_probe, nxt = _probe_k1(args, run_steps, red_dev, args.warmup)
        if args.k1 == "auto" and not k1_probe:
            form = "tile"
        k1_opts[0] = K1_FORMS[form]
        for s in range(nxt, nxt + 2):
            step(s)
        nxt += 2
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        l0 = fab.stats()["kernel_launches"]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            start.record(stream)
            for s in range(nxt, nxt + args.steps):
                step(s)
            end.record(stream)
            torch.cuda.synchronize()
        dist.barrier()
        launches = fab.stats()["kernel_launches"] - l0
        nxt += args.steps
    verified = None
    total_payload = sum(it.rows * rb for q in reqs for it in q.items)
    e2e = _e2e_phase(args, step, stream, red_dev, total_payload,
                     [src_buf] if producer else [],
                     (lambda s: batches[s % sets]) if not producer else None,
                     first=nxt, n_requests=len(reqs))
    if not producer:
        for b in batches:
            st = b.status_host()
            assert (st == 0).all(), st
        if args.verify:
            local_b = DataPlaneBatch(fab, batch.lay.requests, rules, rank, rank, chunk_rows=chunk_rows)
            local_b.synth_inputs()
            assert local_b.alloc()
            local_b.forward(host_notify=False)
            local_b.merge()
            torch.cuda.synchronize()
            ok = all(bool(torch.equal(local_b.embeds, b.embeds)) for b in batches)
            local_b.release()
            verified = ok
            assert ok, "fan-in merged embeddings differ from the local reference pass"
    ms = torch.tensor([start.elapsed_time(end)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    tot_launch = torch.tensor([launches], dtype=torch.float64, device=red_dev)
    dist.all_reduce(tot_launch)
    okt = torch.tensor([0.0 if verified is False else 1.0], dtype=torch.float64, device=red_dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    verified = bool(args.verify) and okt.item() == 1.0
    # per-encoder egress and per-LLM ingress bytes of a step (NVLink direction bound)
    io = torch.tensor([my_bytes if producer else batch.lay.payload_bytes], dtype=torch.float64,
                      device=red_dev)
    io_all = [torch.zeros_like(io) for _ in range(world)]
    dist.all_gather(io_all, io)
    ms_step = ms.item() / args.steps
    if rank == 0:
        egress = [io_all[r].item() for r in pl.producers]
        ingress = [io_all[r].item() for r in pl.consumers]
        busiest = max(egress + ingress) / (ms_step * 1e-3) / 1e9
        fan_out = [len(pl.consumers_of(p)) for p in range(len(pl.producers))]
        fan_in = [len(pl.producers_of(c)) for c in range(len(pl.consumers))]
        line = {
            "metric": METRIC, "value": round(total_payload / (ms_step * 1e-3) / 1e9, 2),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "merged_req_per_s": round(len(reqs) / (ms_step * 1e-3), 1),
            "config": {"workload": CONFIGS[CONFIG]["workload"],
                       "placement": "encoders on even ranks -> LLM replicas on odd ranks, reference "
                                    "TaskDispatcher placement (fan-out / fan-in over NVLink), "
                                    f"K1 ({form}), early-start merge",
                       "requests_per_step": len(reqs), "requests_per_encoder": args.requests,
                       "encoders": len(pl.producers), "llms": len(pl.consumers),
                       "fan_out": fan_out, "fan_in": fan_in,
                       "egress_bytes_per_encoder": egress, "ingress_bytes_per_llm": ingress,
                       "chunk_bytes": chunk_rows * rb,
                       "parallelism": f"{len(pl.producers)} encoder GPUs x {len(pl.consumers)} LLM GPUs"},
            "roofline": {"bound": "nvlink", "achieved": round(busiest, 1), "peak": 770.0,
                         "unit": "GB/s", "frac": round(busiest / 770.0, 4), "traffic": None,
                         "what": "busiest GPU's NVLink direction (max encoder egress / LLM ingress)",
                         "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                         "frac_of_nominal_900": round(busiest / 900.0, 4)},
            "k1_forms": {"chosen": form, "probe_ms_per_step": k1_probe},
            "gpu_launches": int(tot_launch.item()),
            "e2e": e2e,
            "verified": verified,
            "pinned_device": pinned,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    fab.close()
    dist.destroy_process_group()


def _e2e_phase(args, step, stream, red_dev, payload_all, src_bufs, recv_batch, first, n_requests):
    """e2e at N > 1 with HOST buffers: every step each sender copies its
    source buffer from pinned host memory onto its GPU (H2D) before pushing
    it (K1 over NVLink); each receiver merges and reads its per-request status
    back (D2H).  Wall clock per step, synchronised per step, max over ranks;
    the flag/token schedule continues after the device-timed steps."""
    import torch
    import torch.distributed as dist

    host = []
    for b in src_bufs:
        h = torch.empty(b.numel(), dtype=torch.uint8, pin_memory=True)
        h.copy_(b)
        host.append(h)
    recv_of = recv_batch if callable(recv_batch) else (lambda s: recv_batch)
    first_recv = recv_of(first)
    nreq = len(first_recv.lay.requests) if first_recv is not None else 0
    status_h = torch.empty(max(nreq, 1), dtype=torch.int32, pin_memory=True)

    def e2e_step(s):
        for h, d in zip(host, src_bufs):
            d.copy_(h, non_blocking=True)
        step(s)
        if recv_batch is not None:
            status_h[:nreq].copy_(recv_of(s).status[:nreq], non_blocking=True)
        stream.synchronize()
        if recv_batch is not None and nreq and int(status_h[:nreq].numpy().max()) != 0:
            raise RuntimeError("merge validation failed in e2e step")

    steps = max(5, min(args.steps, 20))
    with torch.cuda.stream(stream):
        for s in range(first, first + 3):
            e2e_step(s)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for s in range(first + 3, first + 3 + steps):
            e2e_step(s)
        dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    per_step = t.item() / steps
    return {"value": round(payload_all / per_step / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": payload_all, "d2h_bytes_per_step": 4 * n_requests,
            "ms_per_step": round(per_step * 1e3, 3), "steps": steps,
            "path": "senders: pinned host -> own GPU (H2D) -> fsx_forward (K1 over NVLink into the "
                    "receiver's slab); receivers: early-start fsx_merge -> status D2H; wall clock "
                    "per step, max over ranks"}


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks of this
    script with the torchrun environment (RANK, LOCAL_RANK, WORLD_SIZE,
    MASTER_ADDR=127.0.0.1, MASTER_PORT) and wait for all; rank 0 prints the
    line.  Returns the worst exit code."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


def main():
    global CONFIG, REQUESTS, CHUNK_ROWS
    args = parse()
    CONFIG = args.config
    REQUESTS = CONFIGS[CONFIG]["requests"]
    CHUNK_ROWS = args.chunk_rows or CONFIGS[CONFIG]["chunk_rows"]
    if args.requests is None:
        args.requests = REQUESTS
    if args.gpus > 1 and "RANK" not in os.environ and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if CONFIG == "C":
        if rank == 0:
            run_config_c(args)  # a single-GPU decode-step line (channels); no N > 1 form
        return
    if world <= 1:
        run_single(args)
    elif CONFIG == "D":
        run_fanout(args, rank, world)
    else:
        run_pairs(args, rank, world)


if __name__ == "__main__":
    main()
