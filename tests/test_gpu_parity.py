"""GPU parity: the sm_100a kernels through the C ABI against the oracle.

Bar: bit-exact bytes (integer/byte work).  Inputs are the reference's own
synthetic payloads (synth_payload(payload_seed(ref_id, seq))), which include
bf16 NaN/Inf bit patterns.
"""
import hashlib

import time

import numpy as np
import pytest

from paper_2603_12118_b200 import _native as N
from paper_2603_12118_b200 import trace as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fab(gpu):
    from paper_2603_12118_b200.fabric import DeviceFabric

    # two logical GPUs bound to device 0 (1-GPU box): producer 0, consumer 1;
    # gpus 4-7 on node 1 like tests/test_sidecar.cpp:15-20
    f = DeviceFabric({g: (0 if g < 4 else 1) for g in range(8)}, {g: 0 for g in range(8)})
    f.slab_register(1, 1 << 30)
    f.slab_register(2, 64 << 20)
    yield f
    f.close()


def _torch():
    import torch

    return torch


def test_route_and_topology(fab):
    assert fab.route(0, 3) == N.LOCAL_BUFFER
    assert fab.route(0, 0) == N.LOCAL_BUFFER
    assert fab.route(1, 4) == N.NETWORK_STREAM
    with pytest.raises(N.FsxError) as e:
        fab.route(0, 99)
    assert e.value.code == "not_found"


_SYNTH_SIZES = [0, 1, 7, 8, 15, 16, 17, 31, 4096, 4099, 65536 + 5, (1 << 20) + 3]


# every small size at every alignment; the 112 MiB video aligned, and a
# 16 MiB + 3 span through the unaligned path
@pytest.mark.parametrize("n,shift", [(n, sh) for n in _SYNTH_SIZES for sh in (0, 8, 3)] +
                         [(117_440_512, 0), ((16 << 20) + 3, 3), ((16 << 20) + 3, 8)])
def test_synth_matches_reference_stream(fab, oracle_mod, n, shift):
    torch = _torch()
    seed = T.payload_seed("req-000000/r0000", 0)
    buf = torch.zeros(n + 32, dtype=torch.uint8, device="cuda")
    fab.synth(0, seed, buf.data_ptr() + shift, n)
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    want = np.frombuffer(oracle_mod.synth_payload(seed, n), np.uint8)
    assert np.array_equal(got[shift:shift + n], want)
    assert not got[:shift].any() and not got[shift + n:].any()


def test_synth_kat_appendix(fab, kat):
    torch = _torch()
    for case in kat["appendix_a"]:
        buf = torch.empty(case["n"], dtype=torch.uint8, device="cuda")
        fab.synth(0, int(case["seed"], 16), buf.data_ptr(), case["n"])
        torch.cuda.synchronize()
        h = hashlib.sha256(buf.cpu().numpy().tobytes()).hexdigest()
        assert h == case["sha256"], case["case"]


def _forward_check(fab, oracle_mod, n, chunk, src_shift=0, dst_gpu=1, dma=None):
    torch = _torch()
    seed = T.fnv1a64(f"req-x/r{n}")
    src = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    fab.synth(0, seed, src.data_ptr() + src_shift, n)
    off = fab.slab_alloc(dst_gpu, n)
    assert off is not None and off % 64 == 0
    nchunks = 1 if chunk <= 0 or chunk >= n else -(-n // chunk)
    fb = fab.flags_alloc(dst_gpu, nchunks)
    d0 = fab.stats()["dma_forwards"]
    tok = fab.forward(0, src.data_ptr() + src_shift, dst_gpu, off, n, chunk, fb, dma=dma)
    # which form ran: FSX_FWD_DMA / FSX_FWD_KERNEL as asked, else the library's
    # rule (copy engine for one local single-chunk transfer of <= 16 MiB)
    auto_dma = nchunks <= N.FWD_DMA_MAX_CHUNKS and n <= (16 << 20)
    assert fab.stats()["dma_forwards"] - d0 == int(auto_dma if dma is None else dma)
    fab.wait(dst_gpu, fb, nchunks, tok, timeout_us=20_000_000)
    for c in range(nchunks):
        assert fab.chunk_ready(dst_gpu, fb + c, tok)
    got = fab.slab_read(dst_gpu, off, n)
    want = oracle_mod.synth_payload(seed, n)
    assert got == want
    fab.slab_free(dst_gpu, off)


# forms: None = the library's choice, False = K1 forced (FSX_FWD_KERNEL),
# True = the copy-engine form forced (FSX_FWD_DMA)
@pytest.mark.parametrize("dma", [None, False, True], ids=["auto", "kernel", "dma"])
@pytest.mark.parametrize("n", [0, 1, 7, 256, 4096, 65536, 1 << 20, 8 << 20, 64 << 20, 256 << 20])
def test_forward_single_shot_byte_exact(fab, oracle_mod, n, dma):
    # tests/test_sidecar.cpp:60-87 sizes; single-shot = one chunk, one flag
    _forward_check(fab, oracle_mod, n, 0, dma=dma)


@pytest.mark.parametrize("dma", [None, False, True], ids=["auto", "kernel", "dma"])
@pytest.mark.parametrize("n,chunk", [(1 << 20, 65536), (8 << 20, 1 << 20), (7_340_032 * 3 + 48, 7_340_032),
                                     (300_017, 4096), (65536 * 7 + 5, 65536), (4 << 20, 1 << 20)])
def test_forward_chunked_flags(fab, oracle_mod, n, chunk, dma):
    _forward_check(fab, oracle_mod, n, chunk, dma=dma)


@pytest.mark.parametrize("dma", [None, False, True], ids=["auto", "kernel", "dma"])
def test_forward_unaligned_source(fab, oracle_mod, dma):
    _forward_check(fab, oracle_mod, 100_003, 0, src_shift=3, dma=dma)
    _forward_check(fab, oracle_mod, 100_003, 4096, src_shift=5, dma=dma)


def test_forward_dma_form_in_graph_publishes_flags(fab, oracle_mod):
    """The copy-engine form captured in a CUDA graph (memcpy node + memory-op
    flag nodes): every replay lands the bytes and sets each chunk flag to the
    replay's token only after its bytes (an early-start merge / fsx_wait
    consumer sees the same protocol as K1's)."""
    torch = _torch()
    n, chunk = 3 << 20, 1 << 20
    seed = T.fnv1a64("req-dma/graph")
    src = torch.empty(n, dtype=torch.uint8, device="cuda")
    fab.synth(0, seed, src.data_ptr(), n)
    off = fab.slab_alloc(1, n)
    fb = fab.flags_alloc(1, 3)
    s = torch.cuda.Stream()
    tok = (1 << 41) + 7
    g = torch.cuda.CUDAGraph()
    d0 = fab.stats()["dma_forwards"]
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fab.forward(0, src.data_ptr(), 1, off, n, chunk, fb, s, token=tok, dma=True)
    assert fab.stats()["dma_forwards"] - d0 == 1
    want = oracle_mod.synth_payload(seed, n)
    for r in range(3):
        fab.synth(1, seed + 1 + r, fab.slab_ptr(1, off), n)  # scribble over the segment
        torch.cuda.synchronize()
        assert fab.slab_read(1, off, n) != want
        g.replay()
        if r == 0:  # fresh flags: the host mirror turns to tok only behind the bytes
            fab.wait(1, fb, 3, tok, timeout_us=20_000_000)
        else:
            s.synchronize()
        assert all(fab.chunk_ready(1, fb + c, tok) for c in range(3))
        assert fab.slab_read(1, off, n) == want
    fab.slab_free(1, off)


def test_forward_rejects_bad_chunk_and_overrun(fab):
    torch = _torch()
    src = torch.empty(4096, dtype=torch.uint8, device="cuda")
    fb = fab.flags_alloc(1, 4)
    with pytest.raises(N.FsxError) as e:
        fab.forward(0, src.data_ptr(), 1, 0, 4096, 1000, fb)
    assert e.value.code == "validation"
    cap = fab.slab_usage(2)["capacity"]
    with pytest.raises(N.FsxError) as e:
        fab.forward(0, src.data_ptr(), 2, cap - 100, 4096, 0, fb)
    assert e.value.code == "validation"


def test_forward_batch_mixed(fab, oracle_mod):
    """K1 launches over transfers of different sizes, chunkings, alignments
    and destination slabs (more than FSX_FWD_MAX_BATCH, so two launches)."""
    torch = _torch()
    specs = [(n, ch, sh, dst) for n, ch, sh, dst in
             [(0, 0, 0, 1), (1, 0, 0, 2), (4099, 0, 3, 1), (1 << 20, 65536, 0, 2),
              (7_340_032 * 2 + 32, 7_340_032, 0, 1), (65536 * 3, 4096, 0, 2)] * 12]
    assert len(specs) > N.FWD_MAX_BATCH
    srcs, xfers, offs = [], [], []
    for k, (n, ch, sh, dst) in enumerate(specs):
        buf = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
        fab.synth(0, 1000 + k, buf.data_ptr() + sh, n)
        off = fab.slab_alloc(dst, n)
        nch = 1 if ch <= 0 or ch >= n else -(-n // ch)
        fb = fab.flags_alloc(dst, nch)
        srcs.append(buf)
        offs.append((dst, off, fb, nch))
        xfers.append((0, buf.data_ptr() + sh, dst, off, n, ch, fb, 0))
    toks = fab.forward_batch(xfers)
    assert len(set(toks)) == len(toks)
    for k, (n, ch, sh, dst) in enumerate(specs):
        d, off, fb, nch = offs[k]
        fab.wait(d, fb, nch, toks[k], timeout_us=20_000_000)
        assert fab.slab_read(d, off, n) == oracle_mod.synth_payload(1000 + k, n), specs[k]
        fab.slab_free(d, off)


@pytest.mark.parametrize("n,chunk,shift", [(0, 0, 0), (5, 0, 0), (4096, 0, 0), (4099, 0, 0),
                                           (1 << 20, 65536, 0), (7_340_032 * 2 + 40, 7_340_032, 0),
                                           (100_003, 0, 3), (65536 + 9, 4096, 8)])
def test_fused_digest_matches_oracle(fab, oracle_mod, n, chunk, shift):
    """dg64 fused into K1 (aligned path) or the fallback pass (unaligned), and
    fsx_digest over the delivered slab segment, equal the oracle restatement."""
    torch = _torch()
    seed = 4242 + n
    src = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    fab.synth(0, seed, src.data_ptr() + shift, n)
    want = oracle_mod.C.or_digest64(oracle_mod.synth_payload(seed, n), n)
    off = fab.slab_alloc(1, n)
    nch = 1 if chunk <= 0 or chunk >= n else -(-n // chunk)
    fb = fab.flags_alloc(1, nch)
    slot = fab.u64_slot(0)
    (tok,) = fab.forward_batch([(0, src.data_ptr() + shift, 1, off, n, chunk, fb, 0, slot)])
    fab.wait(1, fb, nch, tok, timeout_us=20_000_000)
    torch.cuda.synchronize()
    assert fab.read_u64(0, slot) == want
    assert fab.digest(1, fab.slab_ptr(1, off), n) == want
    fab.slab_free(1, off)


def test_digest_detects_corruption(fab, oracle_mod):
    torch = _torch()
    buf = torch.empty(1 << 16, dtype=torch.uint8, device="cuda")
    fab.synth(0, 9, buf.data_ptr(), buf.numel())
    d0 = fab.digest(0, buf.data_ptr(), buf.numel())
    buf[1000] ^= 1
    assert fab.digest(0, buf.data_ptr(), buf.numel()) != d0
    buf[1000] ^= 1
    swapped = torch.cat([buf[32768:], buf[:32768]])
    assert fab.digest(0, swapped.data_ptr(), swapped.numel()) != d0
    assert fab.digest(0, buf.data_ptr(), buf.numel()) == d0


def test_forward_host_span_path(fab, oracle_mod):
    for n, chunk in [(0, 0), (1, 0), (4097, 0), (3 << 20, 1 << 20)]:
        payload = np.frombuffer(oracle_mod.synth_payload(n + 11, n), np.uint8).copy()
        off = fab.slab_alloc(1, n)
        nchunks = 1 if chunk <= 0 or chunk >= n else -(-n // chunk)
        fb = fab.flags_alloc(1, nchunks)
        tok = fab.forward_host(payload.ctypes.data if n else 0, 1, off, n, chunk, fb)
        fab.wait(1, fb, nchunks, tok, timeout_us=20_000_000)
        assert fab.slab_read(1, off, n) == payload.tobytes()
        fab.slab_free(1, off)


def test_forward_host_digest_matches_oracle(fab, oracle_mod):
    """fsx_forward_host_digest (the drop-in's host-span send): the bytes land
    byte-exact and the returned dg64 -- fused into the staging copy for a
    pageable source >= 4 MiB, computed alongside the DMA otherwise (small
    pageable, pinned) -- equals the oracle's, for unaligned lengths and
    chunked copies."""
    import ctypes as C

    torch = _torch()
    cases = [(1, 0, False), (4097, 0, False), (5 << 20, 0, False), ((17 << 20) + 13, 3 << 20, False),
             ((6 << 20) + 5, 0, True), ((6 << 20) + 5, 0, False), (40 << 20, 7 << 20, False)]
    # (6 MiB + 5 splits into 6 copy-thread parts whose 64-byte-rounded size
    # once left the last 5 bytes uncopied)
    for n, chunk, pinned in cases:
        data = oracle_mod.synth_payload(n + 77, n)
        if pinned:
            buf = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            buf.numpy()[:] = np.frombuffer(data, np.uint8)
            ptr = buf.data_ptr()
        else:
            arr = np.frombuffer(data, np.uint8).copy()
            ptr = arr.ctypes.data
        off = fab.slab_alloc(1, n)
        nchunks = 1 if chunk <= 0 or chunk >= n else -(-n // chunk)
        fb = fab.flags_alloc(1, nchunks)
        tok, dg = C.c_uint64(0), C.c_uint64(0)
        N.call("fsx_forward_host_digest", fab._h, ptr, 1, off, n, chunk, fb, C.byref(tok), None, C.byref(dg))
        fab.wait(1, fb, nchunks, tok.value, timeout_us=20_000_000)
        assert dg.value == oracle_mod.C.or_digest64(data, n), (n, chunk, pinned)
        assert fab.slab_read(1, off, n) == data
        fab.slab_free(1, off)


def test_slab_allocator_replays_reference_nodearena(fab, kat):
    # NodeArena op trace produced by the reference (sidecar.hpp:106-205)
    from paper_2603_12118_b200.fabric import DeviceFabric

    tr = kat["arena_trace"]
    with DeviceFabric({0: 0}, {0: 0}) as f:
        f.slab_register(0, tr["capacity"])
        for op, arg, res, segs, used in tr["ops"]:
            if op == "alloc":
                off = f.slab_alloc(0, arg)
                assert (-1 if off is None else off) == res
            else:
                if res == 0:
                    f.slab_free(0, arg)
                else:
                    with pytest.raises(N.FsxError) as e:
                        f.slab_free(0, arg)
                    assert e.value.code == "internal"
            u = f.slab_usage(0)
            assert (u["segments_in_use"], u["bytes_in_use"]) == (segs, used)


# ---------------------------------------------------------------------------
# Merge


def _expected(oracle_mod, batch):
    """Oracle: same inputs on the host, CPU merge restatement."""
    O = oracle_mod
    lay, rb = batch.lay, batch.rb
    emb = np.concatenate([np.frombuffer(O.synth_payload(T.text_seed(q), q.total_rows * rb), np.uint8)
                          for q in lay.requests]).copy()
    src = [np.frombuffer(O.synth_payload(T.payload_seed(it.ref_id, 0), it.rows * rb), np.uint8)
           for it in lay.items]
    st = O.merge(rb, batch.pid, emb, batch.tok_host, lay.req_row_off, lay.req_item_off, src,
                 lay.item_rows, nthreads=8)
    return emb, st


def _run_batch(fab, reqs, rules, chunk_rows=None, path="serial", tok_override=None):
    """One data-plane pass over `reqs` by `path`: "serial" (K1 register tiles,
    then the merge), "bulk" (bulk-copy K1, then the merge), "early" (K1, then
    the early-start merge following the chunk flags) or "tee" (the fused
    forward + merge, fsx_forward_merge, with host-mirrored flags)."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    b = DataPlaneBatch(fab, reqs, rules, 0, 1, chunk_rows=chunk_rows)
    if tok_override is not None:
        tok_override(b)
    b.synth_inputs()
    assert b.alloc()
    if path == "tee":
        b.tee(mode=N.MERGE_FULL, host_notify=True)
        b.wait_host()  # every chunk flag of every item published
    elif path == "early":
        b.forward()
        b.merge(early_start=True)
    else:
        b.forward(bulk=path == "bulk")
        torch.cuda.synchronize()
        b.merge()
    torch.cuda.synchronize()
    return b


@pytest.mark.parametrize("path", ["serial", "bulk", "tee", "early"])
@pytest.mark.parametrize("config,count,chunk_rows", [("A", 64, None), ("A", 5, 64), ("D", 24, 1024),
                                                     ("B", 1, 1024),
                                                     # the bench batches at full BASELINE size
                                                     ("B", 4, 1024), ("D", 32, 1024)])
def test_merge_bit_exact(fab, oracle_mod, config, count, chunk_rows, path):
    rules = {"A": T.RULES["A"], "B": T.RULES["B"], "D": T.RULES["D"]}[config]
    reqs = T.config_requests(config, count)
    b = _run_batch(fab, reqs, rules, chunk_rows, path)
    want, st = _expected(oracle_mod, b)
    assert (b.status_host() == 0).all() and (st == 0).all()
    got = b.embeds_host()
    assert np.array_equal(got, want)
    # the forwarded slab bytes themselves (ChunkCallback delivery parity)
    for i in sorted({0, 1, len(b.lay.items) // 2, len(b.lay.items) - 1}):
        if not 0 <= i < len(b.lay.items):
            continue
        it = b.lay.items[i]
        exp = oracle_mod.synth_payload(T.payload_seed(it.ref_id, 0), it.rows * b.rb)
        assert b.slab_item_host(i).tobytes() == exp
    b.release()
    assert fab.slab_usage(1)["segments_in_use"] == 0


@pytest.mark.parametrize("path", ["serial", "tee"])
@pytest.mark.parametrize("config", ["A", "B", "D"])
def test_merge_matches_reference_derived_golden(fab, config, path):
    """The GPU pass (K1 into the slab, K3 merge) produces exactly the prompt
    embeddings built from the bytes the REFERENCE SidecarFabric delivered,
    placed in the slot order the reference record() gives the consumer
    (tests/golden/record_dispatch.json, merged_sha256; make_golden.py)."""
    import hashlib
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "record_dispatch.json")) as fh:
        want = json.load(fh)["merged_sha256"][config]
    reqs = T.config_requests(config, want["requests"])
    b = _run_batch(fab, reqs, T.RULES[config], 1024 if config != "A" else None, path)
    assert (b.status_host() == 0).all()
    assert hashlib.sha256(b.embeds_host().tobytes()).hexdigest() == want["sha256"]
    b.release()


def test_follow_merge_waits_for_late_flags(fab, oracle_mod):
    """The early-start merge (merge_follow_kernel, full grid, one chunk-flag
    acquire per row) launched before its flags are set: it must not finish
    until they are, and then merge byte-exact.  The flags are published late
    from the host side with fresh tokens (fsx_signal_flags), standing in for
    a producer on another GPU."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    reqs = T.config_requests("A", 8)  # a grid small enough to be resident at once
    b = DataPlaneBatch(fab, reqs, T.RULES["A"], 0, 1, chunk_rows=64)
    b.synth_inputs()
    assert b.alloc()
    b.forward()
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    b.tokens[:] = (1 << 44) + rng.integers(1, 1 << 30, size=len(b.tokens))  # nobody set these yet
    s2 = torch.cuda.Stream()
    done = torch.cuda.Event()
    with torch.cuda.stream(s2):
        b.merge(s2, early_start=True)
        done.record(s2)
    time.sleep(0.05)
    assert not done.query(), "early-start merge finished before its chunk flags were set"
    for i in range(len(b.lay.items)):
        fab.signal_flags(1, int(b.flag_base[i]), int(b.n_chunks[i]), int(b.tokens[i]), 0)
    done.synchronize()
    want, st = _expected(oracle_mod, b)
    assert (b.status_host() == 0).all() and (st == 0).all()
    assert np.array_equal(b.embeds_host(), want)
    b.release()


def test_merge_early_start_flags(fab, oracle_mod):
    reqs = T.config_requests("D", 12)
    b = _run_batch(fab, reqs, T.RULES["D"], chunk_rows=512, path="early")
    want, _ = _expected(oracle_mod, b)
    assert np.array_equal(b.embeds_host(), want)
    b.release()


@pytest.mark.parametrize("path", ["serial", "tee", "early"])
def test_merge_validation_leaves_request_untouched(fab, oracle_mod, path):
    """A request whose placeholder count does not match its items keeps its
    prompt rows (status validation); the tee still forwards its items."""
    reqs = T.config_requests("A", 10)
    bad = next(r for r, q in enumerate(reqs) if q.items)

    def corrupt(b):
        t0, t1 = int(b.lay.req_row_off[bad]), int(b.lay.req_row_off[bad + 1])
        idx = t0 + int(np.where(b.tok_host[t0:t1] == T.PLACEHOLDER_ID)[0][0])
        b.tok_host = b.tok_host.copy()
        b.tok_host[idx] = 7
        b.tok[idx] = 7

    b = _run_batch(fab, reqs, T.RULES["A"], path=path, tok_override=corrupt)
    want, st = _expected(oracle_mod, b)
    got_st = b.status_host()
    assert got_st[bad] == N.E_VALIDATION and st[bad] == 1
    assert (np.delete(got_st, bad) == 0).all()
    assert np.array_equal(b.embeds_host(), want)
    k = int(b.lay.req_item_off[bad])  # the failed request's first item reached its slab segment
    it = b.lay.items[k]
    assert b.slab_item_host(k).tobytes() == oracle_mod.synth_payload(T.payload_seed(it.ref_id, 0),
                                                                     it.rows * b.rb)
    b.release()


@pytest.mark.parametrize("path", ["serial", "tee", "early"])
def test_merge_edge_cases(fab, oracle_mod, path):
    rules = T.ShapeRules(hidden_dim=8, pixels_per_token=1, default_image_width=1,
                         default_image_height=3, tokens_per_audio_second=1, default_audio_seconds=1)
    reqs = [T.make_request(0, 0, ["image"], rules),              # placeholders only
            T.make_request(1, 4, [], rules),                     # text only
            T.make_request(2, 1, ["image", "audio", "image"], rules),
            T.make_request(3, 37, ["audio"], rules),
            T.make_request(4, 5, ["text", "image", "text"], rules)]  # zero-row items
    for chunk_rows in (None, 2):  # 2: chunks end mid-CTA and mid-item
        b = _run_batch(fab, reqs, rules, chunk_rows, path)
        want, st = _expected(oracle_mod, b)
        assert (b.status_host() == 0).all()
        assert np.array_equal(b.embeds_host(), want)
        for i, it in enumerate(b.lay.items):
            exp = oracle_mod.synth_payload(T.payload_seed(it.ref_id, 0), it.rows * b.rb)
            assert b.slab_item_host(i).tobytes() == exp
        b.release()
    # odd row width (row_bytes not a multiple of 16): byte path
    rules2 = T.ShapeRules(hidden_dim=5, pixels_per_token=4096 * 4096)
    reqs2 = [T.make_request(i, 3 + i, ["image"] * (i % 3), rules2) for i in range(6)]
    b2 = _run_batch(fab, reqs2, rules2, None, path)
    want2, _ = _expected(oracle_mod, b2)
    assert np.array_equal(b2.embeds_host(), want2)
    b2.release()


@pytest.mark.parametrize("config,count,scan_first", [("A", 64, False), ("A", 7, True), ("D", 24, False),
                                                     ("B", 4, True)])
def test_forward_place_bit_exact(fab, oracle_mod, config, count, scan_first):
    """Direct placement (fsx_forward_place): producer rows straight into the
    consumer's placeholder rows == the oracle merge; no slab segment held."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    reqs = T.config_requests(config, count)
    b = DataPlaneBatch(fab, reqs, T.RULES[config], 0, 1)
    b.synth_inputs()
    s0 = fab.stats()
    if scan_first:  # the consumer's scan, then the producer's copy-only placement
        b.scan()
        b.place(mode=N.MERGE_COPY_ONLY)
    else:
        b.place()
    torch.cuda.synchronize()
    want, st = _expected(oracle_mod, b)
    assert (b.status_host() == 0).all() and (st == 0).all()
    assert np.array_equal(b.embeds_host(), want)
    s1 = fab.stats()
    assert s1["forwards"] == s0["forwards"] + 1
    assert s1["bytes_forwarded"] - s0["bytes_forwarded"] == b.lay.total_item_rows * b.rb
    assert fab.slab_usage(1)["segments_in_use"] == 0


def test_forward_place_validation_and_flag(fab, oracle_mod):
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    reqs = T.config_requests("A", 10)
    bad = next(r for r, q in enumerate(reqs) if q.items)
    b = DataPlaneBatch(fab, reqs, T.RULES["A"], 0, 1)
    t0, t1 = int(b.lay.req_row_off[bad]), int(b.lay.req_row_off[bad + 1])
    idx = t0 + int(np.where(b.tok_host[t0:t1] == T.PLACEHOLDER_ID)[0][0])
    b.tok_host = b.tok_host.copy()
    b.tok_host[idx] = 7
    b.tok[idx] = 7
    b.synth_inputs()
    flag = fab.flags_alloc(1, 1)
    mb = b.merge_batch(False, N.MERGE_FULL)
    sb = b.src_buf.data_ptr()
    b.item_src.copy_(torch.from_numpy(b.src_off + sb))
    fab.forward_place(0, 1, mb, done_flag=flag, token=0x5eed)
    fab.wait(1, flag, 1, 0x5eed, timeout_us=10_000_000)
    torch.cuda.synchronize()
    want, st = _expected(oracle_mod, b)
    got_st = b.status_host()
    assert got_st[bad] == N.E_VALIDATION and st[bad] == 1
    assert np.array_equal(b.embeds_host(), want)
    # early-start / discard / scan-only are not placement modes
    for mode in (N.MERGE_SCAN_ONLY, N.MERGE_FULL | N.MERGE_DISCARD):
        mb2 = b.merge_batch(False, mode)
        with pytest.raises(N.FsxError):
            fab.forward_place(0, 1, mb2)


def test_pass_graph_replay_bit_exact(fab, oracle_mod):
    """The stream-ordered pass captured once as a CUDA graph (DataPlaneBatch
    capture / run_graph, bench.py's config-A schedule) and replayed: merged
    rows == the oracle; a moved slab offset triggers a re-capture."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    reqs = T.config_requests("A", 24)
    b = DataPlaneBatch(fab, reqs, T.RULES["A"], 0, 1)
    b.synth_inputs()
    s = torch.cuda.Stream()
    assert b.alloc()
    b.capture(s)
    assert b.graph_kernels >= 3  # K1 + scan + merge
    for _ in range(3):
        b.run_graph(s)
    b.release()
    hold = fab.slab_alloc(1, 4096)  # the next alloc lands elsewhere: re-capture
    assert b.alloc()
    b.run_graph(s)
    s.synchronize()
    want, _ = _expected(oracle_mod, b)
    assert (b.status_host() == 0).all()
    assert np.array_equal(b.embeds_host(), want)
    for i in range(min(2, len(b.lay.items))):
        it = b.lay.items[i]
        assert b.slab_item_host(i).tobytes() == oracle_mod.synth_payload(T.payload_seed(it.ref_id, 0),
                                                                         it.rows * b.rb)
    b.release()
    fab.slab_free(1, hold)


@pytest.mark.parametrize("kind", ["tee", "tee_pipelined"])
@pytest.mark.parametrize("config,count", [("A", 24), ("D", 8)])
def test_tee_pass_graph_bit_exact(fab, oracle_mod, config, count, kind):
    """The fused forward + merge (scan, then fsx_forward_merge) captured once
    as a CUDA graph and replayed several times: merged rows and slab segments
    == the oracle, and the graph-baked counter / flag ranges are pinned (eager
    forwards in between never reuse them).  tee_pipelined: two graphs, each
    the tee of one scan slot || the scan of the other (the bench's form)."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    reqs = T.config_requests(config, count)
    b = DataPlaneBatch(fab, reqs, T.RULES[config], 0, 1, chunk_rows=512 if config == "D" else None)
    b.synth_inputs()
    s = torch.cuda.Stream()
    assert b.alloc()
    b.capture(s, kind=kind)
    assert b.graph_kernels >= 2  # scan + tee
    if kind == "tee_pipelined":
        b.scan(s, slot=0)
    baked = b.flag_base.copy()
    other = DataPlaneBatch(fab, T.config_requests("A", 4), T.RULES["A"], 0, 1)
    other.synth_inputs()
    for _ in range(3):
        b.run_graph(s)
        assert other.alloc()  # eager traffic between replays draws fresh ranges
        other.forward()
        other.wait_host()
        assert not set(other.flag_base.tolist()) & set(baked.tolist())
        other.release()
    s.synchronize()
    want, _ = _expected(oracle_mod, b)
    assert (b.status_host() == 0).all()
    assert np.array_equal(b.embeds_host(), want)
    for i in range(min(3, len(b.lay.items))):
        it = b.lay.items[i]
        assert b.slab_item_host(i).tobytes() == oracle_mod.synth_payload(T.payload_seed(it.ref_id, 0),
                                                                         it.rows * b.rb)
    b.release()


def test_forward_merge_validation(fab):
    """fsx_forward_merge rejects a transfer count that is not the item count,
    item bytes that are not whole rows, chunks that are not whole rows, and
    early-start / discard mode bits."""
    import ctypes as C

    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    b = DataPlaneBatch(fab, T.config_requests("B", 1), T.RULES["B"], 0, 1, chunk_rows=1024)
    b.synth_inputs()
    assert b.alloc()
    b._prep_transfers(None, None)
    mb = b.merge_batch(False, N.MERGE_FULL)
    mb.d_item_src = b._direct_src().data_ptr()
    with pytest.raises(N.FsxError) as e:
        N.call("fsx_forward_merge", fab._h, 0, b._xfers, C.byref(mb), 0, None)
    assert e.value.code == "validation"
    b._xview["chunk_bytes"] = 1000 * 16  # not whole 7168-byte rows
    with pytest.raises(N.FsxError):
        N.call("fsx_forward_merge", fab._h, 1, b._xfers, C.byref(mb), 0, None)
    b._xview["chunk_bytes"] = 1024 * b.rb
    for bits in (N.MERGE_DISCARD, N.MERGE_SCAN_ONLY):
        bad = b.merge_batch(False, N.MERGE_FULL | bits)
        with pytest.raises(N.FsxError):
            N.call("fsx_forward_merge", fab._h, 1, b._xfers, C.byref(bad), 0, None)
    b.release()


def test_forward_place_edge_cases(fab, oracle_mod):
    """Direct placement on the merge edge cases: placeholder-only, text-only
    and multi-item requests, and a row width that is not a multiple of 16
    bytes (byte path)."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    rules = T.ShapeRules(hidden_dim=8, pixels_per_token=1, default_image_width=1,
                         default_image_height=3, tokens_per_audio_second=1, default_audio_seconds=1)
    reqs = [T.make_request(0, 0, ["image"], rules), T.make_request(1, 4, [], rules),
            T.make_request(2, 1, ["image", "audio", "image"], rules),
            T.make_request(3, 37, ["audio"], rules)]
    rules2 = T.ShapeRules(hidden_dim=5, pixels_per_token=4096 * 4096)
    reqs2 = [T.make_request(i, 3 + i, ["image"] * (i % 3), rules2) for i in range(6)]
    for rq, ru in ((reqs, rules), (reqs2, rules2)):
        b = DataPlaneBatch(fab, rq, ru, 0, 1)
        b.synth_inputs()
        b.place()
        torch.cuda.synchronize()
        want, st = _expected(oracle_mod, b)
        assert (b.status_host() == 0).all()
        assert np.array_equal(b.embeds_host(), want)


def test_stats_and_launch_count(fab):
    s = fab.stats()
    assert s["forwards"] > 0 and s["merges"] > 0 and s["kernel_launches"] > 0


def test_small_put_batch_roundtrip(fab, oracle_mod):
    """fsx_put_small (config C per-token messages through the drop-in's host
    span path): many messages published on the small-message lane; every slab
    segment holds the bytes, the returned bytes equal them, and both device
    digests (bytes moved, segment read back) equal the oracle's dg64.  Sizes
    cover 4 B codes, unaligned tails and the 64 KiB limit; over-limit and empty
    puts decline (ticket -1)."""
    import ctypes as C

    sizes = [4, 1, 7, 15, 16, 17, 2048, 7168, 4099, 65536] * 4
    msgs = [oracle_mod.synth_payload(1000 + i, n) for i, n in enumerate(sizes)]
    offs, tickets = [], []
    for m in msgs:
        off = fab.slab_alloc(2, len(m))
        t = C.c_int64(-2)
        N.call("fsx_put_small", fab._h, 2, off, m, len(m), C.byref(t))
        assert t.value >= 0
        offs.append(off)
        tickets.append(t.value)
    for m, off, t in zip(msgs, offs, tickets):
        p, d = C.c_void_p(), C.c_uint64()
        N.call("fsx_ticket_wait", fab._h, t, C.byref(p), C.byref(d))
        assert C.string_at(p.value, len(m)) == m
        assert d.value == oracle_mod.C.or_digest64(m, len(m))
        sent, landed = C.c_uint64(), C.c_uint64()
        N.call("fsx_ticket_digests", fab._h, t, C.byref(sent), C.byref(landed))
        assert sent.value == landed.value == d.value
        assert fab.slab_read(2, off, len(m)) == m
        N.call("fsx_ticket_free", fab._h, t)
        fab.slab_free(2, off)
    for n in (0, 65537):
        t = C.c_int64(-2)
        N.call("fsx_put_small", fab._h, 2, 0, b"\0" * max(n, 1), n, C.byref(t))
        assert t.value == -1
    with pytest.raises(N.FsxError):
        N.call("fsx_ticket_wait", fab._h, tickets[0], None, None)  # already freed


def test_small_lane_idle_exit_and_relaunch(fab, oracle_mod):
    """The lane's service kernel exits after 200 us without work and is
    relaunched by the next publish: bursts separated by idle gaps (and by a
    device-wide synchronize, which must return) are all served, byte-exact;
    interleaved waits and publishes never lose a message."""
    import ctypes as C

    for burst in range(6):
        msgs = [oracle_mod.synth_payload(5000 + 37 * burst + i, 7168 - 3 * i) for i in range(33)]
        offs, tickets = [], []
        for i, m in enumerate(msgs):
            off = fab.slab_alloc(2, len(m))
            t = C.c_int64(-2)
            N.call("fsx_put_small", fab._h, 2, off, m, len(m), C.byref(t))
            assert t.value >= 0
            offs.append(off)
            tickets.append(t.value)
            if i % 8 == 7:  # wait on an earlier message while later ones are in flight
                N.call("fsx_ticket_wait", fab._h, tickets[i - 4], None, None)
        for i, (m, off, t) in enumerate(zip(msgs, offs, tickets)):
            sent, landed = C.c_uint64(), C.c_uint64()
            if i % 2:  # wait + copy out + digests + free in one call (the drop-in's delivery)
                out = C.create_string_buffer(len(m))
                N.call("fsx_ticket_take", fab._h, t, out, len(m), C.byref(sent), C.byref(landed))
                assert out.raw == m
            else:
                N.call("fsx_ticket_digests", fab._h, t, C.byref(sent), C.byref(landed))
                N.call("fsx_ticket_free", fab._h, t)
            assert sent.value == landed.value == oracle_mod.C.or_digest64(m, len(m))
            assert fab.slab_read(2, off, len(m)) == m  # served: the bytes are in the slab
            fab.slab_free(2, off)
        with pytest.raises(N.FsxError):
            N.call("fsx_ticket_take", fab._h, tickets[1], None, 0, None, None)  # already taken
        if burst % 2:
            _torch().cuda.synchronize()  # waits at most for the idle exit
        else:
            time.sleep(0.002)  # >> 200 us: the kernel has exited, the next publish relaunches
    # publishes racing the idle exit: gaps around the 200 us idle time
    rng = np.random.default_rng(7)
    m = oracle_mod.synth_payload(99, 4096)
    off = fab.slab_alloc(2, 3 * 4096)
    for it in range(300):
        ts = []
        for j in range(1 + it % 3):
            t = C.c_int64(-2)
            N.call("fsx_put_small", fab._h, 2, off + 4096 * j, m, 4096, C.byref(t))
            ts.append(t.value)
        for t in ts:
            sent, landed = C.c_uint64(), C.c_uint64()
            N.call("fsx_ticket_take", fab._h, t, None, 0, C.byref(sent), C.byref(landed))
            assert sent.value == landed.value
        deadline = time.perf_counter() + float(rng.uniform(150e-6, 260e-6))
        while time.perf_counter() < deadline:
            pass
    fab.slab_free(2, off)


def test_small_lane_device_source(fab, oracle_mod):
    """fsx_put_small_device: a row already on the GPU is moved by the lane
    kernel straight from device memory (no host staging): slab bytes, sent and
    landed digests equal the oracle's; no host bytes from fsx_ticket_wait;
    fsx_ticket_take copies the landed segment out."""
    import ctypes as C

    torch = _torch()
    sizes = [4, 17, 2048, 7168, 4099, 65536]
    msgs = [oracle_mod.synth_payload(7000 + i, n) for i, n in enumerate(sizes)]
    dev = [torch.frombuffer(bytearray(m), dtype=torch.uint8).cuda() for m in msgs]
    torch.cuda.synchronize()
    offs, tickets = [], []
    for m, d in zip(msgs, dev):
        off = fab.slab_alloc(2, len(m))
        t = C.c_int64(-2)
        N.call("fsx_put_small_device", fab._h, 2, off, d.data_ptr(), len(m), C.byref(t))
        assert t.value >= 0
        offs.append(off)
        tickets.append(t.value)
    for i, (m, off, t) in enumerate(zip(msgs, offs, tickets)):
        p, dg = C.c_void_p(1), C.c_uint64()
        N.call("fsx_ticket_wait", fab._h, t, C.byref(p), C.byref(dg))
        assert not p.value  # device source: nothing staged on the host
        sent, landed = C.c_uint64(), C.c_uint64()
        out = C.create_string_buffer(len(m))
        N.call("fsx_ticket_take", fab._h, t, out, len(m), C.byref(sent), C.byref(landed))
        assert out.raw == m
        assert sent.value == landed.value == dg.value == oracle_mod.C.or_digest64(m, len(m))
        assert fab.slab_read(2, off, len(m)) == m
        fab.slab_free(2, off)


def test_small_lane_alloc_and_publish(fab, oracle_mod):
    """fsx_put_small_alloc: the slab segment (NodeArena first fit, as
    fsx_slab_alloc) and the lane publish in one call, host and device
    sources; the offsets are the allocator's, the bytes land, declines keep
    the segment; a full slab returns -1 without publishing."""
    import ctypes as C

    torch = _torch()
    msgs = [oracle_mod.synth_payload(8100 + i, 1000 + 700 * i) for i in range(6)]
    placed = []
    for i, m in enumerate(msgs):
        off, t = C.c_int64(-2), C.c_int64(-2)
        if i % 2:
            d = torch.frombuffer(bytearray(m), dtype=torch.uint8).cuda()
            torch.cuda.synchronize()
            N.call("fsx_put_small_alloc", fab._h, 2, d.data_ptr(), len(m), 1, C.byref(off), C.byref(t))
            placed.append((m, off.value, t.value, d))
        else:
            N.call("fsx_put_small_alloc", fab._h, 2, m, len(m), 0, C.byref(off), C.byref(t))
            placed.append((m, off.value, t.value, None))
        assert off.value >= 0 and t.value >= 0
    offs = [p[1] for p in placed]
    assert len(set(offs)) == len(offs)
    for m, off, t, _ in placed:
        sent, landed = C.c_uint64(), C.c_uint64()
        N.call("fsx_ticket_take", fab._h, t, None, 0, C.byref(sent), C.byref(landed))
        assert sent.value == landed.value == oracle_mod.C.or_digest64(m, len(m))
        assert fab.slab_read(2, off, len(m)) == m
        fab.slab_free(2, off)
    # a segment the slab cannot hold: nothing allocated, nothing published
    before = fab.slab_usage(2)
    hog = fab.slab_alloc(2, (64 << 20) - 4096)
    if hog >= 0:  # the fixture slab (64 MiB) is empty between tests
        off, t = C.c_int64(-2), C.c_int64(-2)
        N.call("fsx_put_small_alloc", fab._h, 2, b"x" * 8192, 8192, 0, C.byref(off), C.byref(t))
        assert off.value == -1 and t.value == -1
        fab.slab_free(2, hog)
        after = fab.slab_usage(2)
        assert {k: after[k] for k in ("segments_in_use", "bytes_in_use")} == \
            {k: before[k] for k in ("segments_in_use", "bytes_in_use")}


def test_small_lane_ticket_held_across_ring_turns(fab, oracle_mod):
    """The lane's descriptor ring has 4,096 slots; a ticket held while more
    than a full turn of messages is published after it (an orphaned or parked
    message) keeps its digests -- the publisher that reuses its slot copies
    them into the ticket first -- and everything published meanwhile is served
    byte-exact.  Also 4,100 tickets outstanding at once."""
    import ctypes as C

    held_msg = oracle_mod.synth_payload(4242, 7000)
    held_off = fab.slab_alloc(2, len(held_msg))
    held = C.c_int64(-2)
    N.call("fsx_put_small", fab._h, 2, held_off, held_msg, len(held_msg), C.byref(held))
    assert held.value >= 0
    off = fab.slab_alloc(2, 64 * 4200)
    for turn in range(2):  # two full turns, freed as they go
        pending = []
        for i in range(4100):
            m = ((i + turn) % 251).to_bytes(1, "little") * 48
            t = C.c_int64(-2)
            N.call("fsx_put_small", fab._h, 2, off + 64 * i, m, len(m), C.byref(t))
            assert t.value >= 0
            pending.append(t.value)
            if len(pending) > 64:
                N.call("fsx_ticket_free", fab._h, pending.pop(0))
        for t in pending:
            N.call("fsx_ticket_free", fab._h, t)
    got = fab.slab_read(2, off, 64 * 4100)
    for i in range(4100):
        assert got[64 * i:64 * i + 48] == ((i + 1) % 251).to_bytes(1, "little") * 48
    sent, landed = C.c_uint64(), C.c_uint64()
    out = C.create_string_buffer(len(held_msg))
    N.call("fsx_ticket_take", fab._h, held.value, out, len(held_msg), C.byref(sent), C.byref(landed))
    assert out.raw == held_msg
    assert sent.value == landed.value == oracle_mod.C.or_digest64(held_msg, len(held_msg))
    assert fab.slab_read(2, held_off, len(held_msg)) == held_msg
    # 4,100 tickets outstanding at once (more than the ring): all served
    tickets = []
    for i in range(4100):
        m = (i % 251).to_bytes(1, "little") * 48
        t = C.c_int64(-2)
        N.call("fsx_put_small", fab._h, 2, off + 64 * i, m, len(m), C.byref(t))
        assert t.value >= 0
        tickets.append(t.value)
    for i, t in enumerate(tickets):
        N.call("fsx_ticket_take", fab._h, t, None, 0, C.byref(sent), C.byref(landed))
        m = (i % 251).to_bytes(1, "little") * 48
        assert sent.value == landed.value == oracle_mod.C.or_digest64(m, len(m))
    fab.slab_free(2, off)
    fab.slab_free(2, held_off)


@pytest.mark.parametrize("config,count,chunk_rows", [("B", 2, 1024), ("D", 16, 512), ("A", 12, 64)])
def test_merge_colocated_pipeline_discard(fab, oracle_mod, config, count, chunk_rows):
    """The N=1 bench pass: K1 on one stream, the early-start merge on another
    running concurrently on the same GPU (FSX_MERGE_COLOCATED, one CTA per
    SM), discarding each slab row's L2 lines after reading it
    (FSX_MERGE_DISCARD).  Merged embeddings stay bit-exact with the oracle,
    repeated passes over the same slab segments included."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    rules = T.RULES[config]
    b = DataPlaneBatch(fab, T.config_requests(config, count), rules, 0, 1, chunk_rows=chunk_rows)
    b.synth_inputs()
    torch.cuda.synchronize()
    want, st = _expected(oracle_mod, b)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    mode = N.MERGE_FULL | N.MERGE_DISCARD | N.MERGE_COLOCATED
    for _ in range(3):
        assert b.alloc()
        b.forward(s1, host_notify=False, l2_keep=True)
        with torch.cuda.stream(s2):
            b.merge(s2, early_start=True, mode=mode)
        torch.cuda.synchronize()
        assert (b.status_host() == 0).all() and (st == 0).all()
        assert np.array_equal(b.embeds_host(), want)
        b.release()


def test_merge_mode_bits_validated(fab):
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    b = DataPlaneBatch(fab, T.config_requests("A", 2), T.RULES["A"], 0, 1)
    mb = b.merge_batch(False, N.MERGE_FULL | N.MERGE_COLOCATED)  # colocated needs item flags
    with pytest.raises(N.FsxError):
        fab.merge(1, mb)
    mb = b.merge_batch(False, N.MERGE_FULL | 0x4000)
    with pytest.raises(N.FsxError):
        fab.merge(1, mb)


def test_spin_watchdog_traps_instead_of_hanging(gpu):
    """A device wait on a flag that never arrives (a dead producer) must fail
    the launch after FSX_SPIN_TIMEOUT_S instead of hanging the GPU.  Run in a
    subprocess: the trap leaves that process's CUDA context unusable."""
    import os
    import subprocess
    import sys
    import time

    code = (
        "import sys, torch\n"
        "sys.path.insert(0, %r)\n"
        "from paper_2603_12118_b200.fabric import DeviceFabric\n"
        "f = DeviceFabric({0: 0, 1: 0}, {0: 0, 1: 0})\n"
        "f.slab_register(1, 1 << 20)\n"
        "fb = f.flags_alloc(1, 1)\n"
        "f.stream_wait_flags(1, fb, 1, 0xdead, None)\n"
        "try:\n"
        "    torch.cuda.synchronize()\n"
        "except Exception as e:\n"
        "    print('TRAPPED', type(e).__name__)\n"
        "    sys.exit(0)\n"
        "print('NO ERROR')\n"
        "sys.exit(1)\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    t0 = time.time()
    p = subprocess.run([sys.executable, "-c", code], env={**os.environ, "FSX_SPIN_TIMEOUT_S": "1"},
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and "TRAPPED" in p.stdout, (p.stdout + p.stderr)[-2000:]
    assert time.time() - t0 < 90


def test_forward_host_coalesced_batch_bit_exact(fab, oracle_mod):
    """The host-span batch path with back-to-back items (one pinned buffer, one
    H2D copy for the whole run of single-chunk items, shared flag) followed by
    the early-start merge: merged rows equal the oracle."""
    from paper_2603_12118_b200.dataplane import DataPlaneBatch

    torch = _torch()
    reqs = T.config_requests("A", 16)
    b = DataPlaneBatch(fab, reqs, T.RULES["A"], 0, 1)
    b.synth_inputs()
    torch.cuda.synchronize()
    want, st = _expected(oracle_mod, b)
    pinned = torch.empty(b.src_buf.numel(), dtype=torch.uint8, pin_memory=True)
    pinned.copy_(b.src_buf)
    host = [pinned[int(b.src_off[i]):int(b.src_off[i]) + int(b.item_bytes[i])].numpy()
            for i in range(len(b.lay.items))]
    for _ in range(2):
        assert b.alloc()
        b.forward_host(host)
        assert len(set(b.tokens.tolist())) < len(b.lay.items)  # items were coalesced
        b.merge(early_start=True)
        torch.cuda.synchronize()
        assert (b.status_host() == 0).all() and (st == 0).all()
        assert np.array_equal(b.embeds_host(), want)
        b.release()


def test_fsx_close_returns_every_device_allocation(gpu):
    """Device-slab leak check (the reference's shm-unlink check,
    test_sidecar.cpp:340-350, has no device counterpart): device memory free
    before fsx_open equals free memory after fsx_close, after slabs, flag
    rings, counters, scratch, channels and the small-message lane were all
    used, three open/close cycles in a row (after one warm-up cycle)."""
    import ctypes as C

    from paper_2603_12118_b200.dataplane import DataPlaneBatch
    from paper_2603_12118_b200.fabric import DeviceFabric

    torch = _torch()
    free0 = None
    # cycle 0 is a warm-up: the first use of a kernel in the process loads its
    # module (lazy loading), which keeps device memory for the process's life
    for cycle in range(4):
        if cycle == 1:
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            free0, _ = torch.cuda.mem_get_info()
        fab = DeviceFabric({0: 0, 1: 0, 2: 0}, {0: 0, 1: 0, 2: 0})
        fab.slab_register(1, 256 << 20)
        fab.slab_register(2, 64 << 20)
        b = DataPlaneBatch(fab, T.config_requests("A", 6), T.RULES["A"], 0, 1, chunk_rows=64)
        b.synth_inputs()
        assert b.alloc()
        b.tee(mode=N.MERGE_FULL, host_notify=True)
        b.wait_host()
        b.release()
        assert b.alloc()
        b.forward()
        b.merge(early_start=True)
        torch.cuda.synchronize()
        b.release()
        ch = fab.channel_open(0, 2, 7168, 8)
        rows = torch.zeros(7168, dtype=torch.uint8, device="cuda")
        fab.channel_push([ch], rows.data_ptr(), 7168)
        fab.channel_pull([ch], rows.data_ptr(), 7168)
        fab.channel_close(ch)
        off = fab.slab_alloc(2, 4096)
        t = C.c_int64(-1)
        N.call("fsx_put_small", fab._h, 2, off, b"x" * 4096, 4096, C.byref(t))
        assert t.value >= 0
        N.call("fsx_ticket_wait", fab._h, t.value, None, None)
        N.call("fsx_ticket_free", fab._h, t.value)
        fab.slab_free(2, off)
        slot = fab.u64_slot(1)
        assert slot
        del b, rows
        torch.cuda.synchronize()
        fab.close()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        free1, _ = torch.cuda.mem_get_info()
        # CUDA keeps a few MiB of context-level bookkeeping; a leaked slab is >= 64 MiB
        assert free0 is None or free0 - free1 < (8 << 20), (cycle, free0 - free1)
