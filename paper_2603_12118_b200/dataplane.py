"""One data-plane pass over a request batch on the device fabric.

A pass is what the reference does per request between the encoder's
``emit_output`` (executor_sim.hpp:221-229, 321-336) and the LLM's admission
(executor_sim.hpp:382-392), plus the merge the reference leaves out:

  1. the producer's embeddings live on the producer GPU (K0 synthesises them
     as ``synth_payload(payload_seed(ref_id, 0))``, executor_sim.hpp:330-331);
  2. each item gets a segment of the consumer GPU's slab (fsx_slab_alloc,
     NodeArena policy sidecar.hpp:149-163) and a run of chunk flags;
  3. K1 pushes each item into its segment chunk by chunk (fsx_forward);
  4. K3 merges all items of the batch into the prompt embedding (fsx_merge);
  5. the segments are released (the ack, sidecar.hpp:287-290, 547).

torch provides device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np
import torch

from . import _native as N
from .fabric import DeviceFabric, _stream_ptr
from .trace import (PLACEHOLDER_ID, BatchLayout, Request, ShapeRules, layout, payload_seed,
                    prompt_tokens, text_seed)

ALIGN = 256


def _align(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


class DataPlaneBatch:
    def __init__(self, fab: DeviceFabric, requests: List[Request], rules: ShapeRules,
                 src_gpu: int, dst_gpu: int, placeholder_id: int = PLACEHOLDER_ID,
                 chunk_rows: Optional[int] = None):
        self.fab = fab
        self.rules = rules
        self.rb = rules.row_bytes
        self.lay: BatchLayout = layout(requests, self.rb)
        self.src_gpu, self.dst_gpu = src_gpu, dst_gpu
        self.pid = placeholder_id
        self.chunk_rows = chunk_rows
        self.src_dev = torch.device("cuda", fab.device_of(src_gpu))
        self.dst_dev = torch.device("cuda", fab.device_of(dst_gpu))
        lay = self.lay
        M = len(lay.items)
        # Producer side: one buffer, each item at a 256 B aligned offset.
        self.src_off = np.zeros(M, dtype=np.int64)
        at = 0
        for i, it in enumerate(lay.items):
            self.src_off[i] = at
            at += _align(it.rows * self.rb)
        self.src_buf = torch.empty(max(at, ALIGN), dtype=torch.uint8, device=self.src_dev)
        # Consumer side: prompt embedding, token ids, merge descriptors.
        self.embeds = torch.empty(max(lay.total_rows * self.rb, 16), dtype=torch.uint8,
                                  device=self.dst_dev)
        tok = np.concatenate([prompt_tokens(q, placeholder_id) for q in requests]) \
            if requests else np.zeros(0, np.int32)
        self.tok_host = tok
        self.tok = torch.from_numpy(tok).to(self.dst_dev) if len(tok) else \
            torch.zeros(1, dtype=torch.int32, device=self.dst_dev)
        self.req_row_off = torch.from_numpy(lay.req_row_off).to(self.dst_dev)
        self.req_item_off = torch.from_numpy(lay.req_item_off).to(self.dst_dev)
        self.item_row_off = torch.from_numpy(lay.item_row_off).to(self.dst_dev)
        self.scratch = torch.empty(max(lay.total_item_rows, 1), dtype=torch.int32,
                                   device=self.dst_dev)
        self.status = torch.full((max(len(requests), 1),), -1, dtype=torch.int32,
                                 device=self.dst_dev)
        self.item_src = torch.zeros(max(M, 1), dtype=torch.int64, device=self.dst_dev)
        self.item_flag = torch.zeros(max(M, 1), dtype=torch.int64, device=self.dst_dev)
        self.item_token = torch.zeros(max(M, 1), dtype=torch.int64, device=self.dst_dev)
        self.item_chunk_rows = torch.zeros(max(M, 1), dtype=torch.int64, device=self.dst_dev)
        self.slab_off: Optional[np.ndarray] = None
        self.flag_base = np.zeros(M, dtype=np.int64)
        self.tokens = np.zeros(M, dtype=np.uint64)
        # per-item geometry, fixed for the batch
        self.item_bytes = np.array([it.rows * self.rb for it in lay.items], dtype=np.int64)
        self.item_chunk = np.array([self.chunk_bytes(it) for it in lay.items], dtype=np.int64)
        self.n_chunks = np.array([1 if (cb <= 0 or cb >= nb) else -(-nb // cb)
                                  for nb, cb in zip(self.item_bytes, self.item_chunk)],
                                 dtype=np.int64)
        self.chunk_prefix = np.concatenate([[0], np.cumsum(self.n_chunks)[:-1]]).astype(np.int64) \
            if M else np.zeros(0, np.int64)
        self._xfers = (N.Transfer * max(M, 1))()
        sb = self.src_buf.data_ptr()
        for i in range(M):
            self._xfers[i] = N.Transfer(src_gpu, dst_gpu, sb + int(self.src_off[i]), 0,
                                        int(self.item_bytes[i]), int(self.item_chunk[i]), 0, 0, None)
        self._xview = np.frombuffer(self._xfers, dtype=N.TRANSFER_DTYPE, count=max(M, 1))[:M]

    # -- inputs ---------------------------------------------------------------
    def synth_inputs(self, stream=None) -> None:
        """K0: producer payloads and the pre-filled prompt embeddings."""
        base = self.src_buf.data_ptr()
        for i, it in enumerate(self.lay.items):
            self.fab.synth(self.src_gpu, payload_seed(it.ref_id, 0), base + int(self.src_off[i]),
                           it.rows * self.rb, stream)
        eb = self.embeds.data_ptr()
        for r, q in enumerate(self.lay.requests):
            self.fab.synth(self.dst_gpu, text_seed(q), eb + int(self.lay.req_row_off[r]) * self.rb,
                           q.total_rows * self.rb, stream)

    # -- slab -------------------------------------------------------------------
    def alloc(self) -> bool:
        """One slab segment per item (one all-or-nothing call); False (nothing
        held) if the slab is full."""
        offs = self.fab.slab_alloc_n(self.dst_gpu, self.item_bytes)
        if offs is None:
            return False
        self.slab_off = offs
        # first fit hands back the same offsets step after step: upload the
        # slab views only when they change.  A merge still in flight (an
        # early-start merge of the previous pass on another stream) reads
        # item_src, so the device is drained first and the upload is
        # synchronous: rare, and correct whatever streams the caller uses.
        key = offs.tobytes()
        if len(offs) and key != getattr(self, "_uploaded_offs", None):
            base = self.fab.slab_ptr(self.dst_gpu, 0)
            torch.cuda.synchronize(self.dst_dev)
            self.item_src.copy_(torch.from_numpy(offs + base))
            torch.cuda.synchronize(self.dst_dev)
            self._uploaded_offs = key
        return True

    def release(self) -> None:
        if self.slab_off is not None:
            self.fab.slab_free_n(self.dst_gpu, self.slab_off)
            self.slab_off = None

    # -- K1 ---------------------------------------------------------------------
    def chunk_bytes(self, it) -> int:
        if not self.chunk_rows:
            return 0
        return self.chunk_rows * self.rb

    def forward(self, stream=None, host_notify: bool = True, l2_keep: bool = False,
                bulk: bool = False, flag_base0: Optional[int] = None,
                tokens: Optional[np.ndarray] = None, peer_gpu_count: bool = False,
                tile: bool = False) -> int:
        """Push every item into its slab segment (one fsx_forward_batch call,
        one K1 launch per N.FWD_MAX_BATCH items); returns the launches.  host_notify=False
        when only device work (stream order / early-start merge) waits on the
        chunk flags.  K1 form: bulk = the bulk-copy tiles, tile = the register
        tiles (FSX_FWD_KERNEL), neither = the library's choice (fsx.h)."""
        assert self.slab_off is not None, "alloc() first"
        M = len(self.lay.items)
        if M == 0:
            return 0
        self._prep_transfers(flag_base0, tokens)  # numpy view of the fsx_transfer array
        view = self._xview
        opts = (N.FWD_HOST_NOTIFY if host_notify else 0) | (N.FWD_L2_KEEP if l2_keep else 0) | \
            (N.FWD_BULK if bulk else 0) | (N.FWD_PEER_GPU_COUNT if peer_gpu_count else 0) | \
            (N.FWD_KERNEL if tile else 0)
        N.call("fsx_forward_batch", self.fab._h, M, self._xfers, opts, _stream_ptr(stream))
        self.tokens[:] = view["token"]
        return -(-M // N.FWD_MAX_BATCH)

    def _prep_transfers(self, flag_base0: Optional[int], tokens: Optional[np.ndarray]) -> None:
        """Slab offsets, flag ranges and tokens of this pass into the
        fsx_transfer array (no per-item Python); token 0 = drawn by the fabric."""
        fb0 = flag_base0 if flag_base0 is not None else \
            self.fab.flags_alloc(self.dst_gpu, int(self.n_chunks.sum()))
        self.flag_base[:] = fb0 + self.chunk_prefix
        view = self._xview
        view["dst_off"] = self.slab_off
        view["flag_base"] = self.flag_base
        view["token"] = 0 if tokens is None else tokens

    def tee(self, stream=None, mode: int = N.MERGE_COPY_ONLY, slot: int = 0,
            host_notify: bool = False, l2_keep: bool = False, flag_base0: Optional[int] = None,
            tokens: Optional[np.ndarray] = None) -> int:
        """The forward and the merge as one kernel (fsx_forward_merge): every
        item row is read once from the producer's buffer and stored into its
        slab segment (chunk flags set as K1 would) and into its placeholder
        row (as K3 would).  mode MERGE_COPY_ONLY uses the positions of a
        scan(slot) ordered before it; MERGE_FULL scans first.  Returns the
        launches of the copy (one per 64 items)."""
        assert self.slab_off is not None, "alloc() first"
        M = len(self.lay.items)
        self._prep_transfers(flag_base0, tokens)
        cache = self.__dict__.setdefault("_tee_cache", {})
        b = cache.get((mode, slot))
        if b is None:
            b = self.merge_batch(False, mode, slot)
            b.d_item_src = self._direct_src().data_ptr()
            cache[(mode, slot)] = b
        opts = (N.FWD_HOST_NOTIFY if host_notify else 0) | (N.FWD_L2_KEEP if l2_keep else 0)
        N.call("fsx_forward_merge", self.fab._h, M, self._xfers, C.byref(b), opts,
               _stream_ptr(stream))
        self.tokens[:] = self._xview["token"]
        return max(1, -(-M // N.FWD_MAX_BATCH))

    def _direct_src(self) -> torch.Tensor:
        """Device array of the producer's item pointers (direct placement and
        the tee read the producer's buffers, not slab segments)."""
        if not hasattr(self, "item_src_direct"):
            sb = self.src_buf.data_ptr()
            self.item_src_direct = torch.from_numpy(self.src_off + sb).to(self.dst_dev) \
                if len(self.src_off) else torch.zeros(1, dtype=torch.int64, device=self.dst_dev)
        return self.item_src_direct

    def forward_host(self, host_payload: List[np.ndarray], stream=None) -> None:
        """The host-span send path (sidecar.hpp:302): payload bytes from host
        memory straight into the consumer slab.  Single-chunk items whose host
        buffers and slab segments are both back to back go as ONE copy (every
        host->device copy costs a fixed copy-engine gap); they then share that
        copy's flag and token."""
        assert self.slab_off is not None, "alloc() first"
        if not self.chunk_rows and len(self.lay.items) > 1:
            self._forward_host_coalesced(host_payload, stream)
            return
        for i, it in enumerate(self.lay.items):
            nb = it.rows * self.rb
            cb = self.chunk_bytes(it)
            n = 1 if (cb <= 0 or cb >= nb) else -(-nb // cb)
            self.n_chunks[i] = n
            self.flag_base[i] = self.fab.flags_alloc(self.dst_gpu, n)
            self.tokens[i] = self.fab.forward_host(host_payload[i].ctypes.data, self.dst_gpu,
                                                   int(self.slab_off[i]), nb, cb,
                                                   int(self.flag_base[i]), stream)

    def _forward_host_coalesced(self, host_payload: List[np.ndarray], stream=None) -> None:
        M = len(self.lay.items)
        i = 0
        while i < M:
            j, nb = i, int(self.item_bytes[i])
            while (j + 1 < M and
                   host_payload[j + 1].ctypes.data == host_payload[j].ctypes.data + int(self.item_bytes[j]) and
                   int(self.slab_off[j + 1]) == int(self.slab_off[j]) + int(self.item_bytes[j])):
                j += 1
                nb += int(self.item_bytes[j])
            fb = self.fab.flags_alloc(self.dst_gpu, 1)
            tok = self.fab.forward_host(host_payload[i].ctypes.data, self.dst_gpu, int(self.slab_off[i]),
                                        nb, 0, fb, stream)
            for k in range(i, j + 1):
                self.n_chunks[k] = 1
                self.flag_base[k] = fb
                self.tokens[k] = tok
            i = j + 1

    def wait_host(self, timeout_us: int = 30_000_000) -> None:
        for i in range(len(self.lay.items)):
            self.fab.wait(self.dst_gpu, int(self.flag_base[i]), int(self.n_chunks[i]),
                          int(self.tokens[i]), timeout_us)

    # -- K3 ---------------------------------------------------------------------
    def _scan_slot(self, slot: int):
        """(scratch, status) of scan slot `slot`: slot 0 is the batch's own
        pair; slot 1 a second pair so the scan of the next pass can run while
        the current pass still reads slot 0 (software pipelining)."""
        if slot == 0:
            return self.scratch, self.status
        if not hasattr(self, "_slot1"):
            self._slot1 = (torch.empty_like(self.scratch), torch.full_like(self.status, -1))
        return self._slot1

    def merge_batch(self, early_start: bool = False, mode: int = N.MERGE_FULL,
                    slot: int = 0) -> N.MergeBatch:
        lay = self.lay
        scratch, status = self._scan_slot(slot)
        b = N.MergeBatch()
        b.mode = mode
        b.num_requests = len(lay.requests)
        b.num_items = len(lay.items)
        b.row_bytes = self.rb
        b.placeholder_id = self.pid
        b.d_embeds = self.embeds.data_ptr()
        b.d_token_ids = self.tok.data_ptr()
        b.d_req_row_off = self.req_row_off.data_ptr()
        b.d_req_item_off = self.req_item_off.data_ptr()
        b.d_item_src = self.item_src.data_ptr()
        b.d_item_row_off = self.item_row_off.data_ptr()
        b.d_scratch = scratch.data_ptr()
        b.d_status = status.data_ptr()
        b.total_rows = lay.total_rows
        b.total_item_rows = lay.total_item_rows
        if early_start and len(lay.items):
            M = len(lay.items)
            if not hasattr(self, "_es"):
                # flags are one contiguous u64 ring per slab; chunk rows are
                # fixed for the batch (uploaded once)
                self._flag0 = self.fab.flag_ptr(self.dst_gpu, 0)
                cr = [self.chunk_rows or it.rows for it in lay.items]
                self.item_chunk_rows.copy_(torch.tensor(cr, dtype=torch.int64))
                # a ring of pinned staging buffers of (flag pointer, token) per
                # item: uploaded with a non-blocking copy on the current
                # stream, each reused only once its previous copy has run (the
                # host may run a few passes ahead of the GPU)
                self._es = [(torch.empty((2, M), dtype=torch.int64, pin_memory=True),
                             torch.empty((2, M), dtype=torch.int64, device=self.dst_dev),
                             torch.cuda.Event()) for _ in range(4)]
                self._es_next = 0
            host, dev, ev = self._es[self._es_next]
            self._es_next = (self._es_next + 1) % len(self._es)
            if not getattr(self, "es_device_idle", False):  # caller synchronized the device
                ev.synchronize()
            hv = host.numpy()
            hv[0] = self._flag0 + 8 * self.flag_base
            hv[1] = self.tokens.astype(np.int64)
            dev.copy_(host, non_blocking=True)
            ev.record()
            b.d_item_flag = dev[0].data_ptr()
            b.d_item_token = dev[1].data_ptr()
            b.d_item_chunk_rows = self.item_chunk_rows.data_ptr()
        return b

    def merge(self, stream=None, early_start: bool = False, mode: int = N.MERGE_FULL,
              slot: int = 0) -> None:
        if early_start:  # flag pointers / tokens change every step
            b = self.merge_batch(True, mode, slot)
        else:  # descriptors are fixed for the batch: build once
            cache = self.__dict__.setdefault("_mb_cache", {})
            b = cache.get((mode, slot))
            if b is None:
                b = cache[(mode, slot)] = self.merge_batch(False, mode, slot)
        self.fab.merge(self.dst_gpu, b, stream)

    def place(self, stream=None, mode: int = N.MERGE_FULL, slot: int = 0) -> None:
        """Direct placement instead of forward + merge (fsx_forward_place):
        the producer writes each item's rows from its own buffer straight into
        the consumer's placeholder rows -- no slab segment, no chunk flags, the
        payload crosses memory once.  mode MERGE_COPY_ONLY uses the positions
        of a scan(slot) ordered before it."""
        cache = self.__dict__.setdefault("_place_cache", {})
        b = cache.get((mode, slot))
        if b is None:
            b = self.merge_batch(False, mode, slot)
            b.d_item_src = self._direct_src().data_ptr()
            cache[(mode, slot)] = b
        self.fab.forward_place(self.src_gpu, self.dst_gpu, b, stream=stream)

    # -- CUDA-graph form of a pass ------------------------------------------------
    def capture(self, stream, kind: str = "serial", bulk: bool = True, l2_keep: bool = False) -> None:
        """Record one pass once as a CUDA graph for the current slab offsets;
        run_graph() replays it.  kind "serial": K1 then the merge (FULL) in
        stream order; "tee": the scan then the fused forward + merge.  For
        launch-bound batches (config A): segment offsets, flag ranges and
        tokens are baked in (the ranges are pinned by the fabric) -- first fit
        returns the same offsets pass after pass, and nothing in stream order
        waits on the flags."""
        assert self.slab_off is not None, "alloc() first"
        if kind in ("tee", "tee_pipelined") and not hasattr(self, "item_src_direct"):
            self._direct_src()  # a device upload: not inside the capture
        if kind == "tee_pipelined":
            # two graphs, one per scan slot k: the tee of this pass reads the
            # positions of slot k (scanned by the previous replay) while a
            # forked branch scans slot 1 - k for the next pass -- the eager
            # schedule's one-pass-ahead scan, inside the graph.  The caller
            # scans slot 0 once before the first replay.
            side = torch.cuda.Stream(device=stream.device)
            graphs = []
            l0 = self.fab.stats()["kernel_launches"]
            for k in (0, 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    side.wait_stream(stream)
                    self.scan(side, slot=1 - k)
                    self.tee(stream, mode=N.MERGE_COPY_ONLY, slot=k, l2_keep=l2_keep)
                    stream.wait_stream(side)
                graphs.append(g)
            self.graph_kernels = (self.fab.stats()["kernel_launches"] - l0) // 2
            self._graphs = graphs
            self._graph = graphs[0]
            self._replays = 0
        else:
            g = torch.cuda.CUDAGraph()
            l0 = self.fab.stats()["kernel_launches"]
            with torch.cuda.graph(g, stream=stream):
                if kind == "tee":
                    self.tee(stream, mode=N.MERGE_FULL, l2_keep=l2_keep)
                else:
                    self.forward(stream, host_notify=False, l2_keep=l2_keep, bulk=bulk)
                    self.merge(stream)
            self.graph_kernels = self.fab.stats()["kernel_launches"] - l0  # fsx kernels per replay
            self._graph = g
            self._graphs = None
        self._graph_key = (self.slab_off.tobytes(), kind, bulk, l2_keep)

    def run_graph(self, stream) -> None:
        """Replay the captured pass (alloc() first; re-captured if the slab
        handed back different offsets)."""
        assert self.slab_off is not None, "alloc() first"
        key = (self.slab_off.tobytes(),) + self._graph_key[1:]
        if key != self._graph_key:
            self.capture(stream, *self._graph_key[1:])
        with torch.cuda.stream(stream):
            if self._graphs:  # tee_pipelined: alternate the scan slots
                self._graphs[self._replays % 2].replay()
                self._replays += 1
            else:
                self._graph.replay()

    def scan(self, stream=None, slot: int = 0) -> None:
        """Phase 1 of K3 only: needs just the token ids, so it can run while
        the payload is still being forwarded (or, pipelined, during the
        previous pass)."""
        self.merge(stream, mode=N.MERGE_SCAN_ONLY, slot=slot)

    # -- readback -----------------------------------------------------------------
    def embeds_host(self) -> np.ndarray:
        return self.embeds[: self.lay.total_rows * self.rb].cpu().numpy()

    def status_host(self, slot: int = 0) -> np.ndarray:
        return self._scan_slot(slot)[1][: len(self.lay.requests)].cpu().numpy()

    def slab_item_host(self, i: int) -> np.ndarray:
        it = self.lay.items[i]
        raw = self.fab.slab_read(self.dst_gpu, int(self.slab_off[i]), it.rows * self.rb)
        return np.frombuffer(raw, dtype=np.uint8)
