"""Python handle over the libfsx C ABI (include/fsx.h).

``DeviceFabric`` is the device layer the reference's SidecarFabric would sit
on: the logical GPU map (sidecar.hpp:242-260), per-consumer-GPU
receive slabs with the NodeArena allocation policy (sidecar.hpp:106-205),
chunk flags, the K1 forward, the K3 merge and K0 synthesis.  The C++
SidecarFabric-compatible engine is include/fsx/fabric.hpp; this class exists
so the Python tests and bench.py can drive the same C ABI.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Optional

from . import _native as N


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the per-device legacy default stream


def _stream_ptr(stream) -> Optional[int]:
    """cudaStream_t for the C ABI.  None means torch's current stream (so fsx
    work is ordered with the surrounding torch ops, e.g. the copy that fills a
    source buffer); torch's default stream has handle 0, which the C ABI would
    read as "the fabric's own stream", so it is passed as cudaStreamLegacy.
    Pass an explicit stream when the call targets another device than the
    current one."""
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    if isinstance(stream, int):
        return stream
    h = int(stream.cuda_stream)  # torch.cuda.Stream
    return h if h else CUDA_STREAM_LEGACY


class DeviceFabric:
    def __init__(self, gpu_to_node: Dict[int, int], devices: Optional[Dict[int, int]] = None):
        gpus = sorted(gpu_to_node)
        n = len(gpus)
        ids = (C.c_int * n)(*gpus)
        nodes = (C.c_int * n)(*[gpu_to_node[g] for g in gpus])
        devs = (C.c_int * n)(*[(devices or {}).get(g, -1) for g in gpus])
        h = C.c_void_p()
        N.call("fsx_open", n, ids, nodes, devs, C.byref(h))
        self._h = h
        self.gpus = gpus

    # -- lifetime -----------------------------------------------------------
    def close(self) -> None:
        if self._h:
            N.call("fsx_close", self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- topology (sidecar.hpp:250-260) ---------------------------------------
    def node_of(self, gpu: int) -> int:
        v = C.c_int()
        N.call("fsx_node_of", self._h, gpu, C.byref(v))
        return v.value

    def route(self, src: int, dst: int) -> int:
        v = C.c_int()
        N.call("fsx_route", self._h, src, dst, C.byref(v))
        return v.value

    def device_of(self, gpu: int) -> int:
        v = C.c_int()
        N.call("fsx_device_of", self._h, gpu, C.byref(v))
        return v.value

    # -- slabs ----------------------------------------------------------------
    def slab_register(self, gpu: int, nbytes: int) -> None:
        N.call("fsx_slab_register", self._h, gpu, nbytes)

    def slab_alloc(self, gpu: int, nbytes: int) -> Optional[int]:
        off = C.c_int64()
        N.call("fsx_slab_alloc", self._h, gpu, nbytes, C.byref(off))
        return None if off.value < 0 else off.value

    def slab_free(self, gpu: int, off: int) -> None:
        N.call("fsx_slab_free", self._h, gpu, off)

    def slab_alloc_n(self, gpu: int, lens):
        """All-or-nothing segment allocation for a batch; None if it does not fit."""
        import numpy as np

        ln = np.ascontiguousarray(lens, dtype=np.int64)
        offs = np.empty(len(ln), dtype=np.int64)
        if len(ln):
            N.call("fsx_slab_alloc_n", self._h, gpu, len(ln), ln.ctypes.data, offs.ctypes.data)
            if offs[0] < 0:
                return None
        return offs

    def slab_free_n(self, gpu: int, offs) -> None:
        import numpy as np

        o = np.ascontiguousarray(offs, dtype=np.int64)
        if len(o):
            N.call("fsx_slab_free_n", self._h, gpu, len(o), o.ctypes.data)

    def slab_ptr(self, gpu: int, off: int = 0) -> int:
        p = C.c_void_p()
        N.call("fsx_slab_ptr", self._h, gpu, off, C.byref(p))
        return p.value or 0

    def slab_usage(self, gpu: int) -> dict:
        v = [C.c_int64() for _ in range(4)]
        N.call("fsx_slab_usage", self._h, gpu, *[C.byref(x) for x in v])
        return dict(zip(["segments_in_use", "bytes_in_use", "peak_bytes", "capacity"],
                        [x.value for x in v]))

    def slab_read(self, gpu: int, off: int, nbytes: int, stream=None) -> bytes:
        buf = (C.c_uint8 * max(nbytes, 1))()
        N.call("fsx_slab_read", self._h, gpu, off, buf, nbytes, _stream_ptr(stream))
        return bytes(buf)[:nbytes]

    def slab_export(self, gpu: int) -> tuple:
        buf = (C.c_uint8 * 64)()
        nb = C.c_int64()
        N.call("fsx_slab_export", self._h, gpu, buf, C.byref(nb))
        return bytes(buf), nb.value

    def slab_import(self, gpu: int, handle: bytes, nbytes: int) -> None:
        buf = (C.c_uint8 * 64)(*handle)
        N.call("fsx_slab_import", self._h, gpu, buf, nbytes)

    # -- flags ------------------------------------------------------------------
    def flags_alloc(self, gpu: int, n: int) -> int:
        v = C.c_int64()
        N.call("fsx_flags_alloc", self._h, gpu, n, C.byref(v))
        return v.value

    def flag_ptr(self, gpu: int, idx: int) -> int:
        p = C.c_void_p()
        N.call("fsx_flag_ptr", self._h, gpu, idx, C.byref(p))
        return p.value or 0

    def chunk_ready(self, gpu: int, idx: int, token: int) -> bool:
        v = C.c_int()
        N.call("fsx_chunk_ready", self._h, gpu, idx, token, C.byref(v))
        return bool(v.value)

    def wait(self, gpu: int, flag_base: int, n: int, token: int, timeout_us: int = -1) -> None:
        N.call("fsx_wait", self._h, gpu, flag_base, n, token, timeout_us)

    def stream_wait_flags(self, gpu: int, flag_base: int, n: int, token: int, stream=None) -> None:
        N.call("fsx_stream_wait_flags", self._h, gpu, flag_base, n, token, _stream_ptr(stream))

    def signal_flags(self, dst_gpu: int, flag_base: int, n: int, token: int, src_gpu: int,
                     stream=None) -> None:
        N.call("fsx_signal_flags", self._h, dst_gpu, flag_base, n, token, src_gpu,
               _stream_ptr(stream))

    # -- data movement ----------------------------------------------------------
    def forward(self, src_gpu: int, src_ptr: int, dst_gpu: int, dst_off: int, nbytes: int,
                chunk_bytes: int, flag_base: int, stream=None, token: int = 0,
                host_notify: bool = True, bulk: bool = False, peer_gpu_count: bool = False,
                dma: bool | None = None) -> int:
        """K1.  host_notify mirrors chunk flags to host memory (fsx_wait);
        device-only consumers (stream order, early-start merge) skip it.
        bulk: the bulk-copy tile kernel (FSX_FWD_BULK); peer_gpu_count: peer
        chunks counted at gpu scope, published once at system scope.
        dma: None = the library's choice (the copy-engine form for a local
        transfer of at most FWD_DMA_MAX_CHUNKS chunks), True = the copy-engine
        form (FSX_FWD_DMA), False = always the K1 kernel (FSX_FWD_KERNEL)."""
        tok = C.c_uint64(token)
        opts = (N.FWD_HOST_NOTIFY if host_notify else 0) | (N.FWD_BULK if bulk else 0) | \
            (N.FWD_PEER_GPU_COUNT if peer_gpu_count else 0) | \
            (0 if dma is None else (N.FWD_DMA if dma else N.FWD_KERNEL))
        N.call("fsx_forward_ex", self._h, src_gpu, src_ptr, dst_gpu, dst_off, nbytes, chunk_bytes,
               flag_base, C.byref(tok), opts, _stream_ptr(stream))
        return tok.value

    def forward_batch(self, transfers, stream=None, host_notify: bool = True):
        """K1 over several transfers of one source device in one launch.
        `transfers`: sequence of (src_gpu, src_ptr, dst_gpu, dst_off, nbytes,
        chunk_bytes, flag_base, token); returns the tokens used."""
        n = len(transfers)
        arr = (N.Transfer * max(n, 1))()
        for i, t in enumerate(transfers):
            sg, sp, dg, do, nb, cb, fb, tok = t[:8]
            arr[i] = N.Transfer(sg, dg, sp, do, nb, cb, fb, tok, t[8] if len(t) > 8 else None)
        N.call("fsx_forward_batch", self._h, n, arr, N.FWD_HOST_NOTIFY if host_notify else 0,
               _stream_ptr(stream))
        return [arr[i].token for i in range(n)]

    def forward_host(self, host_ptr: int, dst_gpu: int, dst_off: int, nbytes: int,
                     chunk_bytes: int, flag_base: int, stream=None, token: int = 0) -> int:
        tok = C.c_uint64(token)
        N.call("fsx_forward_host", self._h, host_ptr, dst_gpu, dst_off, nbytes, chunk_bytes,
               flag_base, C.byref(tok), _stream_ptr(stream))
        return tok.value

    # -- dg64 integrity digest ---------------------------------------------------
    def u64_slot(self, gpu: int, stream=None) -> int:
        p = C.c_void_p()
        N.call("fsx_u64_slot", self._h, gpu, C.byref(p), _stream_ptr(stream))
        return p.value

    def read_u64(self, gpu: int, ptr: int, stream=None) -> int:
        v = C.c_uint64()
        N.call("fsx_read_u64", self._h, gpu, ptr, C.byref(v), _stream_ptr(stream))
        return v.value

    def digest(self, gpu: int, ptr: int, nbytes: int, stream=None) -> int:
        """dg64 of device bytes (synchronous convenience)."""
        slot = self.u64_slot(gpu, stream)
        N.call("fsx_digest", self._h, gpu, ptr, nbytes, slot, _stream_ptr(stream))
        return self.read_u64(gpu, slot, stream)

    # -- streaming channels (config C) ---------------------------------------
    def channel_open(self, src_gpu: int, dst_gpu: int, row_bytes: int, slots: int = 64) -> int:
        ch = C.c_int32()
        N.call("fsx_channel_open", self._h, src_gpu, dst_gpu, row_bytes, slots, C.byref(ch))
        return ch.value

    def channel_close(self, ch: int) -> None:
        N.call("fsx_channel_close", self._h, ch)

    @staticmethod
    def _chs(chs):
        return (C.c_int32 * max(len(chs), 1))(*chs)

    def channel_push(self, chs, rows_ptr: int, stride: int, stream=None) -> None:
        N.call("fsx_channel_push", self._h, len(chs), self._chs(chs), rows_ptr, stride,
               _stream_ptr(stream))

    def channel_pull(self, chs, out_ptr: int, stride: int, stream=None) -> None:
        N.call("fsx_channel_pull", self._h, len(chs), self._chs(chs), out_ptr, stride,
               _stream_ptr(stream))

    def _groups(self, groups):
        """[(channels, rows_ptr, stride), ...] -> a ChanGroup array (the
        channel arrays are kept alive on the array object)."""
        arr = (N.ChanGroup * max(len(groups), 1))()
        keep = []
        for i, (chs, ptr, stride) in enumerate(groups):
            a = self._chs(chs)
            keep.append(a)
            arr[i] = N.ChanGroup(len(chs), C.cast(a, C.POINTER(C.c_int32)), ptr, stride)
        arr._keep = keep
        return arr

    def channel_push_groups(self, groups, stream=None) -> None:
        """One push launch for several channel groups (fsx_channel_push_groups):
        groups = [(channels, rows_ptr, stride), ...]."""
        N.call("fsx_channel_push_groups", self._h, len(groups), self._groups(groups), _stream_ptr(stream))

    def channel_pull_groups(self, groups, stream=None) -> None:
        """One pull launch for several channel groups (fsx_channel_pull_groups)."""
        N.call("fsx_channel_pull_groups", self._h, len(groups), self._groups(groups), _stream_ptr(stream))

    def channel_progress(self, ch: int):
        p, c = C.c_uint64(), C.c_uint64()
        N.call("fsx_channel_progress", self._h, ch, C.byref(p), C.byref(c))
        return p.value, c.value

    def merge(self, gpu: int, batch: N.MergeBatch, stream=None) -> None:
        N.call("fsx_merge", self._h, gpu, C.byref(batch), _stream_ptr(stream))

    def forward_place(self, src_gpu: int, dst_gpu: int, batch: N.MergeBatch, done_flag: int = -1,
                      token: int = 0, stream=None) -> None:
        """Direct placement (fsx_forward_place): producer rows straight into
        the consumer's placeholder rows, one launch on src_gpu's device."""
        N.call("fsx_forward_place", self._h, src_gpu, dst_gpu, C.byref(batch), done_flag, token,
               _stream_ptr(stream))

    def synth(self, gpu: int, seed: int, dst_ptr: int, nbytes: int, stream=None) -> None:
        N.call("fsx_synth_payload", self._h, gpu, seed, dst_ptr, nbytes, _stream_ptr(stream))

    def stats(self) -> dict:
        s = N.Stats()
        N.call("fsx_get_stats", self._h, C.byref(s))
        return {k: getattr(s, k) for k, _ in N.Stats._fields_}

    def synchronize(self) -> None:
        N.call("fsx_synchronize", self._h)
