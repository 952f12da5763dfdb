"""ctypes binding of libfsx.so (include/fsx.h).

This is plumbing for the Python tests and bench: the product is the C ABI and
the C++ fabric on top of it.  Loading fails loudly when the library is missing;
every data-moving call raises FsxError when the C ABI reports a non-zero status
(1 + fissim::ErrorCode ordinal, include/fissim/common.hpp:29-47).  There is no
Python or CPU fallback for any operation.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfsx.so")

# fissim::ErrorCode names in ordinal order (common.hpp:29-47).
ERROR_CODES = [
    "validation", "duplicate_app", "not_found", "placement", "oom", "determinism_hazard",
    "determinism_violation", "dangling_ref", "dispatch", "integrity", "protocol", "timeout",
    "infeasible", "config", "connection", "cancelled", "internal",
]

OK = 0
E_VALIDATION = 1
E_NOT_FOUND = 3
E_OOM = 5
E_INTEGRITY = 10
E_PROTOCOL = 11
E_TIMEOUT = 12
E_CONFIG = 14
E_INTERNAL = 17

LOCAL_BUFFER = 0
NETWORK_STREAM = 1

FWD_HOST_NOTIFY = 1
FWD_L2_KEEP = 2
FWD_BULK = 4
FWD_PEER_GPU_COUNT = 16
FWD_DMA = 32  # copy-engine form (cudaMemcpyAsync + cuStreamWriteValue64 flags)
FWD_KERNEL = 64  # force K1 (no automatic copy-engine form)
FWD_DMA_MAX_CHUNKS = 1
FWD_MAX_BATCH = 64  # FSX_FWD_MAX_BATCH: transfers per K1 launch

MERGE_FULL = 0
MERGE_SCAN_ONLY = 1
MERGE_COPY_ONLY = 2
MERGE_DISCARD = 0x100
MERGE_COLOCATED = 0x200


class FsxError(RuntimeError):
    """Mirror of fissim::Error: carries the stable code name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERROR_CODES[status - 1] if 0 < status <= len(ERROR_CODES) else "unknown"
        super().__init__(f"{self.code}: {message}")


class MergeBatch(C.Structure):
    _fields_ = [
        ("num_requests", C.c_int32),
        ("num_items", C.c_int32),
        ("row_bytes", C.c_int64),
        ("placeholder_id", C.c_int32),
        ("mode", C.c_int32),
        ("d_embeds", C.c_void_p),
        ("d_token_ids", C.c_void_p),
        ("d_req_row_off", C.c_void_p),
        ("d_req_item_off", C.c_void_p),
        ("d_item_src", C.c_void_p),
        ("d_item_row_off", C.c_void_p),
        ("d_scratch", C.c_void_p),
        ("d_status", C.c_void_p),
        ("d_item_flag", C.c_void_p),
        ("d_item_token", C.c_void_p),
        ("d_item_chunk_rows", C.c_void_p),
        ("total_rows", C.c_int64),
        ("total_item_rows", C.c_int64),
    ]


class Transfer(C.Structure):
    _fields_ = [
        ("src_gpu", C.c_int32),
        ("dst_gpu", C.c_int32),
        ("d_src", C.c_void_p),
        ("dst_off", C.c_int64),
        ("bytes", C.c_int64),
        ("chunk_bytes", C.c_int64),
        ("flag_base", C.c_int64),
        ("token", C.c_uint64),
        ("d_digest", C.c_void_p),
    ]


def _transfer_dtype():
    import numpy as np

    kinds = {C.c_int32: "<i4", C.c_void_p: "<u8", C.c_int64: "<i8", C.c_uint64: "<u8"}
    return np.dtype({"names": [n for n, _ in Transfer._fields_],
                     "formats": [kinds[t] for _, t in Transfer._fields_],
                     "offsets": [getattr(Transfer, n).offset for n, _ in Transfer._fields_],
                     "itemsize": C.sizeof(Transfer)})


TRANSFER_DTYPE = _transfer_dtype()


class ChanGroup(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("channels", C.POINTER(C.c_int32)),
        ("d_rows", C.c_void_p),
        ("stride", C.c_int64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("forwards", C.c_int64),
        ("bytes_forwarded", C.c_int64),
        ("merges", C.c_int64),
        ("merged_rows", C.c_int64),
        ("segments_in_use", C.c_int64),
        ("bytes_in_use", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("dma_forwards", C.c_int64),
    ]


# name -> (argtypes); every function returns int status except the two strings.
_SIGS = {
    "fsx_device_count": [C.POINTER(C.c_int)],
    "fsx_abi_sizes": [C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    "fsx_open": [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)],
    "fsx_close": [C.c_void_p],
    "fsx_node_of": [C.c_void_p, C.c_int, C.POINTER(C.c_int)],
    "fsx_route": [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int)],
    "fsx_device_of": [C.c_void_p, C.c_int, C.POINTER(C.c_int)],
    "fsx_slab_register": [C.c_void_p, C.c_int, C.c_int64],
    "fsx_slab_alloc": [C.c_void_p, C.c_int, C.c_int64, C.POINTER(C.c_int64)],
    "fsx_slab_free": [C.c_void_p, C.c_int, C.c_int64],
    "fsx_slab_alloc_n": [C.c_void_p, C.c_int, C.c_int32, C.c_void_p, C.c_void_p],
    "fsx_slab_free_n": [C.c_void_p, C.c_int, C.c_int32, C.c_void_p],
    "fsx_slab_ptr": [C.c_void_p, C.c_int, C.c_int64, C.POINTER(C.c_void_p)],
    "fsx_slab_usage": [C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "fsx_slab_read": [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p],
    "fsx_slab_export": [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_int64)],
    "fsx_slab_import": [C.c_void_p, C.c_int, C.c_void_p, C.c_int64],
    "fsx_slab_write": [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p],
    "fsx_ipc_open": [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)],
    "fsx_ipc_close": [C.c_void_p, C.c_void_p],
    "fsx_put_small": [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)],
    "fsx_ticket_wait": [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)],
    "fsx_ticket_digests": [C.c_void_p, C.c_int64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
    "fsx_ticket_free": [C.c_void_p, C.c_int64],
    "fsx_put_small_device": [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)],
    "fsx_put_small_alloc": [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int, C.POINTER(C.c_int64),
                            C.POINTER(C.c_int64)],
    "fsx_ticket_take": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_uint64),
                        C.POINTER(C.c_uint64)],
    "fsx_flush_small": [C.c_void_p],
    "fsx_flags_alloc": [C.c_void_p, C.c_int, C.c_int32, C.POINTER(C.c_int64)],
    "fsx_flag_ptr": [C.c_void_p, C.c_int, C.c_int64, C.POINTER(C.c_void_p)],
    "fsx_forward": [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                    C.c_int64, C.POINTER(C.c_uint64), C.c_void_p],
    "fsx_forward_ex": [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                       C.c_int64, C.POINTER(C.c_uint64), C.c_uint32, C.c_void_p],
    "fsx_forward_batch": [C.c_void_p, C.c_int32, C.POINTER(Transfer), C.c_uint32, C.c_void_p],
    "fsx_forward_host": [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                         C.c_int64, C.POINTER(C.c_uint64), C.c_void_p],
    "fsx_forward_host_digest": [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                C.c_int64, C.POINTER(C.c_uint64), C.c_void_p, C.POINTER(C.c_uint64)],
    "fsx_chunk_ready": [C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.POINTER(C.c_int)],
    "fsx_wait": [C.c_void_p, C.c_int, C.c_int64, C.c_int32, C.c_uint64, C.c_int64],
    "fsx_stream_wait_flags": [C.c_void_p, C.c_int, C.c_int64, C.c_int32, C.c_uint64, C.c_void_p],
    "fsx_signal_flags": [C.c_void_p, C.c_int, C.c_int64, C.c_int32, C.c_uint64, C.c_int,
                         C.c_void_p],
    "fsx_merge": [C.c_void_p, C.c_int, C.POINTER(MergeBatch), C.c_void_p],
    "fsx_forward_place": [C.c_void_p, C.c_int, C.c_int, C.POINTER(MergeBatch), C.c_int64,
                          C.c_uint64, C.c_void_p],
    "fsx_forward_merge": [C.c_void_p, C.c_int32, C.POINTER(Transfer), C.POINTER(MergeBatch),
                          C.c_uint32, C.c_void_p],
    "fsx_channel_open": [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int32, C.POINTER(C.c_int32)],
    "fsx_channel_close": [C.c_void_p, C.c_int32],
    "fsx_channel_push": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "fsx_channel_pull": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "fsx_channel_push_groups": [C.c_void_p, C.c_int32, C.POINTER(ChanGroup), C.c_void_p],
    "fsx_channel_pull_groups": [C.c_void_p, C.c_int32, C.POINTER(ChanGroup), C.c_void_p],
    "fsx_channel_progress": [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
    "fsx_synth_payload": [C.c_void_p, C.c_int, C.c_uint64, C.c_void_p, C.c_int64, C.c_void_p],
    "fsx_digest": [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p],
    "fsx_u64_slot": [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.c_void_p],
    "fsx_read_u64": [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p],
    "fsx_pointer_device": [C.c_void_p, C.POINTER(C.c_int)],
    "fsx_pointer_kind": [C.c_void_p, C.POINTER(C.c_int)],
    "fsx_copy_to_host": [C.c_void_p, C.c_void_p, C.c_int64],
    "fsx_copy_engine": [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "fsx_get_stats": [C.c_void_p, C.POINTER(Stats)],
    "fsx_synchronize": [C.c_void_p],
}

EXPORTED = sorted(list(_SIGS) + ["fsx_last_error", "fsx_version"])

_lib = None


def lib():
    """Load libfsx.so (built in-tree by __graft_entry__.build / make)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libfsx.so not built at {LIB_PATH}: run `make` or "
                              "__graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.fsx_last_error.restype = C.c_char_p
        L.fsx_last_error.argtypes = []
        L.fsx_version.restype = C.c_char_p
        L.fsx_version.argtypes = []
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != OK:
        raise FsxError(status, lib().fsx_last_error().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def device_count() -> int:
    n = C.c_int(0)
    call("fsx_device_count", C.byref(n))
    return n.value
