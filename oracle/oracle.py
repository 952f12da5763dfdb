"""ctypes bindings for the oracle libraries.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module, and only as the checker or as
the timed CPU baseline.  The product package never imports it.

* ``C``   -> oracle/libfsx_oracle.so  (plain-C restatement, fsx_oracle.c)
* ``REF`` -> oracle/_ref/libref_oracle.so (the reference headers compiled
  unmodified, ref_oracle.cpp); None when it was not built.
"""
from __future__ import annotations

import ctypes as C_
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libfsx_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_oracle.so")

u8p = C_.POINTER(C_.c_uint8)
i32p = C_.POINTER(C_.c_int32)
i64p = C_.POINTER(C_.c_int64)


def build(ref: bool = True) -> None:
    """Compile the restatement (and the reference shim when the reference
    headers are present).  Building the checker is not using it."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    inc = os.environ.get("FISSIM_REF_INCLUDE", "/root/reference/proj/include")
    if ref and os.path.exists(os.path.join(inc, "fissim", "sidecar.hpp")):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref", f"FISSIM_REF_INCLUDE={inc}"])


class ShapeRules(C_.Structure):
    _fields_ = [
        ("pixels_per_token", C_.c_int64),
        ("default_image_width", C_.c_int64),
        ("default_image_height", C_.c_int64),
        ("tokens_per_frame", C_.c_int64),
        ("default_video_frames", C_.c_int64),
        ("tokens_per_audio_second", C_.c_int64),
        ("default_audio_seconds", C_.c_double),
        ("hidden_dim", C_.c_int64),
        ("embed_elem_bytes", C_.c_int64),
    ]


def _load_c():
    if not os.path.exists(ORACLE_SO):
        build(ref=False)
    lib = C_.CDLL(ORACLE_SO)
    lib.or_splitmix64.restype = C_.c_uint64
    lib.or_splitmix64.argtypes = [C_.POINTER(C_.c_uint64)]
    lib.or_fnv1a64.restype = C_.c_uint64
    lib.or_fnv1a64.argtypes = [C_.c_char_p, C_.c_size_t]
    lib.or_checksum64.restype = C_.c_uint64
    lib.or_checksum64.argtypes = [C_.c_void_p, C_.c_size_t]
    lib.or_synth_payload_into.restype = None
    lib.or_synth_payload_into.argtypes = [C_.c_uint64, C_.c_void_p, C_.c_size_t]
    lib.or_digest64.restype = C_.c_uint64
    lib.or_digest64.argtypes = [C_.c_void_p, C_.c_size_t]
    lib.or_payload_seed.restype = C_.c_uint64
    lib.or_payload_seed.argtypes = [C_.c_char_p, C_.c_size_t, C_.c_int64]
    lib.or_shape_rules_default.argtypes = [C_.POINTER(ShapeRules)]
    lib.or_item_tokens.restype = C_.c_int64
    lib.or_item_tokens.argtypes = [C_.POINTER(ShapeRules), C_.c_int, C_.c_int64, C_.c_int64,
                                   C_.c_int64, C_.c_double]
    lib.or_arena_new.restype = C_.c_void_p
    lib.or_arena_new.argtypes = [C_.c_int64]
    lib.or_arena_delete.argtypes = [C_.c_void_p]
    lib.or_arena_alloc.restype = C_.c_int64
    lib.or_arena_alloc.argtypes = [C_.c_void_p, C_.c_int64]
    lib.or_arena_free.restype = C_.c_int
    lib.or_arena_free.argtypes = [C_.c_void_p, C_.c_int64]
    for n in ("segments_in_use", "bytes_in_use", "peak_bytes"):
        f = getattr(lib, "or_arena_" + n)
        f.restype = C_.c_int64
        f.argtypes = [C_.c_void_p]
    lib.or_merge.restype = C_.c_int
    lib.or_merge.argtypes = [C_.c_int32, C_.c_int64, C_.c_int32, C_.c_void_p, C_.c_void_p,
                             C_.c_void_p, C_.c_void_p, C_.c_void_p, C_.c_void_p, C_.c_void_p,
                             C_.c_int]
    lib.or_prompt_tokens.restype = None
    lib.or_prompt_tokens.argtypes = [C_.c_char_p, C_.c_size_t, C_.c_int64, C_.c_int32,
                                     C_.c_void_p, C_.c_int32, C_.c_int32, C_.c_void_p]
    return lib


def _load_ref():
    if not os.path.exists(REF_SO):
        return None
    lib = C_.CDLL(REF_SO)
    lib.ref_last_error.restype = C_.c_char_p
    lib.ref_checksum64.restype = C_.c_uint64
    lib.ref_checksum64.argtypes = [C_.c_void_p, C_.c_size_t]
    lib.ref_synth_payload_into.restype = None
    lib.ref_synth_payload_into.argtypes = [C_.c_uint64, C_.c_void_p, C_.c_size_t]
    lib.ref_fnv1a64.restype = C_.c_uint64
    lib.ref_fnv1a64.argtypes = [C_.c_char_p, C_.c_size_t]
    lib.ref_splitmix64.restype = C_.c_uint64
    lib.ref_splitmix64.argtypes = [C_.POINTER(C_.c_uint64)]
    lib.ref_payload_seed.restype = C_.c_uint64
    lib.ref_payload_seed.argtypes = [C_.c_char_p, C_.c_size_t, C_.c_int64]
    lib.ref_item_tokens.restype = C_.c_int64
    lib.ref_item_tokens.argtypes = [C_.c_char_p, C_.c_char_p]
    lib.ref_embed_bytes.restype = C_.c_int64
    lib.ref_embed_bytes.argtypes = [C_.c_char_p, C_.c_char_p]
    lib.ref_arena_new.restype = C_.c_void_p
    lib.ref_arena_new.argtypes = [C_.c_int64]
    lib.ref_arena_delete.argtypes = [C_.c_void_p]
    lib.ref_arena_alloc.restype = C_.c_int64
    lib.ref_arena_alloc.argtypes = [C_.c_void_p, C_.c_int64]
    lib.ref_arena_free.restype = C_.c_int
    lib.ref_arena_free.argtypes = [C_.c_void_p, C_.c_int64]
    lib.ref_arena_segments_in_use.restype = C_.c_int64
    lib.ref_arena_segments_in_use.argtypes = [C_.c_void_p]
    lib.ref_arena_bytes_in_use.restype = C_.c_int64
    lib.ref_arena_bytes_in_use.argtypes = [C_.c_void_p]
    lib.ref_forward.restype = C_.c_int
    lib.ref_forward.argtypes = [C_.c_int, C_.c_int, C_.c_char_p, C_.c_void_p, C_.c_size_t,
                                C_.c_void_p, C_.c_void_p]
    lib.ref_forward_bench.restype = C_.c_double
    lib.ref_forward_bench.argtypes = [C_.c_size_t, C_.c_int, C_.c_int]
    lib.ref_dataplane_pass.restype = C_.c_double
    lib.ref_dataplane_pass.argtypes = [C_.c_int32, C_.c_int32, C_.c_int64, C_.c_int32,
                                       C_.c_void_p, C_.c_void_p, C_.c_void_p, C_.c_void_p,
                                       C_.c_void_p, C_.c_void_p, C_.c_void_p, C_.c_int, C_.c_int,
                                       C_.c_int, C_.c_void_p]
    lib.ref_dataplane_pass_mt.restype = C_.c_double
    lib.ref_dataplane_pass_mt.argtypes = lib.ref_dataplane_pass.argtypes
    lib.ref_stream_bench.restype = C_.c_double
    lib.ref_stream_bench.argtypes = [C_.c_int64, C_.c_int, C_.c_int]
    lib.ref_generate_workload.restype = C_.c_char_p
    lib.ref_generate_workload.argtypes = [C_.c_char_p, C_.c_double, C_.c_double, C_.c_uint64]
    lib.ref_record.restype = C_.c_char_p
    lib.ref_record.argtypes = [C_.c_char_p] * 5
    lib.ref_dispatch.restype = C_.c_char_p
    lib.ref_dispatch.argtypes = [C_.c_char_p] * 5
    return lib


C = _load_c()
REF = _load_ref()


# ---------------------------------------------------------------------------
# Convenience wrappers (bytes in / bytes out)

def synth_payload(seed: int, n: int, lib=None) -> bytes:
    lib = lib or C
    buf = (C_.c_uint8 * max(n, 1))()
    (lib.or_synth_payload_into if lib is C else lib.ref_synth_payload_into)(seed, buf, n)
    return bytes(buf)[:n]


def checksum64(data: bytes, lib=None) -> int:
    lib = lib or C
    f = lib.or_checksum64 if lib is C else lib.ref_checksum64
    return f(data, len(data))


def fnv1a64(s: str, lib=None) -> int:
    lib = lib or C
    b = s.encode()
    return (lib.or_fnv1a64 if lib is C else lib.ref_fnv1a64)(b, len(b))


def payload_seed(ref_id: str, seq: int, lib=None) -> int:
    lib = lib or C
    b = ref_id.encode()
    return (lib.or_payload_seed if lib is C else lib.ref_payload_seed)(b, len(b), seq)


def prompt_tokens(request_id: str, input_tokens: int, item_rows, placeholder_id: int,
                  text_vocab: int):
    import numpy as np
    rows = np.asarray(item_rows, dtype=np.int64)
    T = int(input_tokens + rows.sum())
    out = np.empty(T, dtype=np.int32)
    b = request_id.encode()
    C.or_prompt_tokens(b, len(b), input_tokens, len(rows), rows.ctypes.data, placeholder_id,
                       text_vocab, out.ctypes.data)
    return out


def merge(row_bytes: int, placeholder_id: int, embeds, token_ids, req_row_off, req_item_off,
          item_src, item_rows, nthreads: int = 1):
    """Run the CPU merge restatement in place on numpy buffers.  ``item_src``
    is a list of numpy uint8 arrays.  Returns the per-request status array."""
    import numpy as np
    R = len(req_row_off) - 1
    ptrs = (C_.c_void_p * max(len(item_src), 1))(*[a.ctypes.data for a in item_src])
    status = np.zeros(max(R, 1), dtype=np.int32)
    rro = np.ascontiguousarray(req_row_off, dtype=np.int64)
    rio = np.ascontiguousarray(req_item_off, dtype=np.int64)
    rows = np.ascontiguousarray(item_rows, dtype=np.int64)
    C.or_merge(R, row_bytes, placeholder_id, embeds.ctypes.data, token_ids.ctypes.data,
               rro.ctypes.data, rio.ctypes.data, ptrs, rows.ctypes.data if len(rows) else None,
               status.ctypes.data, nthreads)
    return status[:R]


def ref_record(kind: str, config: dict, request: dict, rules: dict, request_id: str) -> dict:
    """The reference record() of one request (record_replay.hpp:510-528)."""
    import json
    out = REF.ref_record(kind.encode(), json.dumps(config).encode(), json.dumps(request).encode(),
                         json.dumps(rules).encode(), request_id.encode())
    if out is None:
        raise RuntimeError(REF.ref_last_error().decode())
    return json.loads(out)


def ref_dispatch(kind: str, config: dict, requests, rules: dict, replica_gpus: dict) -> list:
    """The reference TaskDispatcher::dispatch of a batch of (request_id,
    request) pairs (task_dispatcher.hpp:178-266)."""
    import json
    out = REF.ref_dispatch(kind.encode(), json.dumps(config).encode(),
                           json.dumps([[rid, rq] for rid, rq in requests]).encode(),
                           json.dumps(rules).encode(), json.dumps(replica_gpus).encode())
    if out is None:
        raise RuntimeError(REF.ref_last_error().decode())
    return json.loads(out)
