"""The C ABI library (libfsx.so) without a GPU: it loads, exports every
symbol include/fsx.h declares, and fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2603_12118_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fsx.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(fsx_\w+)\s*\(", src, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == N.EXPORTED


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", N.LIB_PATH], text=True)
    exported = set(re.findall(r" T (fsx_\w+)$", out, re.M))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-lelf", N.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_struct_layouts_match_binding():
    m, t, s = C.c_int32(), C.c_int32(), C.c_int32()
    N.call("fsx_abi_sizes", C.byref(m), C.byref(t), C.byref(s))
    assert m.value == C.sizeof(N.MergeBatch)
    assert t.value == C.sizeof(N.Transfer)
    assert s.value == C.sizeof(N.Stats)


def test_version_string():
    assert b"sm_100a" in N.lib().fsx_version()


@pytest.mark.skipif(N.device_count() > 0, reason="host has a GPU")
def test_open_fails_loudly_without_gpu():
    assert N.device_count() == 0
    h = C.c_void_p()
    ids = (C.c_int * 2)(0, 1)
    nodes = (C.c_int * 2)(0, 0)
    with pytest.raises(N.FsxError) as e:
        N.call("fsx_open", 2, ids, nodes, None, C.byref(h))
    assert e.value.code == "config"
    assert "no CPU fallback" in str(e.value)


def test_error_codes_follow_reference_ordinals():
    # include/fissim/common.hpp:29-47, status = 1 + ordinal
    assert N.ERROR_CODES[N.E_VALIDATION - 1] == "validation"
    assert N.ERROR_CODES[N.E_NOT_FOUND - 1] == "not_found"
    assert N.ERROR_CODES[N.E_INTEGRITY - 1] == "integrity"
    assert N.ERROR_CODES[N.E_PROTOCOL - 1] == "protocol"
    assert N.ERROR_CODES[N.E_TIMEOUT - 1] == "timeout"
    assert N.ERROR_CODES[N.E_CONFIG - 1] == "config"
    assert N.ERROR_CODES[N.E_INTERNAL - 1] == "internal"


def test_python_constants_match_header():
    """Every FSX_* constant the bindings restate (status codes, transports,
    forward options, FSX_FWD_MAX_BATCH, merge modes) equals include/fsx.h."""
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hdr = open(os.path.join(root, "include", "fsx.h")).read()
    defs = {m.group(1): int(m.group(2), 0)
            for m in re.finditer(r"#define FSX_(\w+) (0x[0-9a-fA-F]+|\d+)u?\b", hdr)}
    pairs = {"E_VALIDATION": "E_VALIDATION", "E_NOT_FOUND": "E_NOT_FOUND", "E_OOM": "E_OOM",
             "E_INTEGRITY": "E_INTEGRITY", "E_PROTOCOL": "E_PROTOCOL", "E_TIMEOUT": "E_TIMEOUT",
             "E_CONFIG": "E_CONFIG", "E_INTERNAL": "E_INTERNAL",
             "TRANSPORT_LOCAL_BUFFER": "LOCAL_BUFFER", "TRANSPORT_NETWORK_STREAM": "NETWORK_STREAM",
             "FWD_HOST_NOTIFY": "FWD_HOST_NOTIFY", "FWD_L2_KEEP": "FWD_L2_KEEP", "FWD_BULK": "FWD_BULK",
             "FWD_PEER_GPU_COUNT": "FWD_PEER_GPU_COUNT", "FWD_MAX_BATCH": "FWD_MAX_BATCH",
             "FWD_DMA": "FWD_DMA", "FWD_KERNEL": "FWD_KERNEL", "FWD_DMA_MAX_CHUNKS": "FWD_DMA_MAX_CHUNKS",
             "MERGE_FULL": "MERGE_FULL", "MERGE_SCAN_ONLY": "MERGE_SCAN_ONLY",
             "MERGE_COPY_ONLY": "MERGE_COPY_ONLY", "MERGE_DISCARD": "MERGE_DISCARD",
             "MERGE_COLOCATED": "MERGE_COLOCATED"}
    for h, py in pairs.items():
        assert h in defs, h
        assert getattr(N, py) == defs[h], (h, defs[h], getattr(N, py))
