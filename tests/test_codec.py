"""Binary sidecar envelope (include/fsx/envelope_codec.hpp):
round trips against the drop-in fissim::ForwardEnvelope, rejection of
truncated / foreign records, and the per-envelope cost next to the
reference's JSON route.  CPU only; the test binary is built from the
reference headers by `make cpptests` (or here when the reference tree is
present)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_envelope_codec")


def test_binary_envelope_codec():
    if not os.path.exists(BIN):
        if not os.path.exists("/root/reference/proj/include/fissim/common.hpp"):
            pytest.skip("reference tree absent and no prebuilt build/test_envelope_codec")
        subprocess.check_call(["make", "-s", "-C", ROOT, "build/test_envelope_codec"])
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-3000:]
    assert "3 test cases, 0 failed" in out, out[-3000:]
    line = next(l for l in out.splitlines() if l.startswith("{"))
    cost = json.loads(line)
    assert cost["binary_bytes"] < cost["json_bytes"]
    assert cost["binary_ns_per_envelope"] < cost["json_ns_per_envelope"]
