"""The N>1 producer->consumer pair protocol end to end on ONE GPU: two
processes (torchrun, gloo for setup), rank 0 pushes into rank 1's slab through
a CUDA IPC mapping, rank 1 runs the early-start merge and acks each step into
rank 0's ack slab.  Both ranks are pinned to device 0 (FSX_PAIRS_DEVICE), so
this checks the protocol and the bytes, not NVLink bandwidth."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("config,requests,direct", [("B", 1, False), ("A", 16, False),
                                                    ("B", 2, True), ("A", 16, True)])
def test_pairs_protocol_same_device(gpu, config, requests, direct):
    """direct: FSX_PAIRS_DIRECT=1, the producer places rows straight into the
    consumer's IPC-mapped prompt embedding (fsx_forward_place) + done flag."""
    env = dict(os.environ, FSX_PAIRS_DEVICE="0")
    if direct:
        env["FSX_PAIRS_DIRECT"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", "bench.py", "--gpus", "2",
           "--steps", "4", "--warmup", "2", "--config", config, "--requests", str(requests),
           "--verify"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=400)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert lines, p.stdout[-2000:]
    d = json.loads(lines[-1])
    assert d["n_gpus"] == 2 and d["verified"] and d["pinned_device"] == "0"
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert ("direct placement" in d["config"]["transfer"]) == direct


def test_fanout_config_d_four_ranks_same_device(gpu):
    """Config D fan-out (2 encoders -> 2 LLM replicas, reference select_replica
    placement, so both LLMs receive from both encoders) as 4 processes pinned to
    one device: IPC slab imports per edge, batched K1 into several peers'
    slabs, early-start merge with fan-in, per-edge acks; merged embeddings
    verified against a local pass on every LLM rank."""
    env = dict(os.environ, FSX_PAIRS_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", "bench.py", "--gpus", "4",
           "--steps", "3", "--warmup", "2", "--config", "D", "--requests", "6", "--verify"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert lines, p.stdout[-2000:]
    d = json.loads(lines[-1])
    assert d["n_gpus"] == 4 and d["verified"]
    assert d["config"]["encoders"] == 2 and d["config"]["llms"] == 2
    assert max(d["config"]["fan_in"]) == 2 and max(d["config"]["fan_out"]) == 2
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
