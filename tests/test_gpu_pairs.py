"""The N>1 producer->consumer pair protocol end to end on ONE GPU: two
processes (torchrun, gloo for setup), rank 0 pushes into rank 1's slab through
a CUDA IPC mapping, rank 1 runs the early-start merge and acks each step into
rank 0's ack slab.  Both ranks are pinned to device 0 (--pin-device), so
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


def _run(args, timeout=400, launcher="torchrun", nproc=2):
    if launcher == "torchrun":
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr=127.0.0.1", f"--master-port={_port()}", "bench.py"] + args
    else:  # bench.py spawns its own ranks
        cmd = [sys.executable, "bench.py"] + args
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("config,requests,transfer,k1", [("B", 1, "slab", "auto"), ("A", 16, "slab", "tile"),
                                                         ("A", 16, "slab", "gpucount"),
                                                         ("A", 16, "slab", "bulk"),
                                                         ("A", 16, "slab", "dma"),
                                                         ("B", 2, "direct", "auto"), ("A", 16, "direct", "auto")])
def test_pairs_protocol_same_device(gpu, config, requests, transfer, k1):
    """The pair protocol for every peer K1 form (register tiles with a
    system-scope count per tile, gpu-scope count + one system-scope publish
    per chunk, bulk-copy tiles, the copy engine + a flag kernel; auto probes
    all four) and for direct
    placement (fsx_forward_place into the consumer's IPC-mapped prompt + done
    flag): merged embeddings verified bit-exact on the consumer."""
    d = _run(["--gpus", "2", "--pin-device", "0", "--steps", "4", "--warmup", "2", "--config", config,
              "--requests", str(requests), "--transfer", transfer, "--k1", k1])
    assert d["n_gpus"] == 2 and d["verified"] and d["pinned_device"] == 0
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert ("direct placement" in d["config"]["transfer"]) == (transfer == "direct")
    if transfer == "slab":
        forms = d["k1_forms"]
        assert forms["chosen"] == (k1 if k1 != "auto" else min(forms["probe_ms_per_step"],
                                                               key=forms["probe_ms_per_step"].get))
        assert d["copy_engine"]["ms_per_step"] > 0


def test_pairs_litmus_many_small_chunks(gpu):
    """Ordering litmus across processes: 40 steps of config A with 64-row
    (512 KiB) chunks, so thousands of chunk flags are published by the
    producer's K1 (gpu-scope count + system-scope publish) while the consumer's
    early-start merge reads each chunk right after its flag: any chunk read
    before its bytes landed would break the bit-exact check."""
    d = _run(["--gpus", "2", "--pin-device", "0", "--steps", "40", "--warmup", "2", "--config", "A",
              "--requests", "24", "--k1", "gpucount", "--chunk-rows", "64", "--sets", "3"], timeout=600)
    assert d["verified"] and d["config"]["chunk_bytes"] == 64 * 8192


def test_bench_spawns_its_own_ranks(gpu):
    """python bench.py --gpus 2 without torchrun (no RANK/WORLD_SIZE): bench.py
    starts both ranks itself and rank 0 prints the single line."""
    d = _run(["--gpus", "2", "--pin-device", "0", "--steps", "3", "--warmup", "2", "--config", "A",
              "--requests", "8"], launcher="self")
    assert d["n_gpus"] == 2 and d["verified"]


def test_fanout_config_d_four_ranks_same_device(gpu):
    """Config D fan-out (2 encoders -> 2 LLM replicas, reference select_replica
    placement, so both LLMs receive from both encoders) as 4 processes pinned to
    one device: IPC slab imports per edge, batched K1 into several peers'
    slabs, early-start merge with fan-in, per-edge acks; merged embeddings
    verified against a local pass on every LLM rank."""
    d = _run(["--gpus", "4", "--pin-device", "0", "--steps", "3", "--warmup", "2", "--config", "D",
              "--requests", "6"], timeout=600, nproc=4)
    assert d["n_gpus"] == 4 and d["verified"]
    assert d["config"]["encoders"] == 2 and d["config"]["llms"] == 2
    assert max(d["config"]["fan_in"]) == 2 and max(d["config"]["fan_out"]) == 2
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0


def test_bench_single_gpu_line(gpu):
    """bench.py at N = 1 (config A, short): one JSON line whose roofline names
    the timed kernel (the tee) with an event-timed rate, the other schedules
    and kernels measured beside it, and config.workload identical to the
    reference arm's (the driver compares them)."""
    d = _run(["--steps", "5", "--warmup", "3", "--config", "A", "--no-cpu-baseline", "--no-e2e",
              "--colocated"], launcher="self")
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert d["config"]["workload"] == b.CONFIGS["A"]["workload"]
    assert "merge_tee_kernel" in d["roofline"]["kernel"] and 0 < d["roofline"]["frac"] < 1.5
    assert set(d["kernels"]) >= {"tee", "forward", "merge", "follow"}
    assert set(d["schedules"]) >= {"tee", "serial", "colocated", "direct_placement"}
    assert len(d["schedules"]["colocated"]["runs_ms"]) == 5
    assert d["gpu_launches"] >= 5


def test_bench_config_c_line(gpu):
    """bench.py --config C: the Qwen2.5-Omni decode step (32 hidden rows + 16
    codes through the streaming channels as one CUDA graph) prints one line
    with the BASELINE metric, a device per-step time, an e2e from host memory
    and the reference arm's workload name (the rows are checked byte-exact
    inside bench.py)."""
    d = _run(["--config", "C", "--steps", "20", "--warmup", "3", "--no-cpu-baseline"], launcher="self")
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert d["config"]["workload"] == b.CONFIGS["C"]["workload"] and d["metric"] == b.METRIC
    assert d["value"] > 0 and 0 < d["us_per_step"] < 1000
    assert d["e2e"]["h2d_bytes_per_step"] == 32 * 7168 + 16 * 4 and d["e2e"]["value"] > 0
    # one push + one pull launch per step (channel groups), against four per
    # step when each group is pushed and pulled on its own
    assert d["gpu_launches"] == 2 * 20 and d["gpu_launches_per_step"] == 2
    assert d["schedules"]["per_group"]["kernels_per_step"] == 4
