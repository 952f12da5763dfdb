"""Streaming channels (config C) on the GPU: thinker hidden states (one
[hidden_dim] bf16 row per token per request, executor_sim.hpp:556-562) and
talker codes (4 B per chunk, :543-549) delivered in seq order, byte-exact
against the reference payloads synth_payload(payload_seed(ref_id, seq))."""
import numpy as np
import pytest

from paper_2603_12118_b200 import trace as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fab(gpu):
    from paper_2603_12118_b200.fabric import DeviceFabric

    f = DeviceFabric({0: 0, 1: 0, 2: 0}, {0: 0, 1: 0, 2: 0})
    f.slab_register(1, 256 << 20)
    f.slab_register(2, 64 << 20)
    yield f
    f.close()


def _rows(oracle_mod, ref_ids, seq, nbytes):
    return np.stack([np.frombuffer(oracle_mod.synth_payload(T.payload_seed(r, seq), nbytes), np.uint8)
                     for r in ref_ids])


@pytest.mark.parametrize("hidden,batch", [(3584, 32), (1024, 7)])
def test_hidden_state_stream_in_order(fab, oracle_mod, hidden, batch):
    import torch

    nb = hidden * 2
    refs = [f"req-{i:06d}/r0001" for i in range(batch)]
    chs = [fab.channel_open(0, 1, nb, slots=8) for _ in refs]
    rows = torch.empty((batch, nb), dtype=torch.uint8, device="cuda")
    out = torch.empty((batch, nb), dtype=torch.uint8, device="cuda")
    for step in range(12):
        want = _rows(oracle_mod, refs, step, nb)
        rows.copy_(torch.from_numpy(want))
        fab.channel_push(chs, rows.data_ptr(), nb)
        out.zero_()
        fab.channel_pull(chs, out.data_ptr(), nb)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want), step
    for ch in chs:
        assert fab.channel_progress(ch) == (12, 12)
        fab.channel_close(ch)


def test_ring_depth_and_partial_steps(fab, oracle_mod):
    """Several steps in flight before the consumer pulls (up to the ring
    depth), and steps that carry only a subset of the streams."""
    import torch

    nb = 2048
    refs = [f"req-{i:06d}/r0001" for i in range(5)]
    chs = [fab.channel_open(0, 2, nb, slots=4) for _ in refs]
    seqs = [0] * 5
    sent = {i: [] for i in range(5)}
    rows = torch.empty((5, nb), dtype=torch.uint8, device="cuda")
    plan = [[0, 1, 2, 3, 4], [1, 3], [0, 1, 2, 3, 4], [4]]  # <= 3 pending per stream
    for active in plan:
        want = np.stack([np.frombuffer(oracle_mod.synth_payload(T.payload_seed(refs[i], seqs[i]), nb),
                                       np.uint8) for i in active])
        rows[:len(active)].copy_(torch.from_numpy(want))
        fab.channel_push([chs[i] for i in active], rows.data_ptr(), nb)
        for k, i in enumerate(active):
            sent[i].append(want[k])
            seqs[i] += 1
    out = torch.empty((1, nb), dtype=torch.uint8, device="cuda")
    for i in range(5):
        for k in range(len(sent[i])):
            fab.channel_pull([chs[i]], out.data_ptr(), nb)
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy()[0], sent[i][k]), (i, k)
    for ch in chs:
        fab.channel_close(ch)


def test_talker_codes_and_backpressure(fab, oracle_mod):
    """4-byte codes; ring of 2 with 6 steps: pulls queued first on a second
    stream, pushes wait in-kernel for free slots."""
    import torch

    refs = [f"req-{i:06d}/r0002" for i in range(16)]
    chs = [fab.channel_open(1, 2, 4, slots=2) for _ in refs]
    steps = 6
    src = torch.empty((steps, 16, 4), dtype=torch.uint8, device="cuda")
    want = np.stack([_rows(oracle_mod, refs, s, 4) for s in range(steps)])
    src.copy_(torch.from_numpy(want))
    out = torch.zeros((steps, 16, 4), dtype=torch.uint8, device="cuda")
    s_pull, s_push = torch.cuda.Stream(), torch.cuda.Stream()
    for s in range(steps):
        fab.channel_pull(chs, out[s].data_ptr(), 4, s_pull)
    for s in range(steps):
        fab.channel_push(chs, src[s].data_ptr(), 4, s_push)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
    for ch in chs:
        assert fab.channel_progress(ch) == (steps, steps)
        fab.channel_close(ch)


def test_channel_errors(fab):
    from paper_2603_12118_b200 import _native as N

    with pytest.raises(N.FsxError) as e:
        fab.channel_open(0, 7, 64)
    assert e.value.code == "not_found"
    with pytest.raises(N.FsxError) as e:
        fab.channel_push([12345], 0, 64)
    assert e.value.code == "not_found"
    a = fab.channel_open(0, 1, 64)
    b = fab.channel_open(1, 2, 64)
    import torch

    rows = torch.empty((2, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(N.FsxError) as e:  # stride below the row size
        fab.channel_push([a], rows.data_ptr(), 32)
    assert e.value.code == "validation"
    fab.channel_close(a)
    fab.channel_close(b)


def test_channel_groups_one_launch_per_step(fab, oracle_mod):
    """fsx_channel_push_groups / _pull_groups: a decode step's thinker hidden
    rows (gpu 0 -> 1, 7 KiB) and talker codes (gpu 1 -> 2, 4 B) from two
    buffers move in one push and one pull launch, in seq order, byte-exact;
    more than 48 rows in one call split into several launches."""
    import torch

    for nh, nc in [(32, 16), (40, 20)]:  # 48 rows: one launch each way; 60: two
        hb = 3584 * 2
        hrefs = [f"req-{i:06d}/r0002" for i in range(nh)]
        crefs = [f"req-{i:06d}/r0003" for i in range(nc)]
        hch = [fab.channel_open(0, 1, hb, slots=4) for _ in hrefs]
        cch = [fab.channel_open(1, 2, 4, slots=4) for _ in crefs]
        hrows = torch.empty((nh, hb), dtype=torch.uint8, device="cuda")
        crows = torch.empty((nc, 4), dtype=torch.uint8, device="cuda")
        hout, cout = torch.empty_like(hrows), torch.empty_like(crows)
        for step in range(6):
            hw, cw = _rows(oracle_mod, hrefs, step, hb), _rows(oracle_mod, crefs, step, 4)
            hrows.copy_(torch.from_numpy(hw))
            crows.copy_(torch.from_numpy(cw))
            hout.zero_()
            cout.zero_()
            l0 = fab.stats()["kernel_launches"]
            fab.channel_push_groups([(hch, hrows.data_ptr(), hb), (cch, crows.data_ptr(), 4)])
            fab.channel_pull_groups([(hch, hout.data_ptr(), hb), (cch, cout.data_ptr(), 4)])
            assert fab.stats()["kernel_launches"] - l0 == 2 * -(-(nh + nc) // 48)
            torch.cuda.synchronize()
            assert np.array_equal(hout.cpu().numpy(), hw), step
            assert np.array_equal(cout.cpu().numpy(), cw), step
        for ch in hch + cch:
            assert fab.channel_progress(ch) == (6, 6)
            fab.channel_close(ch)


def test_channel_groups_validation(fab):
    import torch

    from paper_2603_12118_b200 import _native as N

    ch = fab.channel_open(0, 1, 64, slots=2)
    rows = torch.empty((2, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(N.FsxError) as e:  # stride below the row size
        fab.channel_push_groups([([ch], rows.data_ptr(), 32)])
    assert e.value.code == "validation"
    with pytest.raises(N.FsxError) as e:
        fab.channel_push_groups([([ch], rows.data_ptr(), 64), ([12345], rows.data_ptr(), 64)])
    assert e.value.code == "not_found"
    assert fab.channel_progress(ch) == (0, 0)  # nothing launched
    fab.channel_close(ch)
