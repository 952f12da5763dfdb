"""Multi-process host logic of the N>1 path on CPU (gloo, world_size 2 and 3):
roles, the per-step flag/token schedule both ranks derive independently, and
the one-time setup exchange."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_12118_b200 import pairs


def test_roles():
    r = [pairs.role(i, 4) for i in range(4)]
    assert [x.producer for x in r] == [True, False, True, False]
    assert [x.peer for x in r] == [1, 0, 3, 2]
    assert (r[2].producer_gpu, r[2].consumer_gpu) == (2, 3)
    odd = pairs.role(2, 3)
    assert odd.alone and odd.producer
    assert pairs.pairs_in(8) == 4 and pairs.pairs_in(3) == 2


def test_schedule_unique_and_windowed():
    chunks = [16, 16, 1, 4]
    seen_tokens = set()
    for s in range(200):
        sch = pairs.schedule(s, chunks)
        bases = [b for b, _ in sch]
        assert bases == sorted(bases)
        for (b, t), n in zip(sch, chunks):
            assert t not in seen_tokens and t != 0
            seen_tokens.add(t)
            assert 0 <= b and b + n <= pairs.FLAG_WINDOW * sum(chunks)
        assert pairs.ack_token(s) not in seen_tokens
    # the same step slot reuses the same flag range with different tokens
    assert [b for b, _ in pairs.schedule(3, chunks)] == [b for b, _ in pairs.schedule(67, chunks)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    me = pairs.role(rank, world)
    # consumer publishes (slab handle, segment offsets); producer its ack slab
    mine = {"rank": rank, "handle": bytes([rank]) * 64,
            "offsets": [0, 117440512] if not me.producer else None}
    got = pairs.exchange(mine)
    chunks = [16, 16]
    sched = [pairs.schedule(s, chunks) for s in range(5)]
    peer_view = got[me.peer] if not me.alone else None
    q.put((rank, me.producer, peer_view["handle"] if peer_view else None,
           peer_view["offsets"] if peer_view else None, sched))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_setup_exchange_and_agreement(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, prod, handle, offs, sched = q.get(timeout=120)
        res[rank] = (prod, handle, offs, sched)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # rank 0 (producer) sees rank 1's slab handle and offsets; rank 1 sees rank 0's ack slab
    assert res[0][1] == bytes([1]) * 64 and res[0][2] == [0, 117440512]
    assert res[1][1] == bytes([0]) * 64 and res[1][2] is None
    # both sides derived the identical flag/token schedule without messaging
    assert res[0][3] == res[1][3]
    if world == 3:
        assert res[2][1] is None  # odd rank out runs alone


def test_fanout_plan_follows_select_replica():
    """Config D placement (paper_2603_12118_b200/fanout.py): least-outstanding
    + round-robin selection per task, many-to-many edges, per-consumer flag
    schedule disjoint across items and steps."""
    from paper_2603_12118_b200 import fanout
    from paper_2603_12118_b200 import trace as T

    reqs = T.config_requests("D", 64)
    pl = fanout.plan(reqs, 8, 1024)
    assert pl.producers == [0, 2, 4, 6] and pl.consumers == [1, 3, 5, 7]
    # with nothing completing inside a step, least-outstanding + RR is exact
    # round robin per task: LLM replicas in request order ...
    assert pl.llm_of == [k % 4 for k in range(64)]
    # ... and each modality's encoder replicas in item order
    for mod in ("image", "video", "audio"):
        seq = [pl.enc_of[k][j] for k, q in enumerate(reqs) for j, it in enumerate(q.items)
               if it.modality == mod]
        assert seq == [i % 4 for i in range(len(seq))]
    # every item is produced by exactly one encoder and lands in exactly one LLM list
    all_items = sorted(kj for p in range(4) for kj in pl.producer_items(p))
    assert all_items == sorted((k, j) for k, q in enumerate(reqs) for j in range(len(q.items)))
    assert sorted(kj for c in range(4) for kj in pl.consumer_items[c]) == all_items
    # fan-out and fan-in both happen
    assert any(len(pl.consumers_of(p)) > 1 for p in range(4))
    assert any(len(pl.producers_of(c)) > 1 for c in range(4))
    # flag ranges of one consumer are disjoint within a step and tokens unique
    for c in range(4):
        for s in (0, 1, 63, 64):
            spans, toks = [], set()
            for idx, (k, j) in enumerate(pl.consumer_items[c]):
                b, t = pl.schedule(s, c, idx)
                spans.append((b, b + pl.chunks[k][j]))
                assert t != 0 and t not in toks
                toks.add(t)
                assert pl.item_slot(k, j) == (c, idx)
            spans.sort()
            assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))


def test_fanout_plan_two_ranks_is_a_pair():
    from paper_2603_12118_b200 import fanout
    from paper_2603_12118_b200 import trace as T

    reqs = T.config_requests("D", 8)
    pl = fanout.plan(reqs, 2, 1024)
    assert pl.producers == [0] and pl.consumers == [1]
    assert set(pl.llm_of) == {0}
    assert all(e == 0 for es in pl.enc_of for e in es)


@pytest.mark.parametrize("world", [3, 5, 6])
def test_fanout_plan_odd_and_uneven_worlds(world):
    """Encoders on the even ranks, LLMs on the odd ones for any world size:
    every item lands in exactly one LLM list, placement stays round robin per
    task, and per-LLM flag ranges stay disjoint."""
    from paper_2603_12118_b200 import fanout
    from paper_2603_12118_b200 import trace as T

    reqs = T.config_requests("D", 40)
    pl = fanout.plan(reqs, world, 1024)
    assert pl.producers == list(range(0, world, 2)) and pl.consumers == list(range(1, world, 2))
    n_llm = len(pl.consumers)
    assert pl.llm_of == [k % n_llm for k in range(40)]
    everything = sorted((k, j) for k, q in enumerate(reqs) for j in range(len(q.items)))
    assert sorted(kj for c in range(n_llm) for kj in pl.consumer_items[c]) == everything
    assert sorted(kj for p in range(len(pl.producers)) for kj in pl.producer_items(p)) == everything
    for c in range(n_llm):
        spans = sorted((pl.schedule(7, c, i)[0], pl.schedule(7, c, i)[0] + pl.chunks[k][j])
                       for i, (k, j) in enumerate(pl.consumer_items[c]))
        assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))


def test_fanout_plan_needs_an_llm_rank():
    from paper_2603_12118_b200 import fanout
    from paper_2603_12118_b200 import trace as T

    with pytest.raises(ValueError):
        fanout.plan(T.config_requests("D", 4), 1, 1024)
