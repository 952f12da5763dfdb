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
