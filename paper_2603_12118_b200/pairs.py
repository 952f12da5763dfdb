"""Producer->consumer pairing across processes (one process per GPU).

The path shards by pair: rank 2k is an encoder (producer) and
rank 2k+1 the LLM (consumer) whose receive slab it writes over NVLink; pairs
never talk to each other, so there is no collective on the data path.  The
only cross-process steps are setup (slab IPC handles and segment offsets,
exchanged once through torch.distributed objects) and the per-step
flag/token schedule, which both ranks derive locally from the step number so
no message is needed per transfer.  The consumer acknowledges each step by
storing a token into the producer's ack flag (fsx_signal_flags) -- the
cross-process form of the reference's ack_raw (sidecar.hpp:287-290).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

FLAG_WINDOW = 64  # steps whose flag ranges may be in flight before reuse


@dataclass(frozen=True)
class PairRole:
    rank: int
    world: int
    pair: int
    producer: bool
    peer: int          # -1 when this rank has no partner (odd world, last rank)
    producer_gpu: int  # logical gpu ids used inside the fabric of both ranks
    consumer_gpu: int

    @property
    def alone(self) -> bool:
        return self.peer < 0


def role(rank: int, world: int) -> PairRole:
    pair = rank // 2
    producer = rank % 2 == 0
    peer = rank + 1 if producer else rank - 1
    if peer >= world:
        peer = -1
    return PairRole(rank, world, pair, producer, peer, 2 * pair, 2 * pair + 1)


def pairs_in(world: int) -> int:
    return (world + 1) // 2


def schedule(step: int, chunks_per_item: Sequence[int], window: int = FLAG_WINDOW
             ) -> List[Tuple[int, int]]:
    """(flag_base, token) per item for `step`.  Flag ranges cycle through
    `window` step slots of the consumer's flag ring; tokens are unique per
    (step, item) and never 0 (0 = empty flag)."""
    per_step = sum(chunks_per_item)
    base = (step % window) * per_step
    out, at = [], 0
    for i, n in enumerate(chunks_per_item):
        out.append((base + at, ((step + 1) << 20) | (i + 1)))
        at += n
    return out


def ack_token(step: int) -> int:
    return ((step + 1) << 20) | 0xFFFFF


def exchange(obj):
    """all_gather_object over the default process group (setup only)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
