"""Config D fan-out placement across one box (BASELINE.json configs[3],
SURVEY.md 8d-D / 8e): encoder replicas on the even ranks, LLM replicas on the
odd ranks, one process per GPU; every encoder GPU hosts one replica of each
modality's encoder task ("encoder.image", "encoder.video", "encoder.audio").
The mllm composite records one encoder invocation per item, in ``items``
order, then the LLM invocation (record_replay.hpp:404-416).  Every request of
a step is dispatched the way the reference's TaskDispatcher does it
(task_dispatcher.hpp:178-221): nodes are assigned in record order, each by
``select_replica`` of its task -- least outstanding invocations, round-robin
tie-break (task_dispatcher.hpp:142-173) -- and the chosen replica's
outstanding count is bumped before the next selection (:209).  All requests
of a step are dispatched before any completes, so within a step the counts
only grow.

The result is a many-to-many pattern: encoder e sends each item to the LLM
replica its request was assigned to, so every LLM receives from several
encoders (fan-in) and every encoder feeds several LLMs (fan-out).  There is
still no collective: each (encoder, LLM) edge is a one-sided K1 push into the
LLM's slab plus per-chunk flags, and every LLM acks each encoder that fed it.

Everything here is pure host logic, computed identically on every rank from
the same trace, so no per-step messages exist; tests/test_pairs_gloo.py covers
it on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

from .pairs import FLAG_WINDOW


class ReplicaSelector:
    """select_replica (task_dispatcher.hpp:142-173) without locality
    preference: among the replicas with the fewest outstanding invocations,
    the first at or after the round-robin cursor; the cursor moves past it."""

    def __init__(self, n: int):
        self.outstanding = [0] * n
        self.rr = 0

    def select(self) -> int:
        n = len(self.outstanding)
        best = min(self.outstanding)
        for probe in range(n):
            ep = (self.rr + probe) % n
            if self.outstanding[ep] == best:
                self.rr = (self.rr + probe + 1) % n
                self.outstanding[ep] += 1  # dispatch bumps it (task_dispatcher.hpp:209)
                return ep
        raise AssertionError("unreachable")


@dataclass
class Plan:
    producers: List[int]            # ranks of the encoder replicas
    consumers: List[int]            # ranks of the LLM replicas
    enc_of: List[List[int]]         # per request, per item: encoder ordinal
    llm_of: List[int]               # per request: LLM ordinal
    chunks: List[List[int]]         # per request, per item: number of flagged chunks
    # per consumer ordinal: [(request, item)] in the consumer's merge order
    consumer_items: List[List[Tuple[int, int]]] = field(default_factory=list)
    # per consumer ordinal: chunk prefix of each of its items, and the total
    consumer_chunk_prefix: List[List[int]] = field(default_factory=list)
    consumer_chunks: List[int] = field(default_factory=list)

    def consumer_requests(self, c: int) -> List[int]:
        return [k for k, l in enumerate(self.llm_of) if l == c]

    def producer_items(self, p: int) -> List[Tuple[int, int]]:
        """(request, item) pairs encoder p produces, in dispatch order."""
        return [(k, j) for k, es in enumerate(self.enc_of) for j, e in enumerate(es) if e == p]

    def item_slot(self, k: int, j: int) -> Tuple[int, int]:
        """(consumer ordinal, index of item (k, j) in that consumer's list)."""
        c = self.llm_of[k]
        return c, self._index[c][(k, j)]

    def consumers_of(self, p: int) -> List[int]:
        return sorted({self.llm_of[k] for k, _ in self.producer_items(p)})

    def producers_of(self, c: int) -> List[int]:
        return sorted({self.enc_of[k][j] for k, j in self.consumer_items[c]})

    def schedule(self, step: int, c: int, idx: int, window: int = FLAG_WINDOW) -> Tuple[int, int]:
        """(flag_base, token) of consumer c's item idx at `step`: flag ranges
        cycle through `window` step slots of c's flag ring; tokens are unique
        per (step, item) and never 0 (0 = empty flag)."""
        base = (step % window) * self.consumer_chunks[c] + self.consumer_chunk_prefix[c][idx]
        return base, ((step + 1) << 20) | (idx + 1)


def plan(requests: Sequence, world: int, chunk_rows: int) -> Plan:
    producers = list(range(0, world, 2))
    consumers = list(range(1, world, 2))
    if not consumers:
        raise ValueError("fan-out needs at least one LLM rank (world >= 2)")
    enc: Dict[str, ReplicaSelector] = {}  # one replica set per encoder task (modality)
    llm = ReplicaSelector(len(consumers))
    enc_of, llm_of, chunks = [], [], []
    for q in requests:
        es = []
        for it in q.items:  # record order: the item encoders, then the LLM
            sel = enc.setdefault(it.modality, ReplicaSelector(len(producers)))
            es.append(sel.select())
        enc_of.append(es)
        llm_of.append(llm.select())
        chunks.append([max(1, -(-it.rows // chunk_rows)) for it in q.items])
    pl = Plan(producers, consumers, enc_of, llm_of, chunks)
    pl._index: Dict[int, Dict[Tuple[int, int], int]] = {}
    for c in range(len(consumers)):
        items = [(k, j) for k in pl.consumer_requests(c) for j in range(len(chunks[k]))]
        pre, at = [], 0
        for k, j in items:
            pre.append(at)
            at += chunks[k][j]
        pl.consumer_items.append(items)
        pl.consumer_chunk_prefix.append(pre)
        pl.consumer_chunks.append(max(at, 1))
        pl._index[c] = {kj: i for i, kj in enumerate(items)}
    return pl
