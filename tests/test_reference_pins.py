"""The merge's inputs and the config-D placement pinned to the reference's own
record / dispatch (tests/golden/record_dispatch.json, written by
tests/golden/make_golden.py from oracle/_ref: record() record_replay.hpp:510-528
with invoke_mllm :404-420, TaskDispatcher::dispatch task_dispatcher.hpp:178-266,
SidecarFabric delivery sidecar.hpp:302-563)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2603_12118_b200 import fanout
from paper_2603_12118_b200 import trace as T

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "record_dispatch.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("cfg", ["A", "B", "D"])
def test_layout_items_are_the_reference_consumer_slots(golden, cfg):
    """trace.layout's items of request r (ref id, rows, row bytes, order) are the
    DataRef inputs the reference records for the consumer LLM, in slot order:
    slot 0 is the request literal, slot 1 + i the embedding of item i, produced
    by the encoder task of its modality as output 0."""
    g = golden["record"][cfg]
    assert T.ShapeRules.from_json(g["rules"]) == T.RULES[cfg]
    reqs = T.config_requests(cfg, len(g["requests"]))
    lay = T.layout(reqs, T.RULES[cfg].row_bytes)
    flat = []
    for q, row in zip(reqs, g["requests"]):
        assert q.request_id == row["request_id"]
        assert q.input_tokens == row["input_tokens"]
        assert [s[0] for s in row["slots"]] == list(range(1, len(q.items) + 1))
        assert [(s[1], s[4], s[5]) for s in row["slots"]] == \
            [(it.ref_id, it.rows, T.RULES[cfg].row_bytes) for it in q.items]
        assert [s[2] for s in row["slots"]] == ["encoder." + it.modality for it in q.items]
        assert all(s[3] == 0 for s in row["slots"])
        flat.extend(s[1] for s in row["slots"])
    assert [it.ref_id for it in lay.items] == flat


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("n", [32, 128])
def test_fanout_plan_is_the_reference_dispatch(golden, world, n):
    """fanout.plan's encoder/LLM replica per node equals the reference
    TaskDispatcher's assignment for the same batch, and every encoder output
    is routed to the home GPU of its request's LLM replica (dest_gpus)."""
    g = golden["dispatch"][f"world{world}_n{n}"]
    reqs = T.config_requests("D", n)
    pl = fanout.plan(reqs, world, chunk_rows=1024)
    for k, (q, row) in enumerate(zip(reqs, g["requests"])):
        assert row["request_id"] == q.request_id
        assign = row["assign"]
        *encs, llm = assign  # record order: the item encoders, then the LLM
        assert [e[1] for e in encs] == ["encoder." + it.modality for it in q.items]
        assert [e[2] for e in encs] == pl.enc_of[k]
        assert [e[3] for e in encs] == [pl.producers[p] for p in pl.enc_of[k]]
        assert llm[1] == "llm" and llm[2] == pl.llm_of[k]
        assert llm[3] == pl.consumers[pl.llm_of[k]]
        routes = dict((inv, r) for inv, r in row["routes"])
        for e in encs:
            assert routes[e[0]] == [[0, [llm[3]]]]


@pytest.mark.parametrize("cfg", ["A", "B", "D"])
def test_oracle_merge_hashes_to_reference_derived_golden(oracle_mod, golden, cfg):
    """The CPU merge restatement over trace.layout produces exactly the prompt
    embeddings built from the reference's delivered bytes placed in the
    reference's slot order (merged_sha256, make_golden.py)."""
    O = oracle_mod
    want = golden["merged_sha256"][cfg]
    rules = T.RULES[cfg]
    rb = rules.row_bytes
    reqs = T.config_requests(cfg, want["requests"])
    lay = T.layout(reqs, rb)
    emb = np.concatenate([np.frombuffer(O.synth_payload(T.text_seed(q), q.total_rows * rb), np.uint8)
                          for q in reqs]).copy()
    tok = np.concatenate([T.prompt_tokens(q) for q in reqs])
    src = [np.frombuffer(O.synth_payload(T.payload_seed(it.ref_id, 0), it.rows * rb), np.uint8)
           for it in lay.items]
    st = O.merge(rb, T.PLACEHOLDER_ID, emb, tok, lay.req_row_off, lay.req_item_off, src,
                 lay.item_rows, nthreads=4)
    assert (st == 0).all()
    assert hashlib.sha256(emb.tobytes()).hexdigest() == want["sha256"]
