"""Host-side logic of the path on CPU: request/ref id formats, batch layouts,
the placeholder layout contract and the bench helpers."""
import importlib.util
import os

import numpy as np
import pytest

from paper_2603_12118_b200 import trace as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_id_formats_follow_reference():
    # control_plane.hpp:731-733 (req-%06llu), record_replay.hpp:383-387 (/r%04zu)
    q = T.make_request(12, 100, ["image", "audio"], T.RULES["D"])
    assert q.request_id == "req-000012"
    assert [it.ref_id for it in q.items] == ["req-000012/r0000", "req-000012/r0001"]
    assert [it.rows for it in q.items] == [784, 200]


@pytest.mark.parametrize("config", ["A", "B", "D"])
def test_layout_offsets(config):
    reqs = T.config_requests(config)
    rules = T.RULES[config]
    lay = T.layout(reqs, rules.row_bytes)
    assert lay.req_row_off[0] == 0 and lay.req_item_off[0] == 0 and lay.item_row_off[0] == 0
    assert np.all(np.diff(lay.req_row_off) == [q.total_rows for q in reqs])
    assert np.all(np.diff(lay.req_item_off) == [len(q.items) for q in reqs])
    assert lay.total_item_rows == sum(q.placeholder_rows for q in reqs)
    assert lay.payload_bytes == lay.total_item_rows * rules.row_bytes
    # items are listed request by request, in input-slot order
    flat = [it.ref_id for q in reqs for it in q.items]
    assert [it.ref_id for it in lay.items] == flat


def test_config_b_sizes():
    reqs = T.config_requests("B")
    assert len(reqs) == 4
    assert all(q.input_tokens == 1800 and q.items[0].rows == 16384 for q in reqs)
    lay = T.layout(reqs, T.RULES["B"].row_bytes)
    assert lay.payload_bytes == 4 * 117_440_512


@pytest.mark.parametrize("config", ["A", "D"])
def test_prompt_layout_contract(config):
    for q in T.config_requests(config, 16):
        tok = T.prompt_tokens(q)
        assert len(tok) == q.total_rows
        ph = tok == T.PLACEHOLDER_ID
        assert int(ph.sum()) == q.placeholder_rows
        assert (tok[~ph] < T.TEXT_VOCAB).all() and (tok[~ph] >= 0).all()
        # placeholder runs appear in item order with the documented text split
        m = len(q.items)
        base, rem = divmod(q.input_tokens, m + 1)
        t = 0
        for seg in range(m + 1):
            seglen = base + (1 if seg < rem else 0)
            assert not ph[t:t + seglen].any()
            t += seglen
            if seg < m:
                assert ph[t:t + q.items[seg].rows].all()
                t += q.items[seg].rows
        assert t == len(tok)


def test_shape_rules_from_json_ignores_unknown():
    r = T.ShapeRules.from_json({"hidden_dim": 2048, "something_else": 1})
    assert r.hidden_dim == 2048 and r.row_bytes == 4096


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_bench_clock_summary_and_sample():
    b = _bench()
    cs = b.ClockSampler(0)
    cs.rows = [["0", "1965", "1965", "700", "0x0", "Not Active", "Not Active", "Not Active", "Active"],
               ["0", "1950", "1965", "710", "0x0", "Not Active", "Not Active", "Not Active", "Not Active"]]
    s = cs.summary()
    assert s["sm_max_mhz"] == 1965 and s["reasons"] == ["sw_power_cap"]
    b.CONFIG, b.REQUESTS = "B", 4
    # >= 100 MiB and a request per host thread while the batch has them
    assert len(b.cpu_sample(T)) == min(4, max(1, os.cpu_count() or 1))
    b.CONFIG, b.REQUESTS = "A", 64
    sample = b.cpu_sample(T)  # the whole 64-request batch is < 100 MiB
    assert len(sample) == 64


def test_bench_metric_is_baselines():
    """The driver compares the bench line's metric with BASELINE.json's: the
    same string (unicode arrow included), for both arms."""
    import json

    b = _bench()
    with open(os.path.join(ROOT, "BASELINE.json")) as fh:
        assert b.METRIC == json.load(fh)["metric"]
