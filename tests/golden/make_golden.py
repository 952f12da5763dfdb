"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Every value here is computed by the reference's own code, compiled unmodified
from /root/reference/proj/include into oracle/_ref/libref_oracle.so
(oracle/ref_oracle.cpp).  Run in the build container (the reference is not on
the GPU box):

    python tests/golden/make_golden.py

Outputs (committed):
  kat.json                 known-answer vectors: checksum64, synth_payload,
                           fnv1a64, splitmix64, payload_seed, ShapeRules
                           item_tokens/embed_desc, NodeArena op trace, and
                           SidecarFabric delivered-byte digests
  traces/*.json            generate_workload(mix, rate, duration, seed=42)
                           request traces (sizes only) for configs A and D
  record_dispatch.json     the merge's inputs and the config-D placement:
                           record() (record_replay.hpp:510-528) of every
                           request of configs A/B/D -> the consumer's input
                           DataRefs in slot order; TaskDispatcher::dispatch
                           (task_dispatcher.hpp:178-266) of config-D batches
                           at 2/4/8 GPUs -> replica assignments and dest_gpus;
                           SHA-256 of the merged prompt embeddings built from
                           the bytes the reference SidecarFabric delivered,
                           placed in that slot order

    python tests/golden/make_golden.py [--only record]
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

REF = O.REF
MIXES = "/root/reference/proj/mixes"


def synth(seed, n):
    return O.synth_payload(seed, n, REF)


def _consumer_refs(rec: dict) -> list:
    node = next(n for n in rec["graph"]["nodes"] if n["invocation_id"] == rec["consumer"])
    return [(pos, s["ref"]) for pos, s in enumerate(node["inputs"]) if s["kind"] == "ref"]


def _ref_deliver(ref_id: str, n: int) -> bytes:
    """The bytes the reference SidecarFabric hands the consumer's ChunkCallback
    for this ref's payload (encoder gpu 0 -> LLM gpu 1, LocalBuffer)."""
    p = synth(O.payload_seed(ref_id, 0, REF), n)
    out = (C.c_uint8 * max(n, 1))()
    stats = (C.c_int64 * 7)()
    rc = REF.ref_forward(0, 1, ref_id.encode(), p, n, out, stats)
    assert rc == 0 and stats[6] == 1, (ref_id, rc, REF.ref_last_error())
    return bytes(out)[:n]


def record_dispatch() -> None:
    import numpy as np

    sys.path.insert(0, ROOT)
    from paper_2603_12118_b200 import trace as T

    doc: dict = {"source": "reference record()/TaskDispatcher/SidecarFabric compiled unmodified "
                           "(oracle/_ref, ref_record / ref_dispatch / ref_forward)",
                 "composite": {"kind": "mllm", "config": T.MLLM_COMPOSITE}}
    # --- record(): consumer input slots (record_replay.hpp:404-420) -------
    counts = {"A": 128, "B": 4, "D": 128}
    rec_out = {}
    for cfg, n in counts.items():
        rules = T.RULES[cfg]
        rows = []
        for k in range(n):
            rid = T.request_id(k)
            rq = T.request_json(cfg, k)
            rec = O.ref_record("mllm", T.MLLM_COMPOSITE, rq, T.rules_json(rules), rid)
            slots = []
            for pos, ref in _consumer_refs(rec):
                shape, eb = ref["desc"]["shape"], ref["desc"]["elem_bytes"]
                slots.append([pos, ref["ref_id"], rec["children"][ref["producer"]],
                              ref["output_index"], shape[0], shape[1] * eb])
            rows.append({"request_id": rid, "consumer": rec["consumer"],
                         "input_tokens": rq["gen"]["input_tokens"], "slots": slots})
        rec_out[cfg] = {"rules": T.rules_json(rules), "requests": rows}
    doc["record"] = rec_out
    # --- TaskDispatcher::dispatch: config-D placement at 2/4/8 GPUs --------
    disp = {}
    for world in (2, 4, 8):
        enc, llm = list(range(0, world, 2)), list(range(1, world, 2))
        gpus = {"encoder.image": enc, "encoder.video": enc, "encoder.audio": enc, "llm": llm}
        for n in (32, 128):
            reqs = [(T.request_id(k), T.request_json("D", k)) for k in range(n)]
            res = O.ref_dispatch("mllm", T.MLLM_COMPOSITE, reqs, T.rules_json(T.RULES["D"]), gpus)
            rows = []
            for r in res:
                inv = sorted(r["assign"])  # map order == record order
                rows.append({"request_id": r["request_id"],
                             "assign": [[i] + r["assign"][i] for i in inv],
                             "routes": [[i, r["routes"][i]] for i in inv]})
            disp[f"world{world}_n{n}"] = {"replica_gpus": gpus, "requests": rows}
    doc["dispatch"] = disp
    # --- merged prompt embeddings from the reference's delivered bytes ------
    merged = {}
    for cfg, n in (("A", 64), ("B", 4), ("D", 32)):
        rules = T.RULES[cfg]
        rb = rules.row_bytes
        h = hashlib.sha256()
        for row in rec_out[cfg]["requests"][:n]:
            slots = row["slots"]
            assert all(s[5] == rb for s in slots)
            req = T.Request(row["request_id"], row["input_tokens"],
                            [T.Item("?", s[4], s[1]) for s in slots])
            tok = T.prompt_tokens(req)  # the prompt layout contract
            emb = np.frombuffer(synth(T.text_seed(req), req.total_rows * rb), np.uint8).copy()
            emb = emb.reshape(-1, rb) if req.total_rows else emb.reshape(0, rb)
            pos = np.flatnonzero(tok == T.PLACEHOLDER_ID)
            if slots:
                got = [np.frombuffer(_ref_deliver(s[1], s[4] * rb), np.uint8) for s in slots]
                emb[pos] = np.concatenate(got).reshape(-1, rb)
            h.update(emb.tobytes())
        merged[cfg] = {"requests": n, "row_bytes": rb, "sha256": h.hexdigest()}
    doc["merged_sha256"] = merged
    with open(os.path.join(HERE, "record_dispatch.json"), "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    print("record/dispatch fixtures written")


def main() -> None:
    if REF is None:
        raise SystemExit("oracle/_ref/libref_oracle.so missing: build it with `make -C oracle ref`")
    kat: dict = {"source": "reference fissim headers compiled unmodified (oracle/_ref)"}

    # --- common.hpp primitives -------------------------------------------
    kat["fnv1a64"] = {s: f"{O.fnv1a64(s, REF):016x}" for s in
                      ["", "a", "req/r0", "req-000000/r0000", "req-000000/r0001",
                       "req-000123/r0042", "acc4/r7"]}
    st = C.c_uint64(0x1234)
    kat["splitmix64_from_0x1234"] = [f"{REF.ref_splitmix64(C.byref(st)):016x}" for _ in range(8)]
    synth_cases = []
    rng = random.Random(7)
    for n in [0, 1, 3, 7, 8, 9, 15, 16, 17, 31, 33, 255, 256, 4096, 4099, 65536 + 5]:
        seed = rng.getrandbits(64)
        p = synth(seed, n)
        synth_cases.append({"seed": f"{seed:016x}", "n": n, "sha256": hashlib.sha256(p).hexdigest(),
                            "head": p[:24].hex(), "checksum64": f"{O.checksum64(p, REF):016x}"})
    kat["synth_payload"] = synth_cases
    seeds = []
    for ref_id in ["req-000000/r0000", "req-000000/r0001", "req-000000/r0002", "req-000007/r0003",
                   "soak/r5"]:
        for seq in [0, 1, 5, 127]:
            seeds.append({"ref_id": ref_id, "seq": seq,
                          "seed": f"{O.payload_seed(ref_id, seq, REF):016x}"})
    kat["payload_seed"] = seeds
    # SURVEY.md Appendix A cases (recomputed by the reference here)
    appendix = []
    for name, ref_id, seq, n in [
        ("A image 256x4096 bf16", "req-000000/r0000", 0, 256 * 4096 * 2),
        ("B video 16x1024x3584 bf16", "req-000000/r0000", 0, 16 * 1024 * 3584 * 2),
        ("C hidden 1x3584 bf16", "req-000000/r0001", 0, 3584 * 2),
        ("C hidden 1x1024 bf16", "req-000000/r0001", 5, 1024 * 2),
        ("C talker code", "req-000000/r0002", 0, 4),
        ("MLLM image 784x1024 bf16", "req-000000/r0000", 0, 784 * 1024 * 2),
    ]:
        seed = O.payload_seed(ref_id, seq, REF)
        p = synth(seed, n)
        appendix.append({"case": name, "ref_id": ref_id, "seq": seq, "n": n, "seed": f"{seed:016x}",
                         "checksum64": f"{O.checksum64(p, REF):016x}", "head": p[:8].hex(),
                         "sha256": hashlib.sha256(p).hexdigest()})
    kat["appendix_a"] = appendix
    kat["checksum64_empty"] = f"{O.checksum64(b'', REF):016x}"

    # --- ShapeRules (profiles.hpp:256-283) -------------------------------
    rules = {
        "default": {},
        "qwen25-omni": {"pixels_per_token": 1024, "hidden_dim": 1024, "embed_elem_bytes": 2},
        "qwen3-omni": {"pixels_per_token": 1024, "hidden_dim": 2048, "embed_elem_bytes": 2},
        "configA-internvl3": {"pixels_per_token": 784, "hidden_dim": 4096, "embed_elem_bytes": 2},
        "configB-qwen25vl": {"tokens_per_frame": 1024, "hidden_dim": 3584, "embed_elem_bytes": 2},
        "configD-servegen": {"tokens_per_frame": 1024, "hidden_dim": 3584, "embed_elem_bytes": 2},
    }
    items = [{"modality": "image"}, {"modality": "image", "width": 448, "height": 448},
             {"modality": "image", "width": 1920, "height": 1080}, {"modality": "video"},
             {"modality": "video", "frames": 8}, {"modality": "audio"},
             {"modality": "audio", "seconds": 3.3}, {"modality": "text"}]
    shape = []
    for rname, rj in rules.items():
        for it in items:
            rs, js = json.dumps(rj).encode(), json.dumps(it).encode()
            shape.append({"rules": rname, "item": it, "tokens": REF.ref_item_tokens(rs, js),
                          "embed_bytes": REF.ref_embed_bytes(rs, js)})
    kat["shape_rules"] = {"rules": rules, "cases": shape}

    # --- NodeArena op trace (sidecar.hpp:106-205) ------------------------
    cap = 1 << 20
    a = REF.ref_arena_new(cap)
    rng = random.Random(11)
    ops, live = [], []
    for _ in range(600):
        if live and rng.random() < 0.45:
            off = live.pop(rng.randrange(len(live)))
            rc = REF.ref_arena_free(a, off)
            ops.append(["free", off, rc, REF.ref_arena_segments_in_use(a),
                        REF.ref_arena_bytes_in_use(a)])
        else:
            n = rng.choice([0, 1, 63, 64, 65, 1000, 4096, 70000, 200000])
            off = REF.ref_arena_alloc(a, n)
            if off >= 0:
                live.append(off)
            ops.append(["alloc", n, off, REF.ref_arena_segments_in_use(a),
                        REF.ref_arena_bytes_in_use(a)])
    if live:
        ops.append(["free", live[0], REF.ref_arena_free(a, live[0]), REF.ref_arena_segments_in_use(a),
                    REF.ref_arena_bytes_in_use(a)])
        ops.append(["free", live[0], REF.ref_arena_free(a, live[0]), REF.ref_arena_segments_in_use(a),
                    REF.ref_arena_bytes_in_use(a)])  # double free -> -2
    REF.ref_arena_delete(a)
    kat["arena_trace"] = {"capacity": cap, "ops": ops}

    # --- SidecarFabric forwarding: delivered bytes (sidecar.hpp:302-563) --
    fwd = []
    for n in [0, 1, 7, 256, 4096, 65536, 1 << 20, 8 << 20]:
        for dst in (2, 6):  # tests/test_sidecar.cpp:60-87: 0->2 local, 0->6 network
            ref_id = f"req-x/r{n}-{dst}"
            seed = O.fnv1a64(ref_id, REF)
            p = synth(seed, n)
            out = (C.c_uint8 * max(n, 1))()
            stats = (C.c_int64 * 7)()
            rc = REF.ref_forward(0, dst, ref_id.encode(), p, n, out, stats)
            fwd.append({"ref_id": ref_id, "n": n, "dst": dst, "rc": rc,
                        "payload_sha256": hashlib.sha256(p).hexdigest(),
                        "delivered_sha256": hashlib.sha256(bytes(out)[:n]).hexdigest(),
                        "stats": list(stats)})
    kat["forward"] = fwd

    with open(os.path.join(HERE, "kat.json"), "w") as fh:
        json.dump(kat, fh, indent=1)

    # --- request traces (workload.hpp:196-242, seed 42) ------------------
    os.makedirs(os.path.join(HERE, "traces"), exist_ok=True)
    for mix, rate, dur in [("mllm-chat", 20.0, 20.0), ("servegen-like", 20.0, 20.0)]:
        s = REF.ref_generate_workload(f"{MIXES}/{mix}.json".encode(), rate, dur, 42)
        reqs = json.loads(s)
        slim = [{"arrival_ms": round(r["arrival_ms"], 3), "class": r["class"],
                 "items": [it["modality"] for it in r["request"]["items"]],
                 "input_tokens": r["request"]["gen"]["input_tokens"],
                 "output_tokens": r["request"]["gen"]["output_tokens"],
                 "chunks": r["request"]["gen"]["chunks"],
                 "audio_output": r["request"]["audio_output"]} for r in reqs]
        with open(os.path.join(HERE, "traces", f"{mix}_seed42.json"), "w") as fh:
            json.dump({"mix": mix, "rate_per_s": rate, "duration_s": dur, "seed": 42,
                       "generator": "fissim::generate_workload (workload.hpp:196-242)",
                       "requests": slim}, fh)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "record":
        record_dispatch()
    else:
        main()
        record_dispatch()
