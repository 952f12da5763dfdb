"""Synthetic request traces and the host-side shape/layout rules of the path.

* ``ShapeRules`` mirrors fissim::ShapeRules (include/fissim/profiles.hpp:213-296):
  the row count of every forwarded embedding and its byte size.
* Request / ref ids follow the reference formats ``req-%06llu``
  (control_plane.hpp:731-733) and ``<req>/r%04zu`` (record_replay.hpp:383-387).
  In ``invoke_mllm``/``invoke_omni`` (record_replay.hpp:404-445) the encoder
  invocation of item i is recorded first, so item i's embedding is ref r{i}
  and the consumer's input slots are [request literal, item 0, ..., item m-1].
* Payload bytes are ``synth_payload(payload_seed(ref_id, seq))``
  (executor_sim.hpp:231-233, 330-331; common.hpp:247-265).
* The prompt placeholder layout is the new contract of SURVEY.md 8d (see
  DESIGN.md "Merge contract"): input_tokens text rows split into m+1 segments
  as evenly as possible (earlier segments take the remainder) around m
  placeholder runs.

Traces for configs A and D are the reference's own ``generate_workload``
output (workload.hpp:196-242, seed 42) committed under tests/golden/traces/.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRACE_DIR = os.path.join(ROOT, "tests", "golden", "traces")

GOLDEN_GAMMA = 0x9E3779B97F4A7C15
SYNTH_SALT = 0xD6E8FEB86659FD93
MASK64 = (1 << 64) - 1

# Qwen2-VL/2.5-VL "<|image_pad|>"; text ids are drawn below TEXT_VOCAB so they
# never collide with it.
PLACEHOLDER_ID = 151655
TEXT_VOCAB = 151643

MODALITIES = {"text": 0, "image": 1, "video": 2, "audio": 3}


def fnv1a64(s: str) -> int:
    """common.hpp:210-217"""
    h = 0xCBF29CE484222325
    for c in s.encode():
        h ^= c
        h = (h * 0x100000001B3) & MASK64
    return h


def payload_seed(ref_id: str, seq: int) -> int:
    """executor_sim.hpp:231-233"""
    return fnv1a64(ref_id) ^ ((GOLDEN_GAMMA * (seq + 1)) & MASK64)


def splitmix_words(seed_state: int, first: int, count: int) -> np.ndarray:
    """Outputs first+1 .. first+count of splitmix64 started at ``seed_state``
    (common.hpp:203-208): output k is mix(state + k * gamma)."""
    k = np.arange(first + 1, first + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed_state) + k * np.uint64(GOLDEN_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


@dataclass(frozen=True)
class ShapeRules:
    """fissim::ShapeRules (profiles.hpp:213-226 defaults)."""
    pixels_per_token: int = 1024
    default_image_width: int = 896
    default_image_height: int = 896
    tokens_per_frame: int = 196
    default_video_frames: int = 16
    tokens_per_audio_second: int = 25
    default_audio_seconds: float = 8.0
    hidden_dim: int = 1024
    embed_elem_bytes: int = 2
    audio_samples_per_chunk: int = 960

    @staticmethod
    def from_json(j: dict) -> "ShapeRules":
        return replace(ShapeRules(), **{k: v for k, v in j.items() if k in ShapeRules.__dataclass_fields__})

    def item_tokens(self, item: dict) -> int:
        """profiles.hpp:256-276"""
        m = item.get("modality", "image")
        if m == "image":
            w = item.get("width", self.default_image_width)
            h = item.get("height", self.default_image_height)
            return (w * h + self.pixels_per_token - 1) // self.pixels_per_token
        if m == "video":
            return item.get("frames", self.default_video_frames) * self.tokens_per_frame
        if m == "audio":
            return int(math.ceil(item.get("seconds", self.default_audio_seconds) *
                                 self.tokens_per_audio_second))
        return 0

    def embed_bytes(self, item: dict) -> int:
        """embed_desc(item).total_bytes() (profiles.hpp:278-283)"""
        return self.item_tokens(item) * self.hidden_dim * self.embed_elem_bytes

    @property
    def row_bytes(self) -> int:
        return self.hidden_dim * self.embed_elem_bytes


# Shape rules of the BASELINE.json configs.
RULES = {
    # InternVL3: 448x448 tiles, 14 px patches, 0.5 pixel shuffle -> 256 tokens, D = 4096
    "A": ShapeRules(pixels_per_token=784, default_image_width=448, default_image_height=448,
                    hidden_dim=4096),
    # Qwen2.5-VL video: 16 frames x 1024 tokens, D = 3584
    "B": ShapeRules(tokens_per_frame=1024, hidden_dim=3584),
    # Qwen2.5-Omni thinker hidden 3584 (the reference profile uses 1024)
    "C": ShapeRules(hidden_dim=3584),
    "C-ref": ShapeRules(hidden_dim=1024),
    # Fan-out mix: image 896^2/1024 = 784 rows, video 16x1024, audio 8 s x 25 = 200 rows
    "D": ShapeRules(tokens_per_frame=1024, hidden_dim=3584),
}


@dataclass
class Item:
    modality: str
    rows: int
    ref_id: str


@dataclass
class Request:
    request_id: str
    input_tokens: int
    items: List[Item] = field(default_factory=list)

    @property
    def placeholder_rows(self) -> int:
        return sum(i.rows for i in self.items)

    @property
    def total_rows(self) -> int:
        return self.input_tokens + self.placeholder_rows


def request_id(index: int) -> str:
    return f"req-{index:06d}"


def make_request(index: int, input_tokens: int, modalities: List[str], rules: ShapeRules,
                 item_overrides: Optional[List[dict]] = None) -> Request:
    rid = request_id(index)
    items = []
    for i, m in enumerate(modalities):
        spec = {"modality": m}
        if item_overrides:
            spec.update(item_overrides[i])
        items.append(Item(m, rules.item_tokens(spec), f"{rid}/r{i:04d}"))
    return Request(rid, int(input_tokens), items)


def load_trace(mix: str) -> dict:
    with open(os.path.join(TRACE_DIR, f"{mix}_seed42.json")) as fh:
        return json.load(fh)


def requests_from_trace(mix: str, rules: ShapeRules, count: int, start: int = 0) -> List[Request]:
    tr = load_trace(mix)["requests"]
    out = []
    for i in range(start, start + count):
        r = tr[i % len(tr)]
        out.append(make_request(i, r["input_tokens"], r["items"], rules))
    return out


# Composite the BASELINE configs run through (record_replay.hpp:404-420,
# task_model.hpp:259-283): an mllm with encoder fission and one encoder task
# per modality; the embedding consumer is its "llm" child.
MLLM_COMPOSITE = {"model_id": "fsx/mllm", "modalities": ["image", "video", "audio"],
                  "encoder_fission": True}
CONFIG_MIX = {"A": "mllm-chat", "D": "servegen-like"}


def request_json(config: str, index: int) -> dict:
    """The request object of request ``index`` of a config batch, as the
    reference's generate_workload emits it (workload.hpp:226-233).  Config B
    is one video per request with 1800 input tokens."""
    if config == "B":
        return {"class": "video_chat", "text": "q", "items": [{"modality": "video"}],
                "audio_output": False,
                "gen": {"input_tokens": 1800, "output_tokens": 150, "chunks": 0}}
    tr = load_trace(CONFIG_MIX[config])["requests"]
    r = tr[index % len(tr)]
    return {"class": r["class"], "text": "q", "items": [{"modality": m} for m in r["items"]],
            "audio_output": r["audio_output"],
            "gen": {"input_tokens": r["input_tokens"], "output_tokens": r["output_tokens"],
                    "chunks": r["chunks"]}}


def rules_json(rules: ShapeRules) -> dict:
    """ShapeRules::to_json (profiles.hpp:244-255)."""
    from dataclasses import asdict
    return asdict(rules)


def config_requests(config: str, count: Optional[int] = None) -> List[Request]:
    """Request batches of the BASELINE.json configs."""
    if config == "A":
        return requests_from_trace("mllm-chat", RULES["A"], count or 64)
    if config == "B":
        return [make_request(i, 1800, ["video"], RULES["B"]) for i in range(count or 4)]
    if config == "D":
        return requests_from_trace("servegen-like", RULES["D"], count or 32)
    raise ValueError(f"config {config!r} has no merge batch")


def prompt_tokens(req: Request, placeholder_id: int = PLACEHOLDER_ID,
                  text_vocab: int = TEXT_VOCAB) -> np.ndarray:
    """Token ids of the consumer prompt: text ids are splitmix64 words of
    fnv1a64(request_id + "/tok") reduced mod text_vocab, one word per row so
    ids are position-determined; placeholder rows carry placeholder_id."""
    T = req.total_rows
    words = splitmix_words(fnv1a64(req.request_id + "/tok") ^ SYNTH_SALT, 0, T)
    ids = (words % np.uint64(text_vocab)).astype(np.int32)
    m = len(req.items)
    base, rem = divmod(req.input_tokens, m + 1)
    t = 0
    for seg in range(m + 1):
        t += base + (1 if seg < rem else 0)
        if seg < m:
            ids[t:t + req.items[seg].rows] = placeholder_id
            t += req.items[seg].rows
    return ids


def text_seed(req: Request) -> int:
    """Seed of the pre-filled prompt embedding."""
    return fnv1a64(req.request_id + "/text")


@dataclass
class BatchLayout:
    """Packed offsets of a merge batch (fsx_merge_batch, include/fsx.h)."""
    requests: List[Request]
    row_bytes: int
    req_row_off: np.ndarray   # [R+1]
    req_item_off: np.ndarray  # [R+1]
    item_row_off: np.ndarray  # [M+1]
    item_rows: np.ndarray     # [M]
    items: List[Item]

    @property
    def total_rows(self) -> int:
        return int(self.req_row_off[-1])

    @property
    def total_item_rows(self) -> int:
        return int(self.item_row_off[-1])

    @property
    def payload_bytes(self) -> int:
        return self.total_item_rows * self.row_bytes


def layout(requests: List[Request], row_bytes: int) -> BatchLayout:
    R = len(requests)
    rro = np.zeros(R + 1, dtype=np.int64)
    rio = np.zeros(R + 1, dtype=np.int64)
    items: List[Item] = []
    for r, q in enumerate(requests):
        rro[r + 1] = rro[r] + q.total_rows
        rio[r + 1] = rio[r] + len(q.items)
        items.extend(q.items)
    rows = np.array([i.rows for i in items], dtype=np.int64)
    iro = np.zeros(len(items) + 1, dtype=np.int64)
    if len(items):
        iro[1:] = np.cumsum(rows)
    return BatchLayout(requests, row_bytes, rro, rio, iro, rows, items)


def summarize(requests: List[Request], rules: ShapeRules) -> Dict[str, float]:
    lay = layout(requests, rules.row_bytes)
    return {"requests": len(requests), "items": len(lay.items), "prompt_rows": lay.total_rows,
            "placeholder_rows": lay.total_item_rows, "payload_bytes": lay.payload_bytes}
