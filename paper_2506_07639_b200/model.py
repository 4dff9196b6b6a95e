"""The 7B-shaped ECoT decoder the engine serves: shapes, framing, init.

The reference has no model (SURVEY.md finding 0.1); its requests cross the
boundary as (context, prefix, step, prev_content).  This module fixes the
builder-defined parts that both the B200 engine and the CPU oracle must agree
on bit for bit:

* `ModelConfig` presets: `tiny` (BASELINE config 1, CPU-runnable),
  `7b` (Llama-2-7B decoder + 256 vision tokens, configs 2-5) and
  `7b_2layer` (all 7B kernel shapes at 1/16 of the depth, for parity runs);
* the model-input framing:
  ``[BOS] + [VIS]*n_vision + ctx.encoded%32000 + prefix%32000 + [TAG(step)]``;
  the step tag sits *after* the prefix so every branch of a timestep shares
  the trunk's KV pages; greedy decode over the 32000 text ids, lowest index
  wins ties; the emitted length is the synthetic backend's length decision
  (`backends.length_plan`);
* counter-based weight / vision-embedding init (splitmix64 -> 24-bit uniform,
  exact in fp32), regenerated on each device so no 27 GB host copy is needed;
* the RoPE table, computed once in float64 on the host and handed to both
  implementations.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .refapi import backends as _rb
from .refapi import trace as _rt

stable_digest = _rb.stable_digest
Context, StepSpec, TokenSeq = _rt.Context, _rt.StepSpec, _rt.TokenSeq

TEXT_VOCAB = 32000
VOCAB = 32064
BOS_ID = 32000
VIS_ID = 32001
TAG_BASE = 32002
TAG_SLOTS = VOCAB - TAG_BASE
PAGE_TOKENS = 64           # KV page size == canonical attention chunk
ROPE_MAX_POS = 8192

# tensor ids of the counter-based init
T_EMBED, T_LM_HEAD, T_FINAL_NORM, T_VISION = 1, 2, 3, 4
T_LAYER_BASE, T_LAYER_STRIDE = 16, 16
(L_ATTN_NORM, L_WQ, L_WK, L_WV, L_WO, L_FFN_NORM, L_WGATE, L_WUP, L_WDOWN) = range(9)

LINEAR_MULT = np.float32(2.0 * 0.02 * np.sqrt(3.0))   # U(-a, a), std 0.02
VISION_MULT = np.float32(2.0 * np.sqrt(3.0))          # std 1
NORM_MULT = np.float32(0.2)                           # 1 + U(-0.1, 0.1)


@dataclass(frozen=True)
class ModelConfig:
    name: str
    d_model: int
    n_layers: int
    n_heads: int
    head_dim: int
    d_ffn: int
    n_vision: int
    vocab: int = VOCAB
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0

    def __post_init__(self):
        assert self.n_heads * self.head_dim == self.d_model
        assert self.d_model % 8 == 0 and self.d_ffn % 8 == 0
        assert self.head_dim in (64, 128)

    @property
    def linear_params(self) -> int:
        d, f = self.d_model, self.d_ffn
        return self.n_layers * (4 * d * d + 3 * d * f) + self.vocab * d

    def weight_bytes(self, elem: int) -> int:
        """Bytes one decode iteration streams (linear + lm_head)."""
        return self.linear_params * elem

    def kv_bytes_per_token(self, elem: int) -> int:
        return 2 * self.n_layers * self.d_model * elem


PRESETS = {
    "tiny": ModelConfig("tiny", 256, 4, 4, 64, 688, 16),
    "small": ModelConfig("small", 1024, 4, 8, 128, 2752, 64),
    "7b_2layer": ModelConfig("7b_2layer", 4096, 2, 32, 128, 11008, 256),
    "7b": ModelConfig("7b", 4096, 32, 32, 128, 11008, 256),
}


@dataclass(frozen=True)
class VisionConfig:
    """Vision tower + projector (csrc/vision.cu; oracle `or_vision_encode`):
    a pre-LayerNorm ViT over an img x img synthetic image, patch `patch`, then
    a 2-layer GELU projector into the LLM width; img / patch squared must be
    the LLM's n_vision."""
    name: str
    img: int
    patch: int
    d: int
    layers: int
    heads: int
    mlp: int
    proj_hidden: int
    eps: float = 1e-6

    @property
    def patches(self) -> int:
        return (self.img // self.patch) ** 2


VISION_PRESETS = {
    # DINOv2-L/14-shaped tower at 224 px: 256 patches (OpenVLA's VIS count)
    "vit_l14": VisionConfig("vit_l14", 224, 14, 1024, 24, 16, 4096, 4096),
    "vit_l14_2layer": VisionConfig("vit_l14_2layer", 224, 14, 1024, 2, 16, 4096, 4096),
    # small towers for the tiny / small LLMs (16 / 64 patches)
    "vit_tiny": VisionConfig("vit_tiny", 56, 14, 128, 2, 2, 256, 256),
    "vit_small": VisionConfig("vit_small", 112, 14, 256, 2, 4, 512, 512),
}
DEFAULT_VISION = {"tiny": "vit_tiny", "small": "vit_small", "7b_2layer": "vit_l14_2layer", "7b": "vit_l14"}


def get_vision(name_or_cfg, llm) -> VisionConfig:
    """The tower for an LLM config: a preset name, a VisionConfig, or True
    (the LLM's default tower)."""
    llm = get_config(llm)
    v = VISION_PRESETS[DEFAULT_VISION[llm.name]] if name_or_cfg is True else (
        name_or_cfg if isinstance(name_or_cfg, VisionConfig) else VISION_PRESETS[name_or_cfg])
    if v.patches != llm.n_vision:
        raise ValueError(f"vision tower {v.name} makes {v.patches} rows, {llm.name} frames {llm.n_vision}")
    return v


def get_config(name_or_cfg) -> ModelConfig:
    return name_or_cfg if isinstance(name_or_cfg, ModelConfig) else PRESETS[name_or_cfg]


# --- framing -----------------------------------------------------------------

def vision_seed(observation: bytes) -> int:
    return stable_digest("vision", observation)


def context_ids(ctx: Context, cfg: ModelConfig) -> list[int]:
    return [BOS_ID] + [VIS_ID] * cfg.n_vision + [int(e) % TEXT_VOCAB for e in ctx.encoded]


def text_ids(tokens: TokenSeq) -> list[int]:
    return [int(t) % TEXT_VOCAB for t in tokens]


def step_tag(step: StepSpec) -> int:
    return TAG_BASE + stable_digest("tag", step.name) % TAG_SLOTS


# --- counter-based init (numpy restatement of csrc/init.cu) -------------------

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def tensor_key(seed: int, tensor_id: int) -> int:
    s = _splitmix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))
    return int(_splitmix64(s ^ np.uint64(tensor_id))[0])


def layer_tensor(layer: int, which: int) -> int:
    return T_LAYER_BASE + T_LAYER_STRIDE * layer + which


def uniform_centered(key: int, start: int, count: int) -> np.ndarray:
    """(u24 * 2^-24 - 0.5) as float32 for element indices [start, start+count)."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _splitmix64(np.uint64(key) + idx)
    u = (h >> np.uint64(40)).astype(np.float32)
    return u * np.float32(2.0 ** -24) - np.float32(0.5)


def init_linear(seed: int, tensor_id: int, rows: int, cols: int) -> np.ndarray:
    return (uniform_centered(tensor_key(seed, tensor_id), 0, rows * cols) * LINEAR_MULT).reshape(rows, cols)


def init_norm(seed: int, tensor_id: int, n: int) -> np.ndarray:
    return np.float32(1.0) + uniform_centered(tensor_key(seed, tensor_id), 0, n) * NORM_MULT


def vision_embeddings(vseed: int, n_vision: int, d: int) -> np.ndarray:
    key = tensor_key(vseed, T_VISION)
    return (uniform_centered(key, 0, n_vision * d) * VISION_MULT).reshape(n_vision, d)


def rope_table(cfg: ModelConfig, max_pos: int = ROPE_MAX_POS) -> np.ndarray:
    """[max_pos, 2, head_dim/2] float32 (cos, sin), computed in float64."""
    half = cfg.head_dim // 2
    inv = cfg.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.ascontiguousarray(np.stack([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32))
