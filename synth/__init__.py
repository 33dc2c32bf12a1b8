"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module holds NO arithmetic of the method (no norm, no routing, no GEMM):
only random draws, the bf16 rounding of draws into the storage format the
GPU path consumes, and the workload shapes. Both sides — ``oracle/`` and the
CUDA path under ``paper_2511_11505_b200/`` — receive exactly the arrays built
here, so neither imports the other (task rule ③).

Input recipe (SURVEY.md §8(d) "Synthetic inputs"):
  x      ~ N(0, 1)               fp32 [T, d]       (residual stream, per rank)
  gamma  = 1 + 0.1 N(0, 1)       fp32 [d]          (RMSNorm weight)
  W_R    ~ N(0, 1/d)             fp32 [E, d]       (router, replicated)
  W1, W2 ~ N(0, 1/d)  -> bf16    [E, c, d]         (up / gate)
  W3     ~ N(0, 1/c)  -> bf16    [E, d, c]         (down)
  shared expert likewise with c_s; attention weights ~ N(0, 1/d_in) -> bf16.
Every draw is keyed by (seed, layer, tensor kind, expert or rank) through a
numpy SeedSequence, so one rank can regenerate only its own experts.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Optional

import numpy as np

# --------------------------------------------------------------------------
# bf16 storage helpers (format conversion, not method arithmetic)
# --------------------------------------------------------------------------


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (round-to-nearest-even) and return the uint16 bits."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Widen bf16 bits exactly to fp32."""
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    """Widen bf16 bits exactly to fp64 (what the oracle consumes)."""
    return bf16_bits_to_f32(b).astype(np.float64)


# --------------------------------------------------------------------------
# Workloads (BASELINE.json "configs")
# --------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class MoeShape:
    name: str
    d: int            # hidden size
    n_experts: int    # E routed experts
    top_k: int        # k
    ffn: int          # c, routed expert FFN width
    shared_ffn: int   # c_s, shared expert width (0 = none); n shared experts = concatenated width
    tokens: int       # T tokens per rank (prefill)
    n_layers: int = 1
    # attention filler shapes (SURVEY.md §8(a) assumptions, C-amb-18)
    n_heads: int = 0
    n_kv_heads: int = 0
    head_dim: int = 0
    seq_len: int = 4096


CONFIGS: Dict[str, MoeShape] = {
    # configs[0]: "tiny 2-layer MoE: hidden 64, 4 experts top-2, expert FFN 128, 32 tokens"
    "tiny": MoeShape("tiny", d=64, n_experts=4, top_k=2, ffn=128, shared_ffn=0, tokens=32,
                     n_layers=2, n_heads=4, n_kv_heads=2, head_dim=16, seq_len=16),
    # configs[1]: DeepSeek-V2-Lite: hidden 2048, 64 routed top-6 + 2 shared (2x1408), FFN 1408, 8192 tokens
    "dsv2lite": MoeShape("dsv2lite", d=2048, n_experts=64, top_k=6, ffn=1408, shared_ffn=2816,
                         tokens=8192, n_heads=16, n_kv_heads=16, head_dim=128),
    # configs[2]: Qwen3-30B-A3B: hidden 2048, 128 experts top-8, FFN 768, 48 layers, 16384 tokens
    "qwen3": MoeShape("qwen3", d=2048, n_experts=128, top_k=8, ffn=768, shared_ffn=0,
                      tokens=16384, n_layers=48, n_heads=32, n_kv_heads=4, head_dim=128),
    # configs[3]: Llama-4-Scout: hidden 5120, 16 experts top-1 + shared, FFN 8192, 8192 tokens
    "scout": MoeShape("scout", d=5120, n_experts=16, top_k=1, ffn=8192, shared_ffn=8192,
                      tokens=8192, n_heads=40, n_kv_heads=8, head_dim=128),
}


def decode_shape(base: str, tokens: int) -> MoeShape:
    """configs[4]: decode regime, Qwen3/Scout shapes at 64-512 tokens/step."""
    s = CONFIGS[base]
    return dataclasses.replace(s, name=f"{base}_decode{tokens}", tokens=tokens)


# --------------------------------------------------------------------------
# Seeded draws
# --------------------------------------------------------------------------

_KIND = {"x": 1, "gamma": 2, "w_router": 3, "w1": 4, "w2": 5, "w3": 6,
         "ws1": 7, "ws2": 8, "ws3": 9, "attn_gamma": 10, "w_qkv": 11, "w_o": 12,
         "skew_mean": 13}


def _rng(seed: int, layer: int, kind: str, sub: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, layer, _KIND[kind], sub])))


def _normal(seed, layer, kind, sub, shape, std) -> np.ndarray:
    g = _rng(seed, layer, kind, sub)
    return (g.standard_normal(shape, dtype=np.float32) * np.float32(std)).astype(np.float32)


SKEW_DEFAULT = 0.15   # the skewed-load variant's max/mean expert load ~1.5-2x


def tokens(shape: MoeShape, seed: int = 0, rank: int = 0, T: Optional[int] = None,
           layer: int = 0, skew: float = 0.0) -> np.ndarray:
    """x ~ N(0,1) fp32 [T, d] for one rank.

    skew > 0 is the skewed-load variant (reading C-amb-21):
    every token gets the same mean vector m ~ N(0, skew^2) (one draw per (seed, layer),
    shared by all ranks), x = z + m. The router stays the paper's pure linear map
    G(A) = s(A W_R^T); the shift adds to expert e's logit the offset
    r (m . gamma W_R[e]), ~N(0, skew^2) relative to the token part, so the same
    experts are hot on every rank. Measured max/mean expert load (4096 tokens):
    skew 0.15 (SKEW_DEFAULT) 1.9x DS-V2-Lite, 1.9x Qwen3, 1.65x Scout; skew 0.5:
    5-6x (stress)."""
    T = shape.tokens if T is None else T
    x = _normal(seed, layer, "x", rank, (T, shape.d), 1.0)
    if skew:
        x = (x + _normal(seed, layer, "skew_mean", 0, (shape.d,), skew)).astype(np.float32)
    return x


@dataclasses.dataclass
class MoeWeights:
    """One MoE layer's weights for experts [e0, e0+E_loc) (bf16 as uint16 bits)."""
    gamma: np.ndarray      # fp32 [d]
    w_router: np.ndarray   # fp32 [E, d]
    w1: np.ndarray         # u16 [E_loc, c, d]   up      (PAPER.md:73-76 W1)
    w2: np.ndarray         # u16 [E_loc, c, d]   gate    (W2, g = SiLU on this branch)
    w3: np.ndarray         # u16 [E_loc, d, c]   down    (W3)
    ws1: Optional[np.ndarray]  # u16 [c_s, d] or None
    ws2: Optional[np.ndarray]
    ws3: Optional[np.ndarray]  # u16 [d, c_s]
    e0: int = 0


def moe_weights(shape: MoeShape, seed: int = 0, layer: int = 0, e0: int = 0,
                e_loc: Optional[int] = None, zero_experts: bool = False) -> MoeWeights:
    d, E, c, cs = shape.d, shape.n_experts, shape.ffn, shape.shared_ffn
    e_loc = E if e_loc is None else e_loc
    gamma = (1.0 + 0.1 * _normal(seed, layer, "gamma", 0, (d,), 1.0)).astype(np.float32)
    w_router = _normal(seed, layer, "w_router", 0, (E, d), 1.0 / np.sqrt(d))
    w1 = np.empty((e_loc, c, d), np.uint16)
    w2 = np.empty((e_loc, c, d), np.uint16)
    w3 = np.empty((e_loc, d, c), np.uint16)
    for i in range(e_loc):
        e = e0 + i
        w1[i] = f32_to_bf16_bits(_normal(seed, layer, "w1", e, (c, d), 1.0 / np.sqrt(d)))
        w2[i] = f32_to_bf16_bits(_normal(seed, layer, "w2", e, (c, d), 1.0 / np.sqrt(d)))
        w3[i] = f32_to_bf16_bits(_normal(seed, layer, "w3", e, (d, c), 1.0 / np.sqrt(c)))
    if zero_experts:
        w1[:] = 0
        w2[:] = 0
        w3[:] = 0
    ws1 = ws2 = ws3 = None
    if cs > 0:
        ws1 = f32_to_bf16_bits(_normal(seed, layer, "ws1", 0, (cs, d), 1.0 / np.sqrt(d)))
        ws2 = f32_to_bf16_bits(_normal(seed, layer, "ws2", 0, (cs, d), 1.0 / np.sqrt(d)))
        ws3 = f32_to_bf16_bits(_normal(seed, layer, "ws3", 0, (d, cs), 1.0 / np.sqrt(cs)))
    return MoeWeights(gamma, w_router, w1, w2, w3, ws1, ws2, ws3, e0)


@dataclasses.dataclass
class AttnWeights:
    gamma: np.ndarray   # fp32 [d]
    w_qkv: np.ndarray   # u16 [(Hq + 2 Hkv) * hd, d]  rows: q heads, then k heads, then v heads
    w_o: np.ndarray     # u16 [d, Hq * hd]
    n_heads: int
    n_kv_heads: int
    head_dim: int
    rope_theta: float = 10000.0


def attn_weights(shape: MoeShape, seed: int = 0, layer: int = 0, zero_o: bool = False) -> AttnWeights:
    d, hq, hkv, hd = shape.d, shape.n_heads, shape.n_kv_heads, shape.head_dim
    gamma = (1.0 + 0.1 * _normal(seed, layer, "attn_gamma", 0, (d,), 1.0)).astype(np.float32)
    w_qkv = f32_to_bf16_bits(_normal(seed, layer, "w_qkv", 0, ((hq + 2 * hkv) * hd, d), 1.0 / np.sqrt(d)))
    w_o = f32_to_bf16_bits(_normal(seed, layer, "w_o", 0, (d, hq * hd), 1.0 / np.sqrt(hq * hd)))
    if zero_o:
        w_o[:] = 0
    return AttnWeights(gamma, w_qkv, w_o, hq, hkv, hd)
