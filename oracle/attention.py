"""fp64 oracle of the attention sub-block used as the stack's overlap filler — TEST INFRASTRUCTURE.

The paper splits attention into (a) q,k,v preparation and (b) core attention +
output projection (§4.1) and uses MLA for DeepSeek; MLA is out of
scope, so the filler is standard causal multi-head attention with grouped KV
heads and rotary position embedding (C-amb-18):

  h      = rmsnorm(x, gamma)                          ("layer-norm")
  q,k,v  = h W_qkv^T split into Hq, Hkv, Hkv heads of width hd
  q,k    <- RoPE(q,k; pos = t mod seq_len, theta)     (rotate-half pairs (i, i+hd/2))
  o_h    = softmax(q_h k_g^T / sqrt(hd) + causal mask within the packed sequence) v_g,
           g = h // (Hq / Hkv)
  out    = concat_h(o_h) W_o^T
Parity of this filler against the paper is unpinned beyond the textbook
special cases in tests/test_oracle_stack.py (T=1, zero weights, causality,
sequence packing, RoPE invariants).
"""
from __future__ import annotations

import numpy as np

from .moe import rmsnorm


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """Rotary embedding on the last axis (rotate-half convention); x [T, H, hd]."""
    hd = x.shape[-1]
    half = hd // 2
    inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / hd)
    ang = pos[:, None].astype(np.float64) * inv[None, :]          # [T, half]
    c = np.cos(ang)[:, None, :]
    s = np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def attention_qkv(x, gamma, w_qkv, n_heads, n_kv_heads, head_dim, seq_len, theta=10000.0):
    """Part (a) of P:198: norm + q,k,v projections + RoPE."""
    T = x.shape[0]
    h = rmsnorm(x, gamma)
    qkv = h @ np.asarray(w_qkv, np.float64).T
    q = qkv[:, : n_heads * head_dim].reshape(T, n_heads, head_dim)
    k = qkv[:, n_heads * head_dim:(n_heads + n_kv_heads) * head_dim].reshape(T, n_kv_heads, head_dim)
    v = qkv[:, (n_heads + n_kv_heads) * head_dim:].reshape(T, n_kv_heads, head_dim)
    pos = np.arange(T) % seq_len
    return rope(q, pos, theta), rope(k, pos, theta), v


def attention_core(q, k, v, w_o, seq_len):
    """Part (b) of P:198: causal attention within each packed sequence + W_o."""
    T, Hq, hd = q.shape
    Hkv = k.shape[1]
    grp = Hq // Hkv
    o = np.zeros((T, Hq, hd), np.float64)
    for s0 in range(0, T, seq_len):
        s1 = min(T, s0 + seq_len)
        n = s1 - s0
        mask = np.tril(np.ones((n, n), bool))
        for h in range(Hq):
            g = h // grp
            sc = q[s0:s1, h] @ k[s0:s1, g].T / np.sqrt(hd)
            sc = np.where(mask, sc, -np.inf)
            sc = sc - sc.max(axis=1, keepdims=True)
            p = np.exp(sc)
            p = p / p.sum(axis=1, keepdims=True)
            o[s0:s1, h] = p @ v[s0:s1, g]
    return o.reshape(T, Hq * hd) @ np.asarray(w_o, np.float64).T


def attention_block(x, aw, seq_len: int):
    """attn-out = Attn(rmsnorm(x)) for an fp64-widened AttnWeights-like object."""
    q, k, v = attention_qkv(x, aw.gamma, aw.w_qkv, aw.n_heads, aw.n_kv_heads, aw.head_dim,
                            seq_len, aw.rope_theta)
    return attention_core(q, k, v, aw.w_o, seq_len)
