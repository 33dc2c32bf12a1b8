"""Test/bench helpers: move synth arrays onto the device as the C ABI expects.
(Pure data movement; no arithmetic of the method.)"""
from __future__ import annotations

import numpy as np
import torch

import synth


def dev_bf16(u16: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(u16).view(np.int16)).to(device).view(torch.bfloat16)


def dev_f32(a: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device)


def host_bf16_to_f64(t: torch.Tensor) -> np.ndarray:
    u = t.detach().cpu().view(torch.int16).numpy().view(np.uint16)
    return synth.bf16_bits_to_f64(u)


def moe_weights_dev(w: synth.MoeWeights, device="cuda"):
    from paper_2511_11505_b200 import MoeWeights
    ws = [None if a is None else dev_bf16(a, device) for a in (w.ws1, w.ws2, w.ws3)]
    return MoeWeights(dev_f32(w.gamma, device), dev_f32(w.w_router, device), dev_bf16(w.w1, device),
                      dev_bf16(w.w2, device), dev_bf16(w.w3, device), *ws)


def attn_weights_dev(a: synth.AttnWeights, device="cuda"):
    from paper_2511_11505_b200 import AttnWeights
    return AttnWeights(dev_f32(a.gamma, device), dev_bf16(a.w_qkv, device), dev_bf16(a.w_o, device), a.n_heads,
                       a.n_kv_heads, a.head_dim, a.rope_theta)


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
