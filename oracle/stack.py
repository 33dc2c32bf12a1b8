"""fp64 oracle of the L-layer stack in Regular and Hybrid (FarSkip) wiring — TEST INFRASTRUCTURE.

Regular (Eq. 6, read per C-amb-1):
    attn_in_k = o_{k-1};  mlp_in_k = o_{k-1} + attn_out_k
    o_k = ((o_{k-1} + attn_out_k) + shared_out_k) + routed_out_k
Hybrid FarSkip (boundary C-amb-6):
    attn_in_k = o_{k-2} + attn_out_{k-1} + shared_out_{k-1}   (attn_in_1 = o_0; o_{-1} := o_0 at k=2)
    mlp_in_k  = o_{k-1}                                        (outdated, Eq. 8a)
    o_k       = attn_in_{k+1} + routed_out_k, attn_in_{k+1} = (mlp_in_k + attn_out_k) + shared_out_k
In every mode o_k - o_{k-1} = attn_out_k + shared_out_k + routed_out_k.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np

from .attention import attention_block
from .moe import EpLayer, moe_block

REGULAR = 0
HYBRID = 1


@dataclasses.dataclass
class LayerCache:
    attn_in: np.ndarray
    mlp_in: np.ndarray
    attn_out: np.ndarray
    shared_out: np.ndarray
    routed_out: np.ndarray
    o: np.ndarray
    router: object = None


def stack_forward(o0: np.ndarray, attn_layers: Sequence, moe_layers: Sequence[EpLayer],
                  modes: Sequence[int], seq_len: int,
                  teacher_inputs: Optional[Sequence] = None,
                  routers: Optional[Sequence] = None) -> List[LayerCache]:
    """Run L layers; returns the per-layer ActivationCache.

    ``teacher_inputs[k] = (attn_in_k, mlp_in_k)`` (optional) overrides the
    layer inputs with the GPU's own (per-layer teacher forcing, R-4);
    ``routers[k]`` (optional) fixes layer k's selection (R-1 adoption)."""
    L = len(moe_layers)
    if len(modes) != L or len(attn_layers) != L:
        raise ValueError("modes length mismatch (S:220 config error)")
    o_prev = np.asarray(o0, np.float64)       # o_{k-1}
    o_prev2 = o_prev                          # o_{k-2}
    cache: List[LayerCache] = []
    for k in range(L):
        if modes[k] == REGULAR or k == 0:
            attn_in = o_prev
        else:
            c = cache[k - 1]
            attn_in = (o_prev2 + c.attn_out) + c.shared_out
        if teacher_inputs is not None:
            attn_in = np.asarray(teacher_inputs[k][0], np.float64)
        attn_out = attention_block(attn_in, attn_layers[k], seq_len)
        if modes[k] == REGULAR:
            mlp_in = attn_in + attn_out
        else:
            mlp_in = o_prev
        if teacher_inputs is not None:
            mlp_in = np.asarray(teacher_inputs[k][1], np.float64)
        sh, ro, r = moe_block(mlp_in, moe_layers[k],
                              None if routers is None else routers[k])
        if modes[k] == REGULAR:
            o = ((attn_in + attn_out) + sh) + ro
        else:
            o = ((mlp_in + attn_out) + sh) + ro
        cache.append(LayerCache(attn_in, mlp_in, attn_out, sh, ro, o, r))
        o_prev2, o_prev = o_prev, o
    return cache
