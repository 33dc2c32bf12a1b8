"""fp64 oracle of the MoE block BACKWARD pass — TEST INFRASTRUCTURE ONLY.

SURVEY §8(f) NEXT-2 (the backward of the FarSkip MoE layer, P:207-211 and the
Tab. 3 backward column). Written ahead of any kernel, as the oracle the
future dgrad / wgrad grouped GEMMs and gradient all-to-all will be checked against.

Forward being differentiated (oracle/moe.py, EP=1 semantics; readings C-amb-2,4,5,7):
    r_t   = (mean_i x_ti^2 + eps)^-1/2,  xn_t = gamma (.) x_t r_t           (RMSNorm)
    l_t   = xn_t W_R^T,  S_t = top-k(l_t),  g_tj = softmax_{j in S_t}(l_tj)  (router)
    u = xn W1_e^T, v = xn W2_e^T, h = u (.) SiLU(v), y_e = h W3_e^T       (expert e)
    routed_t = sum_{j in S_t} g_tj y_{e_j}(xn_t),  shared_t = SwiGLU_s(xn_t)
    out_t = x_t + shared_t + routed_t
Given G = dL/dout, returns dL/dx, dL/dgamma, dL/dW_R and the expert / shared weight
gradients. The selection S_t is piecewise constant in the inputs, so the unselected
logits get no gradient (the derivative exists away from top-k boundary ties).
Every step is the chain rule written out per token and slot; no blocking or fusion.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from .moe import RMS_EPS, EpLayer, route, silu


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def silu_grad(z: np.ndarray) -> np.ndarray:
    """d SiLU / dz = s(z) (1 + z (1 - s(z))), s = logistic."""
    s = _sigmoid(z)
    return s * (1.0 + z * (1.0 - s))


def swiglu_backward(a: np.ndarray, w1, w2, w3, dy: np.ndarray):
    """Backward of y = (a W1^T (.) SiLU(a W2^T)) W3^T for a row block a [B,d]:
    returns (da [B,d], dW1 [c,d], dW2 [c,d], dW3 [d,c])."""
    u = a @ w1.T
    v = a @ w2.T
    sv = silu(v)
    h = u * sv
    dW3 = dy.T @ h                      # [d,c]
    dh = dy @ w3                        # [B,c]
    du = dh * sv
    dv = dh * u * silu_grad(v)
    dW1 = du.T @ a
    dW2 = dv.T @ a
    da = du @ w1 + dv @ w2
    return da, dW1, dW2, dW3


@dataclasses.dataclass
class MoeGrads:
    dx: np.ndarray
    dgamma: np.ndarray
    dw_router: np.ndarray
    dw1: np.ndarray
    dw2: np.ndarray
    dw3: np.ndarray
    dws1: Optional[np.ndarray]
    dws2: Optional[np.ndarray]
    dws3: Optional[np.ndarray]


def moe_block_backward(x: np.ndarray, layer: EpLayer, G: np.ndarray, eps: float = RMS_EPS) -> MoeGrads:
    """Gradients of out = x + shared(xn) + routed(xn) (see the module docstring)."""
    x = np.asarray(x, np.float64)
    G = np.asarray(G, np.float64)
    T, d = x.shape
    gamma = np.asarray(layer.gamma, np.float64)
    r = 1.0 / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + eps)     # [T,1]
    xn = x * r * gamma
    rt = route(xn, layer.w_router, layer.top_k)
    E, k = layer.n_experts, layer.top_k
    dxn = np.zeros_like(xn)
    dw1 = np.zeros_like(np.asarray(layer.w1, np.float64))
    dw2 = np.zeros_like(dw1)
    dw3 = np.zeros_like(np.asarray(layer.w3, np.float64))
    dwr = np.zeros((E, d))
    for t in range(T):
        dg = np.zeros(k)
        for j in range(k):
            e = int(rt.idx[t, j])
            w1, w2, w3 = (np.asarray(layer.w1[e], np.float64), np.asarray(layer.w2[e], np.float64),
                          np.asarray(layer.w3[e], np.float64))
            a = xn[t:t + 1]
            y = (a @ w1.T * silu(a @ w2.T)) @ w3.T                 # expert output [1,d]
            dg[j] = float(G[t] @ y[0])                             # routed = sum_j g_j y_j
            da, g1, g2, g3 = swiglu_backward(a, w1, w2, w3, rt.gates[t, j] * G[t:t + 1])
            dxn[t] += da[0]
            dw1[e] += g1
            dw2[e] += g2
            dw3[e] += g3
        # gates = softmax over the selected logits: dl_j = g_j (dg_j - sum_i g_i dg_i)
        gt = rt.gates[t]
        dl = gt * (dg - float(gt @ dg))
        for j in range(k):
            e = int(rt.idx[t, j])
            dwr[e] += dl[j] * xn[t]
            dxn[t] += dl[j] * np.asarray(layer.w_router[e], np.float64)
    dws1 = dws2 = dws3 = None
    if layer.ws1 is not None:
        da, dws1, dws2, dws3 = swiglu_backward(xn, np.asarray(layer.ws1, np.float64),
                                               np.asarray(layer.ws2, np.float64),
                                               np.asarray(layer.ws3, np.float64), G)
        dxn += da
    # RMSNorm: xn = gamma (.) x r,  r = (mean x^2 + eps)^-1/2
    dgamma = np.sum(dxn * x * r, axis=0)
    q = dxn * gamma                                            # dL/d(x r)
    dx_norm = r * q - x * r ** 3 * np.sum(q * x, axis=1, keepdims=True) / d
    return MoeGrads(G + dx_norm, dgamma, dwr, dw1, dw2, dw3, dws1, dws2, dws3)
