"""fp64 oracle of the expert-parallel MoE block forward — TEST INFRASTRUCTURE ONLY.

Cites PAPER.md (P:<line>) and, for interface details the paper leaves open,
SPEC.md (S:<line>) through the readings C-amb-n listed in DESIGN.md.
Nothing here is blocked, fused or reordered beyond the definitions.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

RMS_EPS = 1e-6  # C-amb-5: RMSNorm, eps 1e-6


# ---------------------------------------------------------------------------
# Elementwise / row primitives
# ---------------------------------------------------------------------------

def rmsnorm(x: np.ndarray, gamma: np.ndarray, eps: float = RMS_EPS) -> np.ndarray:
    """Pre-norm 'layer-norm' of P:103, read as RMSNorm (C-amb-5):
    y = x / sqrt(mean(x^2) + eps) * gamma, in fp64."""
    x = np.asarray(x, np.float64)
    r = np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x / r * np.asarray(gamma, np.float64)


def softmax_rows(l: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction; the router's s() (C-amb-2)."""
    l = np.asarray(l, np.float64)
    z = np.exp(l - l.max(axis=-1, keepdims=True))
    return z / z.sum(axis=-1, keepdims=True)


def silu(z: np.ndarray) -> np.ndarray:
    """g = SiLU(z) = z / (1 + e^-z) (C-amb-4)."""
    z = np.asarray(z, np.float64)
    return z / (1.0 + np.exp(-z))


def swiglu(a: np.ndarray, w1: np.ndarray, w2: np.ndarray, w3: np.ndarray) -> np.ndarray:
    """Gated MLP of P:73-76: MLP(A) = sigma(A W1^T . g(A W2^T)) W3^T with
    sigma = identity and g = SiLU on the W2 branch (C-amb-4).
    Shapes: a [B,d], w1,w2 [c,d], w3 [d,c] -> [B,d]."""
    a = np.asarray(a, np.float64)
    u = a @ np.asarray(w1, np.float64).T
    g = silu(a @ np.asarray(w2, np.float64).T)
    return (u * g) @ np.asarray(w3, np.float64).T


# ---------------------------------------------------------------------------
# Router G(A) = s(A W_R^T)
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class RouterOutput:
    idx: np.ndarray      # int32 [T,k], ascending expert id per token (C-amb-3 slot order)
    gates: np.ndarray    # fp64 [T,k], renormalised over the selected set (sum 1)
    logits: np.ndarray   # fp64 [T,E] = xn W_R^T
    probs: np.ndarray    # fp64 [T,E] = softmax(logits)
    gap: np.ndarray      # fp64 [T]  l_(k) - l_(k+1) in descending logit order; +inf if k == E


def route(xn: np.ndarray, w_router: np.ndarray, top_k: int) -> RouterOutput:
    """Router of P:96 with s() read as softmax over E, top-k, renormalise (C-amb-2).

    1. l = xn W_R^T (fp64; W_R fp32 widened exactly);
    2. p = softmax(l);
    3. S_t = the k largest p, exact ties to the lower expert index (C-amb-3);
    4. g = p_S / sum(p_S);
    5. slots ordered by ascending expert id (C-amb-3).
    Also reports the boundary gap used by the near-tie rule R-1.
    """
    E = w_router.shape[0]
    if not 1 <= top_k <= E:
        raise ValueError(f"top_k={top_k} outside [1, E={E}]")
    l = np.asarray(xn, np.float64) @ np.asarray(w_router, np.float64).T
    p = softmax_rows(l)
    T = l.shape[0]
    order = np.argsort(-p, axis=1, kind="stable")          # descending p, ties -> lower index
    sel = np.sort(order[:, :top_k], axis=1)                # slot order = ascending expert id
    ps = np.take_along_axis(p, sel, axis=1)
    gates = ps / ps.sum(axis=1, keepdims=True)
    ls = -np.sort(-l, axis=1)
    gap = np.full(T, np.inf) if top_k == E else ls[:, top_k - 1] - ls[:, top_k]
    return RouterOutput(sel.astype(np.int32), gates, l, p, gap)


# ---------------------------------------------------------------------------
# Permutation maps ("grouped and mapped ... requiring permutation of A"; R_i of P:98-100)
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class PermMaps:
    counts: np.ndarray   # int64 [E]   #{(t,j): idx[t,j] == e}
    offsets: np.ndarray  # int64 [E+1] exclusive prefix of counts
    pos: np.ndarray      # int64 [T,k] destination row of copy (t,j) in the expert-sorted buffer
    src_row: np.ndarray  # int64 [T*k] token whose copy sits in row p


def permutation_maps(idx: np.ndarray, n_experts: int) -> PermMaps:
    """Stable counting sort of the (token, slot) copies by expert (C-amb-11):
    counts[e]; offsets = exclusive scan; within an expert, copies keep ascending
    token order, so pos[t,j] = offsets[e] + #{t' < t : e in S_t'}."""
    idx = np.asarray(idx)
    T, k = idx.shape
    flat = idx.reshape(-1)
    counts = np.zeros(n_experts, np.int64)
    for e in flat:
        counts[e] += 1
    offsets = np.zeros(n_experts + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    pos = np.empty(T * k, np.int64)
    src_row = np.empty(T * k, np.int64)
    for e in range(n_experts):
        members = np.nonzero(flat == e)[0]           # ascending (t, j) flat order -> ascending t
        rows = offsets[e] + np.arange(members.size)
        pos[members] = rows
        src_row[rows] = members // k
    return PermMaps(counts, offsets, pos.reshape(T, k), src_row)


# ---------------------------------------------------------------------------
# Expert parallel dispatch / combine simulation
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class EpLayer:
    """Full (unsharded) MoE layer parameters as fp64 (bf16 widened exactly)."""
    gamma: np.ndarray
    w_router: np.ndarray
    w1: np.ndarray   # [E, c, d]
    w2: np.ndarray   # [E, c, d]
    w3: np.ndarray   # [E, d, c]
    ws1: Optional[np.ndarray] = None   # [c_s, d]
    ws2: Optional[np.ndarray] = None
    ws3: Optional[np.ndarray] = None   # [d, c_s]
    top_k: int = 1

    @property
    def n_experts(self) -> int:
        return self.w1.shape[0]


def expert_owner(e: int, n_experts: int, n_ranks: int) -> int:
    """Contiguous placement: rank p owns experts [p E/P, (p+1) E/P) (C-amb-9)."""
    return e // (n_experts // n_ranks)


def dispatch_sim(xn_per_rank: Sequence[np.ndarray], idx_per_rank: Sequence[np.ndarray],
                 n_experts: int, n_ranks: int):
    """Dispatch of P:97-100: A_i = R_i x A placed on rank i.

    Receive layout on rank p (C-amb-11): expert-major over p's local experts,
    then source rank, then ascending token. Returns per destination rank the
    receive buffer [R_p, d], the per-local-expert row counts, and for every
    source rank s the map (dst rank, dst row) of each copy (t, j)."""
    if n_experts % n_ranks:
        raise ValueError("E not divisible by n_ranks (C-amb-9 config error)")
    e_loc = n_experts // n_ranks
    P = n_ranks
    # counts matrix cnt[s, e]: how many copies source s sends to expert e
    cnt = np.zeros((P, n_experts), np.int64)
    for s in range(P):
        for e in np.asarray(idx_per_rank[s]).reshape(-1):
            cnt[s, e] += 1
    recv_bufs, recv_counts = [], []
    dst_row = [np.empty(np.asarray(i).shape, np.int64) for i in idx_per_rank]
    dst_rank = [np.empty(np.asarray(i).shape, np.int64) for i in idx_per_rank]
    for p in range(P):
        rows = []
        local_counts = np.zeros(e_loc, np.int64)
        r = 0
        for el in range(e_loc):
            e = p * e_loc + el
            for s in range(P):
                idx = np.asarray(idx_per_rank[s])
                T, k = idx.shape
                for t in range(T):
                    for j in range(k):
                        if idx[t, j] == e:
                            rows.append(np.asarray(xn_per_rank[s][t], np.float64))
                            dst_row[s][t, j] = r
                            dst_rank[s][t, j] = p
                            r += 1
                            local_counts[el] += 1
        d = np.asarray(xn_per_rank[0]).shape[1]
        recv_bufs.append(np.array(rows, np.float64).reshape(-1, d))
        recv_counts.append(local_counts)
    return recv_bufs, recv_counts, dst_rank, dst_row, cnt


def experts_on_rank(recv: np.ndarray, local_counts: np.ndarray, layer: EpLayer, p: int,
                    n_ranks: int) -> np.ndarray:
    """Routed expert computation on rank p: each local expert's contiguous row
    segment through its SwiGLU (P:198 step 6)."""
    e_loc = layer.n_experts // n_ranks
    y = np.zeros_like(recv)
    r = 0
    for el in range(e_loc):
        e = p * e_loc + el
        m = int(local_counts[el])
        if m:
            y[r:r + m] = swiglu(recv[r:r + m], layer.w1[e], layer.w2[e], layer.w3[e])
        r += m
    return y


def combine_sim(y_per_rank: Sequence[np.ndarray], gates: np.ndarray, dst_rank: np.ndarray,
                dst_row: np.ndarray) -> np.ndarray:
    """Combine of P:100: the dual all-to-all brings each copy back to its source
    token, which sums the gate-weighted expert outputs in slot order:
    routed[t] = sum_j g[t,j] * y_{p(t,j)}[row(t,j)] (C-amb-12: sum starts at 0)."""
    T, k = gates.shape
    d = y_per_rank[0].shape[1] if len(y_per_rank[0]) else None
    if d is None:
        d = next(y.shape[1] for y in y_per_rank if y.ndim == 2)
    out = np.zeros((T, d), np.float64)
    for t in range(T):
        acc = np.zeros(d, np.float64)
        for j in range(k):
            acc = acc + gates[t, j] * y_per_rank[dst_rank[t, j]][dst_row[t, j]]
        out[t] = acc
    return out


# ----------------------------------------------------------------------------
# FP8 dispatch payload (the paper's inference runs FP8)
# ----------------------------------------------------------------------------
E4M3_MAX = 448.0
FP8_BLOCK = 128


def e4m3_rne(v: np.ndarray) -> np.ndarray:
    """Round to the nearest OCP FP8 E4M3 value, ties to even, saturating to +-448
    (cvt.rn.satfinite.e4m3). Normals 2^-6 .. 1.75 * 2^8 with 3 mantissa bits;
    subnormals k * 2^-9, k = 1..7."""
    v = np.asarray(v, np.float64)
    a = np.abs(v)
    with np.errstate(divide="ignore"):
        e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    e = np.maximum(e, -6.0)                                   # below 2^-6: the subnormal quantum 2^-9
    quantum = np.exp2(e - 3.0)
    q = np.rint(a / quantum) * quantum                        # rint = round half to even
    q = np.minimum(q, E4M3_MAX)
    return np.sign(v) * q


def f32(x):
    return np.asarray(x, np.float32)


def bf16_rne(x) -> np.ndarray:
    """Round float32 values to bfloat16, nearest-even (the kernels' cvt.rn.bf16.f32),
    returned as float64. Finite inputs only."""
    u = f32(x).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def fp8_dispatch_payload(xn_bf16: np.ndarray) -> np.ndarray:
    """The FP8 dispatch payload as the receiving rank's GEMM sees it: per row and per
    128-column block b, s_b = fp32(amax_b / 448) (1 if amax_b = 0), q = e4m3(fp32(x / s_b)),
    x_hat = bf16(fp32(q * s_b)). Input: the bf16 rows (as float values)."""
    x = f32(xn_bf16)
    T, d = x.shape
    if d % FP8_BLOCK:
        raise ValueError("d must be a multiple of 128 for the FP8 payload")
    xb = x.reshape(T, d // FP8_BLOCK, FP8_BLOCK)
    amax = np.abs(xb).max(axis=2, keepdims=True)
    s = np.where(amax > 0, f32(amax) / f32(E4M3_MAX), f32(1.0)).astype(np.float32)
    q = e4m3_rne((xb / s).astype(np.float32))
    xh = (f32(q) * s).astype(np.float32)
    return bf16_rne(xh.reshape(T, d))


def moe_block_ep_fp8(x_per_rank: Sequence[np.ndarray], layer: EpLayer, n_ranks: int):
    """moe_block_ep with the FP8 dispatch payload: the rows sent to the experts are
    fp8_dispatch_payload(bf16(xn)) instead of xn; the shared expert (local) and the
    combine are unchanged. Returns [(shared_out_s, routed_out_s, RouterOutput_s)]."""
    xns = [rmsnorm(x, layer.gamma) for x in x_per_rank]
    routers = [route(xn, layer.w_router, layer.top_k) for xn in xns]
    payload = [fp8_dispatch_payload(bf16_rne(xn)) for xn in xns]
    recv, rc, dst_rank, dst_row, _ = dispatch_sim(payload, [r.idx for r in routers], layer.n_experts, n_ranks)
    ys = [experts_on_rank(recv[p], rc[p], layer, p, n_ranks) for p in range(n_ranks)]
    return [(shared_expert(xns[s], layer), combine_sim(ys, routers[s].gates, dst_rank[s], dst_row[s]), routers[s])
            for s in range(n_ranks)]


def shared_expert(xn: np.ndarray, layer: EpLayer) -> np.ndarray:
    """Shared experts 'process all tokens' on the same xn (C-amb-7);
    n shared experts == one SwiGLU of concatenated width. Width 0 -> exact zeros."""
    if layer.ws1 is None:
        return np.zeros(np.asarray(xn).shape, np.float64)
    return swiglu(xn, layer.ws1, layer.ws2, layer.ws3)


def moe_block_ep(x_per_rank: Sequence[np.ndarray], layer: EpLayer, n_ranks: int,
                 routers: Optional[Sequence[RouterOutput]] = None):
    """MoE block forward with EP over n_ranks simulated ranks.

    Per rank s: xn = rmsnorm(x_s); router; dispatch; experts; combine.
    Returns [(shared_out_s, routed_out_s, RouterOutput_s)] for every rank s,
    shared and routed SEPARATELY. ``routers[s]`` (optional) fixes rank
    s's selection (the near-tie adoption rule R-1)."""
    if len(x_per_rank) != n_ranks:
        raise ValueError("one token block per rank")
    xns = [rmsnorm(x, layer.gamma) for x in x_per_rank]
    if routers is None:
        routers = [route(xn, layer.w_router, layer.top_k) for xn in xns]
    recv, rc, dst_rank, dst_row, _ = dispatch_sim(xns, [r.idx for r in routers],
                                                   layer.n_experts, n_ranks)
    ys = [experts_on_rank(recv[p], rc[p], layer, p, n_ranks) for p in range(n_ranks)]
    out = []
    for s in range(n_ranks):
        routed = combine_sim(ys, routers[s].gates, dst_rank[s], dst_row[s])
        out.append((shared_expert(xns[s], layer), routed, routers[s]))
    return out


def moe_block_allreduce(x: np.ndarray, layer: EpLayer, n_ranks: int):
    """Inference variant of the EP MoE block (vLLM): the activations x
    are replicated on every rank, rank p evaluates only its contiguous expert
    block E_p (C-amb-9) and the partial outputs are summed by an all-reduce.

    Per rank p: partial_p[t] = sum over slots j with e_j in E_p of g_tj MLP^{e_j}(xn_t);
    result = sum_p partial_p (rank order). Returns (shared_out, routed_out, router,
    [partial_p]); the shared expert is evaluated replicated (no collective)."""
    if layer.n_experts % n_ranks:
        raise ValueError(f"n_experts={layer.n_experts} not divisible by n_ranks={n_ranks} (S:178)")
    xn = rmsnorm(x, layer.gamma)
    r = route(xn, layer.w_router, layer.top_k)
    e_loc = layer.n_experts // n_ranks
    partials = []
    for p in range(n_ranks):
        part = np.zeros_like(xn)
        for j in range(layer.top_k):
            for t in range(x.shape[0]):
                e = int(r.idx[t, j])
                if p * e_loc <= e < (p + 1) * e_loc:
                    part[t] += r.gates[t, j] * swiglu(xn[t:t + 1], layer.w1[e], layer.w2[e], layer.w3[e])[0]
        partials.append(part)
    routed = np.zeros_like(xn)
    for part in partials:
        routed = routed + part
    return shared_expert(xn, layer), routed, r, partials


def moe_block(x: np.ndarray, layer: EpLayer, router: Optional[RouterOutput] = None):
    """Single-rank MoE block (EP=1) -> (shared_out, routed_out, RouterOutput).

    The gate-weighted routed sum is MoE(A) = sum_j G(A)_j MLP^j(A) over
    the selected set, evaluated through the expert-sorted permutation
    and the combine sum in slot order. If ``router`` is given its selection is
    used (the near-tie adoption rule R-1 of SURVEY §8(c) O-3)."""
    xn = rmsnorm(x, layer.gamma)
    r = route(xn, layer.w_router, layer.top_k) if router is None else router
    maps = permutation_maps(r.idx, layer.n_experts)
    xs = xn[maps.src_row]
    y = np.zeros_like(xs)
    for e in range(layer.n_experts):
        a, b = maps.offsets[e], maps.offsets[e + 1]
        if b > a:
            y[a:b] = swiglu(xs[a:b], layer.w1[e], layer.w2[e], layer.w3[e])
    T, k = r.idx.shape
    routed = np.zeros_like(xn)
    for j in range(k):
        routed = routed + r.gates[:, j:j + 1] * y[maps.pos[:, j]]
    return shared_expert(xn, layer), routed, r


def moe_block_dense(x: np.ndarray, layer: EpLayer):
    """Brute force (BASELINE.json north star): every token through every
    expert, masked by its top-k gates; no permutation, no dispatch."""
    xn = rmsnorm(x, layer.gamma)
    r = route(xn, layer.w_router, layer.top_k)
    T, E = r.logits.shape
    mask = np.zeros((T, E), np.float64)
    for j in range(r.idx.shape[1]):
        mask[np.arange(T), r.idx[:, j]] = r.gates[:, j]
    routed = np.zeros_like(xn)
    for e in range(E):
        routed += mask[:, e:e + 1] * swiglu(xn, layer.w1[e], layer.w2[e], layer.w3[e])
    return shared_expert(xn, layer), routed, r


def adopt_router(layer: EpLayer, x: np.ndarray, gpu_idx: np.ndarray, margin: float = 1e-6):
    """Near-tie rule R-1: tokens whose oracle boundary gap is
    below ``margin`` take the GPU's selected set (gates recomputed in fp64 from
    the oracle's own probabilities). Returns (RouterOutput, excluded_mask)."""
    xn = rmsnorm(x, layer.gamma)
    r = route(xn, layer.w_router, layer.top_k)
    excl = r.gap < margin
    if excl.any():
        idx = r.idx.copy()
        idx[excl] = np.sort(np.asarray(gpu_idx)[excl], axis=1)
        ps = np.take_along_axis(r.probs, idx.astype(np.int64), axis=1)
        gates = ps / ps.sum(axis=1, keepdims=True)
        r = RouterOutput(idx, gates, r.logits, r.probs, r.gap)
    return r, excl


def layer_from_synth(w, top_k: int) -> EpLayer:
    """Widen a synth.MoeWeights (bf16 bits) to fp64 exactly."""
    def wid(b):
        return None if b is None else (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return EpLayer(np.asarray(w.gamma, np.float64), np.asarray(w.w_router, np.float64),
                   wid(w.w1), wid(w.w2), wid(w.w3), wid(w.ws1), wid(w.ws2), wid(w.ws3), top_k)
