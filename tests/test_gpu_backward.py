"""Backward of the MoE sub-block on the GPU:
the dgrad / SwiGLU-backward / wgrad tcgen05 GEMMs against fp64 definitions on the same
bf16 operands, and fsc_moe_backward (recompute + gradient all-to-all + router / RMSNorm
backward) against the fp64 oracle oracle/moe_backward.py (itself pinned by finite
differences of the forward oracle) at EP = 1 and EP = 2 / 4."""
import dataclasses
import os

import numpy as np
import pytest
import torch

import synth
from oracle import moe as om
from oracle import moe_backward as ob
from tests.gpu_util import dev_bf16, dev_f32, host_bf16_to_f64, moe_weights_dev, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-2   # BJ tolerance (bf16 GEMM operands, fp32 accumulation)


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_11505_b200 import Context, build
    build.build()
    c = Context(d=2048, n_experts=8, top_k=2, ffn=1408, shared_ffn=0, max_tokens=4096)
    yield c
    c.close()


def rb(rng, shape, scale=1.0):
    return synth.f32_to_bf16_bits((rng.standard_normal(shape) * scale).astype(np.float32))


F = synth.bf16_bits_to_f64


# ----------------------------------------------------------------------------- dgrad (MN-major B)
DGRAD = [([1], 64, 64, 0), ([0, 130, 257], 128, 128, 0), ([300, 0, 5], 1408, 2048, 0), ([384], 2048, 1408, 0),
         ([200, 77], 2048, 2 * 1408, 1408 // 64), ([517, 1, 129, 0], 256, 2 * 768, 768 // 64), ([70, 71], 192, 64, 0)]


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("epi", [0, 2])
@pytest.mark.parametrize("counts,N,K,split", DGRAD)
def test_gemm_dgrad_mn_major_b(ctx, counts, N, K, split, epi, cg):
    """out_g = A_g B_g with B_g read [K, N] row-major (MN-major operand: dh = dY W3,
    dX = [dU | dV] [W1 ; W2] with the K range split across two tensors)."""
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(N + K + split)
    G, M = len(counts), sum(counts)
    k0 = split * 64 if split else K
    A = rb(rng, (max(M, 1), K))
    B0 = rb(rng, (G * k0, N), 1 / np.sqrt(K))                   # group g: rows [g k0, (g+1) k0)
    B1 = rb(rng, (G * k0, N), 1 / np.sqrt(K)) if split else None
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    dt = torch.bfloat16 if epi == 0 else torch.float32
    out = torch.zeros(max(M, 1), N, dtype=dt, device="cuda")
    ctx.op_gemm_dgrad(epi, dev_bf16(A), dev_bf16(B0), None if B1 is None else dev_bf16(B1), k0, G, cnt, 0, N, K,
                      split, out)
    torch.cuda.synchronize()
    got = host_bf16_to_f64(out) if epi == 0 else out.cpu().numpy().astype(np.float64)
    r = 0
    for g, m in enumerate(counts):
        if m:
            Bg = F(B0[g * k0:(g + 1) * k0])
            if split:
                Bg = np.concatenate([Bg, F(B1[g * k0:(g + 1) * k0])])
            ref = F(A[r:r + m]) @ Bg
            assert rel_l2(got[r:r + m], ref) < (4e-3 if epi == 0 else 1e-5), (g, rel_l2(got[r:r + m], ref))
        r += m
    ctx.set_gemm_cta_group(0)


# ----------------------------------------------------------------------------- SwiGLU backward epilogue
@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("counts,N,K", [([1], 128, 64), ([0, 130, 257], 128, 128), ([333, 900, 17], 1408, 2048),
                                        ([600, 0, 257], 768, 2048)])
def test_gemm_swiglu_backward(ctx, counts, N, K, cg):
    """Recomputed u = a W1^T, v = a W2^T; h = u SiLU(v); du = g dh SiLU(v);
    dv = g dh u SiLU'(v); g h; and sum_cols h dh (the gate gradient), per row."""
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(3 + N + K)
    G, M = len(counts), sum(counts)
    A = rb(rng, (M, K))
    W1, W2 = rb(rng, (G * N, K), 1 / np.sqrt(K)), rb(rng, (G * N, K), 1 / np.sqrt(K))
    dh = rb(rng, (M, N))
    gate = rng.uniform(0.05, 1.0, M).astype(np.float32)
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    duv = torch.zeros(M, 2 * N, dtype=torch.bfloat16, device="cuda")
    hg = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    dg_ld = 2 * (N // 64) + 2
    dgp = torch.zeros(M, dg_ld, dtype=torch.float32, device="cuda")
    ctx.op_gemm_swiglu_bwd(dev_bf16(A), dev_bf16(W1), dev_bf16(W2), G, cnt, 0, N, K, dev_bf16(dh), dev_f32(gate),
                           duv, hg, dgp, dg_ld)
    torch.cuda.synchronize()
    g_duv, g_hg, g_dg = host_bf16_to_f64(duv), host_bf16_to_f64(hg), dgp.cpu().numpy().astype(np.float64).sum(1)
    r = 0
    for g, m in enumerate(counts):
        if m:
            a = F(A[r:r + m])
            u, v = a @ F(W1[g * N:(g + 1) * N]).T, a @ F(W2[g * N:(g + 1) * N]).T
            sv, dsv = om.silu(v), ob.silu_grad(v)
            gg = gate[r:r + m, None].astype(np.float64)
            d = F(dh[r:r + m])
            assert rel_l2(g_duv[r:r + m, :N], gg * d * sv) < 5e-3
            assert rel_l2(g_duv[r:r + m, N:], gg * d * u * dsv) < 5e-3
            assert rel_l2(g_hg[r:r + m], gg * u * sv) < 5e-3
            assert rel_l2(g_dg[r:r + m], (u * sv * d).sum(1)) < 5e-3
        r += m
    ctx.set_gemm_cta_group(0)


# ----------------------------------------------------------------------------- wgrad
WGRAD = [([1], 128, 64, 0, 0), ([64, 65, 0, 63], 128, 128, 0, 0), ([200, 0, 1, 511], 1408, 2048, 0, 0),
         ([300, 77], 2048, 1408, 0, 0), ([130, 257], 128, 256, 128, 0), ([97], 64, 64, 0, 64),
         ([1000, 33], 768, 2048, 768, 0)]


@pytest.mark.parametrize("counts,N1,N2,a0,b0", WGRAD)
@pytest.mark.parametrize("acc", [False, True])
def test_gemm_wgrad(ctx, counts, N1, N2, a0, b0, acc):
    """out_g = A_g^T B_g over each group's (ragged) rows, both operands read MN-major
    from their row-major token layouts; empty groups give zeros; column offsets select
    dU / dV from [dU | dV]."""
    rng = np.random.default_rng(N1 + N2 + a0 + len(counts))
    G, M = len(counts), sum(counts)
    lda, ldb = a0 + N1 + (64 if a0 else 0), b0 + N2
    A = rb(rng, (M, lda))
    B = rb(rng, (M, ldb))
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    init = rng.standard_normal((G, N1, N2)).astype(np.float32)
    out = torch.from_numpy(init.copy()).cuda() if acc else torch.full((G, N1, N2), np.nan, device="cuda")
    ctx.op_gemm_wgrad(cnt, G, 0, N1, N2, dev_bf16(A), lda, a0, dev_bf16(B), ldb, b0, out, acc)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    r = 0
    for g, m in enumerate(counts):
        ref = F(A[r:r + m, a0:a0 + N1]).T @ F(B[r:r + m, b0:b0 + N2]) if m else np.zeros((N1, N2))
        if acc:
            ref = ref + init[g]
        if m or acc:
            assert rel_l2(got[g], ref) < 1e-5, (g, rel_l2(got[g], ref))
        else:
            assert np.all(got[g] == 0)
        r += m


# ----------------------------------------------------------------------------- fsc_moe_backward, EP = 1
SHAPES = {
    "tiny": synth.CONFIGS["tiny"],
    "ep_small": synth.MoeShape("ep_small", d=256, n_experts=8, top_k=2, ffn=128, shared_ffn=128, tokens=96),
    "ds_small": dataclasses.replace(synth.CONFIGS["dsv2lite"], d=512, n_experts=16, top_k=4, ffn=256, shared_ffn=512,
                                    tokens=256),
    "qwen_small": dataclasses.replace(synth.CONFIGS["qwen3"], d=512, n_experts=32, top_k=8, ffn=192, tokens=200),
}
GRAD_KEYS = ("dx", "dgamma", "dw_router", "dw1", "dw2", "dw3", "dws1", "dws2", "dws3")


def grad_out(shape, T, seed, rank=0):
    g = np.random.default_rng([seed, rank, 77])
    return g.standard_normal((T, shape.d)).astype(np.float32)


def run_backward(ctx, shape, w, x, G, e_loc):
    d, c, cs = shape.d, shape.ffn, shape.shared_ffn
    T = x.shape[0]
    z = lambda *sh: torch.full(sh, float("nan"), dtype=torch.float32, device="cuda")  # noqa: E731
    grads = {"dx": z(T, d), "dgamma": z(d), "dw_router": z(shape.n_experts, d), "dw1": z(e_loc, c, d),
             "dw2": z(e_loc, c, d), "dw3": z(e_loc, d, c)}
    if cs:
        grads.update({"dws1": z(cs, d), "dws2": z(cs, d), "dws3": z(d, cs)})
    ctx.moe_backward(moe_weights_dev(w), dev_f32(x), dev_f32(G), grads)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in grads.items()}


def check_grads(got, ref, shape, e_sl=slice(None)):
    pairs = [("dx", ref.dx), ("dgamma", ref.dgamma), ("dw_router", ref.dw_router), ("dw1", ref.dw1[e_sl]),
             ("dw2", ref.dw2[e_sl]), ("dw3", ref.dw3[e_sl])]
    if shape.shared_ffn:
        pairs += [("dws1", ref.dws1), ("dws2", ref.dws2), ("dws3", ref.dws3)]
    errs = {}
    for k, rv in pairs:
        errs[k] = rel_l2(got[k], rv)
        assert np.all(np.isfinite(got[k])), k
        assert errs[k] < TOL, (k, errs[k])
    return errs


@pytest.mark.parametrize("name", list(SHAPES))
def test_moe_backward_matches_oracle(name):
    from paper_2511_11505_b200 import Context, build
    build.build()
    shape = SHAPES[name]
    T = shape.tokens
    w = synth.moe_weights(shape, seed=3)
    x = synth.tokens(shape, seed=3, T=T)
    G = grad_out(shape, T, 3)
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T)
    got = run_backward(ctx, shape, w, x, G, shape.n_experts)
    got2 = run_backward(ctx, shape, w, x, G, shape.n_experts)       # repeatable (workspace reuse)
    os.environ["FSC_PERMUTE_GATHER"] = "0"                          # recompute permute by source token
    try:
        got3 = run_backward(ctx, shape, w, x, G, shape.n_experts)
    finally:
        del os.environ["FSC_PERMUTE_GATHER"]
    ctx.close()
    for k in got:
        np.testing.assert_array_equal(got[k], got2[k])
        np.testing.assert_array_equal(got[k], got3[k])
    ref = ob.moe_block_backward(x, om.layer_from_synth(w, shape.top_k), G)
    errs = check_grads(got, ref, shape)
    print(name, {k: f"{v:.1e}" for k, v in errs.items()})


# ----------------------------------------------------------------------------- EP > 1
def _bwd_worker(rank, world, port, shape, seed, outdir):
    from tests.test_gpu_ep import _init_pg
    dist = _init_pg(rank, world, port)
    from paper_2511_11505_b200 import Context
    e_loc = shape.n_experts // world
    w = synth.moe_weights(shape, seed=seed, e0=rank * e_loc, e_loc=e_loc)
    x = synth.tokens(shape, seed=seed, rank=rank)
    G = grad_out(shape, x.shape[0], seed, rank)
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=x.shape[0], rank=rank, ep_size=world, device=0)
    ctx.connect()
    got = run_backward(ctx, shape, w, x, G, e_loc)
    # a forward between two backward calls (epochs, shared buffers) changes nothing
    out = torch.empty(x.shape, dtype=torch.float32, device="cuda")
    ctx.moe_forward_blocking(moe_weights_dev(w), dev_f32(x), out)
    got2 = run_backward(ctx, shape, w, x, G, e_loc)
    for k in got:
        np.testing.assert_array_equal(got[k], got2[k])
    np.savez(os.path.join(outdir, f"{rank}.npz"), **got)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_moe_backward_ep_matches_oracle(world):
    """Gradient all-to-all (dispatch of G rows, combine of dX rows and gate gradients) over
    the peer-memory transport: per rank dx / dgamma / dW_R / shared grads against the
    oracle on that rank's tokens, and each rank's expert gradients against the sum of the
    oracle's over every rank's tokens."""
    from paper_2511_11505_b200 import build
    from tests.test_gpu_ep import _spawn
    build.build()
    shape = SHAPES["ds_small"]
    res = _spawn(_bwd_worker, world, shape, 4)
    lay = om.layer_from_synth(synth.moe_weights(shape, seed=4), shape.top_k)
    refs = [ob.moe_block_backward(synth.tokens(shape, seed=4, rank=r), lay, grad_out(shape, shape.tokens, 4, r))
            for r in range(world)]
    tot = {k: sum(getattr(rf, k) for rf in refs) for k in ("dw1", "dw2", "dw3")}
    e_loc = shape.n_experts // world
    for r in range(world):
        g = res[r]
        for k in ("dx", "dgamma", "dw_router", "dws1", "dws2", "dws3"):
            assert rel_l2(g[k], getattr(refs[r], k)) < TOL, (r, k)
        for k in ("dw1", "dw2", "dw3"):
            assert rel_l2(g[k], tot[k][r * e_loc:(r + 1) * e_loc]) < TOL, (r, k)
