"""Per-kernel GPU parity through the C ABI op entry points (K1-K5) against the
fp64 oracle / fp64 definitions on the same seeded inputs."""
import numpy as np
import pytest
import torch

import synth
from oracle import moe as om
from tests.gpu_util import dev_bf16, dev_f32, host_bf16_to_f64, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2511_11505_b200 import build
    build.build()
    from paper_2511_11505_b200 import Context
    c = Context(d=5120, n_experts=128, top_k=8, ffn=1408, shared_ffn=0, max_tokens=16384)
    c.set_router_int8(False)   # K1 tests below: the fp32 SIMT router (ctx_i8: the tensor-core one)
    yield c
    c.close()


def rand_bf16(rng, shape, scale=1.0):
    return synth.f32_to_bf16_bits((rng.standard_normal(shape) * scale).astype(np.float32))


# ----------------------------------------------------------------------------- K4 grouped GEMM
GEMM_CASES = [
    # (counts, N, K)
    ([1], 256, 64),
    ([128], 64, 64),
    ([0, 130, 257], 256, 128),
    ([300, 0, 0, 5], 128, 2048),
    ([517, 64, 1, 129, 0, 255, 256, 1000], 2048, 1408),
    ([200, 77], 5120, 192),
    ([384], 1408, 2048),   # N % 256 != 0 -> BN = 128
    ([70, 71], 192, 64),   # N % 128 != 0 -> BN = 64
]


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("counts,N,K", GEMM_CASES)
def test_grouped_gemm_bf16(ctx, counts, N, K, cg):
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(len(counts) * 1000 + N + K)
    G, M = len(counts), sum(counts)
    A = rand_bf16(rng, (max(M, 1), K))
    B = rand_bf16(rng, (G * N, K), 1.0 / np.sqrt(K))
    out = torch.zeros(max(M, 1), N, dtype=torch.bfloat16, device="cuda")
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    ctx.op_grouped_gemm(0, dev_bf16(A[:M] if M else A), dev_bf16(B), None, G, cnt, 0, N, K, out)
    torch.cuda.synchronize()
    got = host_bf16_to_f64(out)[:M]
    Af, Bf = synth.bf16_bits_to_f64(A), synth.bf16_bits_to_f64(B)
    r = 0
    for g, m in enumerate(counts):
        if m:
            ref = Af[r:r + m] @ Bf[g * N:(g + 1) * N].T
            assert rel_l2(got[r:r + m], ref) < 4e-3, (g, rel_l2(got[r:r + m], ref))
            assert np.max(np.abs(got[r:r + m] - ref)) <= 1e-2 * np.max(np.abs(ref)) + 1e-6
        r += m


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("epi,counts,N,K", [(0, [517, 64, 1, 129, 0, 255, 256, 1000], 2048, 1408),
                                            (0, [70, 71], 192, 64), (1, [600, 0, 257, 255], 768, 2048),
                                            (2, [777], 2048, 256), (0, [0, 0], 256, 64)])
def test_grouped_gemm_dynamic_schedule_bitwise(ctx, epi, counts, N, K, cg):
    """The dynamic tile schedule (atomic claims, shared-memory tile queue, DSMEM hand-off to
    the peer CTA) computes every tile exactly as the static stride does: bitwise equal
    outputs, on the full grid and on a small grid (many tiles per CTA), twice in a row
    (the last CTA out resets the counters)."""
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(21 + N + K + epi)
    G, M = len(counts), sum(counts)
    A = dev_bf16(rand_bf16(rng, (max(M, 1), K)))
    B0 = dev_bf16(rand_bf16(rng, (G * N, K), 1.0 / np.sqrt(K)))
    B1 = dev_bf16(rand_bf16(rng, (G * N, K), 1.0 / np.sqrt(K))) if epi == 1 else None
    resid = dev_f32(rng.standard_normal((max(M, 1), N)).astype(np.float32)) if epi == 2 else None
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda") if epi != 2 else None
    dt = torch.float32 if epi == 2 else torch.bfloat16
    outs = []
    try:
        for dyn, ctas in [(False, 148), (True, 148), (True, 148), (True, 20)]:
            ctx.set_gemm_dynamic(dyn)
            ctx.set_gemm_ctas(ctas)
            out = torch.zeros(max(M, 1), N, dtype=dt, device="cuda")
            ctx.op_grouped_gemm(epi, A, B0, B1, G, cnt, M if epi == 2 else 0, N, K, out, resid)
            torch.cuda.synchronize()
            outs.append(out.cpu())
    finally:
        ctx.set_gemm_dynamic(None)
        ctx.set_gemm_ctas(148)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("counts,N,K", [([1], 128, 64), ([0, 130, 257], 128, 128), ([333, 900, 17], 1408, 2048),
                                        ([40], 64, 64), ([256, 1], 8192, 128), ([600, 0, 257, 255], 768, 2048)])
@pytest.mark.parametrize("cg", [1, 2])
def test_grouped_gemm_swiglu(ctx, counts, N, K, cg):
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(7 + N + K)
    G, M = len(counts), sum(counts)
    A = rand_bf16(rng, (M, K))
    W1 = rand_bf16(rng, (G * N, K), 1.0 / np.sqrt(K))
    W2 = rand_bf16(rng, (G * N, K), 1.0 / np.sqrt(K))
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    ctx.op_grouped_gemm(1, dev_bf16(A), dev_bf16(W1), dev_bf16(W2), G, cnt, 0, N, K, out)
    torch.cuda.synchronize()
    got = host_bf16_to_f64(out)
    Af = synth.bf16_bits_to_f64(A)
    r = 0
    for g, m in enumerate(counts):
        if m:
            u = Af[r:r + m] @ synth.bf16_bits_to_f64(W1[g * N:(g + 1) * N]).T
            gt = Af[r:r + m] @ synth.bf16_bits_to_f64(W2[g * N:(g + 1) * N]).T
            ref = u * om.silu(gt)     # the gated branch of P:73-76
            assert rel_l2(got[r:r + m], ref) < 5e-3
        r += m


@pytest.mark.parametrize("counts,N,K,src", [([1], 128, 64, 5), ([0, 130, 257], 128, 128, 100),
                                            ([333, 900, 17], 1408, 2048, 700), ([600, 0, 257, 255], 768, 2048, 1111),
                                            ([517, 64, 1, 129, 0, 255, 256, 1000], 256, 1408, 300)])
@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("epi", [0, 1])
def test_grouped_gemm_gather(ctx, counts, N, K, src, cg, epi):
    """Fused permute (EP = 1): row r of the grouped GEMM reads A[a_idx[r]] through TMA
    gather4; equals the GEMM of the explicitly permuted rows."""
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(11 + N + K + epi)
    G, M = len(counts), sum(counts)
    A = rand_bf16(rng, (src, K))
    a_idx = rng.integers(0, src, size=M).astype(np.int32)
    W1 = rand_bf16(rng, (G * N, K), 1.0 / np.sqrt(K))
    W2 = rand_bf16(rng, (G * N, K), 1.0 / np.sqrt(K)) if epi == 1 else None
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    ctx.op_grouped_gemm_gather(epi, dev_bf16(A), torch.from_numpy(a_idx).cuda(), dev_bf16(W1),
                               dev_bf16(W2) if W2 is not None else None, G, cnt, 0, N, K, out)
    torch.cuda.synchronize()
    got = host_bf16_to_f64(out)
    Af = synth.bf16_bits_to_f64(A)[a_idx]
    r = 0
    for g, m in enumerate(counts):
        if m:
            u = Af[r:r + m] @ synth.bf16_bits_to_f64(W1[g * N:(g + 1) * N]).T
            ref = u * om.silu(Af[r:r + m] @ synth.bf16_bits_to_f64(W2[g * N:(g + 1) * N]).T) if epi == 1 else u
            assert rel_l2(got[r:r + m], ref) < 5e-3, (g, rel_l2(got[r:r + m], ref))
        r += m


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("with_resid", [True, False])
def test_gemm_resid_f32_single_group(ctx, with_resid, cg):
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(3)
    M, N, K = 777, 2048, 2816
    A = rand_bf16(rng, (M, K))
    B = rand_bf16(rng, (N, K), 1.0 / np.sqrt(K))
    resid = rng.standard_normal((M, N)).astype(np.float32)
    out = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    ctx.op_grouped_gemm(2, dev_bf16(A), dev_bf16(B), None, 1, None, M, N, K, out,
                        dev_f32(resid) if with_resid else None)
    torch.cuda.synchronize()
    ref = synth.bf16_bits_to_f64(A) @ synth.bf16_bits_to_f64(B).T
    if with_resid:
        ref = ref + resid
    # fp32 accumulation of exact bf16 products: the only error source
    assert rel_l2(out.cpu().numpy(), ref) < 1e-5


@pytest.mark.parametrize("cg", [1, 2])
def test_gemm_inplace_resid(ctx, cg):
    ctx.set_gemm_cta_group(cg)
    rng = np.random.default_rng(4)
    M, N, K = 300, 512, 64
    A = rand_bf16(rng, (M, K)); B = rand_bf16(rng, (N, K))
    r0 = rng.standard_normal((M, N)).astype(np.float32)
    buf = dev_f32(r0)
    ctx.op_grouped_gemm(2, dev_bf16(A), dev_bf16(B), None, 1, None, M, N, K, buf, buf)
    torch.cuda.synchronize()
    ref = r0 + synth.bf16_bits_to_f64(A) @ synth.bf16_bits_to_f64(B).T
    assert rel_l2(buf.cpu().numpy(), ref) < 1e-5


# ----------------------------------------------------------------------------- K1 router
# T < 148*32 tokens run the split-d path (partials over d, fixed-order finish kernel);
# larger T the single-pass kernel with balanced waves (two CTAs per SM)
# ... and the full BASELINE batch sizes the bench runs (T = 8192 / 16384 / 8192)
ROUTER_CASES = [("tiny", 32), ("tiny", 1), ("dsv2lite", 700), ("qwen3", 513), ("scout", 256), ("dsv2lite", 64),
                ("qwen3", 2400), ("dsv2lite", 4800), ("qwen3", 6000), ("scout", 5000),
                ("dsv2lite", 8192), ("qwen3", 16384), ("scout", 8192)]


@pytest.fixture(scope="module")
def ctx_i8():
    """E <= 128 and d % 128 == 0: the exact fused tensor-core router (router_tc_kernel)."""
    from paper_2511_11505_b200 import Context
    c = Context(d=5120, n_experts=128, top_k=8, ffn=128, shared_ffn=0, max_tokens=16384)
    c.set_router_int8(True)
    c.set_router_f64(False)   # the tensor-core kernel at every T (auto would pick fp64 at T <= 1024)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_f64():
    """The fp64 small-batch router (router_f64_kernel), forced at every T."""
    from paper_2511_11505_b200 import Context
    c = Context(d=5120, n_experts=128, top_k=8, ffn=128, shared_ffn=0, max_tokens=16384)
    c.set_router_f64(True)
    yield c
    c.close()


@pytest.mark.parametrize("name,T", ROUTER_CASES)
def test_router_parity(ctx, name, T):
    _router_parity(ctx, name, T)


@pytest.mark.parametrize("name,T,skew", [("dsv2lite", 8192, synth.SKEW_DEFAULT), ("qwen3", 16384, 0.5)])
def test_router_parity_skewed(ctx, name, T, skew):
    """Skewed-load tokens: a shared mean shift makes some experts hot."""
    _router_parity(ctx, name, T, skew)


@pytest.mark.parametrize("name,T", [c for c in ROUTER_CASES if c[0] != "tiny"] + [("dsv2lite", 129), ("qwen3", 1)])
def test_router_parity_int8(ctx_i8, name, T):
    """Exact fused tensor-core path (int8 digit planes, tcgen05 kind::i8): same bit-exact
    indices; the logits' rigorous error bound is ~1e-4 of their scale (three 7-bit digits,
    one-signed truncation), so few tokens need the fp64 refinement."""
    nref, e_max = _router_parity(ctx_i8, name, T)
    assert e_max < 5e-5
    # refinement is the exception, not the rule: the boundary gaps shrink with E (Qwen3,
    # E = 128, k = 8: ~4.4% of the tokens are within the band)
    E = synth.CONFIGS[name].n_experts
    assert nref <= max(4, T * E // 1600), (nref, T, E)


@pytest.mark.parametrize("name,T", ROUTER_CASES + [("qwen3", 7), ("dsv2lite", 33), ("scout", 65), ("qwen3", 1000),
                                                 ("qwen3", 1025), ("scout", 512), ("dsv2lite", 300)])
def test_router_parity_f64(ctx_f64, name, T):
    """fp64 router (every product and sum in fp64, fixed order): the oracle's selection
    with no refinement; logits are fp64 values rounded once to fp32."""
    nref, e_max = _router_parity(ctx_f64, name, T)
    assert nref == 0
    assert e_max < 2e-6


@pytest.mark.parametrize("simt", ["0", "1"])
@pytest.mark.parametrize("plan", ["4,1", "4,2", "2,4", "1,8", "1,16", "2,16"])
def test_router_f64_every_tile_and_cluster_shape(ctx_f64, plan, simt, monkeypatch):
    """Every (token-tile height, cluster size) the cost model can pick, forced through
    FSC_ROUTER_F64_PLAN, on ragged batches of the Qwen3 / DS / Scout router shapes, with
    the fp64 tensor-core (DMMA) contraction and the DFMA one (FSC_ROUTER_F64_SIMT)."""
    monkeypatch.setenv("FSC_ROUTER_F64_PLAN", plan)
    monkeypatch.setenv("FSC_ROUTER_F64_SIMT", simt)
    for name, T in (("qwen3", 77), ("dsv2lite", 45), ("scout", 70)):
        _router_parity(ctx_f64, name, T)


@pytest.mark.parametrize("skew", [synth.SKEW_DEFAULT])
def test_router_parity_f64_skewed(ctx_f64, skew):
    _router_parity(ctx_f64, "dsv2lite", 512, skew)


def _router_parity(ctx, name, T, skew=0.0):
    shape = synth.CONFIGS[name]
    w = synth.moe_weights(dataclass_replace_small(shape), seed=1)
    x = synth.tokens(shape, seed=1, T=T, skew=skew)
    d, E, k = shape.d, shape.n_experts, shape.top_k
    xn = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, k, dtype=torch.float32, device="cuda")
    logits = torch.empty(T, E, dtype=torch.float32, device="cuda")
    nref = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.op_router(dev_f32(x), dev_f32(w.gamma), dev_f32(w.w_router), k, xn, idx, gw, logits, nref)
    torch.cuda.synchronize()
    lay = om.EpLayer(w.gamma.astype(np.float64), w.w_router.astype(np.float64), None, None, None, top_k=k)
    xo = om.rmsnorm(x, lay.gamma)
    r = om.route(xo, lay.w_router, k)
    gi = idx.cpu().numpy()
    excl = r.gap < 1e-6                                   # near-tie rule R-1
    np.testing.assert_array_equal(gi[~excl], r.idx[~excl])
    # R-2: the fp32 logits' error, and the exactness claim it supports
    e_max = np.max(np.abs(logits.cpu().numpy() - r.logits))
    assert e_max < 5e-5
    gsel = np.take_along_axis(r.probs, gi.astype(np.int64), axis=1)
    gates_ref = gsel / gsel.sum(1, keepdims=True)
    np.testing.assert_allclose(gw.cpu().numpy(), gates_ref, rtol=0, atol=2e-5)
    np.testing.assert_allclose(gw.cpu().numpy().sum(1), 1.0, atol=2e-6)
    assert np.all(gw.cpu().numpy() > 0)
    # xn is the bf16 rounding of the fp64 normalised row (<= 1 ulp from double rounding)
    got = host_bf16_to_f64(xn)
    assert np.all(np.abs(got - xo) <= np.abs(xo) * 2.0 ** -7 + 1e-30)
    print(f"{name} T={T}: excluded={int(excl.sum())} refined={int(nref.item())} e_max={e_max:.2e}")
    return int(nref.item()), e_max


def dataclass_replace_small(shape):
    import dataclasses
    # router test only needs gamma / W_R: a 1-wide expert FFN keeps generation cheap
    return dataclasses.replace(shape, ffn=1, shared_ffn=0)


@pytest.mark.parametrize("which", ["simt", "tc", "f64"])
def test_router_exact_ties_go_to_lower_index(ctx, ctx_i8, ctx_f64, which):
    ctx = {"simt": ctx, "tc": ctx_i8, "f64": ctx_f64}[which]
    rng = np.random.default_rng(5)
    T, d, E, k = 64, 128, 16, 3
    x = rng.standard_normal((T, d)).astype(np.float32)
    gamma = np.ones(d, np.float32)
    W = (rng.standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    W[9] = W[2]       # experts 2 and 9 tie exactly for every token
    W[12] = W[5]
    xn = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, k, dtype=torch.float32, device="cuda")
    ctx.op_router(dev_f32(x), dev_f32(gamma), dev_f32(W), k, xn, idx, gw)
    torch.cuda.synchronize()
    r = om.route(om.rmsnorm(x, gamma), W.astype(np.float64), k)
    np.testing.assert_array_equal(idx.cpu().numpy(), r.idx)


def test_router_all_experts_tied(ctx_i8):
    """Every router row equal: every logit of a token ties, every token is ambiguous and its
    band is all E experts - more (token, expert) pairs than the fused kernel's pair list, so
    its overflow path runs too. The exact answer: experts 0..k-1 (ties -> lower id), gates 1/k."""
    rng = np.random.default_rng(6)
    T, d, E, k = 300, 256, 128, 8
    x = rng.standard_normal((T, d)).astype(np.float32)
    gamma = (1.0 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    W = np.repeat((rng.standard_normal((1, d)) / np.sqrt(d)).astype(np.float32), E, axis=0)
    xn = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, k, dtype=torch.float32, device="cuda")
    nref = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx_i8.op_router(dev_f32(x), dev_f32(gamma), dev_f32(W), k, xn, idx, gw, None, nref)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.cpu().numpy(), np.tile(np.arange(k, dtype=np.int32), (T, 1)))
    np.testing.assert_allclose(gw.cpu().numpy(), 1.0 / k, rtol=0, atol=1e-6)
    assert int(nref.item()) == T


def test_router_f64_all_tied_and_non_finite(ctx_f64):
    """fp64 router: every logit of a token tied -> experts 0..k-1, gates 1/k; a token with a
    non-finite input still gets k valid, distinct ids and finite gates summing to 1."""
    rng = np.random.default_rng(6)
    T, d, E, k = 300, 256, 128, 8
    x = rng.standard_normal((T, d)).astype(np.float32)
    gamma = (1.0 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    W = np.repeat((rng.standard_normal((1, d)) / np.sqrt(d)).astype(np.float32), E, axis=0)
    xn = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, k, dtype=torch.float32, device="cuda")
    ctx_f64.op_router(dev_f32(x), dev_f32(gamma), dev_f32(W), k, xn, idx, gw)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.cpu().numpy(), np.tile(np.arange(k, dtype=np.int32), (T, 1)))
    np.testing.assert_allclose(gw.cpu().numpy(), 1.0 / k, rtol=0, atol=1e-7)
    W = (rng.standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    x[3, 7] = np.nan
    x[5, 1] = np.inf
    ctx_f64.op_router(dev_f32(x), dev_f32(gamma), dev_f32(W), k, xn, idx, gw)
    torch.cuda.synchronize()
    gi, g = idx.cpu().numpy(), gw.cpu().numpy()
    assert np.all((gi >= 0) & (gi < E))
    assert all(len(set(row)) == k and list(row) == sorted(row) for row in gi)
    assert np.all(np.isfinite(g)) and np.allclose(g.sum(1), 1.0, atol=1e-6)


# ----------------------------------------------------------------------------- K2 / K3 / K5
# T <= 1024 with E <= 128 runs the single-CTA fused kernel, larger T the three-kernel path
@pytest.mark.parametrize("T,E,k,hot", [(1, 4, 2, 0), (32, 4, 2, 0), (33, 8, 3, 0), (1000, 64, 6, 0), (4096, 128, 8, 0),
                                       (777, 16, 1, 0), (512, 128, 8, 0), (1024, 128, 8, 0), (1025, 128, 8, 0),
                                       (1024, 128, 8, 1), (3000, 64, 6, 1), (300, 64, 10, 0), (700, 32, 12, 1)])
def test_perm_maps_exact(ctx, T, E, k, hot):
    rng = np.random.default_rng(T + E)
    if hot:   # every token on the same k experts (extreme skew): one expert block holds all copies
        idx = np.tile(np.arange(E - k, E, dtype=np.int32), (T, 1))
    else:
        idx = np.stack([np.sort(rng.choice(E, k, replace=False)) for _ in range(T)]).astype(np.int32)
    di = torch.from_numpy(idx).cuda()
    counts = torch.empty(E, dtype=torch.int32, device="cuda")
    offs = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    pos = torch.empty(T, k, dtype=torch.int32, device="cuda")
    src = torch.empty(T * k, dtype=torch.int32, device="cuda")
    ctx.op_perm_maps(di, E, counts, offs, pos, src)
    torch.cuda.synchronize()
    m = om.permutation_maps(idx, E)
    np.testing.assert_array_equal(counts.cpu().numpy(), m.counts)
    np.testing.assert_array_equal(offs.cpu().numpy(), m.offsets)
    np.testing.assert_array_equal(pos.cpu().numpy(), m.pos)
    np.testing.assert_array_equal(src.cpu().numpy(), m.src_row)


def test_permute_and_unpermute(ctx):
    rng = np.random.default_rng(9)
    T, d, E, k = 300, 256, 8, 3
    idx = np.stack([np.sort(rng.choice(E, k, replace=False)) for _ in range(T)]).astype(np.int32)
    m = om.permutation_maps(idx, E)
    xn = rand_bf16(rng, (T, d))
    xs = torch.empty(T * k, d, dtype=torch.bfloat16, device="cuda")
    ctx.op_permute(dev_bf16(xn), torch.from_numpy(m.src_row.astype(np.int32)).cuda(), xs)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(xs.cpu().view(torch.int16).numpy().view(np.uint16), xn[m.src_row])
    y = rand_bf16(rng, (T * k, d))
    w = rng.random((T, k)).astype(np.float32)
    resid = rng.standard_normal((T, d)).astype(np.float32)
    out = torch.empty(T, d, dtype=torch.float32, device="cuda")
    pos = torch.from_numpy(m.pos.astype(np.int32)).cuda()
    for res in (resid, None):
        ctx.op_unpermute(dev_bf16(y), pos, dev_f32(w), dev_f32(res) if res is not None else None, out)
        torch.cuda.synchronize()
        yf = synth.bf16_bits_to_f64(y)
        ref = sum(w[:, j:j + 1].astype(np.float64) * yf[m.pos[:, j]] for j in range(k))
        if res is not None:
            ref = ref + res
        assert rel_l2(out.cpu().numpy(), ref) < 1e-6
