"""End-to-end MoE sub-block parity on the GPU (EP = 1) against the fp64 oracle,
blocking vs FarSkip identity, and full-size sampled parity."""
import dataclasses

import numpy as np
import pytest
import torch

import synth
from oracle import moe as om
from tests.gpu_util import dev_f32, moe_weights_dev, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-2  # BASELINE.json north star: max relative L2 error 1e-2 (bf16 GEMM, fp32 accumulate)


def make_ctx(shape, T):
    from paper_2511_11505_b200 import build
    build.build()
    from paper_2511_11505_b200 import Context
    return Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                   shared_ffn=shape.shared_ffn, max_tokens=T)


def run_blocking(ctx, wd, x, dbg_fields=True):
    from paper_2511_11505_b200 import MoeDebug
    T, d = x.shape
    k = ctx.cfg.top_k
    E = ctx.cfg.n_experts
    xin = dev_f32(x)
    out = torch.empty_like(xin)
    dbg = MoeDebug(topk_idx=torch.empty(T, k, dtype=torch.int32, device="cuda"),
                   topk_w=torch.empty(T, k, dtype=torch.float32, device="cuda"),
                   counts=torch.empty(E, dtype=torch.int32, device="cuda"),
                   pos=torch.empty(T, k, dtype=torch.int32, device="cuda"),
                   shared_out=torch.empty(T, d, dtype=torch.float32, device="cuda"),
                   routed_out=torch.empty(T, d, dtype=torch.float32, device="cuda"),
                   n_refined=torch.zeros(1, dtype=torch.int32, device="cuda")) if dbg_fields else None
    ctx.moe_forward_blocking(wd, xin, out, dbg)
    torch.cuda.synchronize()
    return out.cpu().numpy(), (None if dbg is None else {k2: v.cpu().numpy() for k2, v in dbg.tensors.items()})


def check_against_oracle(shape, lay, x, out, dbg):
    r, excl = om.adopt_router(lay, x, dbg["topk_idx"])
    sh, ro, _ = om.moe_block(x, lay, router=r)
    np.testing.assert_array_equal(dbg["topk_idx"], r.idx)             # bit-exact routing (R-1 adopted)
    assert dbg["counts"].sum() == x.shape[0] * shape.top_k              # conservation
    m = om.permutation_maps(r.idx, shape.n_experts)
    np.testing.assert_array_equal(dbg["counts"], m.counts)
    np.testing.assert_array_equal(dbg["pos"], m.pos)
    np.testing.assert_allclose(dbg["topk_w"], r.gates, rtol=0, atol=2e-5)
    ref = (x.astype(np.float64) + sh) + ro
    e_out = rel_l2(out, ref)
    e_ro = rel_l2(dbg["routed_out"], ro)
    assert e_out < TOL and e_ro < TOL, (e_out, e_ro)
    if shape.shared_ffn:
        assert rel_l2(dbg["shared_out"], sh) < TOL
    else:
        assert np.all(dbg["shared_out"] == 0)
    return e_out, e_ro, int(excl.sum())


SMALL = [("tiny", 32, 0), ("tiny", 1, 1), ("tiny", 100, 2), ("dsv2lite", 320, 0), ("qwen3", 256, 0),
         ("dsv2lite", 33, 3)]


@pytest.mark.parametrize("name,T,seed", SMALL)
def test_moe_blocking_parity(name, T, seed):
    shape = synth.CONFIGS[name]
    ctx = make_ctx(shape, T)
    w = synth.moe_weights(shape, seed=seed)
    x = synth.tokens(shape, seed=seed, T=T)
    out, dbg = run_blocking(ctx, moe_weights_dev(w), x)
    lay = om.layer_from_synth(w, shape.top_k)
    e_out, e_ro, ex = check_against_oracle(shape, lay, x, out, dbg)
    print(f"{name} T={T}: rel_l2 out={e_out:.2e} routed={e_ro:.2e} excluded={ex}")
    ctx.close()


def test_moe_zero_experts_and_no_shared():
    shape = synth.CONFIGS["tiny"]
    ctx = make_ctx(shape, 32)
    w = synth.moe_weights(shape, seed=4, zero_experts=True)
    x = synth.tokens(shape, seed=4, T=32)
    out, dbg = run_blocking(ctx, moe_weights_dev(w), x)
    assert np.all(dbg["routed_out"] == 0) and np.all(dbg["shared_out"] == 0)
    np.testing.assert_array_equal(out, x)      # out = (x + 0) + 0 exactly
    ctx.close()


@pytest.mark.parametrize("name,T", [("tiny", 32), ("dsv2lite", 200)])
def test_farskip_equals_blocking_bitwise(name, T):
    """At EP=1 the FarSkip sub-block (partial := x_in) computes the same numbers in
    the same order: (x + shared) + routed (BJ: 'FarSkip and blocking give the same
    numbers whatever the stream timing')."""
    shape = synth.CONFIGS[name]
    ctx = make_ctx(shape, T)
    w = synth.moe_weights(shape, seed=2)
    wd = moe_weights_dev(w)
    x = synth.tokens(shape, seed=2, T=T)
    out_b, _ = run_blocking(ctx, wd, x, dbg_fields=False)
    xin = dev_f32(x)
    partial = xin.clone()
    phases = []

    def cb(phase, stream):
        phases.append(phase)
        # perturb the stream timing while the collective is 'in flight'
        torch.cuda._sleep(200000)

    h = ctx.moe_forward_farskip(wd, xin, partial, callback=cb)
    full = torch.empty_like(xin)
    ctx.moe_wait(h, partial, full)
    torch.cuda.synchronize()
    assert phases == [0, 1]
    np.testing.assert_array_equal(full.cpu().numpy(), out_b)
    from paper_2511_11505_b200 import FscError
    with pytest.raises(FscError):
        ctx.moe_wait(h, partial, full)        # a handle completes once
    ctx.close()


def test_farskip_handle_depth_is_one():
    from paper_2511_11505_b200 import FscError
    shape = synth.CONFIGS["tiny"]
    ctx = make_ctx(shape, 32)
    wd = moe_weights_dev(synth.moe_weights(shape, seed=0))
    x = dev_f32(synth.tokens(shape, T=32))
    p = x.clone()
    h = ctx.moe_forward_farskip(wd, x, p)
    with pytest.raises(FscError):
        ctx.moe_forward_farskip(wd, x, p)
    with pytest.raises(FscError):
        ctx.moe_forward_blocking(wd, x, p)
    ctx.moe_wait(h, p, p)
    torch.cuda.synchronize()
    ctx.close()


def check_full_routing(shape, lay, x, dbg):
    """Every token of the batch: the selection equals the fp64 oracle's (R-1 exclusions
    counted), gates within 2e-5, counts / positions equal the oracle's stable maps."""
    r, excl = om.adopt_router(lay, x, dbg["topk_idx"])
    np.testing.assert_array_equal(dbg["topk_idx"], r.idx)
    np.testing.assert_allclose(dbg["topk_w"], r.gates, rtol=0, atol=2e-5)
    m = om.permutation_maps(r.idx, shape.n_experts)
    np.testing.assert_array_equal(dbg["counts"], m.counts)
    np.testing.assert_array_equal(dbg["pos"], m.pos)
    return r, excl


@pytest.mark.parametrize("name,skew", [("dsv2lite", 0.0), ("qwen3", 0.0), ("dsv2lite", synth.SKEW_DEFAULT),
                                       ("qwen3", 0.5)])
def test_full_size_parity(name, skew):
    """BASELINE config sizes (T = 8192 / 16384) in the bench's launch configuration:
    routing, gates, counts and positions of EVERY token against the fp64 oracle; the
    outputs of a token sample recomputed by the oracle one by one (the block is
    token-independent). skew > 0: the skewed-load token recipe."""
    shape = synth.CONFIGS[name]
    T = shape.tokens
    ctx = make_ctx(shape, T)
    w = synth.moe_weights(shape, seed=0)
    x = synth.tokens(shape, seed=0, T=T, skew=skew)
    out, dbg = run_blocking(ctx, moe_weights_dev(w), x)
    assert dbg["counts"].sum() == T * shape.top_k
    lay = om.layer_from_synth(w, shape.top_k)
    r_all, excl = check_full_routing(shape, lay, x, dbg)
    rng = np.random.default_rng(0)
    sample = np.sort(np.concatenate([[0, T - 1], rng.choice(T, 62, replace=False)]))
    r, _ = om.adopt_router(lay, x[sample], dbg["topk_idx"][sample])
    sh, ro, _ = om.moe_block(x[sample], lay, router=r)
    ref = (x[sample].astype(np.float64) + sh) + ro
    assert rel_l2(out[sample], ref) < TOL
    assert rel_l2(dbg["routed_out"][sample], ro) < TOL
    load = dbg["counts"].max() / dbg["counts"].mean()
    print(f"{name} skew={skew}: refined={int(dbg['n_refined'][0])} excluded={int(excl.sum())} "
          f"max/mean load={load:.2f}")
    ctx.close()


def _layer_f32(w, top_k):
    """EpLayer holding exact fp32 widenings of the bf16 weights (the oracle widens
    each expert to fp64 when it uses it) - keeps Scout-sized layers in memory."""
    f = lambda b: None if b is None else synth.bf16_bits_to_f32(b)  # noqa: E731
    return om.EpLayer(w.gamma.astype(np.float64), w.w_router.astype(np.float64), f(w.w1), f(w.w2), f(w.w3),
                      f(w.ws1), f(w.ws2), f(w.ws3), top_k)


def test_scout_full_size_sampled_parity():
    """Llama-4-Scout-shaped layer (d=5120, 16 experts top-1, FFN 8192 + shared 8192)
    at the full 8192 tokens; 16 sampled tokens recomputed by the oracle."""
    shape = synth.CONFIGS["scout"]
    T = shape.tokens
    ctx = make_ctx(shape, T)
    w = synth.moe_weights(shape, seed=0)
    x = synth.tokens(shape, seed=0, T=T)
    out, dbg = run_blocking(ctx, moe_weights_dev(w), x)
    ctx.close()
    lay = _layer_f32(w, shape.top_k)
    del w
    assert dbg["counts"].sum() == T
    # every token's routing (fp64 router over the whole batch: rmsnorm + x W_R^T only)
    xn = om.rmsnorm(x, lay.gamma)
    rt = om.route(xn, lay.w_router, shape.top_k)
    ok = rt.gap >= 1e-6                                       # R-1
    np.testing.assert_array_equal(dbg["topk_idx"][ok], rt.idx[ok])
    m = om.permutation_maps(dbg["topk_idx"], shape.n_experts)
    np.testing.assert_array_equal(dbg["counts"], m.counts)
    np.testing.assert_array_equal(dbg["pos"], m.pos)
    sample = np.array([0, 1, 777, 4095, 4096, 6000, 8190, 8191] + list(range(100, 108)))
    r, excl = om.adopt_router(lay, x[sample], dbg["topk_idx"][sample])
    np.testing.assert_array_equal(dbg["topk_idx"][sample], r.idx)
    assert np.all(dbg["topk_w"][sample] == 1.0)          # top-1: the renormalised gate is exactly 1
    sh, ro, _ = om.moe_block(x[sample], lay, router=r)
    assert rel_l2(out[sample], (x[sample].astype(np.float64) + sh) + ro) < TOL
    assert rel_l2(dbg["routed_out"][sample], ro) < TOL
    assert rel_l2(dbg["shared_out"][sample], sh) < TOL


@pytest.mark.parametrize("base,T", [("qwen3", 64), ("qwen3", 512), ("scout", 64), ("dsv2lite", 128)])
def test_decode_regime_parity(base, T):
    """configs[4]: decode-sized batches (64-512 tokens per step)."""
    shape = synth.decode_shape(base, T)
    ctx = make_ctx(shape, T)
    w = synth.moe_weights(shape, seed=5)
    x = synth.tokens(shape, seed=5, T=T)
    out, dbg = run_blocking(ctx, moe_weights_dev(w), x)
    ctx.close()
    lay = _layer_f32(w, shape.top_k)
    r, _ = om.adopt_router(lay, x, dbg["topk_idx"])
    np.testing.assert_array_equal(dbg["topk_idx"], r.idx)
    sh, ro, _ = om.moe_block(x, lay, router=r)
    assert rel_l2(out, (x.astype(np.float64) + sh) + ro) < TOL


@pytest.mark.parametrize("name,T", [("dsv2lite", 300), ("qwen3", 512)])
def test_fused_gather_permute_is_bitwise_identical(name, T):
    """fsc_set_gemm_gather: GEMM1 gathers the xn rows through src_row (TMA gather4)
    instead of reading the explicitly permuted buffer; the same operand rows reach
    the same MMA, so the layer output is bit-identical."""
    shape = synth.CONFIGS[name]
    ctx = make_ctx(shape, T)
    w = moe_weights_dev(synth.moe_weights(shape, seed=9))
    x = synth.tokens(shape, seed=9, T=T)
    out0, _ = run_blocking(ctx, w, x)
    ctx.set_gemm_gather(True)
    out1, _ = run_blocking(ctx, w, x)
    ctx.close()
    assert np.array_equal(out0, out1)


@pytest.mark.parametrize("name,T", [("tiny", 33), ("dsv2lite", 700), ("qwen3", 2049), ("scout", 200)])
def test_permute_scatter_equals_gather(name, T, monkeypatch):
    """EP = 1 permute by source token (scatter: xs[pos[t, j]] = xn[t]) and by destination
    row (gather: xs[r] = xn[src_row[r]]) write the same buffer: forward output and the
    backward's gradients bitwise equal."""
    shape = synth.CONFIGS[name]
    ctx = make_ctx(shape, T)
    w = moe_weights_dev(synth.moe_weights(shape, seed=10))
    x = synth.tokens(shape, seed=10, T=T)
    outs = []
    for g in ("0", "1"):
        monkeypatch.setenv("FSC_PERMUTE_GATHER", g)
        outs.append(run_blocking(ctx, w, x)[0])
    ctx.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("name,T", [("tiny", 32), ("dsv2lite", 300), ("qwen3", 257), ("scout", 200)])
def test_fused_unpermute_is_bitwise_identical(name, T):
    """Blocking EP = 1 fuses the gate-weighted unpermute into the down GEMM's epilogue
    (last-arriving copy finishes the token); it must equal the separate unpermute
    kernel bit for bit, in slot order (C-amb-12), on repeated calls (counters reset)."""
    shape = synth.CONFIGS[name]
    ctx = make_ctx(shape, T)
    w = moe_weights_dev(synth.moe_weights(shape, seed=4))
    x = synth.tokens(shape, seed=4, T=T)
    ctx.set_fused_unpermute(False)
    ref, _ = run_blocking(ctx, w, x)
    ctx.set_fused_unpermute(True)
    for _ in range(3):
        got, _ = run_blocking(ctx, w, x)
        assert np.array_equal(got, ref)
    ctx.close()


@pytest.mark.parametrize("router", ["tc", "f64"])
@pytest.mark.parametrize("name,T", [("dsv2lite", 512), ("scout", 300), ("qwen3", 2048)])
def test_int8_router_moe_parity(name, T, router):
    """The whole MoE block with the int8 tensor-core router: routing bit-exact against
    the fp64 oracle and the output within tolerance; identical to the SIMT-router run
    whenever both select the same experts (they do here: both equal the oracle)."""
    shape = synth.CONFIGS[name]
    ctx = make_ctx(shape, T)
    w = synth.moe_weights(shape, seed=6)
    wd = moe_weights_dev(w)
    x = synth.tokens(shape, seed=6, T=T)
    ctx.set_router_int8(False)                          # fp32 SIMT router
    ref_out, ref_dbg = run_blocking(ctx, wd, x)
    ctx.set_router_int8(True)
    ctx.set_router_f64(router == "f64")                 # fp64 router / tensor-core router at any T
    out, dbg = run_blocking(ctx, wd, x)
    ctx.close()
    np.testing.assert_array_equal(dbg["topk_idx"], ref_dbg["topk_idx"])
    lay = _layer_f32(w, shape.top_k)
    r, _ = om.adopt_router(lay, x, dbg["topk_idx"])
    np.testing.assert_array_equal(dbg["topk_idx"], r.idx)
    sh, ro, _ = om.moe_block(x, lay, router=r)
    assert rel_l2(out, (x.astype(np.float64) + sh) + ro) < TOL
    assert rel_l2(out, ref_out) < 1e-5


def test_error_paths_are_status_codes_not_crashes():
    """Every misuse is reported through the C ABI status (FscError in Python) before
    anything is enqueued, and the context stays usable afterwards."""
    from paper_2511_11505_b200 import FSC_EP_ALLREDUCE, FscError
    shape = synth.CONFIGS["tiny"]
    T = 32
    ctx = make_ctx(shape, T)
    wd = moe_weights_dev(synth.moe_weights(shape, seed=0))
    x = dev_f32(synth.tokens(shape, T=T))
    out = torch.empty_like(x)
    big = dev_f32(np.zeros((T + 1, shape.d), np.float32))
    with pytest.raises(FscError):                       # T > max_tokens (FSC_ERR_CONFIG)
        ctx.moe_forward_blocking(wd, big, torch.empty_like(big))
    raw = torch.empty(T * shape.d + 1, dtype=torch.float32, device="cuda")
    mis = raw[1:].view(T, shape.d)                      # 4-byte aligned only
    with pytest.raises(FscError):                       # misaligned activation (FSC_ERR_SHAPE)
        ctx.moe_forward_blocking(wd, mis, out)
    with pytest.raises(FscError):                       # d = 64: no FP8 payload (d % 128)
        ctx.set_dispatch_fp8(True)
    with pytest.raises(FscError):                       # int8 router needs d % 128 == 0
        ctx.set_router_int8(True)
    with pytest.raises(FscError):
        ctx.set_gemm_cta_group(3)
    ctx.set_ep_mode(FSC_EP_ALLREDUCE)                   # EP = 1: accepted, no effect
    ctx.moe_forward_blocking(wd, x, out)                # still usable
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    ctx.close()


@pytest.mark.parametrize("name", ["dsv2lite", "qwen3", "scout"])
def test_bench_launch_configuration_graph_replay(name):
    """Exactly what bench.py times: the full BASELINE-size layer captured as CUDA graphs
    with the GEMM1 timing event nodes (fsc_set_timing_mask) and replayed back to back
    with an L2 flush between steps. Every replay equals the eager run bit for bit, and
    sampled tokens match the fp64 oracle."""
    shape = synth.CONFIGS[name]
    T = shape.tokens
    ctx = make_ctx(shape, T)
    w = synth.moe_weights(shape, seed=3)
    wd = moe_weights_dev(w)
    x = synth.tokens(shape, seed=3, T=T)
    xin = dev_f32(x)
    eager = torch.empty_like(xin)
    ctx.moe_forward_blocking(wd, xin, eager)
    torch.cuda.synchronize()
    outs = [torch.empty_like(xin) for _ in range(2)]
    ctx.set_timing_mask(["gemm1"])
    graphs = []
    for o in outs:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ctx.moe_forward_blocking(wd, xin, o)
        graphs.append(g)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for i in range(4):
        flush.fill_(float(i))
        graphs[i % 2].replay()
    torch.cuda.synchronize()
    log = ctx.timing_log(64)
    ctx.set_timing(False)
    assert log and all(n == "gemm1" and ms > 0 for n, ms in log)
    for o in outs:
        assert torch.equal(o, eager)
    sample = np.array([0, 1, T // 2, T - 1])
    lay = om.layer_from_synth(w, shape.top_k)
    idx = torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda")
    from paper_2511_11505_b200 import MoeDebug
    ctx.moe_forward_blocking(wd, xin, torch.empty_like(xin), MoeDebug(topk_idx=idx))
    r, _ = om.adopt_router(lay, x[sample], idx.cpu().numpy()[sample])
    sh, ro, _ = om.moe_block(x[sample], lay, router=r)
    assert rel_l2(outs[0].cpu().numpy()[sample], (x[sample].astype(np.float64) + sh) + ro) < TOL
    ctx.close()


def test_debug_finiteness_check():
    """fsc_set_debug_checks: a non-finite output is reported as FSC_ERR_NONFINITE
    (SPEC S:29 error class) instead of propagating silently; finite runs pass."""
    from paper_2511_11505_b200 import FSC_ERR_NONFINITE, FscError
    shape = synth.CONFIGS["tiny"]
    T = 32
    ctx = make_ctx(shape, T)
    wd = moe_weights_dev(synth.moe_weights(shape, seed=0))
    x = synth.tokens(shape, T=T)
    ctx.set_debug_checks(True)
    xin = dev_f32(x)
    out = torch.empty_like(xin)
    ctx.moe_forward_blocking(wd, xin, out)
    x[3, 5] = np.inf
    with pytest.raises(FscError) as ei:
        ctx.moe_forward_blocking(wd, dev_f32(x), out)
    assert ei.value.code == FSC_ERR_NONFINITE
    ctx.moe_forward_blocking(wd, xin, out)          # not sticky
    torch.cuda.synchronize()
    ctx.close()
