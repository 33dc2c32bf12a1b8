"""Layer-stack parity on the GPU (EP = 1): Regular / Hybrid wiring, BLOCKING vs
OVERLAPPED schedules, per-layer teacher-forced comparison with the fp64 oracle
(SURVEY §8(c) R-4), and the FarSkip identities of P:175 on the GPU's own
activations."""
import dataclasses

import numpy as np
import pytest
import torch

import synth
from oracle import moe as om
from oracle import stack as ost
from tests.gpu_util import attn_weights_dev, dev_f32, moe_weights_dev, rel_l2

pytestmark = pytest.mark.gpu
R, H = ost.REGULAR, ost.HYBRID


class AWf:
    """fp64 view of synth.AttnWeights for the oracle."""

    def __init__(self, a):
        self.gamma = a.gamma.astype(np.float64)
        self.w_qkv = synth.bf16_bits_to_f64(a.w_qkv)
        self.w_o = synth.bf16_bits_to_f64(a.w_o)
        self.n_heads, self.n_kv_heads, self.head_dim, self.rope_theta = a.n_heads, a.n_kv_heads, a.head_dim, a.rope_theta


SMALL_DS = dataclasses.replace(synth.CONFIGS["dsv2lite"], d=512, n_experts=16, top_k=4, ffn=256, shared_ffn=512,
                               tokens=256, n_heads=4, n_kv_heads=2, head_dim=128, seq_len=128, n_layers=3)


def run_stack(shape, modes, schedule, seed=0, T=None, cache=True):
    from paper_2511_11505_b200 import Context, build
    build.build()
    T = shape.tokens if T is None else T
    L = len(modes)
    mws = [synth.moe_weights(shape, seed=seed, layer=k) for k in range(L)]
    aws = [synth.attn_weights(shape, seed=seed, layer=k) for k in range(L)]
    x = synth.tokens(shape, seed=seed, T=T)
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T)
    mwd = [moe_weights_dev(w) for w in mws]
    awd = [attn_weights_dev(a) for a in aws]
    o0 = dev_f32(x)
    oL = torch.empty_like(o0)
    caches = None
    if cache:
        caches = [{k: torch.full_like(o0, float("nan")) for k in
                   ("attn_in", "mlp_in", "attn_out", "shared_out", "routed_out", "o")} for _ in range(L)]
    ctx.layer_stack_forward(awd, mwd, T, shape.seq_len, modes, schedule, o0, oL, caches)
    torch.cuda.synchronize()
    out = oL.cpu().numpy()
    cc = None if caches is None else [{k: v.cpu().numpy() for k, v in c.items()} for c in caches]
    ctx.close()
    return x, mws, aws, out, cc


@pytest.mark.parametrize("shape", [synth.CONFIGS["tiny"], SMALL_DS], ids=["tiny", "small_ds"])
@pytest.mark.parametrize("modes", [(H, H), (R, R), (R, H), (H, R), (H, H, H)])
def test_stack_teacher_forced_parity(shape, modes):
    from paper_2511_11505_b200 import FSC_OVERLAPPED
    x, mws, aws, out, cc = run_stack(shape, list(modes), FSC_OVERLAPPED)
    lays = [om.layer_from_synth(w, shape.top_k) for w in mws]
    awf = [AWf(a) for a in aws]
    teacher = [(c["attn_in"], c["mlp_in"]) for c in cc]
    ref = ost.stack_forward(x, awf, lays, list(modes), shape.seq_len, teacher_inputs=teacher)
    for k, (c, r) in enumerate(zip(cc, ref)):
        for key, rv in (("attn_out", r.attn_out), ("routed_out", r.routed_out), ("o", r.o)):
            e = rel_l2(c[key], rv)
            assert e < 1e-2, (k, key, e)
        if shape.shared_ffn:
            assert rel_l2(c["shared_out"], r.shared_out) < 1e-2
    np.testing.assert_array_equal(out, cc[-1]["o"])
    # the wiring itself, on the GPU's own activations
    np.testing.assert_array_equal(cc[0]["attn_in"], x)
    for k in range(1, len(modes)):
        prev, cur = cc[k - 1], cc[k]
        if modes[k] == H:
            # mlp-in_k = attn-in_k + routed-exp-out_{k-1}, bitwise; and = o_{k-1} (Eq. 8a)
            np.testing.assert_array_equal(cur["mlp_in"], (cur["attn_in"] + prev["routed_out"]).astype(np.float32))
            np.testing.assert_array_equal(cur["mlp_in"], prev["o"])
        else:
            np.testing.assert_array_equal(cur["attn_in"], prev["o"])           # Eq. 6: attn-in_k = o_{k-1}
    for k, m in enumerate(modes):
        if m == R:
            np.testing.assert_array_equal(cc[k]["mlp_in"], (cc[k]["attn_in"] + cc[k]["attn_out"]).astype(np.float32))


@pytest.mark.parametrize("modes", [(H, H, H), (R, R, R), (R, H, H)])
def test_blocking_equals_overlapped_bitwise(modes):
    from paper_2511_11505_b200 import FSC_BLOCKING, FSC_OVERLAPPED
    _, _, _, a, ca = run_stack(SMALL_DS, list(modes), FSC_BLOCKING)
    _, _, _, b, cb = run_stack(SMALL_DS, list(modes), FSC_OVERLAPPED)
    np.testing.assert_array_equal(a, b)
    for x, y in zip(ca, cb):
        for k in x:
            np.testing.assert_array_equal(x[k], y[k])


def test_all_regular_free_running_is_prenorm_transformer():
    """Far-skip disabled -> the standard pre-norm transformer (BJ north star)."""
    from paper_2511_11505_b200 import FSC_OVERLAPPED
    shape = synth.CONFIGS["tiny"]
    x, mws, aws, out, _ = run_stack(shape, [R, R], FSC_OVERLAPPED, cache=False)
    lays = [om.layer_from_synth(w, shape.top_k) for w in mws]
    ref = ost.stack_forward(x, [AWf(a) for a in aws], lays, [R, R], shape.seq_len)
    assert rel_l2(out, ref[-1].o) < 1e-2


def test_zero_wo_makes_hybrid_equal_regular():
    """W_O = 0 (attn_out = 0): the dropped connections carry zero, so the Hybrid
    and Regular stacks compute the same numbers (oracle pin, reproduced on GPU)."""
    from paper_2511_11505_b200 import Context, FSC_OVERLAPPED
    shape = SMALL_DS
    T, L = shape.tokens, 2
    mws = [synth.moe_weights(shape, seed=1, layer=k) for k in range(L)]
    aws = [synth.attn_weights(shape, seed=1, layer=k, zero_o=True) for k in range(L)]
    x = synth.tokens(shape, seed=1, T=T)
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T)
    outs = []
    for modes in ([H, H], [R, R]):
        o0 = dev_f32(x)
        oL = torch.empty_like(o0)
        ctx.layer_stack_forward([attn_weights_dev(a) for a in aws], [moe_weights_dev(w) for w in mws], T,
                                shape.seq_len, modes, FSC_OVERLAPPED, o0, oL)
        torch.cuda.synchronize()
        outs.append(oL.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    ctx.close()


@pytest.mark.parametrize("T,Hq,Hkv,seq_len", [(640, 4, 2, 256), (600, 2, 1, 256), (384, 3, 3, 128), (1024, 2, 2, 1024),
                                              (130, 1, 1, 128)])
def test_attention_core_parity(T, Hq, Hkv, seq_len):
    """Core attention (P:198 part (b) without W_o) on the GPU - the tcgen05 kernel for
    hd = 128 - against oracle.attention_core with W_o = I on the same bf16 q, k, v: causal
    within packed sequences, GQA head sharing, ragged last tile."""
    from oracle import attention as oa
    from paper_2511_11505_b200 import Context
    from tests.gpu_util import dev_bf16, host_bf16_to_f64
    hd = 128
    rng = np.random.default_rng(T + Hq)
    qkv = synth.f32_to_bf16_bits((rng.standard_normal((T, (Hq + 2 * Hkv) * hd)) * 1.5).astype(np.float32))
    ctx = Context(d=128, n_experts=4, top_k=2, ffn=128, shared_ffn=0, max_tokens=T)
    out = torch.zeros(T, Hq * hd, dtype=torch.bfloat16, device="cuda")
    ctx.op_attention(dev_bf16(qkv), out, Hq, Hkv, hd, seq_len)
    torch.cuda.synchronize()
    f = synth.bf16_bits_to_f64(qkv)
    q = f[:, :Hq * hd].reshape(T, Hq, hd)
    k = f[:, Hq * hd:(Hq + Hkv) * hd].reshape(T, Hkv, hd)
    v = f[:, (Hq + Hkv) * hd:].reshape(T, Hkv, hd)
    ref = oa.attention_core(q, k, v, np.eye(Hq * hd), seq_len)
    got = host_bf16_to_f64(out)
    assert rel_l2(got, ref) < 1e-2, rel_l2(got, ref)
    ctx.close()
