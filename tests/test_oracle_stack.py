"""Pins of the oracle's attention filler, residual wiring and schedule replay."""
import json
import math
import os

import numpy as np
import pytest

from oracle import attention as oa
from oracle import moe as om
from oracle import schedule as osch
from oracle import stack as ost

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


class AW:
    def __init__(self, d, hq, hkv, hd, seed, zero_o=False):
        g = np.random.default_rng(seed)
        self.gamma = 1 + 0.1 * g.standard_normal(d)
        self.w_qkv = g.standard_normal(((hq + 2 * hkv) * hd, d)) / math.sqrt(d)
        self.w_o = np.zeros((d, hq * hd)) if zero_o else g.standard_normal((d, hq * hd)) / math.sqrt(hq * hd)
        self.n_heads, self.n_kv_heads, self.head_dim, self.rope_theta = hq, hkv, hd, 10000.0


def lay(d, E, k, c, cs, seed, zero=False):
    g = np.random.default_rng(seed)
    w = lambda *s: (0 if zero else 1) * g.standard_normal(s) / math.sqrt(s[-1])  # noqa: E731
    return om.EpLayer(1 + 0.1 * g.standard_normal(d), w(E, d), w(E, c, d), w(E, c, d), w(E, d, c),
                      w(cs, d) if cs else None, w(cs, d) if cs else None, w(d, cs) if cs else None, k)


# ------------------------------------------------------------------ attention
def test_attention_single_token_is_v_projection():
    aw = AW(16, 4, 2, 8, 0)
    x = np.random.default_rng(1).standard_normal((1, 16))
    h = om.rmsnorm(x, aw.gamma)
    v = (h @ aw.w_qkv.T)[:, (4 + 2) * 8:].reshape(1, 2, 8)
    vfull = np.repeat(v, 2, axis=1).reshape(1, 32)          # each q head reads its group's v
    np.testing.assert_allclose(oa.attention_block(x, aw, 8), vfull @ aw.w_o.T, rtol=1e-13)


def test_attention_zero_and_causal_and_packing():
    aw = AW(16, 4, 4, 4, 2)
    x = np.random.default_rng(3).standard_normal((12, 16))
    aw0 = AW(16, 4, 4, 4, 2, zero_o=True)
    assert np.all(oa.attention_block(x, aw0, 12) == 0)
    y = oa.attention_block(x, aw, 12)
    for t in range(12):
        x2 = x.copy(); x2[t] += 5.0
        y2 = oa.attention_block(x2, aw, 12)
        np.testing.assert_array_equal(y2[:t], y[:t])        # exact causality
        assert not np.allclose(y2[t], y[t])
    # packing: sequences of 6 equal two independent runs of 6 tokens
    yp = oa.attention_block(x, aw, 6)
    np.testing.assert_allclose(yp[:6], oa.attention_block(x[:6], aw, 6), rtol=1e-14)
    np.testing.assert_allclose(yp[6:], oa.attention_block(x[6:], aw, 6), rtol=1e-13)


def test_rope_rotation_properties():
    g = np.random.default_rng(4)
    q = g.standard_normal((5, 3, 8)); k = g.standard_normal((5, 3, 8))
    pos = np.arange(5)
    rq = oa.rope(q, pos, 10000.0)
    # norm-preserving rotation; identity at position 0
    np.testing.assert_allclose(np.linalg.norm(rq, axis=-1), np.linalg.norm(q, axis=-1), rtol=1e-14)
    np.testing.assert_allclose(rq[0], q[0], rtol=0, atol=0)
    # relative position: <R(m)q, R(n)k> depends only on m - n
    for s in (1, 7, 100):
        a = np.einsum("thd,thd->th", oa.rope(q, pos + s, 1e4), oa.rope(k[::-1], pos[::-1] + s, 1e4))
        b = np.einsum("thd,thd->th", oa.rope(q, pos, 1e4), oa.rope(k[::-1], pos[::-1], 1e4))
        np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-12)
    # hd = 2, theta irrelevant: plain 2-D rotation by angle = position (freq 1)
    v = np.array([[[1.0, 0.0]]])
    np.testing.assert_allclose(oa.rope(v, np.array([1]), 10000.0)[0, 0], [math.cos(1), math.sin(1)], rtol=1e-15)


# ------------------------------------------------------------------ stack wiring
def _stack(L=3, d=16, E=4, k=2, c=8, cs=8, zero_o=False, zero_moe=False, T=10):
    aws = [AW(d, 4, 2, 4, 10 + i, zero_o=zero_o) for i in range(L)]
    mls = [lay(d, E, k, c, cs, 20 + i, zero=zero_moe) for i in range(L)]
    x = np.random.default_rng(5).standard_normal((T, d))
    return x, aws, mls


def test_all_regular_is_straight_line_prenorm_transformer():
    x, aws, mls = _stack()
    cache = ost.stack_forward(x, aws, mls, [ost.REGULAR] * 3, seq_len=5)
    # textbook pre-norm transformer: h += Attn(h); h += MoE(h)
    h = x.copy()
    for a, m in zip(aws, mls):
        h = h + oa.attention_block(h, a, 5)
        sh, ro, _ = om.moe_block(h, m)
        h = h + sh + ro
    np.testing.assert_allclose(cache[-1].o, h, rtol=0, atol=1e-12)


def test_hybrid_identity_and_accumulation():
    x, aws, mls = _stack(L=4)
    cache = ost.stack_forward(x, aws, mls, [ost.HYBRID] * 4, seq_len=5)
    prev = x
    for kk, c in enumerate(cache):
        if kk >= 1:
            # mlp-in_k = attn-in_k + routed-exp-out_{k-1}, bitwise (C-amb-12 order)
            assert np.array_equal(c.mlp_in, c.attn_in + cache[kk - 1].routed_out)
            assert np.array_equal(c.mlp_in, cache[kk - 1].o)          # outdated input, Eq. 8a
        else:
            assert np.array_equal(c.attn_in, x) and np.array_equal(c.mlp_in, x)   # C-amb-6
        # S:154 output accumulation in every mode
        np.testing.assert_allclose(c.o - prev, c.attn_out + c.shared_out + c.routed_out, rtol=0, atol=1e-12)
        prev = c.o
    # the hybrid genuinely differs from the regular stack (the connections are dropped)
    reg = ost.stack_forward(x, aws, mls, [ost.REGULAR] * 4, seq_len=5)
    assert not np.allclose(reg[-1].o, cache[-1].o)


@pytest.mark.parametrize("which", ["zero_o", "zero_moe"])
def test_hybrid_reduces_to_regular(which):
    # W_O = 0 (attn_out = 0) or all MoE weights = 0 (shared = routed = 0) make the
    # dropped connections carry zero, so Hybrid == Regular exactly.
    x, aws, mls = _stack(L=3, **{which: True})
    a = ost.stack_forward(x, aws, mls, [ost.HYBRID] * 3, seq_len=5)
    b = ost.stack_forward(x, aws, mls, [ost.REGULAR] * 3, seq_len=5)
    np.testing.assert_array_equal(a[-1].o, b[-1].o)


def test_mixed_modes_first_n():
    # partial conversion: first layer Regular == REGULAR prefix
    x, aws, mls = _stack(L=3)
    a = ost.stack_forward(x, aws, mls, [ost.REGULAR, ost.HYBRID, ost.HYBRID], seq_len=5)
    b = ost.stack_forward(x, aws, mls, [ost.REGULAR] * 3, seq_len=5)
    np.testing.assert_array_equal(a[0].o, b[0].o)
    with pytest.raises(ValueError):
        ost.stack_forward(x, aws, mls, [ost.REGULAR] * 2, seq_len=5)


def test_teacher_forcing_reproduces_free_run():
    x, aws, mls = _stack(L=3)
    free = ost.stack_forward(x, aws, mls, [ost.HYBRID] * 3, seq_len=5)
    forced = ost.stack_forward(x, aws, mls, [ost.HYBRID] * 3, seq_len=5,
                               teacher_inputs=[(c.attn_in, c.mlp_in) for c in free])
    for a, b in zip(free, forced):
        np.testing.assert_array_equal(a.o, b.o)


# ------------------------------------------------------------------ schedule replay
def test_schedule_golden_l2():
    with open(os.path.join(GOLDEN, "schedule_l2.json")) as f:
        gold = json.load(f)
    for name, want in gold["results"].items():
        end, exposed, t = osch.replay(name, 2, gold["durations"])
        assert (end, exposed) == (want["end"], want["exposed"]), name
        if name == "farskip":
            assert {k: list(v) for k, v in t.items()} == gold["farskip_intervals"]
    # FarSkip never loses to Regular; zero-comm makes them equal
    z = dict(gold["durations"], dispatch=0, combine=0)
    assert osch.replay("farskip", 2, z)[0] == osch.replay("regular", 2, z)[0]
    for L in (1, 3, 6):
        assert osch.replay("farskip", L)[0] <= osch.replay("regular", L)[0]


def test_schedule_eq9_bound():
    # Eq. 9: if T_dispatch + T_combine <= T_layer - (T_routed + T_gate) the interior
    # collectives are hidden; dispatch=core-sized and combine=shared-sized are feasible
    d = dict(osch.DEFAULT_DUR, dispatch=4, combine=4)
    end, exposed, t = osch.replay("farskip", 3, d)
    # only the last layer's combine may stay exposed
    assert exposed == 0
    d = dict(osch.DEFAULT_DUR, dispatch=6, combine=3)     # dispatch longer than core: 2 exposed per layer
    assert osch.replay("farskip", 2, d)[1] == 4
