"""Pins of the fp64 oracle's MoE functions against what the paper and the
mathematics fix (task rule ③). None of these re-types an oracle formula: each
check is a closed form, a special case, an invariant, a library routine used
as an independent definition, or a brute force."""
import itertools
import math

import numpy as np
import pytest

from oracle import moe as om
import synth


def rng(s=0):
    return np.random.default_rng(s)


# --------------------------------------------------------------- rmsnorm
def test_rmsnorm_constant_row_is_sign():
    x = np.full((2, 8), 3.0)
    x[1] = -0.25
    y = om.rmsnorm(x, np.ones(8))
    # closed form: c / sqrt(c^2 + eps)
    np.testing.assert_allclose(y[0], 3.0 / math.sqrt(9.0 + 1e-6), rtol=0, atol=1e-15)
    np.testing.assert_allclose(y[1], -0.25 / math.sqrt(0.0625 + 1e-6), rtol=0, atol=1e-15)


def test_rmsnorm_gamma_zero_and_unit_rms():
    x = rng().standard_normal((4, 64)) * 3
    assert np.all(om.rmsnorm(x, np.zeros(64)) == 0)
    y = om.rmsnorm(x, np.ones(64))
    ms = (x * x).mean(axis=1)
    # RMS(y) = sqrt(ms / (ms + eps))  (closed form)
    np.testing.assert_allclose(np.sqrt((y * y).mean(axis=1)), np.sqrt(ms / (ms + 1e-6)), rtol=1e-14)
    # scale invariance (x -> a x) up to the eps term; exact homogeneity in gamma
    g = rng(1).standard_normal(64)
    np.testing.assert_allclose(om.rmsnorm(x, 2 * g), 2 * om.rmsnorm(x, g), rtol=1e-15)


# --------------------------------------------------------------- softmax
def test_softmax_special_cases():
    np.testing.assert_allclose(om.softmax_rows(np.zeros((1, 3))), [[1 / 3] * 3], rtol=1e-15)
    s = om.softmax_rows(np.array([[1000.0, 0.0]]))
    assert abs(s[0, 0] - 1) < 1e-12 and s[0, 1] < 1e-300 + 1e-12
    l = rng().standard_normal((5, 7))
    s = om.softmax_rows(l)
    np.testing.assert_allclose(s.sum(1), 1, atol=1e-12)
    np.testing.assert_allclose(om.softmax_rows(l + 17.5), s, rtol=1e-13)
    # two-class softmax is the logistic function
    a = rng(2).standard_normal(9)
    two = om.softmax_rows(np.stack([a, np.zeros_like(a)], 1))
    np.testing.assert_allclose(two[:, 0], 1 / (1 + np.exp(-a)), rtol=1e-14)


# --------------------------------------------------------------- SiLU / SwiGLU
def test_silu_values():
    assert om.silu(np.array(0.0)) == 0
    # sigma(1) = 0.7310585786300049 (logistic function table value)
    assert abs(om.silu(np.array(1.0)) - 0.7310585786300049) < 1e-15
    assert abs(om.silu(np.array(-1.0)) - (-1 + 0.7310585786300049)) < 1e-15  # silu(-z) = silu(z) - z
    assert abs(om.silu(np.array(40.0)) - 40.0) < 1e-12


def test_swiglu_examples():
    z = np.zeros((3, 4))
    assert np.all(om.swiglu(rng().standard_normal((2, 4)), np.zeros((5, 4)), np.zeros((5, 4)), np.zeros((4, 5))) == 0)
    # d=c=1, A=[[1]], W1=[[2]], W2=[[0]], W3=[[1]] -> g(0)=0 -> 0
    assert om.swiglu(np.array([[1.0]]), np.array([[2.0]]), np.array([[0.0]]), np.array([[1.0]]))[0, 0] == 0
    # d=c=1, a=1, W1=2, W2=1, W3=3: U=2, G=silu(1)=sigma(1), out = 2*sigma(1)*3
    v = om.swiglu(np.array([[1.0]]), np.array([[2.0]]), np.array([[1.0]]), np.array([[3.0]]))[0, 0]
    assert abs(v - 6 * 0.7310585786300049) < 1e-14
    # the gate branch is W2 (C-amb-4): swapping W1/W2 changes the result
    a = rng(3).standard_normal((2, 4)); w1 = rng(4).standard_normal((5, 4)); w2 = rng(5).standard_normal((5, 4))
    w3 = rng(6).standard_normal((4, 5))
    assert not np.allclose(om.swiglu(a, w1, w2, w3), om.swiglu(a, w2, w1, w3))
    # linear in W1 and in W3
    np.testing.assert_allclose(om.swiglu(a, 3 * w1, w2, w3), 3 * om.swiglu(a, w1, w2, w3), rtol=1e-13)
    np.testing.assert_allclose(om.swiglu(a, w1, w2, -2 * w3), -2 * om.swiglu(a, w1, w2, w3), rtol=1e-13)
    # per-row independence and c-additivity (splitting c into halves sums, cf. Eq. 1-2)
    full = om.swiglu(a, w1, w2, w3)
    h1 = om.swiglu(a, w1[:2], w2[:2], w3[:, :2]) + om.swiglu(a, w1[2:], w2[2:], w3[:, 2:])
    np.testing.assert_allclose(full, h1, rtol=1e-13, atol=1e-15)


# --------------------------------------------------------------- router
def test_route_examples():
    # dense limit: top_k = E -> weights are the full softmax row
    xn = rng().standard_normal((6, 8)); wr = rng(1).standard_normal((4, 8))
    r = om.route(xn, wr, 4)
    assert np.all(r.idx == np.arange(4))
    np.testing.assert_allclose(r.gates, om.softmax_rows(xn @ wr.T), rtol=1e-14)
    assert np.all(np.isinf(r.gap))
    # score row [10,0,0,0], top-1 -> expert 0 with weight 1
    r = om.route(np.array([[1.0]]), np.array([[10.0], [0.0], [0.0], [0.0]]), 1)
    assert r.idx[0, 0] == 0 and r.gates[0, 0] == 1.0
    # equal scores, top-2 -> {0,1}, [0.5, 0.5]
    r = om.route(np.array([[1.0]]), np.ones((4, 1)), 2)
    assert list(r.idx[0]) == [0, 1] and list(r.gates[0]) == [0.5, 0.5]
    # tie at the boundary resolves to the lower index, wherever it sits
    r = om.route(np.array([[1.0]]), np.array([[0.0], [3.0], [1.0], [3.0], [1.0]]), 3)
    assert list(r.idx[0]) == [1, 2, 3]
    with pytest.raises(ValueError):
        om.route(xn, wr, 5)


def test_route_brute_force_and_invariants():
    g = rng(7)
    for E, k in [(4, 1), (5, 2), (6, 3), (8, 2)]:
        xn = g.standard_normal((20, 6)); wr = g.standard_normal((E, 6))
        r = om.route(xn, wr, k)
        l = xn @ wr.T
        for t in range(20):
            # brute force over all k-subsets: the chosen set maximises the sum of logits
            best = max(itertools.combinations(range(E), k), key=lambda S: (sum(l[t, list(S)]), [-i for i in S]))
            assert tuple(r.idx[t]) == tuple(sorted(best))
            sel = r.idx[t]
            unsel = [e for e in range(E) if e not in sel]
            # gates: softmax restricted to the selected logits (closed form identity)
            ex = np.exp(l[t, sel] - l[t, sel].max())
            np.testing.assert_allclose(r.gates[t], ex / ex.sum(), rtol=1e-13)
            assert np.all(r.gates[t] > 0) and abs(r.gates[t].sum() - 1) < 1e-12
            assert len(set(sel)) == k and np.all(np.diff(sel) > 0)
            if unsel:
                assert abs(r.gap[t] - (l[t, sel].min() - l[t, unsel].max())) < 1e-12


# --------------------------------------------------------------- permutation
def test_permutation_maps_vs_stable_sort():
    g = rng(11)
    for T, E, k in [(1, 4, 2), (16, 8, 2), (37, 16, 3), (64, 4, 4), (50, 64, 6)]:
        idx = np.stack([np.sort(g.choice(E, k, replace=False)) for _ in range(T)])
        m = om.permutation_maps(idx, E)
        assert m.counts.sum() == T * k                                  # BJ: counts sum to N*k
        np.testing.assert_array_equal(m.counts, np.bincount(idx.reshape(-1), minlength=E))
        assert sorted(m.pos.reshape(-1)) == list(range(T * k))           # bijection
        t_of = np.repeat(np.arange(T), k)
        order = np.argsort((idx.reshape(-1) * T + t_of), kind="stable")  # library stable sort
        np.testing.assert_array_equal(m.src_row, order // k)
        for t in range(T):
            for j in range(k):
                p = m.pos[t, j]
                assert m.src_row[p] == t
                e = idx[t, j]
                assert m.offsets[e] <= p < m.offsets[e + 1]


# --------------------------------------------------------------- dispatch / combine
def _layer(T_unused, d, E, k, c, cs, seed=0):
    g = rng(seed)
    w = lambda *s: g.standard_normal(s) / math.sqrt(s[-1])  # noqa: E731
    return om.EpLayer(1 + 0.1 * g.standard_normal(d), w(E, d), w(E, c, d), w(E, c, d), w(E, d, c),
                      w(cs, d) if cs else None, w(cs, d) if cs else None, w(d, cs) if cs else None, k)


def test_dispatch_forced_example():
    # T=2, E=4, top_1, n_ranks=2, assignments [0,3] -> rank0 {t0}, rank1 {t1}
    xn = np.array([[1.0, 2.0], [3.0, 4.0]])
    idx = np.array([[0], [3]])
    recv, rc, dst_rank, dst_row, cnt = om.dispatch_sim([xn[:2]], [idx], 4, 1)
    assert recv[0].shape == (2, 2)
    # two ranks, each holding one of the tokens as its own
    recv, rc, dst_rank, dst_row, cnt = om.dispatch_sim([xn, xn], [idx, idx], 4, 2)
    np.testing.assert_array_equal(recv[0], [xn[0], xn[0]])    # token0 from both sources
    np.testing.assert_array_equal(recv[1], [xn[1], xn[1]])
    assert list(rc[0]) == [2, 0] and list(rc[1]) == [0, 2]
    with pytest.raises(ValueError):
        om.dispatch_sim([xn] * 3, [idx] * 3, 4, 3)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_ep_invariance(P):
    # random T=16, E=8, top-2; the routed output is identical across n_ranks
    lay = _layer(16, 12, 8, 2, 10, 6, seed=3)
    X = rng(5).standard_normal((16 * P, 12))
    ref = om.moe_block(X, lay)
    outs = om.moe_block_ep([X[s * 16:(s + 1) * 16] for s in range(P)], lay, P)
    routed = np.concatenate([o[1] for o in outs])
    shared = np.concatenate([o[0] for o in outs])
    np.testing.assert_allclose(routed, ref[1], rtol=0, atol=1e-12)
    np.testing.assert_allclose(shared, ref[0], rtol=0, atol=1e-12)


@pytest.mark.parametrize("P", [1, 2, 4])
def test_allreduce_variant_equals_dense_and_partials_are_disjoint(P):
    """P:215-217 inference variant: the all-reduced sum of the per-rank local-expert
    partials is the dense brute-force MoE output (every token through every expert,
    masked by its gates); each partial only holds its own experts' contributions
    (zeroing every other rank's experts leaves it unchanged)."""
    lay = _layer(12, 16, 8, 3, 10, 6, seed=7)
    x = rng(8).standard_normal((12, 16))
    sh, ro, r, parts = om.moe_block_allreduce(x, lay, P)
    sh2, ro2, r2 = om.moe_block_dense(x, lay)
    np.testing.assert_allclose(ro, ro2, rtol=0, atol=1e-12 * max(1, np.abs(ro2).max()))
    np.testing.assert_allclose(sh, sh2, rtol=0, atol=0)
    e_loc = 8 // P
    for p in range(P):
        lay_p = om.EpLayer(lay.gamma, lay.w_router, lay.w1.copy(), lay.w2.copy(), lay.w3.copy(), lay.ws1, lay.ws2,
                           lay.ws3, top_k=lay.top_k)
        mask = np.ones(8, bool)
        mask[p * e_loc:(p + 1) * e_loc] = False
        lay_p.w3[mask] = 0.0                    # other ranks' experts contribute exactly 0
        _, ro_p, _ = om.moe_block(x, lay_p, router=r)
        np.testing.assert_allclose(parts[p], ro_p, rtol=0, atol=1e-12 * max(1, np.abs(ro_p).max()))
    with pytest.raises(ValueError):
        om.moe_block_allreduce(x, lay, 3)


def test_moe_block_equals_dense_brute_force():
    for (T, d, E, k, c, cs) in [(32, 64, 4, 2, 128, 0), (40, 16, 8, 3, 24, 32), (9, 8, 6, 6, 4, 0), (7, 8, 5, 1, 4, 4)]:
        lay = _layer(T, d, E, k, c, cs, seed=T)
        x = rng(T + 1).standard_normal((T, d))
        sh, ro, r = om.moe_block(x, lay)
        sh2, ro2, r2 = om.moe_block_dense(x, lay)
        np.testing.assert_allclose(ro, ro2, rtol=0, atol=1e-12 * max(1, np.abs(ro2).max()))
        np.testing.assert_allclose(sh, sh2, rtol=0, atol=0)


def test_moe_zero_cases():
    lay = _layer(8, 16, 4, 2, 8, 0, seed=1)
    x = rng(2).standard_normal((8, 16))
    sh, ro, _ = om.moe_block(x, lay)
    assert np.all(sh == 0)
    lay.w1[:] = 0; lay.w2[:] = 0; lay.w3[:] = 0
    sh, ro, _ = om.moe_block(x, lay)
    assert np.all(ro == 0)


def test_moe_single_expert_top1_is_dense_mlp():
    # E = k = 1: MoE(A) = G(A)_1 MLP^1(A) with G = 1 -> the plain gated MLP of P:73-76
    lay = _layer(6, 8, 1, 1, 12, 0, seed=9)
    x = rng(3).standard_normal((6, 8))
    _, ro, r = om.moe_block(x, lay)
    assert np.all(r.gates == 1.0)
    np.testing.assert_allclose(ro, om.swiglu(om.rmsnorm(x, lay.gamma), lay.w1[0], lay.w2[0], lay.w3[0]), rtol=1e-14)


def test_near_tie_adoption_rule():
    lay = _layer(8, 8, 4, 2, 8, 0, seed=4)
    x = rng(8).standard_normal((8, 8))
    r0 = om.route(om.rmsnorm(x, lay.gamma), lay.w_router, 2)
    # a 'GPU' answer that differs from the oracle only on excluded tokens is adopted
    r, excl = om.adopt_router(lay, x, r0.idx, margin=10.0)   # every token excluded
    assert excl.all()
    np.testing.assert_array_equal(r.idx, r0.idx)
    r, excl = om.adopt_router(lay, x, r0.idx, margin=0.0)
    assert not excl.any()


def test_synth_bf16_roundtrip_and_layer():
    # bf16 spacing at 1 is 2^-7: 1+2^-7 exact; 1+2^-8 and 1+3*2^-8 are ties -> even mantissa
    a = np.array([1.0, 1.0078125, 1.00390625, 1.01171875, -3.5, 1e-3], np.float32)
    b = synth.f32_to_bf16_bits(a)
    back = synth.bf16_bits_to_f32(b)
    np.testing.assert_array_equal(back[:5], np.array([1.0, 1.0078125, 1.0, 1.015625, -3.5], np.float32))
    assert abs(back[5] - 1e-3) / 1e-3 < 2 ** -8
    w = synth.moe_weights(synth.CONFIGS["tiny"], seed=0)
    lay = om.layer_from_synth(w, 2)
    assert lay.w1.shape == (4, 128, 64) and lay.w3.shape == (4, 64, 128)
    np.testing.assert_array_equal(lay.w1[1], synth.bf16_bits_to_f64(w.w1[1]))
    # experts regenerate identically when drawn per rank slice
    w2 = synth.moe_weights(synth.CONFIGS["tiny"], seed=0, e0=2, e_loc=2)
    np.testing.assert_array_equal(w2.w3, w.w3[2:4])


# ----------------------------------------------------------------------------- FP8 dispatch payload (NEXT-4)
def _e4m3_table():
    """All finite OCP E4M3 values decoded from their bit patterns (the format's
    definition: bias 7, 3 mantissa bits, exponent field 0 = subnormal, S.1111.111 = NaN)."""
    vals = []
    for code in range(256):
        sgn = -1.0 if code & 0x80 else 1.0
        e, m = (code >> 3) & 0xF, code & 0x7
        if e == 0xF and m == 0x7:
            continue                                   # NaN
        v = m * 2.0 ** -9 if e == 0 else (1 + m / 8.0) * 2.0 ** (e - 7)
        vals.append(sgn * v)
    return np.unique(np.array(vals))


def test_e4m3_rne_against_the_format_table():
    table = _e4m3_table()
    assert table.max() == 448.0 and table.min() == -448.0 and len(table) == 253   # +0/-0 merge
    np.testing.assert_array_equal(om.e4m3_rne(table), table)           # representable -> itself
    pos = table[table >= 0]
    mids = (pos[:-1] + pos[1:]) / 2                                      # exact ties
    lo_code_even = np.array([int(round(v / (2.0 ** max(np.floor(np.log2(v)) - 3, -9)))) % 2 == 0
                             if v > 0 else True for v in pos[:-1]])
    want = np.where(lo_code_even, pos[:-1], pos[1:])                     # ties to the even mantissa
    np.testing.assert_array_equal(om.e4m3_rne(mids), want)
    np.testing.assert_array_equal(om.e4m3_rne(-mids), -want)
    # brute force nearest on random values (no ties): the table's closest element
    v = rng(3).uniform(-460, 460, 2000) * rng(4).choice([1, 1e-2, 1e-4], 2000)
    near = table[np.abs(v[:, None] - table[None, :]).argmin(axis=1)]
    np.testing.assert_array_equal(om.e4m3_rne(v), np.clip(near, -448, 448))
    assert om.e4m3_rne(np.array([1e6, -1e6])).tolist() == [448.0, -448.0]   # satfinite


def test_fp8_payload_block_scaling():
    x = om.bf16_rne(rng(6).standard_normal((5, 256)).astype(np.float32))
    x[2, :128] = 0.0                                                    # empty block: scale 1, exact zeros
    xh = om.fp8_dispatch_payload(x)
    assert np.all(xh[2, :128] == 0)
    for t in range(5):
        for b in range(2):
            blk, hb = x[t, 128 * b:128 * (b + 1)], xh[t, 128 * b:128 * (b + 1)]
            if np.abs(blk).max() == 0:
                continue
            i = np.abs(blk).argmax()
            assert abs(hb[i] - blk[i]) <= 2 ** -8 * abs(blk[i])          # amax -> +-448 exactly, then bf16
            big = np.abs(blk) >= np.abs(blk).max() * 2 ** -5             # normal-range e4m3 codes
            rel = np.abs(hb[big] - blk[big]) / np.abs(blk[big])
            assert rel.max() <= 2 ** -4 + 2 ** -8                        # half an e4m3 ulp (+ bf16)


def test_fp8_dispatch_block_matches_exact_block_within_fp8_error():
    lay = _layer(16, 256, 8, 2, 64, 32, seed=2)
    xs = [rng(10 + s).standard_normal((16, 256)) for s in range(2)]
    exact = om.moe_block_ep(xs, lay, 2)
    q = om.moe_block_ep_fp8(xs, lay, 2)
    for (sh0, ro0, r0), (sh1, ro1, r1) in zip(exact, q):
        np.testing.assert_array_equal(r0.idx, r1.idx)
        np.testing.assert_array_equal(sh0, sh1)                          # shared expert: local, unquantised
        err = np.linalg.norm(ro1 - ro0) / np.linalg.norm(ro0)
        assert 1e-3 < err < 8e-2                                         # FP8-level, not exact, not broken


def _bf16_brute_nearest_even(x32):
    """Nearest bf16 by brute force: the two bf16 neighbours of each fp32 value (bit
    truncation and the next bf16 away from zero), the closer one in fp64, exact ties
    to the even bf16 mantissa (IEEE round-to-nearest-even)."""
    u = np.asarray(x32, np.float32).view(np.uint32)
    lo = (u & 0xFFFF0000).astype(np.uint32)
    hi = (lo + 0x10000).astype(np.uint32)
    f = lambda b: b.view(np.float32).astype(np.float64)  # noqa: E731
    x, a, b = np.asarray(x32, np.float32).astype(np.float64), f(lo), f(hi)
    da, db = np.abs(x - a), np.abs(x - b)
    even_lo = ((lo >> 16) & 1) == 0
    pick_lo = (da < db) | ((da == db) & even_lo)
    return np.where(pick_lo, a, b)


def test_bf16_rne_exact_ties_and_brute_force():
    """bf16_rne (the kernels' cvt.rn.bf16.f32) against the format: exact halfway
    cases go to the even mantissa, and random values to the nearest bf16."""
    ulp = 2.0 ** -7                                                   # bf16 spacing in [1, 2)
    ties = np.array([1 + ulp / 2, 1 + 3 * ulp / 2, 2 - ulp / 2, 1.5 + ulp / 2], np.float32)
    want = [1.0, 1 + 2 * ulp, 2.0, 1.5]                               # halfway -> even mantissa
    got = om.bf16_rne(ties)
    assert got.tolist() == want
    np.testing.assert_array_equal(om.bf16_rne(-ties), -got)            # sign symmetric
    assert om.bf16_rne(np.float32(1 + ulp / 2 + 2 ** -20)) == 1 + ulp  # just above the tie: up
    v = (rng(9).standard_normal(20000) * np.exp(rng(10).uniform(-30, 30, 20000))).astype(np.float32)
    v[:200] = ((v[:200].view(np.uint32) & 0xFFFF0000) | 0x8000).view(np.float32)   # 200 exact ties
    np.testing.assert_array_equal(om.bf16_rne(v), _bf16_brute_nearest_even(v))
