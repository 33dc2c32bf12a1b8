"""Pins of the MoE-block backward oracle (oracle/moe_backward.py):
every analytic gradient against central finite differences of the forward oracle
(a definition-level check independent of the chain-rule derivation), plus closed
forms: SiLU' against its difference quotient, the RMSNorm Jacobian's scale
invariance, and zero gradients for unselected router logits."""
import numpy as np
import pytest

from oracle import moe as om
from oracle import moe_backward as ob


def _layer(d, E, k, c, cs, seed):
    g = np.random.default_rng(seed)
    lay = om.EpLayer(1 + 0.1 * g.standard_normal(d), g.standard_normal((E, d)) / np.sqrt(d),
                     g.standard_normal((E, c, d)) / np.sqrt(d), g.standard_normal((E, c, d)) / np.sqrt(d),
                     g.standard_normal((E, d, c)) / np.sqrt(c),
                     g.standard_normal((cs, d)) / np.sqrt(d) if cs else None,
                     g.standard_normal((cs, d)) / np.sqrt(d) if cs else None,
                     g.standard_normal((d, cs)) / np.sqrt(cs) if cs else None, top_k=k)
    return lay


def _loss(x, lay, G):
    sh, ro, r = om.moe_block(x, lay)
    return float(np.sum(G * (x + sh + ro))), r.idx


def _fd(f, arr, idx, h=1e-6):
    old = arr[idx]
    arr[idx] = old + h
    lp, ip = f()
    arr[idx] = old - h
    lm, im = f()
    arr[idx] = old
    return (lp - lm) / (2 * h), np.array_equal(ip, im)


def test_silu_grad_closed_form():
    z = np.linspace(-8, 8, 41)
    h = 1e-6
    np.testing.assert_allclose(ob.silu_grad(z), (om.silu(z + h) - om.silu(z - h)) / (2 * h), rtol=1e-7, atol=1e-9)
    assert ob.silu_grad(np.array([0.0]))[0] == 0.5


@pytest.mark.parametrize("cs", [0, 4])
def test_backward_matches_finite_differences(cs):
    d, E, k, c, T = 8, 4, 2, 6, 5
    lay = _layer(d, E, k, c, cs, seed=3 + cs)
    g = np.random.default_rng(11)
    x = g.standard_normal((T, d))
    G = g.standard_normal((T, d))
    grads = ob.moe_block_backward(x, lay, G)
    f = lambda: _loss(x, lay, G)
    checks = [("dx", x, grads.dx), ("dgamma", lay.gamma, grads.dgamma), ("dw_router", lay.w_router, grads.dw_router),
              ("dw1", lay.w1, grads.dw1), ("dw2", lay.w2, grads.dw2), ("dw3", lay.w3, grads.dw3)]
    if cs:
        checks += [("dws1", lay.ws1, grads.dws1), ("dws2", lay.ws2, grads.dws2), ("dws3", lay.ws3, grads.dws3)]
    for name, arr, ga in checks:
        assert ga.shape == arr.shape, name
        flat = list(np.ndindex(arr.shape))
        pick = [flat[i] for i in g.choice(len(flat), min(len(flat), 40), replace=False)]
        for ix in pick:
            num, same_sel = _fd(f, arr, ix)
            assert same_sel, "perturbation crossed a top-k boundary; choose another seed"
            assert abs(num - ga[ix]) <= 1e-6 * max(1.0, abs(num)), (name, ix, num, ga[ix])


def test_unselected_experts_get_no_weight_gradient():
    d, E, k, c, T = 8, 6, 2, 5, 3
    lay = _layer(d, E, k, c, 0, seed=9)
    x = np.random.default_rng(1).standard_normal((T, d))
    G = np.random.default_rng(2).standard_normal((T, d))
    grads = ob.moe_block_backward(x, lay, G)
    used = set(om.route(om.rmsnorm(x, lay.gamma), lay.w_router, k).idx.reshape(-1).tolist())
    for e in range(E):
        if e not in used:
            assert not grads.dw1[e].any() and not grads.dw2[e].any() and not grads.dw3[e].any()
            assert not grads.dw_router[e].any()


def test_zero_experts_give_the_identity_gradient():
    """With the MoE removed (zero experts, no shared), out = x and dL/dx = G exactly;
    the RMSNorm Jacobian term vanishes (dxn = 0)."""
    d, E, k, c, T = 8, 4, 2, 6, 4
    lay = _layer(d, E, k, c, 0, seed=5)
    lay.w1[:] = 0.0
    lay.w2[:] = 0.0
    lay.w3[:] = 0.0
    x = np.random.default_rng(6).standard_normal((T, d))
    G = np.random.default_rng(7).standard_normal((T, d))
    grads = ob.moe_block_backward(x, lay, G)
    np.testing.assert_array_equal(grads.dx, G)
    assert not grads.dgamma.any() and not grads.dw_router.any()
