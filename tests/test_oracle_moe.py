"""Pins for oracle/moe.py (O7, O8 SwiGLU + Eq. 1, O11 EP).

Pins: T1=1 reduces the layer to the textbook dense top-k MoE (written
independently with einsum); T1=T2=0 gives g0*E0(x); x=0 and W2=0 give 0
(S:463-465); brute force over all experts on the tiny config; the EP sum of
per-rank outputs equals the 1-rank output.
"""
import numpy as np
import pytest

import synthgen
from oracle import formats as fm
from oracle import moe
from oracle import router as rt

SH = synthgen.TINY


def _store(hi=fm.F16, lo=fm.Q4, shape=SH):
    cache = {}

    def blob(layer, e, enc):
        if (layer, e, enc) not in cache:
            w1, w3, w2 = synthgen.expert_weights(shape, layer, e)
            cache[(layer, e, enc)] = fm.quantize_blob(enc, w1, w3, w2)
        return cache[(layer, e, enc)]
    return moe.ExpertStore(blob, shape.hidden, shape.ffn)


@pytest.fixture(scope="module")
def store():
    return _store()


def _x(t=0, layer=0, batch=4):
    return synthgen.hidden_states(SH, t, layer, batch=batch)


def test_t1_one_equals_dense_topk_moe(store):
    """T1 = 1: every selection High (fp16) -> the textbook top-k MoE layer."""
    x = _x(batch=6)
    wg = synthgen.router_weights(SH, 0)
    y, routes = moe.moe_layer(x, wg, store, 0, 2, 1.0, 1.0, fm.F16, fm.Q4)
    experts = [store.get(0, e, fm.F16) for e in range(SH.n_experts)]
    ref = moe.dense_topk_moe(x, wg, experts, 2)
    assert all(d == rt.HIGH for r in routes for d in r.decisions)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


def test_t_zero_gives_top1_only(store):
    """T1 = T2 = 0: rank 1 is always skipped -> y = g0 E_{e0}(x), no renormalisation."""
    x = _x(batch=4)
    wg = synthgen.router_weights(SH, 1)
    y, routes = moe.moe_layer(x, wg, store, 1, 2, 0.0, 0.0, fm.F16, fm.Q4)
    for b, r in enumerate(routes):
        w1, w3, w2 = store.get(1, r.experts[0], fm.F16)
        ref = r.gates[0] * moe.expert_ffn(w1, w3, w2, x[b].astype(np.float64))
        assert r.gates[0] < 1.0
        np.testing.assert_allclose(y[b], ref, rtol=1e-13, atol=1e-14)


def test_zero_input_and_zero_w2():
    """x = 0 -> 0 (silu(0) = 0); W2 = 0 -> 0."""
    st = _store()
    wg = synthgen.router_weights(SH, 0)
    y, _ = moe.moe_layer(np.zeros((2, SH.hidden), np.float16), wg, st, 0, 2, 0.6, 0.9,
                         fm.F16, fm.Q4)
    assert np.all(y == 0)
    w1, w3, _ = synthgen.expert_weights(SH, 0, 0)
    z = np.zeros((SH.hidden, SH.ffn), np.float16)
    blob = fm.quantize_blob(fm.Q4, w1, w3, z)
    W1, W3, W2 = fm.decode_blob(fm.Q4, blob, SH.hidden, SH.ffn)
    assert np.all(moe.expert_ffn(W1, W3, W2, _x()[0].astype(np.float64)) == 0)


def test_brute_force_all_experts(store):
    """Compute all E experts in both encodings, pick by exact sorting of Fraction
    logits and by thresholds on fp64 prefix sums; compare element-wise."""
    from fractions import Fraction
    x = _x(t=3, batch=8)
    wg = synthgen.router_weights(SH, 0)
    t1, t2 = 0.6, 0.9
    y, routes = moe.moe_layer(x, wg, store, 0, 2, t1, t2, fm.F16, fm.Q4)
    xf = x.astype(np.float64)
    outs = {(e, enc): moe.expert_ffn(*store.get(0, e, enc), xf.T).T
            for e in range(SH.n_experts) for enc in (fm.F16, fm.Q4)}
    for b in range(x.shape[0]):
        logits = [sum(Fraction(float(wg[e, h])) * Fraction(float(x[b, h]))
                      for h in range(SH.hidden)) for e in range(SH.n_experts)]
        order = sorted(range(SH.n_experts), key=lambda e: (-logits[e], e))[:2]
        lf = np.array([float(logits[e]) for e in order])
        g = np.exp(lf - lf[0])
        g /= g.sum()
        s1 = g[0]
        ref = g[0] * outs[(order[0], fm.F16)][b]
        if s1 <= t1:
            ref = ref + g[1] * outs[(order[1], fm.F16)][b]
        elif s1 <= t2:
            ref = ref + g[1] * outs[(order[1], fm.Q4)][b]
        assert routes[b].experts == order
        np.testing.assert_allclose(y[b], ref, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ep_partition_sums_to_single_rank(store, world):
    x = _x(t=5, batch=5)
    wg = synthgen.router_weights(SH, 1)
    y1, r1 = moe.moe_layer(x, wg, store, 1, 2, 0.6, 0.9, fm.F16, fm.Q4)
    parts = []
    for rank in range(world):
        yr, rr = moe.moe_layer(x, wg, store, 1, 2, 0.6, 0.9, fm.F16, fm.Q4,
                               rank=rank, world=world)
        assert [r.decisions for r in rr] == [r.decisions for r in r1]
        parts.append(yr)
    np.testing.assert_allclose(np.sum(parts, axis=0), y1, rtol=1e-14, atol=1e-15)


def test_low_uses_quantised_version(store):
    """A Low decision is computed from the lo_enc blob, not the fp16 one."""
    x = _x(t=11, batch=16)
    wg = synthgen.router_weights(SH, 0)
    y, routes = moe.moe_layer(x, wg, store, 0, 2, 0.6, 0.9, fm.F16, fm.Q4)
    b = next(i for i, r in enumerate(routes) if r.decisions[1] == rt.LOW)
    r = routes[b]
    xf = x[b].astype(np.float64)
    want = (r.gates[0] * moe.expert_ffn(*store.get(0, r.experts[0], fm.F16), xf)
            + r.gates[1] * moe.expert_ffn(*store.get(0, r.experts[1], fm.Q4), xf))
    wrong = (r.gates[0] * moe.expert_ffn(*store.get(0, r.experts[0], fm.F16), xf)
             + r.gates[1] * moe.expert_ffn(*store.get(0, r.experts[1], fm.F16), xf))
    np.testing.assert_allclose(y[b], want, rtol=1e-13)
    assert np.abs(y[b] - wrong).max() > 1e-6


def test_silu_closed_form_values():
    """silu(z) = z / (1 + e^-z) = z * sigmoid(z) (reading R10, SwiGLU as in
    Mixtral/Phi).  Values worked from e = 2.718281828459045...:
    sigmoid(1) = 1/(1 + 0.36787944117144233) = 0.7310585786300049, so
    silu(1) = 0.7310585786300049 and silu(-1) = -sigmoid(-1) = -0.2689414213699951;
    silu(4) = 4/(1 + 0.01831563888873418) = 3.928055160151634,
    silu(-4) = -4 * 0.01798620996209156 = -0.07194483984836624.
    A slip such as z/(1 + e^z) gives silu(1) = 0.2689..., caught here; the
    identity silu(z) - silu(-z) = z and silu -> z (z >> 0), -> 0 (z << 0) too."""
    z = np.array([1.0, -1.0, 4.0, -4.0, 0.0])
    ref = np.array([0.7310585786300049, -0.2689414213699951, 3.928055160151634,
                    -0.07194483984836624, 0.0])
    assert np.allclose(moe.silu(z), ref, rtol=1e-15, atol=0)
    w = np.linspace(-30, 30, 601)
    assert np.allclose(moe.silu(w) - moe.silu(-w), w, rtol=0, atol=1e-12)
    assert abs(moe.silu(np.array([40.0]))[0] - 40.0) < 1e-12
    assert abs(moe.silu(np.array([-40.0]))[0]) < 1e-15


def test_dense_reference_activation_matches_silu_independently():
    """The dense top-k reference takes the logistic function from
    scipy.special.expit, not through silu(): the two agree to rounding, and the
    tanh form (1 + tanh(z/2))/2 agrees too away from its cancellation range."""
    from scipy.special import expit
    a = np.linspace(-20, 20, 4001)
    assert np.allclose(a * expit(a), moe.silu(a), rtol=1e-14, atol=0)
    b = np.linspace(-4, 20, 2401)
    assert np.allclose(b * 0.5 * (1.0 + np.tanh(0.5 * b)), moe.silu(b), rtol=1e-12, atol=0)


def test_served_encodings_resident_upgrade_rule():
    """R27 worked example: token 0 selects (e3 High, e5 Low), token 1 (e5 High,
    e3 Low), token 2 (e1 High, e3 Skip), token 3 (e6 High, e2 Low).
    Strict: Low -> lo.  Non-strict: e5's and e3's Low requests are served by hi
    (both touched High in this forward); e2's is not (never High); Skip stays."""
    R = rt.Route
    routes = [R([3, 5], [0.7, 0.3], [rt.HIGH, rt.LOW], None), R([5, 3], [0.6, 0.4], [rt.HIGH, rt.LOW], None),
              R([1, 3], [0.95, 0.05], [rt.HIGH, rt.SKIP], None), R([6, 2], [0.8, 0.2], [rt.HIGH, rt.LOW], None)]
    F, Q = fm.F16, fm.Q4
    assert moe.served_encodings_resident(routes, F, Q, strict=True) == \
        [[F, Q], [F, Q], [F, None], [F, Q]]
    assert moe.served_encodings_resident(routes, F, Q, strict=False) == \
        [[F, F], [F, F], [F, None], [F, Q]]
