"""Pins for oracle/router.py (O2 exact logits, O3 top-k, O4 gates, O5 Eq. 2,
O6 T1/T2 decision).  Pins: SPEC worked examples, a hand example,
Fraction brute force, an independent mpmath computation of the thresholds,
the s-formulation vs the integer gap test, and invariants."""
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import router as rt
from tests.conftest import GOLDEN
import synthgen


def _f16(a):
    return np.asarray(a, dtype=np.float16)


def test_fp16_parts_exact():
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.standard_normal(4000), rng.standard_normal(2000) * 1e-5,
                        [0.0, -0.0, 65504.0, 2 ** -24, -(2 ** -14)]]).astype(np.float16)
    m, e = rt.fp16_parts(v)
    for vi, mi, ei in zip(v, m, e):
        assert Fraction(float(vi)) == Fraction(int(mi)) * Fraction(2) ** int(ei)
        assert -24 <= ei <= 5


def test_exact_logits_equal_fraction_brute_force():
    rng = np.random.default_rng(1)
    x = _f16(rng.standard_normal((3, 64)))
    w = _f16(rng.standard_normal((5, 64)) * 0.1)
    L = rt.exact_logits(x, w)
    for b in range(3):
        for e in range(5):
            exact = sum(Fraction(float(w[e, h])) * Fraction(float(x[b, h])) for h in range(64))
            assert Fraction(L[b][e], 2 ** 48) == exact


def test_hand_example_tie_goes_to_lower_index():
    """x = [1,2], e0 = [0.5, 0.25], e1 = [1, 0]: L0 = L1 = 1.0."""
    x = _f16([[1.0, 2.0]])
    w = _f16([[0.5, 0.25], [1.0, 0.0]])
    L = rt.exact_logits(x, w)[0]
    assert L[0] == L[1] == 2 ** 48
    r = rt.route_token(L, 2, 0.6, 0.9)
    assert r.experts == [0, 1]
    assert r.gates == [0.5, 0.5]
    assert r.decisions == [rt.HIGH, rt.HIGH]     # gap 0 <= Theta(0.6)


def test_spec_compute_gate_examples():
    """unit-basis gates, x = [2, 1]."""
    x = _f16([[2.0, 1.0]])
    w = _f16([[1.0, 0.0], [0.0, 1.0]])
    r1 = rt.route(x, w, 1, 0.6, 0.9)[0]
    assert r1.experts == [0] and r1.gates == [1.0]
    r2 = rt.route(x, w, 2, 0.6, 0.9)[0]
    assert r2.experts == [0, 1]
    assert abs(r2.gates[0] - math.e / (math.e + 1)) < 1e-15
    assert round(r2.gates[0], 4) == 0.7311 and round(r2.gates[1], 4) == 0.2689
    # s_1 = 0.7311 in (0.6, 0.9] -> Low
    assert r2.decisions == [rt.HIGH, rt.LOW]
    # tie at 0 for experts 1 and 3, top_k 1 -> expert 1
    L = [-5, 0, -7, 0]
    assert rt.top_k(L, 1) == [1]


def test_spec_scores_examples():
    """S:124-126 (Eq. 2)."""
    assert rt.scores([1.0]) == [0.0]
    assert rt.scores([0.7, 0.3]) == [0.0, 0.7]
    s = rt.scores([0.4, 0.35, 0.25])
    assert s[0] == 0.0 and s[1] == 0.4 and abs(s[2] - 0.75) < 1e-15


def test_spec_classify_examples():
    """S:133-135 with T1 = 0.6, T2 = 0.9."""
    H, L, S = rt.HIGH, rt.LOW, rt.SKIP
    assert rt.classify([0, 0.7], 0.6, 0.9) == [H, L]
    assert rt.classify([0, 0.95], 0.6, 0.9) == [H, S]
    assert rt.classify([0, 0.5], 0.6, 0.9) == [H, H]
    with pytest.raises(ValueError):
        rt.classify([0, 0.5], 0.9, 0.6)


def test_theta_golden_and_independent_mpmath():
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 60
    with open(os.path.join(GOLDEN, "router_spec_examples.txt")) as f:
        rows = [l.split() for l in f if l.startswith("theta")]
    assert rows
    for _, t, want in rows:
        t = float(t)
        assert rt.theta(t) == int(want)
        T = mpmath.mpf(t)                        # exact binary value of the double
        v = mpmath.log(T / (1 - T)) * mpmath.mpf(2) ** 48
        assert mpmath.floor(v) == int(want)
    # T = 1 -> always High; T = 0 -> never <= (s_1 = g_0 >= 0.5 > 0)
    assert rt.theta(1.0) is None
    assert rt.classify_k2_exact(10 ** 30, 0, 1.0, 1.0) == [rt.HIGH, rt.HIGH]
    assert rt.classify_k2_exact(0, 0, 0.0, 0.0) == [rt.HIGH, rt.SKIP]


def test_gap_test_equals_s_formulation():
    """Integer gap test == classify(scores(softmax)) away from the boundary."""
    rnd = random.Random(5)
    for t1, t2 in ((0.6, 0.9), (0.55, 0.7), (0.8, 0.95), (0.5, 0.5)):
        th1, th2 = math.log(t1 / (1 - t1)), math.log(t2 / (1 - t2))
        n = 0
        while n < 20000:
            gap = abs(rnd.gauss(0, 2.0))
            if min(abs(gap - th1), abs(gap - th2)) < 1e-9:
                continue
            G = int(gap * 2 ** 48)
            L0, L1 = G, 0
            g = rt.gate_weights([L0, L1], [0, 1])
            assert rt.classify_k2_exact(L0, L1, t1, t2) == rt.classify(rt.scores(g), t1, t2)
            n += 1


def test_rank0_always_high_and_monotone_in_t1():
    """P:423 / P:436: rank 0 always High; raising T1 never demotes."""
    rnd = random.Random(9)
    for _ in range(2000):
        k = rnd.randint(1, 6)
        w = [rnd.random() for _ in range(k)]
        g = sorted([v / sum(w) for v in w], reverse=True)
        s = rt.scores(g)
        t2 = rnd.random()
        prev = None
        for t1 in sorted(rnd.random() * t2 for _ in range(5)):
            d = rt.classify(s, t1, t2)
            assert d[0] == rt.HIGH
            if prev is not None:
                assert all(a <= b for a, b in zip(d, prev))
            prev = d


def test_k2_half_high_closed_form():
    """with top-2, all top-1 experts (50% of selections) score 0 -> High."""
    rng = np.random.default_rng(2)
    x = _f16(rng.standard_normal((40, 32)))
    w = _f16(rng.standard_normal((8, 32)) * 0.3)
    for r in rt.route(x, w, 2, 0.0, 0.0):
        assert r.decisions[0] == rt.HIGH and r.decisions[1] == rt.SKIP


def test_workload_mix_matches_paper_split():
    """Workload recipe check (DESIGN.md Inputs): router sigma = 1.5 on E=8
    reproduces the paper's 67/30/3 High/Low/Skip split at T1=0.6, T2=0.9
     within sampling error."""
    shape = synthgen.TINY
    wg = synthgen.router_weights(shape, 0)
    counts = [0, 0, 0]
    n = 0
    for t in range(60):
        x = synthgen.hidden_states(shape, t, 0, batch=32)
        for r in rt.route(x, wg, 2, 0.6, 0.9):
            for d in r.decisions:
                counts[d] += 1
                n += 1
    mix = [c / n for c in counts]
    # 3840 selections: binomial sd ~ 0.8%; allow 4 sd and the one-layer router draw
    assert abs(mix[0] - 0.67) < 0.045 and abs(mix[1] - 0.30) < 0.045 and abs(mix[2] - 0.03) < 0.02, mix
