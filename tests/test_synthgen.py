"""The seeded generator: deterministic, correctly scaled, and the stated recipe."""
import math

import numpy as np

import synthgen as sg


def test_deterministic_and_offsettable():
    k = sg.stream_key(1433, 2, 0, 3, 1)
    a = sg.fill_f16(k, 1000, 0.5)
    b = sg.fill_f16(k, 1000, 0.5)
    assert np.array_equal(a.view(np.uint16), b.view(np.uint16))
    c = sg.fill_f16(k, 400, 0.5, start=600)
    assert np.array_equal(a[600:].view(np.uint16), c.view(np.uint16))
    assert sg.stream_key(1433, 2, 0, 3, 1) != sg.stream_key(1433, 2, 0, 3, 2)


def test_moments_and_bounds():
    v = sg.fill_f16(sg.stream_key(7, 1), 400_000, 2.0).astype(np.float64)
    assert abs(v.mean()) < 0.02
    assert abs(v.std() - 2.0) < 0.01
    assert np.abs(v).max() <= 2.0 * 2.0 * math.sqrt(3.0) * 1.001    # Irwin-Hall(4): 2*sqrt(3) sigma


def test_recipe_scales():
    sh = sg.TINY
    wg = sg.router_weights(sh, 0).astype(np.float64)
    assert abs(wg.std() * math.sqrt(sh.hidden) - sh.sigma_router) < 0.05
    w1, w3, w2 = sg.expert_weights(sh, 1, 3)
    assert w1.shape == (sh.ffn, sh.hidden) and w2.shape == (sh.hidden, sh.ffn)
    assert abs(w2.astype(np.float64).std() * math.sqrt(sh.ffn) - 1) < 0.02


def test_correlated_states_cosine():
    sh = sg.MoEShape("t", 4, 8, 2, 4096, 512, 1.5)
    x = sg.correlated_states(sh, 3, 0.999, 0.5).astype(np.float64)
    for t in range(3):
        for l in range(3):
            a, b = x[t, l], x[t, l + 1]
            cos = a @ b / np.linalg.norm(a) / np.linalg.norm(b)
            assert abs(cos - 0.999) < 0.002
