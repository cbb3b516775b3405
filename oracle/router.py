"""O2-O6: exact router logits, top-k, gate weights, Eq. 2 scores, T1/T2 decision.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: the gating function is "a linear layer followed by a Top-k operation"
(Sec. 2.1, Eq. 1).  Selected experts are ranked by ||G(x)_e||,
normalised, and scored by Eq. 2:
        s_{e_0} = 0,   s_{e_i} = sum_{j<i} ||G(x)_{e_j}||   (i > 0)
An expert is High precision if s <= T1, the first expert always High
(P:423), a second threshold T2 bypasses (skips) the least important;
Mixtral uses T1 = 0.6, T2 = 0.9.

Readings (R1-R3, R9): softmax over the selected top-k logits;
ties broken towards the lower expert index; High s<=T1, Low T1<s<=T2,
Skip s>T2; router logits computed EXACTLY (fp16 x fp16 products summed as
integers on a 2^-48 grid) so that the decision is a deterministic function of
the fp16 inputs.
"""
from __future__ import annotations

import math
from functools import lru_cache
from decimal import Decimal, getcontext

import numpy as np

HIGH, LOW, SKIP = 0, 1, 2
PREC_NAMES = {HIGH: "High", LOW: "Low", SKIP: "Skip"}
LOGIT_SHIFT = 48          # L = logit * 2^48 is an integer for fp16 x fp16


def fp16_parts(v16: np.ndarray):
    """(sign*significand, exponent) of fp16 values: v = m * 2^e exactly."""
    bits = np.asarray(v16, dtype=np.float16).view(np.uint16).astype(np.int64)
    sign = np.where(bits >> 15, -1, 1)
    ex = (bits >> 10) & 0x1F
    man = bits & 0x3FF
    if np.any(ex == 0x1F):
        raise ValueError("inf/nan in router input")
    m = np.where(ex == 0, man, man + 1024) * sign
    e = np.where(ex == 0, -24, ex - 25)
    return m, e


def exact_logits(x16: np.ndarray, wg16: np.ndarray):
    """O2: L[b][e] = sum_h W[e,h]*x[b,h] * 2^48 as exact Python ints.

    x16 [B,H] fp16, wg16 [E,H] fp16.  Every fp16 is m*2^e with e >= -24, so
    each product is an integer multiple of 2^-48 and the sum is exact.
    """
    xm, xe = fp16_parts(x16)
    wm, we = fp16_parts(wg16)
    B, H = xm.shape
    E = wm.shape[0]
    out = []
    for b in range(B):
        row = []
        for e in range(E):
            acc = 0
            for h in range(H):
                p = int(wm[e, h]) * int(xm[b, h])
                if p:
                    acc += p << int(we[e, h] + xe[b, h] + LOGIT_SHIFT)
            row.append(acc)
        out.append(row)
    return out


def top_k(L_row, k: int):
    """O3: experts sorted by (L descending, index ascending); first k."""
    order = sorted(range(len(L_row)), key=lambda e: (-L_row[e], e))
    return order[:k]


def gate_weights(L_row, sel):
    """O4: softmax over the selected logits only (reading R1), fp64."""
    l = [math.ldexp(float(L_row[e]), -LOGIT_SHIFT) for e in sel]
    ex = [math.exp(v - l[0]) for v in l]
    tot = sum(ex)
    return [v / tot for v in ex]


def scores(g):
    """O5, Eq. 2: s_0 = 0, s_i = sum_{j<i} g_j."""
    s = [0.0]
    for i in range(1, len(g)):
        s.append(s[-1] + g[i - 1])
    return s


def classify(s, t1: float, t2: float):
    """O6: rank 0 High; High s<=T1, Low T1<s<=T2, Skip s>T2."""
    if t1 > t2:
        raise ValueError("t1 > t2")
    out = []
    for i, v in enumerate(s):
        if i == 0 or v <= t1:
            out.append(HIGH)
        elif v <= t2:
            out.append(LOW)
        else:
            out.append(SKIP)
    return out


@lru_cache(maxsize=64)
def theta(t: float):
    """Integer gap threshold of T for k=2: floor(ln(T/(1-T)) * 2^48).

    For k=2, s_1 = g_0 = 1/(1+exp(-(l_0-l_1))) is monotone in the gap, so
        s_1 <= T   <=>   L_0 - L_1 <= floor(ln(T/(1-T)) * 2^48)
    with L the exact integer logits.  T is taken as its exact binary value.
    Returns None for T >= 1 (always true) and a very negative int for T <= 0.
    """
    if t >= 1.0:
        return None
    if t <= 0.0:
        return -(1 << 200)
    getcontext().prec = 80
    T = Decimal(t)
    v = (T / (1 - T)).ln() * (Decimal(2) ** LOGIT_SHIFT)
    return int(v.to_integral_value(rounding="ROUND_FLOOR"))


def classify_k2_exact(L0: int, L1: int, t1: float, t2: float):
    """O6 for k=2 as the exact integer gap test (same result as classify())."""
    if t1 > t2:
        raise ValueError("t1 > t2")
    G = L0 - L1
    th1, th2 = theta(t1), theta(t2)
    if th1 is None or G <= th1:
        return [HIGH, HIGH]
    if th2 is None or G <= th2:
        return [HIGH, LOW]
    return [HIGH, SKIP]


class Route:
    """Routing result of one token: experts in rank order, gates, decisions."""

    __slots__ = ("experts", "gates", "decisions", "logits", "degenerate")

    def __init__(self, experts, gates, decisions, logits, degenerate=False):
        self.experts = experts
        self.gates = gates
        self.decisions = decisions
        self.logits = logits
        self.degenerate = degenerate

    def __repr__(self):
        d = [PREC_NAMES[v] for v in self.decisions]
        return f"Route(experts={self.experts}, gates={self.gates}, dec={d})"


MARGIN = 1e-12


def route_token(L_row, k: int, t1: float, t2: float) -> Route:
    """O3-O6 for one token from its exact logits."""
    sel = top_k(L_row, k)
    g = gate_weights(L_row, sel)
    if k == 2:
        dec = classify_k2_exact(L_row[sel[0]], L_row[sel[1]], t1, t2)
        degenerate = False
    else:
        s = scores(g)
        dec = classify(s, t1, t2)
        degenerate = any(abs(v - t) <= MARGIN for v in s[1:] for t in (t1, t2))
    return Route(sel, g, dec, [L_row[e] for e in sel], degenerate)


def route(x16: np.ndarray, wg16: np.ndarray, k: int, t1: float, t2: float):
    """O2-O6 for every token of x16 [B,H]: list of Route."""
    L = exact_logits(x16, wg16)
    return [route_token(row, k, t1, t2) for row in L]
