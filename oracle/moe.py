"""O7 served encoding, O8 SwiGLU experts + Eq. 1 weighted sum, O11 EP partition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 1 (Sec. 2.1):   y = sum_{i=1..K} G(x)_{e_i} E_{e_i}(x)
Experts are FFNs; we read them as SwiGLU, E(x) = W2 (silu(W1 x) * W3 x)
(R10, as in Mixtral / Phi-MoE).  A Low expert is computed from its
low-precision version ("load the low-precision version"), a Skip expert
contributes nothing and the remaining gates are NOT renormalised (R4).
Everything below is fp64 on the exactly decoded weights.
"""
from __future__ import annotations

import numpy as np
from scipy.special import expit

from .formats import decode_blob
from .router import HIGH, LOW, SKIP, route


def silu(z: np.ndarray) -> np.ndarray:
    """silu(z) = z / (1 + e^-z)."""
    with np.errstate(over="ignore"):
        return z / (1.0 + np.exp(-z))


def expert_ffn(w1: np.ndarray, w3: np.ndarray, w2: np.ndarray, x: np.ndarray) -> np.ndarray:
    """O8: E(x) = W2 (silu(W1 x) * (W3 x)), fp64.  x [H] -> [H]."""
    a = w1 @ x
    u = w3 @ x
    h = silu(a) * u
    return w2 @ h


def served_encoding_strict(decision: int, hi_enc: int, lo_enc: int):
    """O7 (strict / fully resident): High -> hi_enc, Low -> lo_enc, Skip -> None."""
    if decision == HIGH:
        return hi_enc
    if decision == LOW:
        return lo_enc
    return None


def served_encodings_resident(routes, hi_enc: int, lo_enc: int, strict: bool = True):
    """O7 for one fully resident forward over a batch of tokens -> served[b][i].

    strict (the benches' default): High -> hi_enc, Low -> lo_enc, Skip -> None.
    Non-strict (R27; SURVEY 8(d) C5 "allow_upgrade = 1, one stream
    per touched expert"; reading A6 "Low is served by High when allow_upgrade"):
    both versions are resident, and a Low selection of expert e is served by
    the hi_enc copy when some token of the SAME forward selected e as High --
    that expert's High weights are streamed anyway, so the Low request costs
    no extra bytes.  Otherwise Low -> lo_enc.
    """
    high = {e for r in routes for e, d in zip(r.experts, r.decisions) if d == HIGH}
    out = []
    for r in routes:
        row = []
        for e, d in zip(r.experts, r.decisions):
            if d == SKIP:
                row.append(None)
            elif d == HIGH or (not strict and e in high):
                row.append(hi_enc)
            else:
                row.append(lo_enc)
        out.append(row)
    return out


class ExpertStore:
    """Decoded fp64 experts, keyed (layer, expert, enc), from a blob provider."""

    def __init__(self, blob_fn, hidden: int, ffn: int):
        self.blob_fn = blob_fn          # (layer, expert, enc) -> uint8 blob
        self.hidden = hidden
        self.ffn = ffn
        self._cache = {}

    def get(self, layer: int, expert: int, enc: int):
        key = (layer, expert, enc)
        if key not in self._cache:
            self._cache[key] = decode_blob(enc, self.blob_fn(layer, expert, enc),
                                           self.hidden, self.ffn)
        return self._cache[key]


def owner(expert: int, world: int) -> int:
    """O11: expert-parallel owner rank, e mod R."""
    return expert % world


def tp_slice(w1: np.ndarray, w3: np.ndarray, w2: np.ndarray, tp_rank: int, tp_world: int):
    """TP-within-expert: rank r of R holds rows [r F/R, (r+1) F/R)
    of W1 and W3 and the same columns of W2.  SwiGLU acts row by row of F and
    W2 h sums over F, so E(x) = sum_r W2[:, s_r] (silu(W1[s_r] x) * W3[s_r] x)."""
    F = w1.shape[0]
    f0, f1 = tp_rank * F // tp_world, (tp_rank + 1) * F // tp_world
    return w1[f0:f1], w3[f0:f1], w2[:, f0:f1]


def ts_dispatch_plan(routes, world: int, capacity: int):
    """Token-sharded EP, dispatch side: a token's non-skipped
    selections go to the owners of their experts, owner(e) = e mod world;
    one ROW per (token, owner) holds the token's selections that owner has
    (rank order); the rows of an owner are in token order.  Returns pos[b][i]
    = dest * capacity + row of selection i's owner (-1 for Skip) and per
    destination the list of rows (token, [(expert, decision, gate), ...])."""
    pos = [[-1] * len(r.experts) for r in routes]
    sent = [[] for _ in range(world)]
    for b, r in enumerate(routes):
        rows = {}
        for i, (e, g, d) in enumerate(zip(r.experts, r.gates, r.decisions)):
            if d == SKIP:
                continue
            q = owner(e, world)
            if q not in rows:
                if len(sent[q]) >= capacity:
                    raise ValueError("token-sharded capacity exceeded")
                rows[q] = len(sent[q])
                sent[q].append((b, []))
            sent[q][rows[q]][1].append((e, d, g))
            pos[b][i] = q * capacity + rows[q]
    return pos, sent


def ts_owner_rows(x_rows: np.ndarray, records, store: ExpertStore, layer: int, hi_enc: int,
                  lo_enc: int) -> np.ndarray:
    """Token-sharded EP, owner side: each received row is the sum of the Eq. 1
    terms g * E_e(x) of its selections (the source's gates, strict encodings)."""
    out = np.zeros((len(records), x_rows.shape[1]), dtype=np.float64)
    for j, (_, sels) in enumerate(records):
        x = x_rows[j].astype(np.float64)
        for e, d, g in sels:
            w1, w3, w2 = store.get(layer, e, served_encoding_strict(d, hi_enc, lo_enc))
            out[j] += g * expert_ffn(w1, w3, w2, x)
    return out


def ts_combine(pos, returned: np.ndarray, H: int) -> np.ndarray:
    """Token-sharded EP, source side: y[b] = the sum of the token's returned
    rows, each owner's row once (returned[dest * capacity + row])."""
    y = np.zeros((len(pos), H), dtype=np.float64)
    for b, row in enumerate(pos):
        for p_ in dict.fromkeys(p for p in row if p >= 0):
            y[b] += returned[p_]
    return y


def moe_layer(x16: np.ndarray, wg16: np.ndarray, store: ExpertStore, layer: int,
              k: int, t1: float, t2: float, hi_enc: int, lo_enc: int,
              rank: int = 0, world: int = 1, served=None, tp_rank: int = 0, tp_world: int = 1):
    """One MoE layer for tokens x16 [B,H] (fp16): returns (y fp64 [B,H], routes).

    served[b][i], if given, overrides O7 with the encoding the cache state
    machine chose (O9); None there means Skip.  With world > 1 only the
    experts this rank owns are computed (O11): the layer output is the sum of
    the per-rank outputs.  With tp_world > 1 every expert is computed on this
    rank's slice of F (tp_slice): the layer output is again the sum over ranks.
    """
    routes = route(x16, wg16, k, t1, t2)
    B, H = x16.shape
    y = np.zeros((B, H), dtype=np.float64)
    for b, r in enumerate(routes):
        x = x16[b].astype(np.float64)
        for i, (e, g, d) in enumerate(zip(r.experts, r.gates, r.decisions)):
            if d == SKIP or owner(e, world) != rank:
                continue
            enc = served[b][i] if served is not None else served_encoding_strict(d, hi_enc, lo_enc)
            if enc is None:
                continue
            w1, w3, w2 = store.get(layer, e, enc)
            if tp_world > 1:
                w1, w3, w2 = tp_slice(w1, w3, w2, tp_rank, tp_world)
            y[b] += g * expert_ffn(w1, w3, w2, x)
    return y, routes


def dense_topk_moe(x16: np.ndarray, wg16: np.ndarray, experts_f64, k: int) -> np.ndarray:
    """Textbook top-k MoE, written independently of O3-O8 for the T1=1 pin.

    Computes ALL experts densely with einsum, softmax over all logits (fp64
    from float logits), keeps the top-k by a stable argsort, renormalises.
    experts_f64: list over experts of (W1, W3, W2) fp64.
    """
    x = x16.astype(np.float64)
    logits = x @ wg16.astype(np.float64).T                       # [B,E]
    W1 = np.stack([w[0] for w in experts_f64])                  # [E,F,H]
    W3 = np.stack([w[1] for w in experts_f64])
    W2 = np.stack([w[2] for w in experts_f64])                  # [E,H,F]
    a = np.einsum("efh,bh->bef", W1, x)
    u = np.einsum("efh,bh->bef", W3, x)
    # SwiGLU activation taken independently of silu() above: the logistic
    # function from scipy.special.expit, so a slip in silu() fails the pin
    h = a * expit(a) * u
    o = np.einsum("ehf,bef->beh", W2, h)                         # [B,E,H]
    p = np.exp(logits - logits.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    order = np.argsort(-logits, axis=1, kind="stable")[:, :k]
    mask = np.zeros_like(p)
    np.put_along_axis(mask, order, 1.0, axis=1)
    w = p * mask
    w /= w.sum(axis=1, keepdims=True)
    return np.einsum("be,beh->bh", w, o)


def algorithmic_bytes(routes, enc_bytes: dict, hi_enc: int, lo_enc: int,
                      n_experts: int, hidden: int, ffn: int, world: int = 1, rank: int = 0):
    """Realised algorithmic bytes of one layer (SURVEY.md 8(d) unit):
    served blob bytes of every computed expert + router weights + x + y + h."""
    total = 2 * n_experts * hidden
    for r in routes:
        total += 2 * hidden + 4 * hidden
        for e, d in zip(r.experts, r.decisions):
            if d == SKIP or owner(e, world) != rank:
                continue
            total += enc_bytes[hi_enc if d == HIGH else lo_enc] + 2 * 4 * ffn
    return total
