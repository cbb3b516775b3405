"""Eq. 3 weight calibration and the policy comparison of fig:cache-policy-verify
("weights ... calibrated by minimising the miss
penalty", P:1040 LRU/LFU/LHU/FLD vs the combined policy, normalised by Random).

CPU only: the library's own cache state machine (hbc_*, the code the offload
path runs) replays synthetic C4 decode traces -- Mixtral shapes (32 layers,
8 experts, top-2), gating inputs with layer cosine 0.999 and token locality
rho, pools at 25 % of the F16 expert bytes (cap_high 48,
cap_low 56), decisions from the routers of the seeded workload (fp64 logits;
a tool, not a parity check).  Miss penalty = bytes loaded on demand (High
miss: the F16 blob, Low miss: the Q4 blob).  Prints and writes a markdown
table: every weight vector in {0..3}^4 (grid over the simplex directions),
the Random policy (all-zero weights, R29), and the corners.

    python tools/eq3_calibrate.py [--seqs 6] [--tokens 48] [--rho 0.5] [--p 0] [--out profiles/...]
"""
import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthgen as sg  # noqa: E402
from paper_2411_01433_b200.hobbit import HostCache, blob_bytes, default_config  # noqa: E402

F16, Q4 = 0, 2
HIGH, LOW, SKIP = 0, 1, 2


def decisions(shape, xs, t1=0.6, t2=0.9):
    """[(layer, experts, prec)] per token, from fp64 router logits."""
    th1 = np.log(t1 / (1 - t1)) if t1 < 1 else np.inf
    th2 = np.log(t2 / (1 - t2)) if t2 < 1 else np.inf
    wg = [sg.router_weights(shape, l).astype(np.float64) for l in range(shape.n_layers)]
    out = []
    for t in range(xs.shape[0]):
        tok = []
        for l in range(shape.n_layers):
            lg = wg[l] @ xs[t, l].astype(np.float64)
            order = np.argsort(-lg, kind="stable")[:2]
            gap = lg[order[0]] - lg[order[1]]
            p1 = HIGH if gap <= th1 else (LOW if gap <= th2 else SKIP)
            tok.append((l, [int(order[0]), int(order[1])], [HIGH, p1]))
        out.append(tok)
    return out


def replay(traces, w, caps, p, L):
    cfg = default_config(n_layers=L, n_experts=8, top_k=2, hidden=4096, ffn=14336, hi_enc=F16,
                         lo_enc=Q4, w_lru=w[0], w_lfu=w[1], w_lhu=w[2], w_fld=w[3],
                         cap_high=caps[0], cap_low=caps[1], lookahead_p=p)
    hc = HostCache(cfg)
    bb = {F16: blob_bytes(F16, 4096, 14336), Q4: blob_bytes(Q4, 4096, 14336)}
    loaded = 0
    for seq in traces:
        hc.reset_sequence()
        for tok in seq:
            hc.token_begin()
            for l, ex, pr in tok:
                hc.forward(l, ex, pr)
                if p:
                    pred = [(tok[l + j][1], tok[l + j][2]) for j in range(1, p + 1) if l + j < L]
                    hc.prefetch(l, pred)
            loaded += sum(bb[e[4]] for e in hc.events() if e[0] == 1)
    return loaded


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=6)
    ap.add_argument("--tokens", type=int, default=48)
    ap.add_argument("--rho", type=float, default=0.5)
    ap.add_argument("--p", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_eq3_calibration.md"))
    a = ap.parse_args()
    shape = sg.MIXTRAL
    L = shape.n_layers
    traces = []
    for s in range(a.seqs):
        xs = sg.correlated_states(shape, a.tokens, 0.999, a.rho, seed=sg.DEFAULT_SEED + 17 * s)
        traces.append(decisions(shape, xs))
    caps = (48, 56)
    res = {}
    for w in itertools.product(range(4), repeat=4):
        res[w] = replay(traces, w, caps, a.p, L)
    rnd = res[(0, 0, 0, 0)]
    ranked = sorted((v, w) for w, v in res.items() if w != (0, 0, 0, 0))
    names = {(1, 0, 0, 0): "LRU", (0, 1, 0, 0): "LFU", (0, 0, 1, 0): "LHU", (0, 0, 0, 1): "FLD",
             (1, 1, 1, 1): "equal weights (default)"}
    lines = [f"# r02: Eq. 3 weight calibration on synthetic C4 traces (p = {a.p})", "",
             f"{a.seqs} sequences x {a.tokens} decode tokens, Mixtral shapes, rho = {a.rho}, "
             f"layer cosine 0.999, pools {caps[0]} F16 + {caps[1]} Q4 slots (25 % of the F16 "
             f"expert bytes), the library's host cache (hbc_*).  Miss penalty = bytes loaded "
             f"on demand{' and by prefetch' if a.p else ''}; normalised by the Random policy "
             f"(all-zero weights, R29) as in fig:cache-policy-verify (P:1040).", "",
             "| weights (LRU:LFU:LHU:FLD) | policy | GB loaded | vs Random | vs LRU |",
             "|---|---|---|---|---|"]
    lru = res[(1, 0, 0, 0)]

    def row(w, v):
        return (f"| {':'.join(map(str, w))} | {names.get(w, '')} | {v / 1e9:.2f} | "
                f"{v / rnd:.4f} | {v / lru:.4f} |")
    lines.append(f"| 0:0:0:0 | Random | {rnd / 1e9:.2f} | 1.0000 | {rnd / lru:.4f} |")
    for w in [(1, 0, 0, 0), (0, 1, 0, 0), (0, 0, 1, 0), (0, 0, 0, 1), (1, 1, 1, 1)]:
        lines.append(row(w, res[w]))
    lines += ["", "Best 10 of the 255 non-zero weight vectors in {0..3}^4:", "",
              "| weights | GB loaded | vs Random | vs LRU |", "|---|---|---|---|"]
    for v, w in ranked[:10]:
        lines.append(f"| {':'.join(map(str, w))} | {v / 1e9:.2f} | {v / rnd:.4f} | {v / lru:.4f} |")
    best_w = ranked[0][1]
    lines += ["", f"Calibrated weights (minimum miss penalty): {':'.join(map(str, best_w))} -- "
              f"{100 * (1 - ranked[0][0] / lru):.2f} % fewer bytes than LRU, "
              f"{100 * (1 - ranked[0][0] / rnd):.2f} % fewer than Random.  (The paper reports "
              f"4.69-8.68 % less miss penalty than LRU on its real traces, P:1040; the trace "
              f"statistics here are synthetic.)"]
    txt = "\n".join(lines) + "\n"
    print(txt)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write(txt)


if __name__ == "__main__":
    main()
