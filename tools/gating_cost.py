"""Stacked vs sequential gating cost ("Stacking
Computer", P:1018 fig:predictor-analysis): the next-layer predictions of
layers l+1..l+p from x_l, computed (a) stacked -- one prefetch_next_layer
call with lookahead p (one router launch over the p router matrices) -- or
(b) sequentially -- p calls with lookahead 1, each predicting one layer.
Each call includes the router launch and the blocking read of the
prediction record (the host runs the cache walk).  CUDA-event time on the
compute stream, median over repetitions; Mixtral H and E (F kept small: the
blobs only feed the prefetch copies).

    python tools/gating_cost.py [--reps 200] [--out profiles/r02_gating_cost.md]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402
from tests.gpu_util import gpu_blobs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_gating_cost.md"))
a = ap.parse_args()
torch.cuda.set_device(0)
sh = sg.MoEShape("mixtral-h", 8, 8, 2, 4096, 256, 1.5)


def make(p):
    cfg = h.default_config(n_layers=8, n_experts=8, top_k=2, hidden=4096, ffn=256, hi_enc=0,
                           lo_enc=2, max_batch=1, cap_high=64, cap_low=64, lookahead_p=p)
    ctx = h.Context(cfg)
    for l in range(8):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(8), [0, 2]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())
    return ctx


x = torch.from_numpy(sg.hidden_states(sh, 5, 0)).cuda()
s = torch.cuda.current_stream()
rows = []
seq_ctx = make(1)
for p in (1, 2, 3, 4):
    ctx = make(p)
    st, sq, wst, wsq = [], [], [], []
    for r in range(a.reps):
        ctx.token_begin()
        seq_ctx.token_begin()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        w0 = time.perf_counter()
        e0.record(s)
        ctx.prefetch(0, x)
        e1.record(s)
        w1 = time.perf_counter()
        for j in range(p):
            seq_ctx.prefetch(j, x)
        e2.record(s)
        w2 = time.perf_counter()
        torch.cuda.synchronize()
        st.append(e0.elapsed_time(e1) * 1e3)
        sq.append(e1.elapsed_time(e2) * 1e3)
        wst.append((w1 - w0) * 1e6)
        wsq.append((w2 - w1) * 1e6)
    rows.append((p, statistics.median(st), statistics.median(sq), statistics.median(wst),
                 statistics.median(wsq)))
    ctx.close()
lines = ["# r02: stacked vs sequential gating cost (tools/gating_cost.py)", "",
         "Predictions of layers l+1..l+p from x_l (Mixtral H = 4096, E = 8, batch 1): one "
         "prefetch_next_layer call with lookahead p (the p routers in one launch, P:505) vs p "
         "calls with lookahead 1.  Each call = router launch + blocking read of the prediction "
         f"record + the host cache walk.  Median of {a.reps} repetitions.", "",
         "| p | stacked GPU us | sequential GPU us | stacked host us | sequential host us |",
         "|---|---|---|---|---|"]
for p, a1, b1, c1, d1 in rows:
    lines.append(f"| {p} | {a1:.1f} | {b1:.1f} | {c1:.1f} | {d1:.1f} |")
txt = "\n".join(lines) + "\n"
print(txt)
with open(a.out, "w") as f:
    f.write(txt)
