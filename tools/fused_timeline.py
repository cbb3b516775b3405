"""Phase breakdown of the fused batch-1 decode kernel from its in-kernel
%globaltimer stamps (hb_stamps), on the first `--layers` Mixtral-shape
layers, CUDA-graph replay (the bench's launch configuration).

    python tools/fused_timeline.py [--layers 8] [--model mixtral|phi] [--pair f16q4]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--model", default="mixtral")
ap.add_argument("--pair", default="f16q4")
ap.add_argument("--tokens", type=int, default=16)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
shape = {"mixtral": sg.MIXTRAL, "phi": sg.PHI}[a.model]
hi, lo = bench.PAIRS[a.pair]
L, Hd = a.layers, shape.hidden
ctx, blobs = bench.build_model(h, sg, None, shape, hi, lo, 0, 1, 0, layers=L)
P = a.tokens
X = torch.from_numpy(np.stack([np.stack([sg.hidden_states(shape, 1000 + t, l)[0] for l in range(L)])
                               for t in range(P)])).cuda()
Y = torch.empty(L, Hd, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
ctx.stamps(P * L * (a.reps + 2))
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for t in range(P):
            for l in range(L):
                ctx.forward(l, X[t, l].view(1, Hd), Y[l].view(1, Hd), stream=s)
    g.replay()
    torch.cuda.synchronize()
    ctx.stamps(P * L * (a.reps + 2))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for r in range(a.reps):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (a.reps * P * L)
rec = np.array(ctx.stamps_read(), dtype=np.float64)
print(f"records {len(rec)}, events: {ms * 1000:.2f} us per layer-forward "
      f"({1000.0 / (ms * 32):.1f} tok/s at 32 layers)")
st, dec, k2a, rel, end, wg, lg, jb, hl, hf, d0, d1, d2, d3, nfb = (rec[:, i] for i in range(15))
gap = st[1:] - end[:-1]
def pr(name, v):
    print(f"  {name:28s} mean {np.mean(v) / 1e3:7.2f} us   median {np.median(v) / 1e3:7.2f}  "
          f"p90 {np.percentile(v, 90) / 1e3:7.2f}")
pr("kernel (start->end)", end - st)
pr("router+jobs (start->decided)", dec - st)
if wg.any():
    pr("  start -> W_g landed", wg - st)
    pr("  W_g -> logits", lg - wg)
    pr("  logits -> jobs", jb - lg)
    pr("    logits -> sums/eps", d0 - lg)
    pr("    sums -> ranks", d1 - d0)
    pr("    ranks -> ok", d2 - d1)
    pr("    ok -> jobs built", d3 - d2)
    pr("    jobs built -> jobs stamp", jb - d3)
    print(f"    exact fallbacks: {int(nfb.sum())} of {len(nfb)} forwards")
    pr("  jobs -> decided (y, zero)", dec - jb)
pr("K2a (decided->k2a_done)", k2a - dec)
pr("barrier (k2a_done->released)", rel - k2a)
pr("h + K2b (released->end)", end - rel)
if hl.any():
    pr("  released -> h staged (first CTA)", hf - rel)
    pr("  released -> h staged (last CTA)", hl - rel)
pr("gap end -> next start", gap)
# realised expert bytes per forward (decisions of the same inputs, eager)
nb = []
w13 = {e: sum(h.blob_section(e, Hd, shape.ffn, m, sc)[1] for m in (0, 1) for sc in (0, 1)
              if not (e == 0 and sc == 1)) for e in (hi, lo)}
w2 = {e: h.blob_bytes(e, Hd, shape.ffn) - w13[e] for e in (hi, lo)}
a13 = a2 = 0
with torch.cuda.stream(s):
    for t in range(P):
        for l in range(L):
            ctx.forward(l, X[t, l].view(1, Hd), Y[l].view(1, Hd), stream=s)
            for d in ctx.decisions(1):
                if d.served_enc != 255:
                    a13 += w13[d.served_enc]
                    a2 += w2[d.served_enc]
n = P * L
print(f"  expert bytes per forward: W1+W3 {a13 / n / 1e6:.1f} MB, W2 {a2 / n / 1e6:.1f} MB; "
      f"K2a {a13 / n / np.mean(k2a - dec) :.0f} GB/s, K2b {a2 / n / np.mean(end - rel):.0f} GB/s, "
      f"kernel {(a13 + a2) / n / np.mean(end - st):.0f} GB/s, layer {(a13 + a2) / n / (ms * 1e6):.0f} GB/s")
