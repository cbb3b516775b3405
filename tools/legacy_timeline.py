"""Timeline of the legacy batch-1 decode chain (router kernel -> K2a -> hfin
-> K2b per layer) inside a CUDA-graph replay, from the in-kernel
%globaltimer points of the diagnostic HB_LEGACY_TL build (csrc/tl_stamps.cuh).

    python -m paper_2411_01433_b200.build --variant tl -DHB_LEGACY_TL=1
    HOBBIT_LIB=build/variants/tl/libhobbit.so python tools/legacy_timeline.py [--model phi]

Prints, per layer-forward, the median time of each point after the previous
forward's K2b end (the moment the layer's input would exist in a real model).
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
ap.add_argument("--solo", action="store_true", help="--router labels of the solo router kernel")
ap.add_argument("--router", action="store_true",
                help="the HB_LEGACY_TL=2 build: router sub-steps in fields 8..14 "
                     "(SM cycles of the leader CTA after its wait; 1.965 GHz assumed)")
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
n_rec = P * L * (a.reps + 2)
ctx.stamps(n_rec)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for t in range(P):
            for l in range(L):
                ctx.forward(l, X[t, l].view(1, Hd), Y[l].view(1, Hd), stream=s)
    g.replay()
    torch.cuda.synchronize()
    ctx.stamps(n_rec)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for r in range(a.reps):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (a.reps * P * L)
raw = np.array(ctx.stamps_read(), dtype=np.uint64)
rec = np.where(raw >= np.uint64(1 << 63), ~raw, raw).astype(np.float64)
print(f"records {len(rec)}, events: {ms * 1000:.2f} us per layer-forward "
      f"({1000.0 / (ms * 32):.1f} tok/s at 32 layers)")
pts = [("router CTA entry", 5), ("router past wait", 6), ("router leader done", 7),
       ("router zeroing done", 13), ("K2a CTA entry (first)", 8), ("K2a past wait (first)", 0),
       ("K2a past wait (last)", 1), ("K2a done (first CTA)", 14), ("K2a done (last CTA)", 2),
       ("hfin past wait (first)", 9), ("hfin done (last)", 10), ("K2b CTA entry (first)", 11),
       ("K2b past wait (first)", 12), ("K2b h staged (first)", 3), ("K2b done (last CTA)", 4)]
if a.router:
    pts = [("router CTA entry", 5), ("router past wait", 6), ("  leader: partial logits", 8),
           ("  leader: x_perm written", 9), ("  leader: cluster sync 1", 10),
           ("  leader: DSMEM combine", 11), ("  leader: cluster sync 2", 12),
           ("  leader: decided", 13), ("  leader: job table", 14), ("router leader done", 7),
           ("K2a past wait (first)", 0), ("K2b done (last CTA)", 4)]
if a.solo:
    a.router = True
    pts = [("router CTA entry", 5), ("router past wait", 6), ("  x loaded", 8), ("  logits summed", 9),
           ("  decided", 10), ("  job table", 11), ("router done", 7),
           ("K2a past wait (first)", 0), ("K2b done (last CTA)", 4)]
prev_end = rec[:-1, 4]
cur = rec[1:]
print(f"  {'point (after the previous K2b end)':36s} {'median':>8s} {'p10':>8s} {'p90':>8s}  (us)")
for name, f in pts:
    v = cur[:, f]
    if a.router and 8 <= f <= 14:               # SM cycles after the router's wait
        d = v / 1.965e3 + (cur[:, 6] - prev_end)[:] / 1e3
        print(f"  {name:36s} {np.median(d):8.2f} {np.percentile(d, 10):8.2f} {np.percentile(d, 90):8.2f}"
              f"   ({np.median(v):.0f} cycles after the wait)")
        continue
    ok = v > 0
    if not ok.any():
        continue
    d = (v[ok] - prev_end[ok]) / 1e3
    print(f"  {name:36s} {np.median(d):8.2f} {np.percentile(d, 10):8.2f} {np.percentile(d, 90):8.2f}")
