"""Batched decode / prefill sweep (SURVEY 8(d) C5, configs[4]) on one B200:
K2 (dequant-GEMV) vs K3 (tcgen05 grouped GEMM) per batch size.

    python tools/bench_batched.py [--batches 1,8,32,64,128,256,512] [--layers 8]
                                  [--pair f16q4] [--model mixtral] [--steps 10]

One step = one forward of B tokens through `layers` MoE layers (layers
rotate so the streamed weights stay >> L2).  Per B and path prints one JSON
line: tokens/s, algorithmic bytes per step (each served (expert, encoding)
blob once per layer + X, h, y), GB/s of the whole step and of the K3a/K3b
(or K2a/K2b) kernels from CUDA events, the dense tensor TFLOP/s of the
computed experts, and the HBM roofline fraction against MEASURED_PEAKS.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,8,16,32,64,128,256,512")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--pair", default="f16q4")
    ap.add_argument("--model", default="mixtral")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--strict", type=int, default=1,
                    help="0: SURVEY C5's rule (R27, allow the F16 copy for Low requests)")
    ap.add_argument("--paths", default="k2,k3",
                    help="k2 (GEMV), k3 (tcgen05 GEMM), ts (token-sharded EP at world 1)")
    args = ap.parse_args()
    batches = [int(b) for b in args.batches.split(",")]
    shape = {"mixtral": sg.MIXTRAL, "phi": sg.PHI}[args.model]
    hi, lo = bench.PAIRS[args.pair]
    L, Hd, F = args.layers, shape.hidden, shape.ffn
    torch.cuda.set_device(0)
    ctx, blobs = bench.build_model(h, sg, None, shape, hi, lo, 0, 1, 0, max_batch=max(batches),
                                   layers=L, cfg_extra=None if args.strict else {"strict": 0})
    ctx_ts = None
    if "ts" in args.paths.split(","):
        # token-sharded EP context at world 1: dispatch into the
        # local block, the owner batch through K3, combine -- the overhead of
        # the token-sharded path against the plain batched forward
        ctx_ts, blobs_ts = bench.build_model(h, sg, None, shape, hi, lo, 0, 1, 0,
                                             max_batch=max(batches), layers=L,
                                             cfg_extra={"token_sharded": 1})
        ctx_ts.set_batched_min(1)
    peak, peak_kind = bench.peaks()
    mats = {}
    for enc in (hi, lo):
        w13 = w2 = 0
        for m in range(3):
            for sec in range(2):
                try:
                    n = h.blob_section(enc, Hd, F, m, sec)[1]
                except h.HobbitError:
                    continue
                if m < 2:
                    w13 += n
                else:
                    w2 += n
        mats[enc] = (w13, w2)
    stream = torch.cuda.Stream()
    for B in batches:
        X = torch.from_numpy(np.stack([sg.hidden_states(shape, 5000 + B, l, batch=B)
                                       for l in range(L)])).cuda()
        Y = torch.empty(L, B, Hd, dtype=torch.float32, device="cuda")
        for path in args.paths.split(","):
            if path in ("k3", "ts") and B == 1:
                continue
            if path == "k3":
                ctx.set_batched_min(1)
            elif path == "k2":
                ctx.set_batched_min(0)
            else:
                ctx.set_batched_min(1)         # bytes from the plain K3 forward's decisions
            # decisions -> algorithmic bytes / flops of one step
            a_bytes = b_bytes = 0
            flops = 0
            with torch.cuda.stream(stream):
                for l in range(L):
                    ctx.forward(l, X[l], Y[l], stream=stream)
                    jobs = set()
                    nsel = 0
                    for d in ctx.decisions(B):
                        if d.served_enc != h.HB_ENC_NONE:
                            jobs.add((d.expert, d.served_enc))
                            nsel += 1
                    a_bytes += sum(mats[e][0] for _, e in jobs) + 2 * B * Hd + 2 * nsel * F
                    b_bytes += sum(mats[e][1] for _, e in jobs) + 2 * nsel * F + 4 * B * Hd
                    flops += 2 * 3 * Hd * F * nsel
            cx = ctx_ts if path == "ts" else ctx
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                for l in range(L):                 # warm (allocations) outside the capture
                    cx.forward(l, X[l], Y[l], stream=stream)
                with torch.cuda.graph(g, stream=stream):
                    for l in range(L):
                        cx.forward(l, X[l], Y[l], stream=stream)
                for _ in range(args.warmup):
                    g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.steps):
                    g.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.steps
                cx.profile(L)
                for l in range(L):
                    cx.forward(l, X[l], Y[l], stream=stream)
                prof = cx.profile_read()
                cx.profile(0)
            ka = sum(p[0] for p in prof)
            kb = sum(p[1] for p in prof)
            out = {"B": B, "path": path, "layers": L, "pair": args.pair, "model": args.model,
                   # tokens through all 32 layers of the model (the step runs L layers)
                   "tok_s": round(B * L / 32 * 1000.0 / ms, 1), "ms_per_step": round(ms, 4),
                   "tok_s_L_layers": round(B * 1000.0 / ms, 1),
                   "step_gbs": round((a_bytes + b_bytes) / ms / 1e6, 1),
                   "ka_gbs": round(a_bytes / ka / 1e6, 1), "kb_gbs": round(b_bytes / kb / 1e6, 1),
                   "kab_frac": round((a_bytes + b_bytes) / (ka + kb) / 1e6 / peak, 4),
                   "tflops": round(flops / (ka + kb) / 1e9, 1),
                   "ka_ms": round(ka / L, 4), "kb_ms": round(kb / L, 4),
                   "kernel_share": round((ka + kb) / ms, 4),
                   "bytes_per_step": int(a_bytes + b_bytes), "peak": peak, "peak_kind": peak_kind}
            print(json.dumps(out), flush=True)
        del X, Y
    ctx.set_batched_min(0)


if __name__ == "__main__":
    main()
