"""Benchmark: decode tokens/s of the mixed-precision MoE expert layer (HOBBIT,
arXiv 2411.01433) on B200, Mixtral-8x7B shapes, batch-1 decode.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one decode token through all 32 MoE layers (every row of SURVEY.md
8(a) on the resident path: exact router + top-k + gates + Eq. 2 + T1/T2,
expert lookup in the slot table, W1/W3+SwiGLU and W2+gate-sum GEMVs), with
the Mixtral-8x7B shapes of BASELINE.json configs[1]: E=8, top-2, H=4096,
F=14336, fp16 High / int4 Low, T1=0.6, T2=0.9, all 256
experts resident in both encodings (107.6 GiB).  Inputs per (token, layer)
are seeded synthetic fp16 hidden states (not chained, R23); weights
are seeded synthetic (no checkpoints).  Each token streams ~17 GB of expert
weights, far larger than the 126 MB L2, so no L2 flush is needed.

N > 1 (torchrun): expert-parallel, rank r owns experts e % N == r of every
layer; each layer's partial y is summed with an NCCL all-reduce on the
compute stream.  All ranks process the same token (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "decode tokens/s (Mixtral-8x7B shape) at 1/2/4/8 B200; expert-FFN HBM GB/s vs peak"
UNIT = "tokens/s"
WORKLOAD = "mixtral-8x7b-shapes batch-1 decode, 32 layers, fp16/int4 strict (T1=0.6,T2=0.9), all experts resident"


PAIRS = {"f16q4": (0, 2), "f16q2": (0, 3), "q8q2": (1, 3), "q8q4": (1, 2),
         "f16q2k": (0, 4), "q8q2k": (1, 4)}     # 4 = HB_Q2K (llama.cpp Q2_K arithmetic, R32)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """DRAM bytes (read + write) of one K2a + K2b launch pair of one known
    forward, with that forward's own algorithmic bytes, from the newest
    committed profiles/*_k2pair.json (tools/ncu_k2pair.py); {} if none."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_k2pair.json")))
    if not files:
        return {}
    try:
        with open(files[-1]) as f:
            d = json.load(f)
        return {"traffic": int(d["dram_bytes"]), "traffic_alg_bytes": int(d["alg_bytes"]),
                "traffic_over_alg": round(d["dram_bytes"] / d["alg_bytes"], 4),
                "traffic_source": os.path.relpath(files[-1], ROOT)}
    except Exception:
        return {}


# ------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ our arm
def build_model(h, sg, fm, shape, hi, lo, rank, world, dev, t1=0.6, t2=0.9, max_batch=1, layers=None,
                tp_rank=0, tp_world=1, cfg_extra=None):
    """Random-init weights of the shape (seeded generator), quantised on the
    GPU and registered resident.  EP (world > 1): this rank's experts
    (e % world == rank).  TP-within-expert (tp_world > 1): every expert, rows
    [r F/R, (r+1) F/R) of W1/W3 and those columns of W2."""
    import torch
    H, F = shape.hidden, shape.ffn
    Fs = F // tp_world
    cfg = h.default_config(n_layers=shape.n_layers, n_experts=shape.n_experts, top_k=shape.top_k,
                           hidden=H, ffn=Fs, hi_enc=hi, lo_enc=lo, t1=t1,
                           t2=t2, max_batch=max_batch, rank=rank, world=world,
                           **(cfg_extra or {}))
    ctx = h.Context(cfg, dev)
    tmp = [torch.empty(n * k, dtype=torch.float16, device="cuda")
           for n, k in ((F, H), (F, H), (H, F))]
    f0, f1 = tp_rank * Fs, (tp_rank + 1) * Fs
    blobs = []
    for l in range(shape.n_layers if layers is None else layers):
        ctx.set_router(l, sg.router_weights(shape, l))
        for e in range(shape.n_experts):
            if e % world != rank:
                continue
            for mat, t in enumerate(tmp):
                h.synth_fill(t, sg.expert_key(sg.DEFAULT_SEED, l, e, mat),
                             float(sg.scale_f32(sg.expert_sigma(shape, mat))))
            ws = [tmp[0].view(F, H), tmp[1].view(F, H), tmp[2].view(H, F)]
            if tp_world > 1:
                ws = [ws[0][f0:f1].contiguous(), ws[1][f0:f1].contiguous(),
                      ws[2][:, f0:f1].contiguous()]
            for enc in (hi, lo):
                b = h.quantize_expert(enc, *ws)
                ctx.register_expert(l, e, enc, b)
                blobs.append(b)
            del ws
    del tmp
    torch.cuda.synchronize()
    return ctx, blobs


def run_ours(args):
    import torch
    import torch.distributed as dist

    import synthgen as sg
    from paper_2411_01433_b200 import hobbit as h

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torchrun "
                         f"(python -m torch.distributed.run --nproc-per-node N bench.py --gpus N)")
    # HB_BENCH_SAME_GPU=1 (plumbing check only, never a measurement): every
    # rank on cuda:0, gloo, torch all-reduce -- the N > 1 code path on one GPU
    same_gpu = os.environ.get("HB_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
        os.environ["HB_BENCH_TORCH_ALLREDUCE"] = "1"
    torch.cuda.set_device(local)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = {"mixtral": sg.MIXTRAL, "phi": sg.PHI}[args.model]
    hi, lo = PAIRS[args.pair]
    L, Hd = shape.n_layers, shape.hidden
    # N > 1: TP-within-expert (every rank streams 1/N of every selected
    # expert: batch-1 decode scales with N) when F/N is a multiple of 256,
    # else expert parallelism (e % N; top-2 of 8 caps batch-1 at ~1.5x)
    par = args.parallel
    if par == "auto":
        par = "tp" if world > 1 and (shape.ffn // world) % 256 == 0 and shape.ffn % world == 0 else "ep"
    tp = par == "tp" and world > 1
    t_init = time.time()
    ctx, blobs = build_model(h, sg, None, shape, hi, lo, 0 if tp else rank, 1 if tp else world,
                             local, t1=args.t1, t2=args.t2, tp_rank=rank if tp else 0,
                             tp_world=world if tp else 1)
    # the exchange (A10) inside the library: the forward ends with the NCCL
    # all-reduce of y over the ranks; HB_BENCH_TORCH_ALLREDUCE=1 reduces with
    # torch.distributed instead (eager)
    torch_reduce = world > 1 and os.environ.get("HB_BENCH_TORCH_ALLREDUCE") == "1"
    if world > 1 and not torch_reduce:
        ctx.nccl_init(tp=tp)
    t_init = time.time() - t_init

    # token inputs: a pool of P tokens x 32 layers, resident on the device
    P = 16
    X = torch.from_numpy(np.stack([
        np.stack([sg.hidden_states(shape, 1000 + t, l)[0] for l in range(L)]) for t in range(P)
    ])).cuda()                                                       # [P, L, H] fp16
    Y = torch.empty(L, Hd, dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()

    def step(t, s):
        for l in range(L):
            ctx.forward(l, X[t % P, l].view(1, Hd), Y[l].view(1, Hd), stream=s)
            if world > 1:
                if torch_reduce:
                    dist.all_reduce(Y[l])

    # ---- realised algorithmic bytes of the pool's tokens (decisions, untimed)
    Fr = shape.ffn // world if tp else shape.ffn          # this rank's F (TP slice)
    blob_b = {hi: h.blob_bytes(hi, Hd, Fr), lo: h.blob_bytes(lo, Hd, Fr)}
    # SURVEY 8(d) unit: served blob bytes + router W_g + x + y + h (write + read)
    bytes_tok = []
    mix = [0, 0, 0]
    for t in range(P):
        tot = 0
        for l in range(L):
            with torch.cuda.stream(stream):
                ctx.forward(l, X[t, l].view(1, Hd), Y[l].view(1, Hd), stream=stream)
            for d in ctx.decisions(1):
                mix[d.prec] += 1
                if d.served_enc != h.HB_ENC_NONE:
                    tot += blob_b[d.served_enc] + 2 * 4 * Fr
            tot += 2 * shape.n_experts * Hd + 2 * Hd + 4 * Hd
        bytes_tok.append(tot)
    torch.cuda.synchronize()
    # per-matrix bytes of one blob (W1+W3 vs W2) from the layout
    def mat_bytes(enc, mats):
        tot = 0
        for m in mats:
            for sec in range(3):
                try:
                    tot += h.blob_section(enc, Hd, Fr, m, sec)[1]
                except h.HobbitError:
                    pass
        return tot
    w13b = {e: mat_bytes(e, (0, 1)) for e in (hi, lo)}
    w2b = {e: mat_bytes(e, (2,)) for e in (hi, lo)}

    # ---- CUDA graphs, one per pool token (32 layers; at N > 1 the in-library
    # NCCL all-reduce of every layer is captured too).  A second set is
    # captured with the in-kernel %globaltimer stamps on (hb_stamps): it is
    # replayed right after the timed region for the roofline, so the headline
    # graphs carry no instrumentation.
    use_graph = not torch_reduce
    graphs, sgraphs = [], []
    launches_per_step = 0
    if use_graph:
        c0 = ctx.launch_count()
        with torch.cuda.stream(stream):
            for t in range(P):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    step(t, stream)
                graphs.append(g)
            launches_per_step = (ctx.launch_count() - c0) // P
            # record capacity fixed before capture (the stamped graphs keep the pointer)
            stamp_cap = max(P, args.steps) * L
            ctx.stamps(stamp_cap)
            for t in range(P):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    step(t, stream)
                sgraphs.append(g)
            ctx.stamps(0)

    def run_step(t, stamped=False):
        if use_graph:
            (sgraphs if stamped else graphs)[t % P].replay()
        else:
            step(t, stream)

    # ---- warmup + timed region
    with torch.cuda.stream(stream), ClockSampler(local) as clk:
        for w in range(args.warmup):
            run_step(w)
        # keep the GPU busy (untimed) until the clock sampler is producing samples
        t_wait = time.time()
        while not clk.lines and time.time() - t_wait < 5.0:
            for w in range(8):
                run_step(w)
            torch.cuda.synchronize()
        n_pre = len(clk.lines)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        c_before = ctx.launch_count()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            run_step(args.warmup + k)
        e1.record(stream)
        torch.cuda.synchronize()
        time.sleep(0.15)
        clk.lines = clk.lines[max(0, n_pre - 1):]   # samples from the timed region on
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    gpu_launches = (launches_per_step * args.steps if use_graph
                    else ctx.launch_count() - c_before)
    tok_s = 1000.0 / ms_step
    steps_tokens = [(args.warmup + k) % P for k in range(args.steps)]
    bytes_step = float(np.mean([bytes_tok[t] for t in steps_tokens]))

    # ---- roofline of the dominant kernels (K2a + K2b): the same K steps
    # replayed from the stamped graphs; per forward the kernels' own in-kernel
    # intervals: K2a = [first CTA past its wait, last CTA done], K2b = [first
    # CTA with h staged, last CTA done]
    roof = {}
    if use_graph and not args.no_roofline:
        with torch.cuda.stream(stream):
            ctx.stamps(stamp_cap)
            e2 = torch.cuda.Event(enable_timing=True)
            e3 = torch.cuda.Event(enable_timing=True)
            e2.record(stream)
            for k in range(args.steps):
                run_step(args.warmup + k, stamped=True)
            e3.record(stream)
            torch.cuda.synchronize()
            rec = np.array(ctx.stamps_read(args.steps * L), dtype=np.float64)
            ctx.stamps(0)
        ms_stamped = e2.elapsed_time(e3) / args.steps
        # bytes per forward of the same (token, layer) sequence, from its decisions
        k2a_b, k2b_b = [], []
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                t = (args.warmup + k) % P
                for l in range(L):
                    ctx.forward(l, X[t, l].view(1, Hd), Y[l].view(1, Hd), stream=stream)
                    a = b = ne = 0
                    for d in ctx.decisions(1):
                        if d.served_enc != h.HB_ENC_NONE:
                            a += w13b[d.served_enc]
                            b += w2b[d.served_enc]
                            ne += 1
                    # SURVEY 8(d) unit split over the two kernels: K2a = W1/W3 +
                    # x + h written (4F per expert); K2b = W2 + h read + y
                    k2a_b.append(a + 2 * Hd + 4 * Fr * ne)
                    k2b_b.append(b + 4 * Fr * ne + 4 * Hd)
        n = min(len(rec), len(k2a_b))
        k2a_ns = rec[:n, 2] - rec[:n, 0]
        k2b_ns = rec[:n, 4] - rec[:n, 3]
        k2_ns = float(np.sum(k2a_ns + k2b_ns))
        gemv_bytes = float(np.sum(k2a_b[:n]) + np.sum(k2b_b[:n]))
        achieved = gemv_bytes / k2_ns                     # bytes/ns = GB/s
        roof = {"achieved": round(achieved, 1),
                "k2a_gbs": round(float(np.sum(k2a_b[:n]) / np.sum(k2a_ns)), 1),
                "k2b_gbs": round(float(np.sum(k2b_b[:n]) / np.sum(k2b_ns)), 1),
                "k2_share_of_step": round(k2_ns / n * L * 1e-6 / ms_stamped, 4),
                "stamped_ms_per_step": round(ms_stamped, 4),
                "alg_bytes_per_launch_pair": int(gemv_bytes / n),
                "forwards": int(n),
                "method": "in-kernel %globaltimer stamps (hb_stamps) over a graph replay of the "
                          "timed steps; bytes from the same forwards' decisions"}
    peak, peak_kind = peaks()
    traffic = ncu_traffic()

    # ---- end to end through the public API with host buffers: every step
    # copies that token's inputs from pinned host memory (H2D) and its result
    # back (D2H) inside the timed region; the 32 forwards and both copies are
    # one CUDA graph per pool token (a user can capture the same calls), or
    # eager when the reduce runs in torch
    Xh = torch.empty(P, L, Hd, dtype=torch.float16, pin_memory=True)
    Xh.copy_(X.cpu())
    Yh = torch.empty(P, L, Hd, dtype=torch.float32, pin_memory=True)
    Xd = torch.empty(L, Hd, dtype=torch.float16, device="cuda")

    def e2e_step(k):
        Xd.copy_(Xh[k % P], non_blocking=True)
        for l in range(L):
            ctx.forward(l, Xd[l].view(1, Hd), Y[l].view(1, Hd), stream=stream)
            if world > 1:
                if torch_reduce:
                    dist.all_reduce(Y[l])
        Yh[k % P].copy_(Y, non_blocking=True)

    egraphs = []
    if use_graph:
        with torch.cuda.stream(stream):
            for t in range(P):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    e2e_step(t)
                egraphs.append(g)
            for w in range(args.warmup):
                egraphs[w % P].replay()
    with torch.cuda.stream(stream):
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e2.record(stream)
        for k in range(args.steps):
            if egraphs:
                egraphs[k % P].replay()
            else:
                e2e_step(k)
        e3.record(stream)
        torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3) / args.steps
    if world > 1:
        tt = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_e2e = float(tt.item())

    # ---- batched decode / prefill through K3 on the same weights (N=1, diagnostic)
    batched = None
    if world == 1 and not args.no_batched:
        batched = batched_leg(h, sg, shape, hi, lo, blobs, local, stream)

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(shape, n_token_layers=args.cpu_sample)

    tot_mix = sum(mix)
    clk_sum = clk.summary()
    out = {
        "metric": METRIC, "value": round(tok_s, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f16 weights / q4 codes, fp32 accumulate", "data": "synthetic",
        "config": {"workload": WORKLOAD if (args.model, args.pair, args.t1, args.t2) == ("mixtral", "f16q4", 0.6, 0.9)
                   else f"DIAGNOSTIC {shape.name} pair {args.pair} (not the headline workload)",
                   "global_batch": 1, "layers": L, "experts": shape.n_experts,
                   "top_k": shape.top_k, "hidden": Hd, "ffn": shape.ffn, "pair": args.pair,
                   "parallelism": f"{'tp' if tp else 'ep'}{world}",
                   "l2": "inputs > L2 (~17 GB of weights per step)",
                   "graph": use_graph},
        "e2e": {"value": round(1000.0 / ms_e2e, 3), "unit": UNIT,
                "h2d_bytes_per_step": L * Hd * 2, "d2h_bytes_per_step": L * Hd * 4,
                "graph": bool(egraphs)},
        "gpu_launches": int(gpu_launches),
        "roofline": dict({"bound": "hbm", "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                          "frac": round(roof["achieved"] / peak, 4) if roof else None,
                          "frac_vs_8000_spec": round(roof["achieved"] / 8000.0, 4) if roof else None,
                          "kernel": "K2a+K2b dequant-GEMV (gemv_kernel<1>, gemv_kernel<0>)"},
                         **roof, **traffic),
        "layer_gbs": round(bytes_step / (ms_step * 1e-3) / 1e9, 1),
        "bytes_per_step": int(bytes_step),
        "precision_mix": [round(v / tot_mix, 4) for v in mix],
        "clocks": clk_sum,
        "init_s": round(t_init, 1),
    }
    if batched is not None:
        out["batched_k3"] = batched          # tok/s normalised to 32-layer tokens
    if cpu is not None:
        out["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------ batched leg (A9)
def batched_leg(h, sg, shape, hi, lo, blobs, dev, stream, Bs=(256, 512), layers=8, steps=5):
    """SURVEY 8(d) C5 on the same resident weights (1 GPU): batched decode (B=256)
    and a 512-token prefill through the tcgen05 grouped-GEMM path K3, first
    `layers` layers rotating (>= 3.6 GB of expert weights per step, >> L2).
    Diagnostic extra of the bench line: tokens/s and step-level GB/s of the
    served blobs (each (expert, encoding) blob once per layer + X + h + y)."""
    import torch
    E, Hd, F = shape.n_experts, shape.hidden, shape.ffn
    bb = {hi: h.blob_bytes(hi, Hd, F), lo: h.blob_bytes(lo, Hd, F)}
    out = {}
    # allow_upgrade = 1, one stream per touched expert
    # (strict = 0, R27); the strict mix (every Low from lo_enc) too
    for strict in (0, 1):
      cfg = h.default_config(n_layers=shape.n_layers, n_experts=E, top_k=shape.top_k, hidden=Hd,
                             ffn=F, hi_enc=hi, lo_enc=lo, max_batch=max(Bs), strict=strict)
      ctx = h.Context(cfg, dev)
      i = 0
      for l in range(shape.n_layers):
          ctx.set_router(l, sg.router_weights(shape, l))
          for e in range(E):
              for enc in (hi, lo):
                  ctx.register_expert(l, e, enc, blobs[i])
                  i += 1
      with torch.cuda.stream(stream):
        for B in Bs:
            X = torch.from_numpy(np.stack([sg.hidden_states(shape, 7000 + B, l, batch=B)
                                           for l in range(layers)])).cuda()
            Y = torch.empty(layers, B, Hd, dtype=torch.float32, device="cuda")
            nbytes = 0
            for l in range(layers):
                ctx.forward(l, X[l], Y[l], stream=stream)
                jobs, nsel = set(), 0
                for d in ctx.decisions(B):
                    if d.served_enc != h.HB_ENC_NONE:
                        jobs.add((d.expert, d.served_enc))
                        nsel += 1
                nbytes += sum(bb[e] for _, e in jobs) + 2 * B * Hd + 2 * 2 * nsel * F + 4 * B * Hd
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for l in range(layers):
                    ctx.forward(l, X[l], Y[l], stream=stream)
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            out[f"B{B}" + ("" if strict == 0 else "_strict")] = {
                "tok_s": round(B * layers / shape.n_layers * 1000.0 / ms, 1),
                "ms_per_step": round(ms, 4), "layers": layers,
                "step_gbs": round(nbytes / ms / 1e6, 1), "path": "K3 tcgen05 GEMM",
                "strict": strict}
            del X, Y, g
      ctx.close()
    return out


# ------------------------------------------------------------ oracle timings
def _oracle_sample(shape, n_token_layers, seed_tok=2000, layer=None):
    """Pre-generate blobs (untimed), then time the oracle as it stands on
    n_token_layers (token, layer) pairs: exact router + decode + fp64 FFN.
    layer=None rotates through the layers; an int keeps one layer (its blobs
    are then generated once for all samples)."""
    import synthgen as sg
    from oracle import formats as fm
    from oracle import moe as om
    from oracle import router as rt
    blobs = {}

    def blob(l, e, enc):
        if (l, e, enc) not in blobs:
            w1, w3, w2 = sg.expert_weights(shape, l, e)
            blobs[(l, e, enc)] = fm.quantize_blob(enc, w1, w3, w2)
        return blobs[(l, e, enc)]

    cases = []
    for i in range(n_token_layers):
        l = i % shape.n_layers if layer is None else layer
        x16 = sg.hidden_states(shape, seed_tok + i, l)
        wg = sg.router_weights(shape, l)
        r = rt.route(x16, wg, 2, 0.6, 0.9)[0]
        for e, d in zip(r.experts, r.decisions):
            if d != rt.SKIP:
                blob(l, e, fm.F16 if d == rt.HIGH else fm.Q4)
        cases.append((l, x16, wg))
    times = []
    for l, x16, wg in cases:
        store = om.ExpertStore(blob, shape.hidden, shape.ffn)      # fresh: decode is timed
        t0 = time.perf_counter()
        om.moe_layer(x16, wg, store, l, 2, 0.6, 0.9, fm.F16, fm.Q4)
        times.append(time.perf_counter() - t0)
    return times


def cpu_baseline(shape, n_token_layers=2):
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits
        ctxm = threadpool_limits(limits=cores)
    except Exception:
        ctxm = None
    times = _oracle_sample(shape, n_token_layers)
    if ctxm is not None:
        ctxm.unregister() if hasattr(ctxm, "unregister") else None
    s_tl = float(np.mean(times))
    return {"value": round(1.0 / (shape.n_layers * s_tl), 6), "unit": UNIT, "cores": cores,
            "kind": "oracle",
            "sample": f"{n_token_layers} token-layers of the Mixtral-shape workload (exact router, "
                      f"blob decode, fp64 SwiGLU + Eq. 1), {s_tl:.2f} s per token-layer; "
                      f"tokens/s extrapolated = 1/(32 * s per token-layer)"}


def run_reference(args):
    """The reference arm (tier rules: the oracle as it stands, on the host
    cores).  One step = ONE token-layer of the workload (1/32 of a decode
    token: exact router, blob decode, fp64 SwiGLU + Eq. 1), so the run is
    --warmup + --steps token-layers of real work (~6 s each); ms_per_step is
    that measured time and value = tokens/s = 1 / (32 * s per token-layer).
    All steps use one layer's blobs (generated once, untimed)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synthgen as sg
    shape = sg.MIXTRAL
    t0 = time.time()
    n = args.warmup + args.steps
    times = _oracle_sample(shape, n, layer=0)
    timed = times[args.warmup:]
    s_tl = float(np.mean(timed))
    ms_step = 1000.0 * s_tl
    cores = len(os.sched_getaffinity(0))
    v = 1.0 / (shape.n_layers * s_tl)
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": UNIT,
           "n_gpus": world, "steps": len(timed), "warmup": args.warmup,
           "ms_per_step": round(ms_step, 1), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD, "global_batch": 1,
                      "step": "one token-layer (1/32 of a decode token) on the CPU oracle"},
           "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": f"each step = 1 token-layer of the workload (layer 0) timed "
                                      f"on the oracle; tokens/s = 1/(32 * s per token-layer); "
                                      f"{len(timed)} steps"},
           "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "wall_s": round(time.time() - t0, 1)}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batched", action="store_true", help="skip the K3 batched/prefill extra")
    ap.add_argument("--no-roofline", action="store_true", help="diagnostics: skip the stamped replay")
    ap.add_argument("--parallel", choices=["auto", "ep", "tp"], default="auto",
                    help="N > 1: expert parallel or TP-within-expert (auto: tp when F/N fits)")
    ap.add_argument("--t1", type=float, default=0.6, help="diagnostics only (1.0/1.0 = all-High)")
    ap.add_argument("--t2", type=float, default=0.9, help="diagnostics only")
    ap.add_argument("--cpu-sample", type=int, default=2)
    ap.add_argument("--model", choices=["mixtral", "phi"], default="mixtral",
                    help="diagnostics only: the headline is mixtral")
    ap.add_argument("--pair", choices=sorted(PAIRS), default="f16q4",
                    help="diagnostics only: the headline is f16q4")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
