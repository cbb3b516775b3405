"""Full decoder step around the MoE layer (first half): model
tokens/s instead of layer tokens/s, batch-1 decode, Mixtral-8x7B shapes.

    python tools/decoder_step.py [--layers 32] [--context 1024] [--tokens 16] [--pair f16q4]

Per layer (the paper runs the whole model in Llama.cpp; the MoE layer
is the method, the rest is the host model):
    h += Wo . attn(rope(Wqkv . rmsnorm(h)), KV cache)      (GQA 32 q / 8 kv heads, d = 128)
    h += moe_layer_forward(rmsnorm(h))                      (this library, exact router, K2 chain)
The attention half runs on library kernels (cuBLAS GEMV for the projections,
cuBLAS batched GEMV over the KV cache for the GQA attention) plus a few
elementwise torch ops; it is the host model around the method, not the
product path.  Weights are random (seeded), the KV cache holds `context`
random positions; one token = all layers, captured in one CUDA graph.
Prints one JSON line: model tok/s, the MoE-only tok/s of the same graph
structure, the bytes per token of both halves and their HBM GB/s.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn.functional as Fn  # noqa: E402

import bench  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402

NQ, NKV, HD = 32, 8, 128            # Mixtral-8x7B attention
THETA, EPS = 1e6, 1e-5


def rmsnorm(x, w):
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + EPS)).half() * w


def rope(t, pos, inv):
    # t [1, n, 1, HD]: rotate halves (Llama / Mixtral convention)
    ang = pos.float() * inv                         # [HD/2]
    c, s = torch.cos(ang).half(), torch.sin(ang).half()
    a, b = t[..., :HD // 2], t[..., HD // 2:]
    return torch.cat([a * c - b * s, a * s + b * c], dim=-1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--context", type=int, default=1024)
    ap.add_argument("--tokens", type=int, default=16)
    ap.add_argument("--pair", default="f16q4")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    base = sg.MIXTRAL
    shape = sg.MoEShape(base.name, a.layers, base.n_experts, base.top_k, base.hidden, base.ffn,
                        base.sigma_router)
    H, L, S = shape.hidden, a.layers, a.context
    hi, lo = bench.PAIRS[a.pair]
    ctx, blobs = bench.build_model(h, sg, None, shape, hi, lo, 0, 1, 0)
    g = torch.Generator(device="cuda").manual_seed(7)
    att = []
    for _ in range(L):
        att.append(dict(
            wqkv=(torch.randn(NQ * HD + 2 * NKV * HD, H, device="cuda", generator=g) / H ** 0.5).half(),
            wo=(torch.randn(H, NQ * HD, device="cuda", generator=g) / (NQ * HD) ** 0.5).half(),
            ln1=torch.ones(H, device="cuda", dtype=torch.float16),
            ln2=torch.ones(H, device="cuda", dtype=torch.float16),
            k=torch.randn(NKV, S, HD, device="cuda", generator=g).half(),
            v=torch.randn(NKV, S, HD, device="cuda", generator=g).half()))
    inv = (1.0 / THETA ** (torch.arange(0, HD, 2, device="cuda").float() / HD))
    hbuf = (torch.randn(1, H, device="cuda", generator=g)).half()
    y = torch.empty(1, H, dtype=torch.float32, device="cuda")
    xin = torch.empty(1, H, dtype=torch.float16, device="cuda")
    pos = torch.tensor([S - 1], device="cuda", dtype=torch.int64)

    def layer(l, moe_only=False):
        nonlocal hbuf
        if not moe_only:
            p = att[l]
            qkv = Fn.linear(rmsnorm(hbuf, p["ln1"]), p["wqkv"])           # cuBLAS GEMV
            q = qkv[:, :NQ * HD].view(1, NQ, 1, HD)
            k = qkv[:, NQ * HD:NQ * HD + NKV * HD].view(1, NKV, 1, HD)
            v = qkv[:, NQ * HD + NKV * HD:].view(NKV, 1, HD)
            q, k = rope(q, pos, inv), rope(k, pos, inv)
            # the token's k, v at its cache position (the cache stays S long: a
            # ring, the same attention work every step)
            p["k"].index_copy_(1, pos, k.view(NKV, 1, HD))
            p["v"].index_copy_(1, pos, v)
            # GQA decode attention as batched GEMV over the cache (cuBLAS):
            # 4 query heads per kv head, one softmax over the S positions
            sc = torch.bmm(q.view(NKV, NQ // NKV, HD), p["k"].transpose(1, 2)) * (HD ** -0.5)
            o = torch.bmm(torch.softmax(sc.float(), dim=-1).half(), p["v"])   # [NKV, 4, HD]
            hbuf = hbuf + Fn.linear(o.reshape(1, NQ * HD), p["wo"])
        xin.copy_(rmsnorm(hbuf, att[l]["ln2"]))
        ctx.forward(l, xin, y, stream=torch.cuda.current_stream())
        hbuf = hbuf + y.half()

    s = torch.cuda.Stream()
    res = {}
    mix = {}
    for mode in ("model", "moe_only"):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for l in range(L):                       # warm-up (allocations, cuBLAS handles)
                layer(l, mode == "moe_only")
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=s):
                for l in range(L):
                    layer(l, mode == "moe_only")
                pos.copy_(torch.remainder(pos + 1, S))     # the next position (ring)
            for _ in range(3):
                graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.tokens):
                graph.replay()
            e1.record(s)
            torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / a.tokens
        d = ctx.decisions(1)
        mix[mode] = [int(v.prec) for v in d]
        assert torch.isfinite(hbuf).all(), "hidden state overflowed"
        del graph
    att_bytes = L * (2 * (NQ * HD + 2 * NKV * HD) * H + 2 * H * NQ * HD + 2 * 2 * NKV * HD * S)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = {"config": "full decoder step (SURVEY 8(f) f4), Mixtral-8x7B shapes, batch-1 decode",
           "layers": L, "context": S, "pair": a.pair, "attention": "cuBLAS GEMV projections + cuBLAS bmm GQA attention (32/8 heads, d 128) + RoPE",
           "model_tok_s": round(1000.0 / res["model"], 2), "model_ms_per_token": round(res["model"], 4),
           "moe_only_tok_s": round(1000.0 / res["moe_only"], 2),
           "moe_only_ms_per_token": round(res["moe_only"], 4),
           "attention_part_ms_per_token": round(res["model"] - res["moe_only"], 4),
           "attention_bytes_per_token": att_bytes,
           "attention_part_gbs": round(att_bytes / ((res["model"] - res["moe_only"]) * 1e-3) / 1e9, 1),
           "hbm_peak_gbs": peak, "last_layer_decisions": mix,
           "data": "synthetic, random-init weights and KV cache"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
