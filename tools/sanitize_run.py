"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
tiny shapes through every path of the library -- batch-1 decode (legacy
chain, fused, split), GEMV batches, the tcgen05 batched path (K3), the
offload path with loads, prefetch and evictions.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402
from tests.gpu_util import gpu_blobs  # noqa: E402

F16, Q4 = 0, 2
sh = sg.MoEShape("tiny4", 4, 8, 2, 256, 512, 1.5)


def resident(max_batch, mode):
    os.environ["HB_DECODE"] = mode
    cfg = h.default_config(n_layers=4, n_experts=8, top_k=2, hidden=256, ffn=512, hi_enc=F16,
                           lo_enc=Q4, max_batch=max_batch)
    ctx = h.Context(cfg)
    keep = []
    for l in range(2):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(8), [F16, Q4]).items():
            ctx.register_expert(l, e, enc, b)
            keep.append(b)
    return ctx, keep


def run(ctx, B, layers=(0, 1), reps=2):
    for r in range(reps):
        for l in layers:
            x = torch.from_numpy(sg.hidden_states(sh, 60 + r, l, batch=B)).cuda()
            y = torch.empty(B, 256, dtype=torch.float32, device="cuda")
            ctx.forward(l, x, y)
    torch.cuda.synchronize()


for mode in ("legacy", "fused", "split"):
    ctx, keep = resident(1, mode)
    run(ctx, 1)
    ctx.close()
os.environ["HB_DECODE"] = "legacy"
ctx, keep = resident(16, "legacy")
ctx.set_batched_min(0)
run(ctx, 3)
ctx.set_batched_min(4)
run(ctx, 16)                                   # K3
ctx.close()
# deterministic mode (GEMV and K3)
cfg = h.default_config(n_layers=4, n_experts=8, top_k=2, hidden=256, ffn=512, hi_enc=F16,
                       lo_enc=Q4, max_batch=16, deterministic=1)
ctx = h.Context(cfg)
keep = []
for l in range(2):
    ctx.set_router(l, sg.router_weights(sh, l))
    for (e, enc), b in gpu_blobs(sh, l, range(8), [F16, Q4]).items():
        ctx.register_expert(l, e, enc, b)
        keep.append(b)
ctx.set_batched_min(0)
run(ctx, 3)
ctx.set_batched_min(4)
run(ctx, 16)
ctx.close()
# token-sharded EP, world 1 (pack, owner batch, combine), K2 and K3
for B, bm in ((2, 0), (12, 4)):
    cfg = h.default_config(n_layers=4, n_experts=8, top_k=2, hidden=256, ffn=512, hi_enc=F16,
                           lo_enc=Q4, max_batch=B, token_sharded=1)
    ctx = h.Context(cfg)
    keep = []
    for l in range(2):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(8), [F16, Q4]).items():
            ctx.register_expert(l, e, enc, b)
            keep.append(b)
    ctx.set_batched_min(bm)
    run(ctx, B)
    ctx.close()
# offload: loads, evictions, prefetch -- host manager, device manager (SM
# copies, small chunks), both-versions prefetch
for dc, both in ((0, 0), (1, 0), (1, 1)):
    if dc:
        os.environ["HB_DC_CHUNK_KB"] = "16"
    cfg = h.default_config(n_layers=4, n_experts=8, top_k=2, hidden=256, ffn=512, hi_enc=F16,
                           lo_enc=Q4, max_batch=1, cap_high=8, cap_low=8, lookahead_p=1,
                           device_cache=dc, prefetch_both=both)
    ctx = h.Context(cfg)
    for l in range(4):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(8), [F16, Q4]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())
    for t in range(3):
        ctx.token_begin()
        for l in range(4):
            x = torch.from_numpy(sg.hidden_states(sh, 70 + t, l)).cuda()
            y = torch.empty(1, 256, dtype=torch.float32, device="cuda")
            ctx.forward(l, x, y)
            ctx.prefetch(l, x)
    torch.cuda.synchronize()
    ctx.events()
    ctx.close()
print("sanitize_run done")
