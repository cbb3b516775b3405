"""One known batch-1 forward (Mixtral F16/Q4, one layer, one token), repeated:
the launch pair ncu captures for the roofline's `traffic` field, with the
forward's own algorithmic bytes (SURVEY 8(d) unit split over K2a / K2b).

    ncu --set full --clock-control none -k regex:gemv_kernel -s 6 -c 2 \\
        -o gpurun_out/k2pair -f python tools/ncu_k2pair.py gpurun_out/k2pair_alg.json
    python tools/ncu_summary.py --tag r02 --full gpurun_out/k2pair.ncu-rep \\
        --k2pair gpurun_out/k2pair_alg.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "k2pair_alg.json"
shape = sg.MIXTRAL
layer, tok = 5, 1003
hi, lo = bench.PAIRS["f16q4"]
H, F = shape.hidden, shape.ffn
cfg = h.default_config(n_layers=shape.n_layers, n_experts=shape.n_experts, top_k=2, hidden=H,
                       ffn=F, hi_enc=hi, lo_enc=lo, max_batch=1)
ctx = h.Context(cfg)
tmp = [torch.empty(n * k, dtype=torch.float16, device="cuda") for n, k in ((F, H), (F, H), (H, F))]
keep = []
ctx.set_router(layer, sg.router_weights(shape, layer))
for e in range(shape.n_experts):
    for mat, t in enumerate(tmp):
        h.synth_fill(t, sg.expert_key(sg.DEFAULT_SEED, layer, e, mat),
                     float(sg.scale_f32(sg.expert_sigma(shape, mat))))
    for enc in (hi, lo):
        b = h.quantize_expert(enc, tmp[0].view(F, H), tmp[1].view(F, H), tmp[2].view(H, F))
        ctx.register_expert(layer, e, enc, b)
        keep.append(b)
x = torch.from_numpy(sg.hidden_states(shape, tok, layer)).cuda()
y = torch.empty(1, H, dtype=torch.float32, device="cuda")
for _ in range(4):
    ctx.forward(layer, x, y)
torch.cuda.synchronize()


def mat_bytes(enc, mats):
    tot = 0
    for m in mats:
        for sec in range(2):
            try:
                tot += h.blob_section(enc, H, F, m, sec)[1]
            except h.HobbitError:
                pass
    return tot


a = b = ne = 0
for d in ctx.decisions(1):
    if d.served_enc != h.HB_ENC_NONE:
        a += mat_bytes(d.served_enc, (0, 1))
        b += mat_bytes(d.served_enc, (2,))
        ne += 1
k2a = a + 2 * H + 4 * F * ne
k2b = b + 4 * F * ne + 4 * H
with open(out_path, "w") as f:
    json.dump({"layer": layer, "token": tok, "experts": [d.expert for d in ctx.decisions(1)],
               "served": [d.served_enc for d in ctx.decisions(1)], "k2a_alg_bytes": k2a,
               "k2b_alg_bytes": k2b, "alg_bytes": k2a + k2b}, f, indent=1)
print("alg bytes", k2a, k2b)
