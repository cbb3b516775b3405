"""Router (K1) cost vs batch size: one layer, resident Mixtral shapes (run under ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402

Bs = [int(b) for b in os.environ.get("BS", "1,16,64,256,512").split(",")]
torch.cuda.set_device(0)
ctx, blobs = bench.build_model(h, sg, None, sg.MIXTRAL, 0, 2, 0, 1, 0, max_batch=max(Bs), layers=1)
for B in Bs:
    x = torch.from_numpy(sg.hidden_states(sg.MIXTRAL, 9, 0, batch=B)).cuda()
    y = torch.empty(B, 4096, dtype=torch.float32, device="cuda")
    ctx.forward(0, x, y)
    torch.cuda.synchronize()
