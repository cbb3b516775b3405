"""Timeline of K3 CTA 0 (build variant with -DHB_K3_TRACE): per raw slot the
producer issue time, the converters' raw_full wake-up, per canonical stage the
converters' can_full arrive and the MMA thread's can_full wake-up (us)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_2411_01433_b200 import _lib  # noqa: E402
from paper_2411_01433_b200 import hobbit as h  # noqa: E402

B = int(os.environ.get("B", "256"))
torch.cuda.set_device(0)
ctx, blobs = bench.build_model(h, sg, None, sg.MIXTRAL, 0, 2, 0, 1, 0, max_batch=B, layers=1)
ctx.set_batched_min(1)
X = torch.from_numpy(sg.hidden_states(sg.MIXTRAL, 7, 0, batch=B)).cuda()
Y = torch.empty(B, 4096, dtype=torch.float32, device="cuda")
for _ in range(3):
    ctx.forward(0, X, Y)
torch.cuda.synchronize()
buf = np.zeros((4, 4096), np.uint64)
assert _lib.lib.hb_k3_trace(C.c_void_p(buf.ctypes.data), C.c_size_t(buf.nbytes)) == 0
t0 = min(int(v) for v in buf.ravel() if v)
names = ["prod_issue", "conv_rawfull", "conv_canfull", "mma_start"]
for ch in range(4):
    v = buf[ch][buf[ch] > 0].astype(np.int64) - t0
    d = np.diff(v)
    print(f"{names[ch]:13s} n={len(v):4d} first={v[:6].tolist()} median_dt={np.median(d) if len(d) else 0:.0f}ns "
          f"p90_dt={np.percentile(d, 90) if len(d) else 0:.0f}ns span={v[-1] if len(v) else 0}ns")
p, r = buf[0][buf[0] > 0].astype(np.int64), buf[1][buf[1] > 0].astype(np.int64)
n = min(len(p), len(r))
print("issue->rawfull latency median", np.median(r[:n] - p[:n]), "ns; p90", np.percentile(r[:n] - p[:n], 90))
c, m = buf[2][buf[2] > 0].astype(np.int64), buf[3][buf[3] > 0].astype(np.int64)
n = min(len(c), len(m))
print("canfull arrive->mma wake median", np.median(m[:n] - c[:n]), "ns")
