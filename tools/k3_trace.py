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
names = ["b_issue", "raw_issue", "conv_arrive_g0", "mma_go"]
v = [buf[ch][buf[ch] > 0].astype(np.int64) - t0 for ch in range(4)]
for ch in range(4):
    d = np.diff(v[ch])
    print(f"{names[ch]:13s} n={len(v[ch]):4d} first={v[ch][:10].tolist()} median_dt={np.median(d):.0f}ns")
n = min(len(v[0]), len(v[3]))
print("b issue -> mma go (median)", np.median(v[3][:n] - v[0][:n]))
for ch in range(4):
    print(names[ch], "last", v[ch][-1] if len(v[ch]) else None)
