"""Per-warp timeline of the GEMV kernels (diagnostic; needs a library built with
-DHB_DBG_TIMELINE, e.g. `python -m paper_2411_01433_b200.build --variant tl
-DHB_DBG_TIMELINE` and HOBBIT_LIB=build/variants/tl/libhobbit.so).

For a few (token, layer) forwards of the bench workload it prints, per kernel,
the spread of warp entry, stage-done, stream-loop-done and publish-done times
relative to the first warp's entry (microseconds)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    import synthgen as sg
    from paper_2411_01433_b200 import _lib
    from paper_2411_01433_b200 import hobbit as h

    model = os.environ.get("TL_MODEL", "mixtral")
    pair = os.environ.get("TL_PAIR", "f16q4")
    shape = {"mixtral": sg.MIXTRAL, "phi": sg.PHI}[model]
    hi, lo = bench.PAIRS[pair]
    torch.cuda.set_device(0)
    t1 = float(os.environ.get("TL_T1", "0.6"))
    t2 = float(os.environ.get("TL_T2", "0.9"))
    ctx, blobs = bench.build_model(h, sg, None, shape, hi, lo, 0, 1, 0, t1, t2)
    lib = _lib.lib
    fn = lib.hb_debug_timeline
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    nw = 148 * 16
    buf = np.zeros((nw, 4), dtype=np.uint64)
    Hd = shape.hidden
    Y = torch.empty(1, Hd, dtype=torch.float32, device="cuda")
    rows = {0: [], 1: []}
    rfn = lib.hb_debug_router_timeline
    rfn.argtypes = [ctypes.c_void_p]
    rbuf = np.zeros(16, dtype=np.uint64)
    rrows = []
    lay = []
    for t in range(4):
        for l in range(0, shape.n_layers, 4):
            x = torch.from_numpy(sg.hidden_states(shape, 1000 + t, l)).cuda()
            for _ in range(3):       # warm; the last launch is recorded
                ctx.forward(l, x.view(1, Hd), Y)
            torch.cuda.synchronize()
            assert rfn(rbuf.ctypes.data) == 0
            rb = rbuf.astype(np.int64)
            rrows.append((rb[1:14] - rb[0]) / 1000.0)
            # absolute layer timeline relative to router entry
            ab = []
            for k in (0, 1):
                assert fn(buf.ctypes.data, k) == 0
                bk = buf.astype(np.int64)
                act = bk[:, 3] > 0
                ab.append(((bk[:, 0].min() - rb[0]) / 1e3, (np.median(bk[act, 2]) - rb[0]) / 1e3,
                           (bk[act, 3].max() - rb[0]) / 1e3))
            lay.append([(rb[6] - rb[0]) / 1e3, *ab[0], *ab[1]])
            for k in (0, 1):
                assert fn(buf.ctypes.data, k) == 0
                b = buf.astype(np.int64)
                act = b[:, 3] > 0
                t0 = b[:, 0].min()
                rel = (b - t0) / 1000.0
                rows[k].append([rel[:, 0].max(), np.median(rel[:, 1]), rel[:, 1].max(),
                                np.median(rel[act, 2]), rel[act, 2].max(),
                                np.median(rel[act, 3]), rel[act, 3].max(), act.sum()])
                if t == 1 and l == 4:
                    os.makedirs("gpurun_out", exist_ok=True)
                    np.save(f"gpurun_out/tl_{model}_{pair}_{k}.npy", b)
                buf[:] = 0
                # clear device copy for the next launch (stale warps would confuse)
    np.set_printoptions(suppress=True, linewidth=200)
    print("router stamps (us after entry: 1 wait, 2 partial, 3-4 combine, 5 decide, 6 jobs, 7 stamp, 8 rank, 9 ballot, 10 gates, 11 gstore, 12 sstore, 13 decide entry):",
          np.median(np.array(rrows), axis=0).round(2))
    print("layer (us from router entry): router_end | K2a entry, first-run med, end | "
          "K2b entry, first-run med, end:", np.median(np.array(lay), axis=0).round(2))
    for k, name in ((0, "K2a"), (1, "K2b")):
        a = np.array(rows[k])
        print(f"{model} {pair} {name}: entry_max {np.median(a[:,0]):.2f}  stage med/max "
              f"{np.median(a[:,1]):.2f}/{np.median(a[:,2]):.2f}  loop med/max "
              f"{np.median(a[:,3]):.2f}/{np.median(a[:,4]):.2f}  publish med/max "
              f"{np.median(a[:,5]):.2f}/{np.median(a[:,6]):.2f}  warps {np.median(a[:,7]):.0f}")
        for r in a[:4]:
            print("   ", " ".join(f"{v:7.2f}" for v in r))


if __name__ == "__main__":
    main()
