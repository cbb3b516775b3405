"""GPU parity of token-sharded expert parallelism (
hb_config.token_sharded) through the C-ABI against the oracle.

Each rank routes its own tokens (exact decisions), packs one row per (token,
owner) -- x and the token's selections that owner holds -- into the owner's
block (e mod world), the owner runs its received rows as one batch through the
K2 (GEMV) or K3 (tcgen05 GEMM) path, and the gate-weighted rows come back to
be summed per token
(oracle: ts_dispatch_plan / ts_owner_rows / ts_combine, pinned by
tests/test_ep_gloo.py against the single-process layer).

  * world 1, one-shot moe_layer_forward (local exchange) and with the
    in-library NCCL exchange (hb_nccl_init, world 1): y = the oracle's layer;
  * two processes on one GPU driving the staged calls (hb_ts_dispatch /
    hb_ts_compute / hb_ts_combine) with gloo all-to-all between them: every
    rank's y = the oracle's layer on that rank's tokens; the dispatched
    records equal the oracle's plan.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthgen as sg  # noqa: E402
from oracle import formats as fm  # noqa: E402
from oracle import moe as om  # noqa: E402
from oracle import router as rt  # noqa: E402
from tests.gpu_util import TOL, OracleStore, rel_err  # noqa: E402
from tests.test_gpu_parity import _resident, _run  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _check_layer(y, x16, sh, l, tol=TOL):
    store = OracleStore(sh)
    ref, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16, fm.Q4)
    for b in range(ref.shape[0]):
        assert rel_err(y[b], ref[b])[0] <= tol, b


@pytest.mark.parametrize("B,bm", [(1, 0), (3, 0), (12, 4), (40, 4)],
                         ids=["B1-K2", "B3-K2", "B12-K3", "B40-K3"])
def test_ts_world1_one_shot(B, bm):
    sh = sg.TINY
    ctx = _resident(sh, [0, 1], fm.F16, fm.Q4, max_batch=B, batched_min=bm, token_sharded=1)
    if B == 1:
        ctx.set_batched_min(bm)
    for l in range(2):
        x16 = sg.hidden_states(sh, 60 + B, l, batch=B)
        _check_layer(_run(ctx, l, x16), x16, sh, l)


def test_ts_world1_nccl_exchange():
    """The one-shot forward through ncclSend/ncclRecv (world 1: to itself)."""
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=20, batched_min=4, token_sharded=1)
    ctx.nccl_init()
    x16 = sg.hidden_states(sh, 64, 0, batch=20)
    _check_layer(_run(ctx, 0, x16), x16, sh, 0)


def _ts_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sh = sg.TINY
    for B, bm in ((3, 0), (24, 4)):
        ctx = _resident(sh, [0, 1], fm.F16, fm.Q4, max_batch=B, batched_min=bm, rank=rank,
                        world=world, token_sharded=1)
        meta_s, rows_s, ret_s = ctx.ts_buffers()
        meta_r, rows_r, ret_r = ctx.ts_buffers()
        for l in range(2):
            x16 = sg.hidden_states(sh, 70 + rank, l, batch=B)
            x = torch.from_numpy(x16).cuda()
            y = torch.empty(B, sh.hidden, dtype=torch.float32, device="cuda")
            ctx.ts_dispatch(l, x, meta_s, rows_s)
            torch.cuda.synchronize()
            for src, dst in ((meta_s, meta_r), (rows_s, rows_r)):
                out = torch.empty_like(src, device="cpu")
                dist.all_to_all_single(out, src.cpu())          # block q -> rank q
                dst.copy_(out)
            np.save(os.path.join(out_dir, f"meta_{B}_{l}_{rank}.npy"), meta_s.cpu().numpy())
            ctx.ts_compute(l, meta_r, rows_r, ret_s)
            torch.cuda.synchronize()
            out = torch.empty_like(ret_s, device="cpu")
            dist.all_to_all_single(out, ret_s.cpu())
            ret_r.copy_(out)
            ctx.ts_combine(ret_r, y)
            torch.cuda.synchronize()
            np.save(os.path.join(out_dir, f"y_{B}_{l}_{rank}.npy"), y.cpu().numpy())
        ctx.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_ts_two_processes_staged(world, tmp_path):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_ts_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    sh = sg.TINY
    for B in (3, 24):
        C = B                                   # one row per (token, owner)
        for l in range(2):
            for r in range(world):
                x16 = sg.hidden_states(sh, 70 + r, l, batch=B)
                y = np.load(tmp_path / f"y_{B}_{l}_{r}.npy")
                _check_layer(y, x16, sh, l)
                # the dispatched rows = the oracle's plan (hb_ts_meta: token, n,
                # expert[8], prec[8] bytes, gate[8] = 20 words)
                routes = rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)
                _, sent = om.ts_dispatch_plan(routes, world, C)
                raw = np.load(tmp_path / f"meta_{B}_{l}_{r}.npy")
                words = raw.view(np.int32).reshape(world, C, 20)
                precs = raw.reshape(world, C, 80)[:, :, 40:48]
                for q in range(world):
                    got = [(int(m[0]), [int(e) for e in m[2:2 + m[1]]], [int(d) for d in pp[:m[1]]])
                           for m, pp in zip(words[q], precs[q]) if m[0] >= 0]
                    want = [(b, [e for e, _, _ in sels], [d for _, d, _ in sels]) for b, sels in sent[q]]
                    assert got == want, (B, l, r, q)
                    assert all(m[0] == -1 for m in words[q][len(sent[q]):])


def test_ts_nonfinite_row_and_all_skip_second_selection():
    """R28 on the token-sharded path: a token whose x has an inf gets a NaN
    row (nothing dispatched for it), the others equal the oracle; and with
    T1 = T2 = 0 every second selection is Skip -- one row per token
    travels."""
    sh = sg.TINY
    B = 6
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=B, batched_min=4, token_sharded=1)
    x16 = sg.hidden_states(sh, 77, 0, batch=B)
    x16[2, 5] = np.float16(np.inf)
    y = _run(ctx, 0, x16)
    assert np.isnan(y[2]).all()
    store = OracleStore(sh)
    ok = [b for b in range(B) if b != 2]
    ref, _ = om.moe_layer(x16[ok], sg.router_weights(sh, 0), store, 0, 2, 0.6, 0.9, fm.F16, fm.Q4)
    for i, b in enumerate(ok):
        assert rel_err(y[b], ref[i])[0] <= TOL
    ctx2 = _resident(sh, [0], fm.F16, fm.Q4, max_batch=B, batched_min=0, token_sharded=1,
                     t1=0.0, t2=0.0)
    x16 = sg.hidden_states(sh, 78, 0, batch=B)
    y = _run(ctx2, 0, x16)
    ref, routes = om.moe_layer(x16, sg.router_weights(sh, 0), store, 0, 2, 0.0, 0.0, fm.F16, fm.Q4)
    assert all(r.decisions[1] == rt.SKIP for r in routes)
    for b in range(B):
        assert rel_err(y[b], ref[b])[0] <= TOL
