"""Expert parallelism (O11) across processes on CPU: world-size-2 `gloo`.

The N>1 path of bench.py shards the experts of every layer by owner(e) =
e mod world: each rank computes the selected experts
it owns and the partial layer outputs are summed by an all-reduce.  Here two
processes run the oracle's per-rank layer (the same partition rule the CUDA
path implements, checked on one GPU by test_gpu_parity::test_ep_partition_on_one_gpu)
and all-reduce over gloo; the sum must equal the single-process layer and the
ranks must split the experts exactly."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthgen as sg
from oracle import formats as fm
from oracle import moe as om
from oracle import router as rt

SH = sg.TINY
LAYER = 1
B = 6


def _store():
    blobs = {}

    def blob(layer, e, enc):
        if (layer, e, enc) not in blobs:
            w1, w3, w2 = sg.expert_weights(SH, layer, e)
            blobs[(layer, e, enc)] = fm.quantize_blob(enc, w1, w3, w2)
        return blobs[(layer, e, enc)]

    return om.ExpertStore(blob, SH.hidden, SH.ffn)


def _worker(rank, world, port, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        x16 = sg.hidden_states(SH, 31, LAYER, batch=B)
        wg = sg.router_weights(SH, LAYER)
        y, routes = om.moe_layer(x16, wg, _store(), LAYER, SH.top_k, 0.6, 0.9, fm.F16, fm.Q4,
                                 rank=rank, world=world)
        owned = sorted({e for r in routes for e, d in zip(r.experts, r.decisions)
                        if d != rt.SKIP and om.owner(e, world) == rank})
        t = torch.from_numpy(np.ascontiguousarray(y))
        dist.all_reduce(t)                      # Eq. 1 summed over ranks
        own = torch.zeros(SH.n_experts, dtype=torch.int64)
        own[owned] = rank + 1
        dist.all_reduce(own)
        if rank == 0:
            np.save(os.path.join(out_dir, "y.npy"), t.numpy())
            np.save(os.path.join(out_dir, "own.npy"), own.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_ep_gloo_allreduce_equals_single_process(world):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        y = np.load(os.path.join(d, "y.npy"))
        own = np.load(os.path.join(d, "own.npy"))
    x16 = sg.hidden_states(SH, 31, LAYER, batch=B)
    ref, routes = om.moe_layer(x16, sg.router_weights(SH, LAYER), _store(), LAYER, SH.top_k,
                               0.6, 0.9, fm.F16, fm.Q4)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    # every served expert was computed by exactly its owner rank (no overlap,
    # no gap): own[e] = owner + 1 for the selected, non-skipped experts
    used = {e for r in routes for e, d in zip(r.experts, r.decisions) if d != rt.SKIP}
    for e in range(SH.n_experts):
        assert own[e] == ((om.owner(e, world) + 1) if e in used else 0), (e, own)


def _tp_worker(rank, world, port, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        x16 = sg.hidden_states(SH, 32, LAYER, batch=B)
        wg = sg.router_weights(SH, LAYER)
        y, _ = om.moe_layer(x16, wg, _store(), LAYER, SH.top_k, 0.6, 0.9, fm.F16, fm.Q4,
                            tp_rank=rank, tp_world=world)
        t = torch.from_numpy(np.ascontiguousarray(y))
        dist.all_reduce(t)                      # partial experts summed over the ranks
        if rank == 0:
            np.save(os.path.join(out_dir, "y.npy"), t.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tp_within_expert_gloo_equals_single_process(world):
    """SURVEY 8(f) f3, TP-within-expert: every rank computes every selected
    expert on its slice of F (rows of W1/W3, columns of W2); the all-reduced
    sum equals the single-process layer (fp64, to rounding)."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_tp_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        y = np.load(os.path.join(d, "y.npy"))
    x16 = sg.hidden_states(SH, 32, LAYER, batch=B)
    ref, _ = om.moe_layer(x16, sg.router_weights(SH, LAYER), _store(), LAYER, SH.top_k,
                          0.6, 0.9, fm.F16, fm.Q4)
    np.testing.assert_allclose(y, ref, rtol=1e-10, atol=1e-12)


def test_tp_slice_is_a_restriction():
    """tp_slice picks rows of W1/W3 and the matching columns of W2 only."""
    w1 = np.arange(8 * 4).reshape(8, 4).astype(float)
    w3 = -w1
    w2 = np.arange(4 * 8).reshape(4, 8).astype(float)
    a, b, c = om.tp_slice(w1, w3, w2, 1, 2)
    assert np.array_equal(a, w1[4:]) and np.array_equal(b, w3[4:]) and np.array_equal(c, w2[:, 4:])


# ------------------------------------------------------- token-sharded EP (f3)
TS_B = 5          # tokens per rank
NSEL = 2          # top_k of the tiny shape


def _ts_worker(rank, world, port, out_dir):
    """Each rank routes ITS tokens, sends one row per (token, owner) with the
    token's selections that owner holds (all_to_all of fixed-capacity blocks),
    computes the rows it received, sends them back and sums them per token."""
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        H = SH.hidden
        C = TS_B
        x16 = sg.hidden_states(SH, 40 + rank, LAYER, batch=TS_B)
        routes = rt.route(x16, sg.router_weights(SH, LAYER), SH.top_k, 0.6, 0.9)
        pos, sent = om.ts_dispatch_plan(routes, world, C)
        rows = np.zeros((world, C, H), dtype=np.float64)
        meta = np.full((world, C, 2 + 3 * NSEL), -1.0)      # token, n, (e, d, g) x NSEL
        for q in range(world):
            for j, (b, sels) in enumerate(sent[q]):
                rows[q, j] = x16[b].astype(np.float64)
                meta[q, j, :2] = (b, len(sels))
                for i, (e, d, g) in enumerate(sels):
                    meta[q, j, 2 + 3 * i:5 + 3 * i] = (e, d, g)
        rrows = torch.empty(world * C * H, dtype=torch.float64)
        rmeta = torch.empty(meta.size, dtype=torch.float64)
        dist.all_to_all_single(rrows, torch.from_numpy(rows.ravel()))
        dist.all_to_all_single(rmeta, torch.from_numpy(meta.ravel()))
        rrows = rrows.numpy().reshape(world * C, H)
        rmeta = rmeta.numpy().reshape(world * C, 2 + 3 * NSEL)
        live = [j for j in range(world * C) if rmeta[j, 0] >= 0]
        recs = []
        for j in live:
            n = int(rmeta[j, 1])
            sels = [(int(rmeta[j, 2 + 3 * i]), int(rmeta[j, 3 + 3 * i]), rmeta[j, 4 + 3 * i])
                    for i in range(n)]
            assert all(om.owner(e, world) == rank for e, _, _ in sels)
            recs.append((int(rmeta[j, 0]), sels))
        out = np.zeros((world * C, H))
        out[live] = om.ts_owner_rows(rrows[live].astype(np.float16), recs, _store(), LAYER,
                                     fm.F16, fm.Q4)
        ret = torch.empty(world * C * H, dtype=torch.float64)
        dist.all_to_all_single(ret, torch.from_numpy(out.ravel()))
        y = om.ts_combine(pos, ret.numpy().reshape(world * C, H), H)
        np.save(os.path.join(out_dir, f"y{rank}.npy"), y)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_token_sharded_gloo_equals_single_process(world):
    """SURVEY 8(f) f3, token-sharded EP: dispatch -> owner compute -> combine
    across two processes equals the single-process layer on each rank's tokens
    (fp64, to rounding); the plan puts every selection at its owner."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_ts_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        ys = [np.load(os.path.join(d, f"y{r}.npy")) for r in range(world)]
    for r in range(world):
        x16 = sg.hidden_states(SH, 40 + r, LAYER, batch=TS_B)
        ref, _ = om.moe_layer(x16, sg.router_weights(SH, LAYER), _store(), LAYER, SH.top_k,
                              0.6, 0.9, fm.F16, fm.Q4)
        np.testing.assert_allclose(ys[r], ref, rtol=1e-10, atol=1e-12)


def test_ts_dispatch_plan_order_and_capacity():
    """One row per (token, owner), rows in token order per owner, selections in
    rank order inside a row; Skip sends nothing; overflow raises."""
    R = rt.Route
    routes = [R(experts=[3, 0], gates=[0.7, 0.3], decisions=[rt.HIGH, rt.LOW], logits=None),
              R(experts=[1, 2], gates=[0.9, 0.1], decisions=[rt.HIGH, rt.SKIP], logits=None),
              R(experts=[2, 0], gates=[0.6, 0.4], decisions=[rt.HIGH, rt.HIGH], logits=None)]
    pos, sent = om.ts_dispatch_plan(routes, 2, 4)
    # owner 0 (even experts): token 0 (e0), token 2 (e2, e0); owner 1: token 0 (e3), token 1 (e1)
    assert pos == [[4, 0], [5, -1], [1, 1]]
    assert [(b, [e for e, _, _ in sels]) for b, sels in sent[0]] == [(0, [0]), (2, [2, 0])]
    assert [(b, [e for e, _, _ in sels]) for b, sels in sent[1]] == [(0, [3]), (1, [1])]
    with pytest.raises(ValueError):
        om.ts_dispatch_plan(routes, 1, 2)
