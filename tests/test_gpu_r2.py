"""GPU parity, round 2: the configurations the kernels take that round 1 left
untested, through the C-ABI against the fp64 / exact oracle.

  * canonical blobs registered straight from the oracle;
  * the non-strict upgrade rule (R27) on the K2 and K3 paths;
  * K2a with x read from global memory (H = 4096, B = 4..8);
  * K3 at the full Mixtral shape with B = 256 and a 512-token prefill
    (the bench's batched launch configuration), sampled tokens incl. Low/Skip;
  * exact logit ties on the device (duplicated router rows);
  * routers with E = 32 and E = 64 experts;
  * expert parallelism through the library in two processes.
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
from tests.test_gpu_parity import _check_routes, _ctx, _resident, _run  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _served(ctx, B):
    return [[None if d.served_enc == 255 else d.served_enc for d in ctx.decisions(B)[b * 2:b * 2 + 2]]
            for b in range(B)]


# ------------------------------------------------------------ canonical blobs
@pytest.mark.parametrize("mode", ["device", "host"])
def test_register_canonical_oracle_blobs_resident(mode):
    """The oracle's own canonical blobs, registered with HB_REG_CANONICAL (the
    library copies them into its HBM and converts them), give the oracle's y."""
    sh = sg.TINY
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=8)
    ctx.set_batched_min(0)
    store = OracleStore(sh)
    for l in range(sh.n_layers):
        ctx.set_router(l, sg.router_weights(sh, l))
        for e in range(sh.n_experts):
            for enc in (fm.F16, fm.Q4):
                b = store._blob(l, e, enc)
                ctx.register_expert(l, e, enc, torch.from_numpy(b).cuda() if mode == "device" else b,
                                    canonical=True)
    for l in range(sh.n_layers):
        x16 = sg.hidden_states(sh, 40, l, batch=8)
        y = _run(ctx, l, x16)
        ref, routes = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16, fm.Q4)
        _check_routes(ctx, routes, 8, 2)
        for b in range(8):
            assert rel_err(y[b], ref[b])[0] <= 1e-4


def test_register_canonical_oracle_blobs_offload():
    """Offload mode: canonical host blobs converted into the library's pinned
    arena; outputs match the oracle with the served encodings."""
    from oracle import cache as oc
    sh = sg.MoEShape("tiny4", 4, 8, 2, 256, 512, 1.5)
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=1, cap_high=6, cap_low=6, lookahead_p=0)
    store = OracleStore(sh)
    for l in range(sh.n_layers):
        ctx.set_router(l, sg.router_weights(sh, l))
        for e in range(sh.n_experts):
            for enc in (fm.F16, fm.Q4):
                ctx.register_expert(l, e, enc, store._blob(l, e, enc), canonical=True)
    ref_cache = oc.ExpertCache(4, 8, 6, 6, (1, 1, 1, 1), fm.F16, fm.Q4)
    for t in range(4):
        ctx.token_begin()
        ref_cache.token_begin()
        for l in range(sh.n_layers):
            x16 = sg.hidden_states(sh, 41 + t, l)
            y = _run(ctx, l, x16)
            route = rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0]
            served = ref_cache.forward(l, route)
            ref, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9,
                                  fm.F16, fm.Q4, served=[served])
            assert rel_err(y[0], ref[0])[0] <= 1e-4
    assert ctx.events() == ref_cache.events


# ------------------------------------------------------------ upgrade rule R27
@pytest.mark.parametrize("B,batched_min", [(6, 0), (48, 1)], ids=["K2", "K3"])
def test_non_strict_upgrade_rule(B, batched_min):
    """strict = 0: a Low selection of an expert some token selected High in the
    same forward is served by hi_enc (one stream per touched expert); the
    served encodings equal oracle O7 (served_encodings_resident) and y the
    oracle's with those encodings."""
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=B, batched_min=batched_min, strict=0)
    store = OracleStore(sh)
    x16 = sg.hidden_states(sh, 43, 0, batch=B)
    y = _run(ctx, 0, x16)
    routes = rt.route(x16, sg.router_weights(sh, 0), 2, 0.6, 0.9)
    served = om.served_encodings_resident(routes, fm.F16, fm.Q4, strict=False)
    assert served != om.served_encodings_resident(routes, fm.F16, fm.Q4, strict=True)
    assert _served(ctx, B) == served
    ref, _ = om.moe_layer(x16, sg.router_weights(sh, 0), store, 0, 2, 0.6, 0.9, fm.F16, fm.Q4,
                          served=served)
    _check_routes(ctx, routes, B, 2)
    bar = 1e-4 if batched_min == 0 else 1e-3
    for b in range(B):
        assert rel_err(y[b], ref[b])[0] <= bar


# ------------------------------------------------------------ K2a global x
@pytest.mark.parametrize("B", [4, 8])
@pytest.mark.parametrize("pair", [(fm.F16, fm.Q4), (fm.Q8, fm.Q2)], ids=["f16q4", "q8q2"])
def test_k2a_global_x_path(B, pair):
    """H = 4096 and B >= 4: x of all tokens no longer fits K2a's CTA stage
    (B*(2H + H/8) > 28 KB), so K2a reads x from global memory."""
    sh = sg.MoEShape("mixtral-h", 1, 8, 2, 4096, 1024, 1.5)
    hi, lo = pair
    ctx = _resident(sh, [0], hi, lo, max_batch=B, batched_min=0)
    store = OracleStore(sh)
    x16 = sg.hidden_states(sh, 43, 0, batch=B)
    y = _run(ctx, 0, x16)
    ref, routes = om.moe_layer(x16, sg.router_weights(sh, 0), store, 0, 2, 0.6, 0.9, hi, lo)
    _check_routes(ctx, routes, B, 2)
    for b in range(B):
        nw, el = rel_err(y[b], ref[b])
        assert nw <= 1e-4, (b, nw, el)


# ------------------------------------------------------------ K3 full size
def test_k3_full_size_b256_and_prefill512():
    """The bench's batched configuration (BASELINE configs[4]): Mixtral shapes,
    B = 256 decode and a 512-token prefill through K3, strict F16/Q4.  The
    oracle checks 10 sampled tokens per batch, chosen to include Low and Skip
    selections; decisions of every token are checked bit-exactly."""
    sh = sg.MoEShape("mixtral", 32, 8, 2, 4096, 14336, 1.5)
    layer = 7
    ctx = _resident(sh, [layer], fm.F16, fm.Q4, max_batch=512, batched_min=32)
    store = OracleStore(sh)
    wg = sg.router_weights(sh, layer)
    for B, tok in ((256, 300), (512, 301)):
        x16 = sg.hidden_states(sh, tok, layer, batch=B)
        y = _run(ctx, layer, x16)
        routes = rt.route(x16, wg, 2, 0.6, 0.9)
        _check_routes(ctx, routes, B, 2)
        low = [b for b, r in enumerate(routes) if r.decisions[1] == rt.LOW]
        skip = [b for b, r in enumerate(routes) if r.decisions[1] == rt.SKIP]
        assert low and skip
        sample = sorted(set([0, B - 1, B // 2] + low[:4] + skip[:3]))
        ref, _ = om.moe_layer(x16[sample], wg, store, layer, 2, 0.6, 0.9, fm.F16, fm.Q4)
        for i, b in enumerate(sample):
            nw, el = rel_err(y[b], ref[i])
            assert nw <= 1e-3, (B, b, nw, el)


# ------------------------------------------------------------ router edge cases
def _tie_router(sh, dup):
    """Router rows where every expert in `dup` has the same row: their exact
    logits tie for every x (scaled up so they are the top candidates)."""
    wg = sg.router_weights(sh, 0).astype(np.float32)
    wg[dup] = wg[dup[0]] * 4.0
    return wg.astype(np.float16)


@pytest.mark.parametrize("dup", [[1, 6], [2, 4, 7]], ids=["pair", "triple"])
@pytest.mark.parametrize("B", [1, 12])
def test_router_exact_ties_on_device(dup, B):
    """Duplicated router rows give exactly tied logits: the lower expert index
    ranks first (reading R2), the gap is 0 -> High (s1 = 0.5 <= T1), and the
    device matches the oracle bit for bit."""
    sh = sg.TINY
    wg = _tie_router(sh, dup)
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=B)
    ctx.set_router(0, wg)
    # a deterministic input whose first token has the duplicated rows on top
    seed = next(t for t in range(44, 400)
                if rt.route(sg.hidden_states(sh, t, 0, batch=1), wg, 2, 0.6, 0.9)[0].experts
                == sorted(dup)[:2])
    x16 = sg.hidden_states(sh, seed, 0, batch=B)
    xt = torch.from_numpy(x16).cuda()
    y = torch.empty(B, sh.hidden, dtype=torch.float32, device="cuda")
    from tests.gpu_util import gpu_blobs
    for (e, enc), b in gpu_blobs(sh, 0, range(8), [fm.F16, fm.Q4]).items():
        ctx.register_expert(0, e, enc, b)
    ctx.forward(0, xt, y)
    torch.cuda.synchronize()
    L = rt.exact_logits(x16, wg)
    assert ctx.logits(B) == L
    routes = [rt.route_token(row, 2, 0.6, 0.9) for row in L]
    ties = [r for r in routes if r.logits[0] == r.logits[1]]
    assert ties, "the duplicated rows must produce exact ties"
    for r in ties:
        assert r.experts == sorted(dup)[:2] and r.decisions == [rt.HIGH, rt.HIGH]
    _check_routes(ctx, routes, B, 2)


@pytest.mark.parametrize("E", [32, 64])
@pytest.mark.parametrize("B", [1, 3, 20])
def test_router_many_experts(E, B):
    """E = 32 and 64 experts (the router's per-task partial table holds up to
    64 rows): exact logits and decisions equal the oracle's."""
    sh = sg.MoEShape(f"e{E}", 1, E, 2, 1024, 256, 1.5)
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=B)
    if B > 1:
        ctx.set_batched_min(0)
    ctx.set_router(0, sg.router_weights(sh, 0))
    from tests.gpu_util import gpu_blobs
    for (e, enc), b in gpu_blobs(sh, 0, range(E), [fm.F16, fm.Q4]).items():
        ctx.register_expert(0, e, enc, b)
    x16 = sg.hidden_states(sh, 45, 0, batch=B)
    _run(ctx, 0, x16)
    L = rt.exact_logits(x16, sg.router_weights(sh, 0))
    assert ctx.logits(B) == L
    _check_routes(ctx, [rt.route_token(row, 2, 0.6, 0.9) for row in L], B, 2)


# ------------------------------------------------------------ EP, two processes
def _ep_worker(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sh = sg.TINY
    results = []
    for B, bm in ((3, 0), (40, 1)):
        ctx = _resident(sh, [0, 1], fm.F16, fm.Q4, max_batch=B, batched_min=bm,
                        rank=rank, world=world)
        for l in range(2):
            x16 = sg.hidden_states(sh, 46, l, batch=B)
            y = torch.from_numpy(_run(ctx, l, x16))
            dist.all_reduce(y)                       # the EP sum of the partial outputs
            results.append(y.numpy())
        ctx.close()
    if rank == 0:
        np.save(out_path, np.concatenate([r.ravel() for r in results]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_ep_two_processes_through_library(world, tmp_path):
    """O11 through the library in two processes (one context per process, same
    GPU, ranks 0 and 1 own the even / odd experts): the gloo sum of the
    per-rank outputs equals the oracle's single-rank layer, for the K2 and K3
    paths."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "ep.npy")
    mp.start_processes(_ep_worker, args=(world, port, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    sh = sg.TINY
    store = OracleStore(sh)
    refs = []
    for B in (3, 40):
        for l in range(2):
            x16 = sg.hidden_states(sh, 46, l, batch=B)
            ref, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9,
                                  fm.F16, fm.Q4)
            refs.append(ref)
    off = 0
    for ref in refs:
        y = got[off:off + ref.size].reshape(ref.shape)
        off += ref.size
        for b in range(ref.shape[0]):
            assert rel_err(y[b], ref[b])[0] <= TOL


# ------------------------------------------------------------ non-finite inputs
@pytest.mark.parametrize("mode", ["legacy", "fused"])
@pytest.mark.parametrize("B,batched_min", [(1, 0), (3, 0), (12, 4), (20, 4), (20, 0)],
                         ids=["B1", "B3", "K3-B12", "K3-B20", "GEMV-B20"])
def test_nonfinite_input_documented_behaviour(mode, B, batched_min, monkeypatch):
    """DESIGN.md R28: a token whose x holds an inf/nan gets Skip decisions
    (expert -1, gate NaN) and a NaN output row; every other token is
    unaffected (equal to the oracle)."""
    monkeypatch.setenv("HB_DECODE", mode)
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=32, batched_min=batched_min)
    store = OracleStore(sh)
    x16 = sg.hidden_states(sh, 47, 0, batch=B)
    bad = B // 2
    x16[bad, 5] = np.float16(np.inf) if B % 2 else np.float16(np.nan)
    y = _run(ctx, 0, x16)
    dec = ctx.decisions(B)
    assert all(d.expert == -1 and d.prec == rt.SKIP and np.isnan(d.gate) for d in dec[2 * bad:2 * bad + 2])
    assert np.all(np.isnan(y[bad]))
    good = [b for b in range(B) if b != bad]
    if good:
        ref, routes = om.moe_layer(x16[good], sg.router_weights(sh, 0), store, 0, 2, 0.6, 0.9,
                                   fm.F16, fm.Q4)
        for i, b in enumerate(good):
            assert [d.expert for d in dec[2 * b:2 * b + 2]] == routes[i].experts
            assert rel_err(y[b], ref[i])[0] <= TOL


# ------------------------------------------------------------ decode variants
@pytest.mark.parametrize("mode", ["fused", "split", "router"])
def test_decode_variants_match_oracle(mode, monkeypatch):
    """The alternative batch-1 decode chains (HB_DECODE):
    decisions, logits and y equal the oracle's on the tiny layers and on one
    full-size Mixtral F16/Q4 layer."""
    monkeypatch.setenv("HB_DECODE", mode)
    sh = sg.TINY
    ctx = _resident(sh, [0, 1], fm.F16, fm.Q4, max_batch=1)
    store = OracleStore(sh)
    for t in range(4):
        for l in range(2):
            x16 = sg.hidden_states(sh, 48 + t, l)
            y = _run(ctx, l, x16)
            ref, routes = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9,
                                       fm.F16, fm.Q4)
            _check_routes(ctx, routes, 1, 2)
            assert ctx.logits(1) == rt.exact_logits(x16, sg.router_weights(sh, l))
            assert rel_err(y[0], ref[0])[0] <= 1e-4
    big = sg.MoEShape("mixtral", 32, 8, 2, 4096, 14336, 1.5)
    ctx = _resident(big, [9], fm.F16, fm.Q4, max_batch=1)
    store = OracleStore(big)
    x16 = sg.hidden_states(big, 49, 9)
    y = _run(ctx, 9, x16)
    ref, routes = om.moe_layer(x16, sg.router_weights(big, 9), store, 9, 2, 0.6, 0.9, fm.F16, fm.Q4)
    _check_routes(ctx, routes, 1, 2)
    assert rel_err(y[0], ref[0])[0] <= 1e-4


# ------------------------------------------------------------ slot WAR ordering
def test_offload_slot_war_ordering():
    """Offload path, pools of 2 slots, two layers with disjoint experts: every
    forward evicts the slots the previous layer's GEMV kernels are still
    reading (F = 4096: tens of microseconds of K2) while its ~100 MB copies
    start on the copy stream right away.  The per-slot 'free' events must
    order each copy after the readers: every output equals the oracle's."""
    from oracle import cache as oc
    sh = sg.MoEShape("war", 2, 8, 2, 4096, 4096, 1.5)
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=1, cap_high=2, cap_low=2, lookahead_p=0)
    store = OracleStore(sh)
    from tests.gpu_util import gpu_blobs
    for l in range(2):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(8), [fm.F16, fm.Q4]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())
    ref_cache = oc.ExpertCache(2, 8, 2, 2, (1, 1, 1, 1), fm.F16, fm.Q4)
    outs, refs = [], []
    for t in range(6):
        ctx.token_begin()
        ref_cache.token_begin()
        for l in range(2):
            x16 = sg.hidden_states(sh, 80 + t, l)
            x = torch.from_numpy(x16).cuda()
            y = torch.empty(1, sh.hidden, dtype=torch.float32, device="cuda")
            ctx.forward(l, x, y)                 # no synchronisation between forwards
            outs.append(y)
            route = rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0]
            served = ref_cache.forward(l, route)
            refs.append((x16, l, served))
    torch.cuda.synchronize()
    evictions = [e for e in ctx.events() if e[0] == 1 and e[6] >= 0]
    assert len(evictions) >= 8, "the trace must evict slots still in use by the previous layer"
    for y, (x16, l, served) in zip(outs, refs):
        ref, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16, fm.Q4,
                              served=[served])
        assert rel_err(y.cpu().numpy()[0], ref[0])[0] <= 1e-4


# ------------------------------------------------------------ TP-within-expert
def _tp_worker(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2411_01433_b200 import hobbit as h
    from tests.gpu_util import gpu_expert_f16
    sh = sg.TINY
    Fs = sh.ffn // world
    f0, f1 = rank * Fs, (rank + 1) * Fs
    results = []
    for B, bm in ((1, 0), (3, 0), (24, 4)):
        cfg = h.default_config(n_layers=2, n_experts=8, top_k=2, hidden=sh.hidden, ffn=Fs,
                               hi_enc=fm.F16, lo_enc=fm.Q4, max_batch=B)
        ctx = h.Context(cfg)
        if B > 1:
            ctx.set_batched_min(bm)
        keep = []
        for l in range(2):
            ctx.set_router(l, sg.router_weights(sh, l))
            for e in range(8):
                w1, w3, w2 = gpu_expert_f16(sh, l, e)
                ws = [w1[f0:f1].contiguous(), w3[f0:f1].contiguous(), w2[:, f0:f1].contiguous()]
                for enc in (fm.F16, fm.Q4):
                    b = h.quantize_expert(enc, *ws)
                    ctx.register_expert(l, e, enc, b)
                    keep.append(b)
        for l in range(2):
            x16 = sg.hidden_states(sh, 90, l, batch=B)
            y = torch.from_numpy(_run(ctx, l, x16))
            dist.all_reduce(y)                       # partial experts summed over the ranks
            results.append(y.numpy())
        ctx.close()
    if rank == 0:
        np.save(out_path, np.concatenate([r.ravel() for r in results]))
    dist.barrier()
    dist.destroy_process_group()


def test_tp_within_expert_two_processes_through_library(tmp_path):
    """two processes (one context each, same GPU), each with
    every expert's F/2 slice (rows of W1/W3, columns of W2, quantised by the
    library); the gloo sum of the partial outputs equals the oracle's layer,
    on the decode (B = 1), GEMV batch and tcgen05 (K3) paths."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "tp.npy")
    mp.start_processes(_tp_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    sh = sg.TINY
    store = OracleStore(sh)
    off = 0
    for B in (1, 3, 24):
        for l in range(2):
            x16 = sg.hidden_states(sh, 90, l, batch=B)
            ref, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16, fm.Q4)
            y = got[off:off + ref.size].reshape(ref.shape)
            off += ref.size
            bar = 1e-4 if B < 4 else 1e-3
            for b in range(B):
                assert rel_err(y[b], ref[b])[0] <= bar


# ------------------------------------------------------------ deterministic mode
@pytest.mark.parametrize("B,bm,shape", [(1, 0, "mixtral"), (5, 0, "tiny"), (40, 4, "tiny")],
                         ids=["B1-K2-mixtral", "B5-K2", "B40-K3"])
def test_deterministic_mode_bit_reproducible(B, bm, shape):
    """hb_config.deterministic (R24): whole row
    tiles per warp, no dynamic chunks, no K split -- repeated forwards give
    bit-identical y, and y still matches the oracle."""
    sh = sg.TINY if shape == "tiny" else sg.MoEShape("mx1", 1, 8, 2, 4096, 14336, 1.5)
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=B, batched_min=bm, deterministic=1)
    x16 = sg.hidden_states(sh, 90 + B, 0, batch=B)
    outs = [_run(ctx, 0, x16) for _ in range(4)]
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    store = OracleStore(sh)
    ref, _ = om.moe_layer(x16, sg.router_weights(sh, 0), store, 0, 2, 0.6, 0.9, fm.F16, fm.Q4)
    tol = 1e-3 if bm else 1e-4
    for b in range(B):
        assert rel_err(outs[0][b], ref[b])[0] <= tol
