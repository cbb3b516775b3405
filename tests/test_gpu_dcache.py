"""GPU parity of the device-resident cache manager with GPU-initiated,
chunk-preemptible loads (hb_config.device_cache = 1).

The state machine runs in HBM (Eq. 3; the prefetch walk),
loads are SM copies from the mapped pinned host blobs, foreground (this
forward's experts) before background (prefetch), background chunks pre-empted
by the next forward.  Checked against the oracle:

  * cache events bit-exact with O9/O10 and y equal to the oracle's computed
    with the served encodings, with tiny chunks and few copier CTAs (many
    chunks per expert, background copiers racing the replacements);
  * large experts (F = H = 4096, ~100 MB F16) in pools of 2 slots with
    lookahead: slots are re-assigned while background copiers still write them;
  * the whole offload token (32-layer-style chain of forwards + prefetches)
    captured ONCE in a CUDA graph and replayed token after token.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthgen as sg  # noqa: E402
from oracle import cache as oc  # noqa: E402
from oracle import formats as fm  # noqa: E402
from oracle import moe as om  # noqa: E402
from oracle import router as rt  # noqa: E402
from tests.gpu_util import TOL, OracleStore, gpu_blobs, rel_err  # noqa: E402
from tests.test_gpu_parity import _ctx  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _dc_ctx(sh, ch, cl, p, w=(1, 1, 1, 1)):
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=1, cap_high=ch, cap_low=cl, lookahead_p=p,
               w_lru=w[0], w_lfu=w[1], w_lhu=w[2], w_fld=w[3], device_cache=1)
    for l in range(sh.n_layers):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(sh.n_experts), [fm.F16, fm.Q4]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())           # HB_REG_HOST_COPY
    return ctx


def _predict(sh, x16, l, p):
    return {l + j: rt.route(x16, sg.router_weights(sh, l + j), 2, 0.6, 0.9)[0]
            for j in range(1, p + 1) if l + j < sh.n_layers}


@pytest.mark.parametrize("w", [(1, 1, 1, 1), (3, 0, 0, 1), (0, 0, 0, 0)])
def test_dcache_small_chunks_many_copiers(w, monkeypatch):
    """16 KB chunks, 3 foreground / 2 background CTAs: every expert is dozens
    of chunks shared between the two copiers; events and outputs exact."""
    monkeypatch.setenv("HB_DC_CHUNK_KB", "16")
    monkeypatch.setenv("HB_DC_FG_CTAS", "3")
    monkeypatch.setenv("HB_DC_BG_CTAS", "2")
    sh = sg.MoEShape("tiny4", 4, 8, 2, 256, 512, 1.5)
    p = 2
    ctx = _dc_ctx(sh, 5, 5, p, w)
    store = OracleStore(sh)
    ref = oc.ExpertCache(sh.n_layers, sh.n_experts, 5, 5, w, fm.F16, fm.Q4)
    xs = sg.correlated_states(sh, 10, 0.999, 0.5)
    outs = []
    for t in range(10):
        ctx.token_begin()
        ref.token_begin()
        for l in range(sh.n_layers):
            x16 = xs[t, l][None, :]
            x = torch.from_numpy(x16).cuda()
            y = torch.empty(1, sh.hidden, dtype=torch.float32, device="cuda")
            ctx.forward(l, x, y)                 # no host synchronisation anywhere
            served = ref.forward(l, rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0])
            outs.append((y, x16, l, served))
            ctx.prefetch(l, x)
            ref.prefetch(l, _predict(sh, x16, l, p))
    torch.cuda.synchronize()
    assert ctx.events() == ref.events
    for y, x16, l, served in outs:
        r, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16, fm.Q4,
                            served=[served])
        assert rel_err(y.cpu().numpy()[0], r[0])[0] <= TOL


def test_dcache_large_experts_slot_reuse_under_background_copies():
    """~100 MB experts in pools of 5 with lookahead 1: prefetch inserts evict
    slots whose background copies are in flight and the next forward's
    on-demand loads evict prefetched slots -- the replacement must wait for
    the copiers holding the slot; every output equals the oracle's."""
    sh = sg.MoEShape("war", 3, 8, 2, 4096, 4096, 1.5)
    # 5 slots: 2 masked (lookahead 1) + 2 current can never exhaust a pool
    ctx = _dc_ctx(sh, 5, 5, 1)
    store = OracleStore(sh)
    ref = oc.ExpertCache(sh.n_layers, sh.n_experts, 5, 5, (1, 1, 1, 1), fm.F16, fm.Q4)
    outs = []
    for t in range(6):
        ctx.token_begin()
        ref.token_begin()
        for l in range(sh.n_layers):
            x16 = sg.hidden_states(sh, 120 + t, l)
            x = torch.from_numpy(x16).cuda()
            y = torch.empty(1, sh.hidden, dtype=torch.float32, device="cuda")
            ctx.forward(l, x, y)
            served = ref.forward(l, rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0])
            outs.append((y, x16, l, served))
            ctx.prefetch(l, x)
            ref.prefetch(l, _predict(sh, x16, l, 1))
    torch.cuda.synchronize()
    ev = ctx.events()
    assert ev == ref.events
    assert sum(1 for e in ev if e[0] == 1 and e[6] >= 0) >= 8
    for y, x16, l, served in outs:
        r, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16, fm.Q4,
                            served=[served])
        assert rel_err(y.cpu().numpy()[0], r[0])[0] <= 1e-4


@pytest.mark.parametrize("p", [0, 1])
def test_dcache_offload_token_graph_captured(p):
    """The offload forward has no host sync in device_cache mode: one whole
    token (every layer's forward + prefetch) is captured once and replayed;
    events and outputs of every replayed token equal the oracle's."""
    sh = sg.MoEShape("tiny6", 6, 8, 2, 256, 512, 1.5)
    ctx = _dc_ctx(sh, 6, 6, p)
    store = OracleStore(sh)
    ref = oc.ExpertCache(sh.n_layers, sh.n_experts, 6, 6, (1, 1, 1, 1), fm.F16, fm.Q4)
    L = sh.n_layers
    xin = torch.zeros(L, 1, sh.hidden, dtype=torch.float16, device="cuda")
    yout = torch.zeros(L, 1, sh.hidden, dtype=torch.float32, device="cuda")
    xs = sg.correlated_states(sh, 9, 0.999, 0.5)
    # token 0 eagerly (warm-up, also exercises the eager path), then capture
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    results = []
    for t in range(9):
        xin.copy_(torch.from_numpy(xs[t][:, None, :]))
        ref.token_begin()
        if t <= 1:
            ctx.token_begin()
        if t == 0:
            for l in range(L):
                ctx.forward(l, xin[l], yout[l])
                ctx.prefetch(l, xin[l])
        else:
            if t == 1:
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for l in range(L):
                        ctx.forward(l, xin[l], yout[l], stream=s)
                        ctx.prefetch(l, xin[l], stream=s)
            g.replay()
        torch.cuda.synchronize()
        ys = yout.cpu().numpy()
        for l in range(L):
            x16 = xs[t, l][None, :]
            served = ref.forward(l, rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0])
            r, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16,
                                fm.Q4, served=[served])
            results.append(rel_err(ys[l, 0], r[0])[0])
            ref.prefetch(l, _predict(sh, x16, l, p))
    assert max(results) <= TOL
    assert ctx.events() == ref.events


@pytest.mark.parametrize("dc", [0, 1])
def test_offload_prefetch_both_versions(dc):
    """R30 (prefetch_both): both versions of each missing predicted expert,
    Low first, on the host manager (dc=0) and the device manager (dc=1):
    events bit-exact with the oracle, outputs equal."""
    sh = sg.MoEShape("tiny4", 4, 8, 2, 256, 512, 1.5)
    p, ch, cl = 2, 9, 9
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=1, cap_high=ch, cap_low=cl, lookahead_p=p,
               device_cache=dc, prefetch_both=1)
    for l in range(sh.n_layers):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(sh.n_experts), [fm.F16, fm.Q4]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())
    store = OracleStore(sh)
    ref = oc.ExpertCache(sh.n_layers, sh.n_experts, ch, cl, (1, 1, 1, 1), fm.F16, fm.Q4,
                         prefetch_both=True)
    xs = sg.correlated_states(sh, 8, 0.999, 0.5)
    outs = []
    for t in range(8):
        ctx.token_begin()
        ref.token_begin()
        for l in range(sh.n_layers):
            x16 = xs[t, l][None, :]
            x = torch.from_numpy(x16).cuda()
            y = torch.empty(1, sh.hidden, dtype=torch.float32, device="cuda")
            ctx.forward(l, x, y)
            served = ref.forward(l, rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0])
            outs.append((y, x16, l, served))
            ctx.prefetch(l, x)
            ref.prefetch(l, _predict(sh, x16, l, p))
    torch.cuda.synchronize()
    ev = ctx.events()
    assert ev == ref.events
    pf = [e for e in ev if e[1] == 1 and e[0] == 1]
    assert any(a[2:4] == b[2:4] and a[4] == fm.Q4 and b[4] == fm.F16 for a, b in zip(pf, pf[1:]))
    for y, x16, l, served in outs:
        r, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16, fm.Q4,
                            served=[served])
        assert rel_err(y.cpu().numpy()[0], r[0])[0] <= TOL


@pytest.mark.parametrize("dc", [0, 1])
def test_offload_capacity_error_is_loud(dc):
    """A pool of one High slot and a token selecting two High experts: the
    second insert has no eligible victim (the first is in use).  The host
    manager fails that forward; the device manager records a sticky
    HB_ECAPACITY that the next call reports (it cannot return it from an
    asynchronous forward)."""
    from paper_2411_01433_b200 import hobbit as H
    sh = sg.MoEShape("tiny4", 4, 8, 2, 256, 512, 1.5)
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=1, cap_high=1, cap_low=4, lookahead_p=0,
               device_cache=dc, t1=1.0, t2=1.0)             # every selection High
    for l in range(sh.n_layers):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(sh.n_experts), [fm.F16, fm.Q4]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())
    ctx.token_begin()
    x = torch.from_numpy(sg.hidden_states(sh, 5, 0)).cuda()
    y = torch.empty(1, sh.hidden, dtype=torch.float32, device="cuda")
    with pytest.raises(H.HobbitError) as ei:
        ctx.forward(0, x, y)
        torch.cuda.synchronize()
        ctx.events()                                   # device manager: reported here
    assert "HB_ECAPACITY" in str(ei.value)


def test_dcache_expert_parallel_rank():
    """The device cache manager on EP rank 1 of 2 (owns the odd experts):
    events bit-exact with the oracle's cache of the same rank."""
    sh = sg.MoEShape("tiny4", 4, 8, 2, 256, 512, 1.5)
    ch, cl, p = 3, 3, 1
    ctx = _ctx(sh, fm.F16, fm.Q4, max_batch=1, cap_high=ch, cap_low=cl, lookahead_p=p,
               device_cache=1, rank=1, world=2)
    for l in range(sh.n_layers):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(1, 8, 2), [fm.F16, fm.Q4]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())
    store = OracleStore(sh)
    ref = oc.ExpertCache(sh.n_layers, sh.n_experts, ch, cl, (1, 1, 1, 1), fm.F16, fm.Q4,
                         rank=1, world=2)
    xs = sg.correlated_states(sh, 6, 0.999, 0.5)
    for t in range(6):
        ctx.token_begin()
        ref.token_begin()
        for l in range(sh.n_layers):
            x16 = xs[t, l][None, :]
            x = torch.from_numpy(x16).cuda()
            y = torch.empty(1, sh.hidden, dtype=torch.float32, device="cuda")
            ctx.forward(l, x, y)
            served = ref.forward(l, rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0])
            r, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16,
                                fm.Q4, rank=1, world=2, served=[served])
            torch.cuda.synchronize()
            assert rel_err(y.cpu().numpy()[0], r[0])[0] <= TOL
            ctx.prefetch(l, x)
            ref.prefetch(l, _predict(sh, x16, l, p))
    torch.cuda.synchronize()
    assert ctx.events() == ref.events
