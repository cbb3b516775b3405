"""GPU parity of K3, the tcgen05 grouped-GEMM path for batched decode / prefill
(SURVEY 8(a) A9), through the C-ABI against the fp64 oracle.

K3 rounds every dequantised weight d*q (+m) to fp16 and h to fp16 (DESIGN.md
R26), so its bar is the north_star tolerance (2e-3 normwise per token), not the
~1e-6 of the exact-code decode path.  Decisions must stay bit-exact.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthgen as sg  # noqa: E402
from oracle import formats as fm  # noqa: E402
from oracle import moe as om  # noqa: E402
from tests.gpu_util import TOL, OracleStore, gpu_blobs, rel_err  # noqa: E402
from tests.test_gpu_parity import _check_routes, _resident, _run  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


PAIRS = [(fm.F16, fm.Q4), (fm.F16, fm.Q2), (fm.Q8, fm.Q2), (fm.Q8, fm.Q4)]


def _check_layer(ctx, sh, layer, x16, hi, lo, tokens=None, store=None):
    y = _run(ctx, layer, x16)
    B = x16.shape[0]
    store = store or OracleStore(sh)
    idx = list(range(B)) if tokens is None else tokens
    ref, routes = om.moe_layer(x16[idx], sg.router_weights(sh, layer), store, layer,
                               sh.top_k, 0.6, 0.9, hi, lo)
    if tokens is None:
        _check_routes(ctx, routes, B, sh.top_k)
    worst = 0.0
    for i, b in enumerate(idx):
        nw, el = rel_err(y[b], ref[i])
        worst = max(worst, nw)
        assert nw <= TOL, (b, nw, el)
    return worst


@pytest.mark.parametrize("pair", PAIRS, ids=lambda p: f"{fm.ENC_NAMES[p[0]]}-{fm.ENC_NAMES[p[1]]}")
@pytest.mark.parametrize("B", [1, 7, 32, 64])
def test_k3_parity_tiny(pair, B):
    sh = sg.TINY
    hi, lo = pair
    ctx = _resident(sh, [0, 1], hi, lo, max_batch=64)
    ctx.set_batched_min(1)                 # force K3 for every batch size
    for l in range(sh.n_layers):
        x16 = sg.hidden_states(sh, 30, l, batch=B)
        worst = _check_layer(ctx, sh, l, x16, hi, lo)
        assert worst <= 1e-3, worst         # fp16 operand rounding only


def test_k3_many_tokens_per_expert():
    """> 128 tokens of one (expert, encoding): several vjob3 per job, ragged tail."""
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=600, batched_min=8)
    x16 = sg.hidden_states(sh, 31, 0, batch=600)
    _check_layer(ctx, sh, 0, x16, fm.F16, fm.Q4)


def test_k3_matches_gemv_path():
    """The same batch through K2 (GEMV) and K3 (GEMM): identical decisions,
    outputs within the tolerance of each other."""
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=48)
    x16 = sg.hidden_states(sh, 32, 0, batch=48)
    ctx.set_batched_min(0)
    y2 = _run(ctx, 0, x16)
    d2 = [(d.token, d.expert, d.sel_rank, d.prec, d.served_enc, d.gate) for d in ctx.decisions(48)]
    ctx.set_batched_min(1)
    y3 = _run(ctx, 0, x16)
    d3 = [(d.token, d.expert, d.sel_rank, d.prec, d.served_enc, d.gate) for d in ctx.decisions(48)]
    assert d2 == d3
    for b in range(48):
        assert rel_err(y3[b], y2[b])[0] <= TOL


@pytest.mark.parametrize("shape,pair,B", [
    (sg.MIXTRAL, (fm.F16, fm.Q4), 64), (sg.MIXTRAL, (fm.Q8, fm.Q2), 40),
    (sg.PHI, (fm.F16, fm.Q4), 48)], ids=["mixtral-f16q4-b64", "mixtral-q8q2-b40", "phi-f16q4-b48"])
def test_k3_parity_full_size(shape, pair, B):
    """BASELINE.json full shapes, batched decode through K3 (the bench's
    batched launch configuration); the oracle checks a sample of tokens."""
    hi, lo = pair
    layer = 3
    sh1 = sg.MoEShape(shape.name, shape.n_layers, shape.n_experts, 2, shape.hidden, shape.ffn,
                      shape.sigma_router)
    ctx = _resident(sh1, [layer], hi, lo, max_batch=B)
    ctx.set_batched_min(32)
    x16 = sg.hidden_states(sh1, 200, layer, batch=B)
    _check_layer(ctx, sh1, layer, x16, hi, lo, tokens=[0, B // 2, B - 1])


@pytest.mark.parametrize("t1,t2", [(1.0, 1.0), (0.0, 0.0), (0.5, 0.5)])
def test_k3_threshold_edges(t1, t2):
    """All-High (dense top-k MoE), all-Skip-but-rank-0, tie edge through K3."""
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, t1=t1, t2=t2, max_batch=32, batched_min=1)
    store = OracleStore(sh)
    x16 = sg.hidden_states(sh, 33, 0, batch=32)
    y = _run(ctx, 0, x16)
    ref, routes = om.moe_layer(x16, sg.router_weights(sh, 0), store, 0, 2, t1, t2, fm.F16, fm.Q4)
    _check_routes(ctx, routes, 32, 2)
    for b in range(32):
        assert rel_err(y[b], ref[b])[0] <= TOL


def test_k3_zero_input():
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=16, batched_min=1)
    y = _run(ctx, 0, np.zeros((16, sh.hidden), np.float16))
    assert np.all(y == 0)


def test_k3_default_threshold_routes_batches():
    """Default context: batch >= 4 takes K3 (launch count says which chain ran)."""
    sh = sg.TINY
    from paper_2411_01433_b200 import hobbit as h
    cfg = h.default_config(n_layers=1, n_experts=8, top_k=2, hidden=256, ffn=512, max_batch=16)
    ctx = h.Context(cfg)
    ctx.set_router(0, sg.router_weights(sh, 0))
    for (e, enc), b in gpu_blobs(sh, 0, range(8), [fm.F16, fm.Q4]).items():
        ctx.register_expert(0, e, enc, b)
    x = torch.from_numpy(sg.hidden_states(sh, 34, 0, batch=16)).cuda()
    y = torch.empty(16, sh.hidden, dtype=torch.float32, device="cuda")
    n0 = ctx.launch_count()
    ctx.forward(0, x[:3], y[:3])
    n1 = ctx.launch_count()
    ctx.forward(0, x, y)
    n2 = ctx.launch_count()
    assert n1 - n0 == 4            # router, K2a, hfin, K2b
    assert n2 - n1 == 6            # router, prep, K3a (F16, Q), K3b (F16, Q)


@pytest.mark.parametrize("world", [2, 4])
def test_k3_ep_partition_on_one_gpu(world):
    """O11 through K3: per-rank contexts (same GPU) sum to the 1-rank output,
    every served expert computed by exactly its owner."""
    sh = sg.TINY
    x16 = sg.hidden_states(sh, 35, 1, batch=24)
    full = _run(_resident(sh, [1], fm.F16, fm.Q4, max_batch=24, batched_min=1), 1, x16)
    parts = []
    for r in range(world):
        ctx = _resident(sh, [1], fm.F16, fm.Q4, max_batch=24, batched_min=1, rank=r, world=world)
        parts.append(_run(ctx, 1, x16))
        d = ctx.decisions(24)
        assert all((v.served_enc == 255) == (v.prec == 2 or v.expert % world != r) for v in d)
    np.testing.assert_allclose(np.sum(parts, axis=0), full, rtol=1e-5, atol=1e-6)


def test_k3_setter_errors():
    from paper_2411_01433_b200 import hobbit
    sh = sg.TINY
    ctx = _resident(sh, [0], fm.F16, fm.Q4, max_batch=1)
    with pytest.raises(hobbit.HobbitError):
        ctx.set_batched_min(1)
    ctx.set_batched_min(0)
