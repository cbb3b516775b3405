"""GPU parity of the k-quant encoding HB_Q2K (llama.cpp's Q2_K arithmetic,
DESIGN.md R32/R33) through the C-ABI against the oracle.

  * quantiser bytes three ways (library quantiser; hb_repack_canonical of the
    oracle's canonical blob; tests/layout_spec.py on the CPU);
  * decode-layer parity for the pairs F16/Q2K and Q8/Q2K at the tiny shape
    (B = 1, 5, 16 on the GEMV path; B = 4, 16, 40 on the tcgen05 path) and at
    the full Mixtral shape; bar 1e-3 normwise: the kernels form each Q2K
    weight in fp16 (the scale products and the fma each round once) where the
    other encodings keep exact integer codes (R34);
  * the offload path: cache events reported with HB_Q2K, bit-exact with O9/O10.
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
from tests.gpu_util import OracleStore, gpu_blobs, rel_err  # noqa: E402
from tests.test_gpu_parity import _check_routes, _ctx, _resident, _run  # noqa: E402
from tests.test_gpu_parity import test_quantiser_bytes_bit_exact as _qbytes  # noqa: E402

TOL_Q2K = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("shape", [sg.TINY, sg.MoEShape("phi-slice", 1, 1, 2, 4096, 6400, 1.8)],
                         ids=["tiny", "phi"])
def test_q2k_quantiser_bytes_bit_exact(shape):
    _qbytes(fm.Q2K, shape)


@pytest.mark.parametrize("hi", [fm.F16, fm.Q8], ids=["F16-Q2K", "Q8-Q2K"])
@pytest.mark.parametrize("B", [1, 5, 16])
def test_q2k_layer_parity_tiny(hi, B):
    sh = sg.TINY
    ctx = _resident(sh, [0, 1], hi, fm.Q2K, max_batch=16)
    store = OracleStore(sh)
    for l in range(sh.n_layers):
        x16 = sg.hidden_states(sh, 30 + B, l, batch=B)
        y = _run(ctx, l, x16)
        ref, routes = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, hi, fm.Q2K)
        _check_routes(ctx, routes, B, 2)
        served = [[d.served_enc for d in ctx.decisions(B)[2 * b:2 * b + 2]] for b in range(B)]
        for b, r in enumerate(routes):
            for i, dec in enumerate(r.decisions):
                want = 255 if dec == rt.SKIP else (hi if dec == rt.HIGH else fm.Q2K)
                assert served[b][i] == want
            assert rel_err(y[b], ref[b])[0] <= TOL_Q2K, b


@pytest.mark.parametrize("hi", [fm.F16, fm.Q8], ids=["F16-Q2K", "Q8-Q2K"])
@pytest.mark.parametrize("B", [4, 16, 40])
def test_q2k_batched_tcgen05_parity(hi, B):
    """The tcgen05 grouped GEMM (K3) with Q2K items: the converters dequantise
    the 20-byte records (R34) into the A operand."""
    sh = sg.TINY
    ctx = _resident(sh, [0], hi, fm.Q2K, max_batch=40, batched_min=4)
    store = OracleStore(sh)
    x16 = sg.hidden_states(sh, 50 + B, 0, batch=B)
    y = _run(ctx, 0, x16)
    ref, routes = om.moe_layer(x16, sg.router_weights(sh, 0), store, 0, 2, 0.6, 0.9, hi, fm.Q2K)
    _check_routes(ctx, routes, B, 2)
    assert sum(d == rt.LOW for r in routes for d in r.decisions) >= 1
    for b in range(B):
        assert rel_err(y[b], ref[b])[0] <= TOL_Q2K, b


def test_q2k_layer_parity_full_size():
    sh1 = sg.MoEShape("mixtral", 32, 8, 2, 4096, 14336, 1.5)
    layer = 5
    ctx = _resident(sh1, [layer], fm.F16, fm.Q2K)
    store = OracleStore(sh1)
    wg = sg.router_weights(sh1, layer)
    lows = 0
    for t in range(3):
        x16 = sg.hidden_states(sh1, 200 + t, layer)
        y = _run(ctx, layer, x16)
        ref, routes = om.moe_layer(x16, wg, store, layer, 2, 0.6, 0.9, fm.F16, fm.Q2K)
        _check_routes(ctx, routes, 1, 2)
        lows += sum(d == rt.LOW for d in routes[0].decisions)
        assert rel_err(y[0], ref[0])[0] <= TOL_Q2K
    assert lows >= 1, "the sample must exercise the Q2K expert"


@pytest.mark.parametrize("dc", [0, 1])
def test_q2k_offload_events(dc):
    sh = sg.MoEShape("tiny4", 4, 8, 2, 256, 512, 1.5)
    ch, cl = 5, 5
    ctx = _ctx(sh, fm.F16, fm.Q2K, max_batch=1, cap_high=ch, cap_low=cl, lookahead_p=1,
               device_cache=dc)
    for l in range(sh.n_layers):
        ctx.set_router(l, sg.router_weights(sh, l))
        for (e, enc), b in gpu_blobs(sh, l, range(sh.n_experts), [fm.F16, fm.Q2K]).items():
            ctx.register_expert(l, e, enc, b.cpu().numpy())
    store = OracleStore(sh)
    ref = oc.ExpertCache(sh.n_layers, sh.n_experts, ch, cl, (1, 1, 1, 1), fm.F16, fm.Q2K)
    xs = sg.correlated_states(sh, 6, 0.999, 0.5)
    for t in range(6):
        ctx.token_begin()
        ref.token_begin()
        for l in range(sh.n_layers):
            x16 = xs[t, l][None, :]
            x = torch.from_numpy(x16).cuda()
            y = _run(ctx, l, x16)
            served = ref.forward(l, rt.route(x16, sg.router_weights(sh, l), 2, 0.6, 0.9)[0])
            r, _ = om.moe_layer(x16, sg.router_weights(sh, l), store, l, 2, 0.6, 0.9, fm.F16,
                                fm.Q2K, served=[served])
            assert rel_err(y[0], r[0])[0] <= TOL_Q2K
            ctx.prefetch(l, x)
            ref.prefetch(l, {l + 1: rt.route(x16, sg.router_weights(sh, l + 1), 2, 0.6, 0.9)[0]}
                         if l + 1 < sh.n_layers else {})
    torch.cuda.synchronize()
    ev = ctx.events()
    assert ev == ref.events
    assert any(e[4] == fm.Q2K for e in ev)


def test_q2k_phi_full_size():
    """Phi shapes (F = 6400: W2 has 25 Q2K groups per row, K2b's unstaged-h path)."""
    sh1 = sg.MoEShape("phi", 32, 16, 2, 4096, 6400, 1.8)
    layer = 3
    ctx = _resident(sh1, [layer], fm.F16, fm.Q2K)
    store = OracleStore(sh1)
    wg = sg.router_weights(sh1, layer)
    lows = 0
    for t in range(4):
        x16 = sg.hidden_states(sh1, 300 + t, layer)
        y = _run(ctx, layer, x16)
        ref, routes = om.moe_layer(x16, wg, store, layer, 2, 0.6, 0.9, fm.F16, fm.Q2K)
        _check_routes(ctx, routes, 1, 2)
        lows += sum(d == rt.LOW for d in routes[0].decisions)
        assert rel_err(y[0], ref[0])[0] <= TOL_Q2K
    assert lows >= 1
