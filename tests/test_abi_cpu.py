"""C-ABI checks that need no GPU: the library loads and exports every symbol
include/hobbit.h declares; host logic (blob layout, Theta, the Eq. 3 cache
state machine and prefetch walk) matches the oracle bit for bit."""
import random

import pytest

from oracle import cache as oc
from oracle import formats as fm
from oracle import router as rt
from paper_2411_01433_b200 import _lib as L
from paper_2411_01433_b200.hobbit import (HostCache, blob_bytes, blob_section, canonical_section,
                                          default_config, theta)
from tests import layout_spec as ls


def test_every_header_symbol_is_exported_and_bound():
    syms = L.header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L.lib, s), s
        assert s in L._SIGS, f"{s} has no ctypes signature"


def test_version_and_error_string():
    assert b"sm_100a" in L.lib.hb_version()
    assert isinstance(L.lib.hb_last_error(None), bytes)


@pytest.mark.parametrize("enc", [fm.F16, fm.Q8, fm.Q4, fm.Q2])
@pytest.mark.parametrize("hf", [(256, 512), (4096, 14336), (4096, 6400), (512, 256)])
def test_blob_layout_matches_oracle(enc, hf):
    """hb_canonical_section = the oracle's canonical sections; hb_blob_section =
    the device layout of tests/layout_spec.py; both the same total size."""
    H, F = hf
    assert blob_bytes(enc, H, F) == fm.blob_bytes(enc, H, F)
    lay, _ = fm.blob_layout(enc, H, F)
    for mat in range(3):
        for sec, name in enumerate(["q", "d", "m"]):
            key = "w" if (enc == fm.F16 and name == "q") else name
            if key not in lay[mat]:
                with pytest.raises(L.HobbitError):
                    canonical_section(enc, H, F, mat, sec)
                continue
            assert canonical_section(enc, H, F, mat, sec) == lay[mat][key]
    secs, total = ls.sections(enc, H, F)
    assert total == blob_bytes(enc, H, F)
    for mat, (q, s) in enumerate(secs):
        assert blob_section(enc, H, F, mat, 0)[0] == q
        if s is None:
            with pytest.raises(L.HobbitError):
                blob_section(enc, H, F, mat, 1)
        else:
            assert blob_section(enc, H, F, mat, 1)[0] == s


def test_blob_layout_rejects_bad_dims():
    assert blob_bytes(fm.Q4, 4096, 14300) == 0
    assert blob_bytes(fm.Q4, 4000, 14336) == 0


def test_theta_matches_oracle():
    rnd = random.Random(1)
    ts = [0.6, 0.9, 0.5, 0.0, 1.0, 0.999999, 1e-9, 0.25] + [rnd.random() for _ in range(2000)]
    for t in ts:
        assert theta(t) == rt.theta(t) or (t <= 0 and theta(t) < -(1 << 100)), t


def _cfg(L_, E, k, ch, cl, w, upgrade=1, rank=0, world=1, p=2, both=0):
    return default_config(n_layers=L_, n_experts=E, top_k=k, hidden=256, ffn=512,
                          hi_enc=fm.F16, lo_enc=fm.Q4, w_lru=w[0], w_lfu=w[1], w_lhu=w[2],
                          w_fld=w[3], cap_high=ch, cap_low=cl, allow_upgrade=upgrade,
                          rank=rank, world=world, lookahead_p=p, prefetch_both=both)


def _rand_route(rnd, E, k):
    ex = rnd.sample(range(E), k)
    dec = [rt.HIGH] + [rnd.choice([rt.HIGH, rt.LOW, rt.LOW, rt.SKIP]) for _ in range(k - 1)]
    return ex, dec


@pytest.mark.parametrize("trial", range(16))
def test_host_cache_matches_oracle_bit_exact(trial):
    """hbc_* (the library's cache) vs oracle O9/O10 on random traces, with
    prefetch walks (predicted precision, or both versions Low first: R30),
    explicit loads, sequence resets and EP ranks."""
    rnd = random.Random(100 + trial)
    both = int(trial >= 12)
    L_, E, k = rnd.choice([(4, 8, 2), (6, 8, 2), (5, 16, 2), (4, 8, 3)])
    world = rnd.choice([1, 1, 2])
    rank = rnd.randrange(world)
    p = rnd.randint(0, 3)
    w = (rnd.randint(0, 3), rnd.randint(0, 3), rnd.randint(0, 3), rnd.randint(1, 3))
    if trial % 4 == 3:
        w = (0, 0, 0, 0)                              # Random policy (R29)
    upgrade = rnd.choice([0, 1])
    ch, cl = rnd.randint(2 * k + 2, 10), rnd.randint(2 * k + 2, 10)
    if both:                                          # masks now reach both pools
        ch, cl = ch + 2 * k, cl + 2 * k
    ref = oc.ExpertCache(L_, E, ch, cl, w, fm.F16, fm.Q4, allow_upgrade=bool(upgrade),
                         rank=rank, world=world, prefetch_both=bool(both))
    hc = HostCache(_cfg(L_, E, k, ch, cl, w, upgrade, rank, world, p, both))
    for _ in range(3):
        e = rnd.randrange(E)
        if e % world == rank:
            l = rnd.randrange(L_)
            enc = rnd.choice([fm.F16, fm.Q4])
            ref.load(l, e, enc)
            hc.load(l, e, enc)
    for tok in range(40):
        if rnd.random() < 0.05:
            ref.reset_sequence()
            hc.reset_sequence()
        ref.token_begin()
        hc.token_begin()
        for l in range(L_):
            ex, dec = _rand_route(rnd, E, k)
            served = ref.forward(l, rt.Route(ex, [1.0 / k] * k, dec, [0] * k))
            assert hc.forward(l, ex, dec) == served
            pred = {}
            for j in range(1, p + 1):
                if l + j < L_:
                    pe, pd = _rand_route(rnd, E, k)
                    pred[l + j] = rt.Route(pe, [1.0 / k] * k, pd, [0] * k)
            got = hc.prefetch(l, [(pred[x].experts, pred[x].decisions) for x in sorted(pred)])
            assert got == ref.prefetch(l, pred)
    assert hc.events() == ref.events


def test_host_cache_capacity_error():
    hc = HostCache(_cfg(2, 8, 2, 1, 1, (1, 1, 1, 1)))
    hc.token_begin()
    with pytest.raises(L.HobbitError) as e:
        hc.forward(0, [0, 1], [rt.HIGH, rt.HIGH])
    assert e.value.code == L.HB_ECAPACITY
