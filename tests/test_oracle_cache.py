"""Pins for oracle/cache.py (O9 Eq. 3 two-pool cache, O10 prefetch walk).

Pins: SPEC worked examples, the simplex corners of Eq. 3 against
independently written pure LRU / LFU / LHU / FLD straight-line replays on
random traces, the mask / current-layer
exclusion invariant, the byte-accounting closed form and the
Fig. fig:predictor walk pattern.
"""
import random

import pytest

from oracle import cache as oc
from oracle.router import HIGH, LOW, SKIP, Route

HI, LO = 0, 2          # hi_enc F16, lo_enc Q4


def _route(experts, decisions, gates=None):
    gates = gates or [1.0 / len(experts)] * len(experts)
    return Route(list(experts), gates, list(decisions), [0] * len(experts))


def _cache(L=32, E=8, ch=4, cl=4, w=(1, 1, 1, 1), **kw):
    return oc.ExpertCache(L, E, ch, cl, w, HI, LO, **kw)


def test_priority_spec_examples():
    """FLD same layer 1.0, next layer 31/32; LRU R=3, T=10 -> 0.3.
    p_t = P / (T * l_n * (a+b+c+d))."""
    c = _cache(w=(0, 0, 0, 1))
    c.T = 7
    k5, k6 = c.key(5, 0), c.key(6, 0)
    assert c.priority(k5, 5) / (c.T * 32 * 1) == 1.0
    assert c.priority(k6, 5) / (c.T * 32 * 1) == 0.96875
    c = _cache(w=(1, 0, 0, 0))
    c.T = 10
    c.R[c.key(0, 3)] = 3
    assert c.priority(c.key(0, 3), 0) / (10 * 32 * 1) == 0.3


def test_on_use_spec_examples():
    """High hit advances R,F,H; Low hit leaves H; two uses in one
    token add 2 to F with R = T."""
    c = _cache()
    c.token_begin()
    c.forward(0, _route([1, 2], [HIGH, LOW]))          # two misses -> loads
    c.token_begin()
    c.forward(0, _route([1, 2], [HIGH, LOW]))          # two hits
    k1, k2 = c.key(0, 1), c.key(0, 2)
    assert (c.R[k1], c.F[k1], c.H[k1]) == (2, 2, 2)
    assert (c.R[k2], c.F[k2], c.H.get(k2, 0)) == (2, 2, 0)
    c.forward(1, _route([1, 2], [HIGH, HIGH]))
    assert c.R[c.key(1, 1)] == 2 and c.F[c.key(1, 1)] == 1


def test_insert_spec_examples():
    """not full -> no eviction; LRU {A:R=1, B:R=4}, T=5 -> evict A;
    {A:R=4, B:R=1} with B masked -> evict A."""
    c = _cache(ch=2, w=(1, 0, 0, 0))
    c.load(0, 0, HI)
    c.load(0, 1, HI)
    assert [e[6] for e in c.events] == [-1, -1]
    A, B = c.key(0, 0), c.key(0, 1)
    c.T, c.R[A], c.R[B] = 5, 1, 4
    c.forward(3, _route([5, 6], [HIGH, SKIP]))
    assert c.events[-1][:2] == (oc.EV_LOAD, oc.K_ONDEMAND) and c.events[-1][6] == A
    c2 = _cache(ch=2, w=(1, 0, 0, 0))
    c2.load(0, 0, HI)
    c2.load(0, 1, HI)
    c2.T, c2.R[A], c2.R[B] = 5, 4, 1
    c2.mask[B] = 9
    c2.forward(3, _route([5, 6], [HIGH, SKIP]))
    assert c2.events[-1][6] == A


def test_reset_sequence_spec_examples():
    """records and T zeroed, pools unchanged; FLD-only priority unchanged."""
    c = _cache(w=(1, 1, 1, 1))
    c.token_begin()
    c.forward(2, _route([0, 3], [HIGH, LOW]))
    pools = {p: list(s) for p, s in c.pools.items()}
    c.reset_sequence()
    assert c.T == 0 and not c.R and not c.F and not c.H
    assert c.pools == pools
    c.T = 4
    assert c.priority(c.key(2, 0), 2) == 1 * 4 * 32        # only the FLD term remains


def test_lookup_spec_examples():
    """Low served by a cached High (upgrade); High never by Low."""
    c = _cache()
    c.token_begin()
    c.load(0, 1, HI)
    served = c.forward(0, _route([4, 1], [HIGH, LOW]))
    assert served == [HI, HI]                      # e1 Low served by its High copy
    assert c.events[-1][0] == oc.EV_HIT and c.events[-1][4] == HI
    c2 = _cache()
    c2.token_begin()
    c2.load(0, 1, LO)
    served = c2.forward(0, _route([1, 3], [HIGH, LOW]))
    assert served[0] == HI and c2.events[-2][0] == oc.EV_LOAD       # High miss
    c3 = _cache(allow_upgrade=False)
    c3.token_begin()
    c3.load(0, 1, HI)
    assert c3.forward(0, _route([4, 1], [HIGH, LOW])) == [HI, LO]


def test_on_miss_tasks_spec_examples():
    """full hit -> no task; [High, Skip] empty pool -> one High task."""
    c = _cache()
    c.token_begin()
    c.forward(0, _route([2, 5], [HIGH, SKIP]))
    loads = [e for e in c.events if e[0] == oc.EV_LOAD]
    assert len(loads) == 1 and loads[0][3] == 2 and loads[0][4] == HI
    n = len(c.events)
    c.token_begin()
    c.forward(0, _route([2, 5], [HIGH, SKIP]))
    assert all(e[0] == oc.EV_HIT for e in c.events[n:])


# ------------------------------------------------- straight-line references

class RefPolicyCache:
    """Independent straight-line two-pool cache with a PURE policy (no Eq. 3):
    'lru' evicts the least recently used, 'lfu' the least frequently used,
    'lhu' the least High-used, 'fld' the farthest layer ahead; ties -> lowest
    (layer, expert)."""

    def __init__(self, policy, L, E, ch, cl):
        self.policy, self.L, self.E = policy, L, E
        self.hp, self.lp = [None] * ch, [None] * cl
        self.last, self.freq, self.hfreq = {}, {}, {}
        self.t = 0
        self.log = []

    def _victim_rank(self, key, layer):
        l, e = divmod(key, self.E)
        if self.policy == "lru":
            v = self.last.get(key, 0)
        elif self.policy == "lfu":
            v = self.freq.get(key, 0)
        elif self.policy == "lhu":
            v = self.hfreq.get(key, 0)
        else:
            v = -((l - layer) % self.L)          # farther ahead = evict first
        return (v, l, e)

    def _put(self, pool, key, layer, busy):
        if None in pool:
            i = pool.index(None)
            pool[i] = key
            return i, -1
        cands = [(self._victim_rank(k, layer), i) for i, k in enumerate(pool) if k not in busy]
        _, i = min(cands)
        v = pool[i]
        pool[i] = key
        return i, v

    def step(self, layer, experts, decisions):
        busy = {layer * self.E + e for e, d in zip(experts, decisions) if d != SKIP}
        for e, d in zip(experts, decisions):
            if d == SKIP:
                continue
            key = layer * self.E + e
            if d == HIGH:
                if key in self.hp:
                    self.log.append(("hit", layer, e, HI))
                else:
                    s, v = self._put(self.hp, key, layer, busy)
                    self.log.append(("load", layer, e, HI, s, v))
                high = True
            else:
                if key in self.lp:
                    self.log.append(("hit", layer, e, LO))
                    high = False
                elif key in self.hp:
                    self.log.append(("hit", layer, e, HI))
                    high = True
                else:
                    s, v = self._put(self.lp, key, layer, busy)
                    self.log.append(("load", layer, e, LO, s, v))
                    high = False
            self.last[key] = self.t
            self.freq[key] = self.freq.get(key, 0) + 1
            if high:
                self.hfreq[key] = self.hfreq.get(key, 0) + 1


def _random_trace(rnd, L, E, n_tok):
    out = []
    for _ in range(n_tok):
        tok = []
        for l in range(L):
            ex = rnd.sample(range(E), 2)
            d1 = rnd.choice([HIGH, HIGH, LOW, LOW, SKIP])
            tok.append((l, ex, [HIGH, d1]))
        out.append(tok)
    return out


def _events_as_ref_log(events):
    log = []
    for ev in events:
        typ, kind, l, e, enc, s, v = ev
        log.append(("hit", l, e, enc) if typ == oc.EV_HIT else ("load", l, e, enc, s, v))
    return log


@pytest.mark.parametrize("policy,w", [("lru", (1, 0, 0, 0)), ("lfu", (0, 1, 0, 0)),
                                      ("lhu", (0, 0, 1, 0)), ("fld", (0, 0, 0, 1))])
def test_simplex_corners_equal_pure_policies(policy, w):
    rnd = random.Random(hash(policy) & 0xFFFF)
    for trial in range(100):
        L, E = rnd.choice([(2, 4), (3, 6), (4, 8)])
        ch, cl = rnd.randint(2, 5), rnd.randint(2, 5)
        c = oc.ExpertCache(L, E, ch, cl, w, HI, LO)
        ref = RefPolicyCache(policy, L, E, ch, cl)
        for tok in _random_trace(rnd, L, E, 50):
            c.token_begin()
            ref.t += 1
            for l, ex, dec in tok:
                c.forward(l, _route(ex, dec))
                ref.step(l, ex, dec)
        assert _events_as_ref_log(c.events) == ref.log, (policy, trial)


def test_masked_and_current_never_victims():
    rnd = random.Random(11)
    for trial in range(50):
        L, E = 6, 8
        c = oc.ExpertCache(L, E, 5, 5, (rnd.randint(0, 3), rnd.randint(0, 3),
                                        rnd.randint(0, 3), rnd.randint(1, 3)), HI, LO)
        for tok in _random_trace(rnd, L, E, 30):
            c.token_begin()
            for l, ex, dec in tok:
                n0 = len(c.events)
                live = {k for k, exp in c.mask.items() if exp >= l}
                c.forward(l, _route(ex, dec))
                cur = {c.key(l, e) for e, d in zip(ex, dec) if d != SKIP}
                for ev in c.events[n0:]:
                    if ev[0] == oc.EV_LOAD and ev[6] >= 0:
                        assert ev[6] not in cur and ev[6] not in live
                if l + 1 < L:
                    pred = {l + 1: _route(rnd.sample(range(E), 2), [HIGH, LOW])}
                    n1 = len(c.events)
                    c.prefetch(l, pred)
                    live = set(c.mask)
                    for ev in c.events[n1:]:
                        if ev[0] == oc.EV_LOAD and ev[6] >= 0:
                            assert ev[6] not in live and ev[6] not in cur


def test_byte_accounting_closed_form():
    """bytes loaded = #High loads * B_hi + #Low loads * B_lo; the miss
    penalty of a Low miss is B_l/B_h of a High miss (1/4 for fp16/int4)."""
    from oracle import formats as fm
    rnd = random.Random(3)
    c = oc.ExpertCache(4, 8, 3, 3, (1, 1, 1, 1), fm.F16, fm.Q4)
    for tok in _random_trace(rnd, 4, 8, 40):
        c.token_begin()
        for l, ex, dec in tok:
            c.forward(l, _route(ex, dec))
    bh, bl = fm.blob_bytes(fm.F16, 4096, 14336), fm.blob_bytes(fm.Q4, 4096, 14336)
    loads = [e for e in c.events if e[0] == oc.EV_LOAD]
    nh = sum(1 for e in loads if e[4] == fm.F16)
    nl = sum(1 for e in loads if e[4] == fm.Q4)
    total = sum(bh if e[4] == fm.F16 else bl for e in loads)
    assert total == nh * bh + nl * bl
    # nominal bit-width ratio 4/16; with block scales 4.5/16
    assert abs(bl / bh - 4.5 / 16) < 1e-12


def test_prefetch_walk_pattern():
    """P:497 / fig:predictor / S:187: layer+1 all cached -> go on; layer+2 has
    a miss -> prefetch layer+2; everything predicted is masked."""
    c = _cache(L=8, E=8, ch=8, cl=8)
    c.token_begin()
    c.forward(0, _route([0, 1], [HIGH, LOW]))
    c.load(1, 2, HI)
    c.load(1, 3, LO)
    pred = {1: _route([2, 3], [HIGH, LOW]), 2: _route([4, 5], [HIGH, LOW]),
            3: _route([6, 7], [HIGH, HIGH])}
    n = len(c.events)
    assert c.prefetch(0, pred) == 2
    new = c.events[n:]
    assert [(e[0], e[1], e[2], e[3], e[4]) for e in new] == [
        (oc.EV_LOAD, oc.K_PREFETCH, 2, 4, HI), (oc.EV_LOAD, oc.K_PREFETCH, 2, 5, LO)]
    assert set(c.mask) == {c.key(1, 2), c.key(1, 3), c.key(2, 4), c.key(2, 5)}
    assert c.R.get(c.key(2, 4)) is None                  # no record update on prefetch
    # all predicted present -> nothing loaded, masks still set
    assert c.prefetch(0, {1: _route([2, 3], [HIGH, LOW])}) == -1


def test_mask_expiry():
    c = _cache(L=8, E=8)
    c.token_begin()
    c.forward(0, _route([0, 1], [HIGH, SKIP]))
    c.prefetch(0, {1: _route([2, 3], [HIGH, SKIP])})
    assert c.key(1, 2) in c.mask
    c.forward(1, _route([2, 3], [HIGH, SKIP]))
    assert c.key(1, 2) in c.mask                          # lives through layer 1
    c.prefetch(1, {})
    assert c.key(1, 2) not in c.mask


def test_capacity_error():
    c = _cache(ch=1, cl=1)
    c.token_begin()
    with pytest.raises(oc.CapacityError):
        c.forward(0, _route([0, 1], [HIGH, HIGH]))


def test_ep_owned_only():
    c = oc.ExpertCache(4, 8, 4, 4, (1, 1, 1, 1), HI, LO, rank=1, world=2)
    c.token_begin()
    served = c.forward(0, _route([2, 3], [HIGH, LOW]))
    assert served == [None, LO]
    assert all(e[3] % 2 == 1 for e in c.events)


def test_random_policy_uniform_and_record_free():
    """R29 (P:1040's Random normaliser): all-zero Eq. 3 weights pick the victim
    uniformly among the eligible members, independently of the records.
    Pool of 4 High slots, one layer of 8 experts: insert the non-member keys
    round robin so every insert evicts; over 4000 evictions each of the 4
    eligible members is chosen 1000 +- 150 times (binomial sd ~ 27)."""
    c = oc.ExpertCache(1, 64, 4, 1, (0, 0, 0, 0), 0, 2)
    c.token_begin()
    for e in range(4):
        c.load(0, e, 0)
    counts = {}
    nxt = 4
    for i in range(4000):
        before = list(c.pools[oc.POOL_HIGH])
        c.load(0, nxt % 64, 0) if (nxt % 64) not in before else None
        after = c.pools[oc.POOL_HIGH]
        for j, (a, b) in enumerate(zip(before, after)):
            if a != b:
                counts[j] = counts.get(j, 0) + 1
        nxt += 1
        if i % 50 == 0:
            c.token_begin()
    assert sorted(counts) == [0, 1, 2, 3]
    assert all(850 <= v <= 1150 for v in counts.values()), counts
    # the records do not matter: two caches with different use histories
    # choose the same victims
    a = oc.ExpertCache(1, 8, 2, 1, (0, 0, 0, 0), 0, 2)
    b = oc.ExpertCache(1, 8, 2, 1, (0, 0, 0, 0), 0, 2)
    for cc in (a, b):
        cc.token_begin()
        cc.load(0, 0, 0)
        cc.load(0, 1, 0)
    b.R[0], b.F[0], b.H[0] = 7, 9, 9
    for e in (2, 3, 4, 5):
        a.load(0, e, 0)
        b.load(0, e, 0)
    assert a.pools == b.pools


def test_prefetch_both_versions_low_first():
    """R30 ("versions ... with different precision levels"):
    prefetch_both loads the Low version of each missing predicted expert, then
    the High one, each only where its pool lacks the key; the walk itself
    (which layer has a miss) is unchanged."""
    c = oc.ExpertCache(8, 8, 8, 8, (1, 1, 1, 1), HI, LO, prefetch_both=True)
    c.token_begin()
    c.forward(0, _route([0, 1], [HIGH, LOW]))
    c.load(1, 3, LO)                                   # expert 3 of layer 1: Low present
    n = len(c.events)
    assert c.prefetch(0, {1: _route([2, 3], [HIGH, HIGH])}) == 1
    new = [(e[0], e[1], e[2], e[3], e[4]) for e in c.events[n:]]
    assert new == [(oc.EV_LOAD, oc.K_PREFETCH, 1, 2, LO), (oc.EV_LOAD, oc.K_PREFETCH, 1, 2, HI),
                   (oc.EV_LOAD, oc.K_PREFETCH, 1, 3, HI)]
    # a predicted-Low miss also brings both versions
    n = len(c.events)
    assert c.prefetch(1, {2: _route([4, 5], [LOW, SKIP])}) == 2
    assert [(e[3], e[4]) for e in c.events[n:]] == [(4, LO), (4, HI)]
    # without the option: the predicted precision only
    d = oc.ExpertCache(8, 8, 8, 8, (1, 1, 1, 1), HI, LO)
    d.token_begin()
    d.forward(0, _route([0, 1], [HIGH, LOW]))
    d.prefetch(0, {1: _route([2, 3], [HIGH, LOW])})
    assert [(e[3], e[4]) for e in d.events if e[1] == oc.K_PREFETCH] == [(2, HI), (3, LO)]
