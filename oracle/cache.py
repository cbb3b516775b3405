"""O9 two-pool expert cache with the Eq. 3 policy, O10 adaptive prefetch walk.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper, Sec. 3.4: separate caches for high- and low-precision
experts; on every use update the LRU/LFU/LHU records (LHU only for High);
on a miss insert and evict the expert of lowest priority
  p_t = w_lru R_t/T + w_lfu F_t/T + w_lhu H_t/T
        + w_fld (1 - ((l_t - l_i + l_n) % l_n)/l_n)                 (Eq. 3)
R_t last-used time, F_t / H_t (High-)use counts in the current sequence,
T current token number, l_i current layer, l_t layer of expert t, l_n layers.
Records reset at each new sequence.
Sec. 3.3: predict the next layer's experts; if all cached, go on to
the following layer, up to p layers; mask predicted experts against eviction;
prefetch the first layer with a miss.

Readings (R5, R6, R13-R20): weights are integer numerators
(a,b,c,d) and the policy is evaluated exactly as
  P = l_n (a R + b F + c H) + d T (l_n - ((l_t - l_i + l_n) mod l_n))
(= T l_n (a+b+c+d) p_t); victim = argmin (P, layer, expert) over members that
are neither masked nor selected (non-skip) at the current layer; lowest free
slot first; a Low request is served by a cached High version when
allow_upgrade; prefetch fetches the PREDICTED precision (parity unpinned:
the paper says "versions ... with different precision levels"); prefetch
inserts do not update records; a mask lives until its layer's prefetch
call (or the next token).
"""
from __future__ import annotations

from .router import HIGH, LOW, SKIP

# event tuple: (type, kind, layer, expert, enc, slot, victim_key)
EV_HIT, EV_LOAD, EV_DROP = 0, 1, 2
K_ONDEMAND, K_PREFETCH, K_EXPLICIT = 0, 1, 2
POOL_HIGH, POOL_LOW = 0, 1


class CapacityError(RuntimeError):
    pass


class ExpertCache:
    def __init__(self, n_layers, n_experts, cap_high, cap_low, weights,
                 hi_enc, lo_enc, allow_upgrade=True, rank=0, world=1, prefetch_both=False):
        self.L = n_layers
        self.E = n_experts
        self.pools = {POOL_HIGH: [None] * cap_high, POOL_LOW: [None] * cap_low}
        self.w = tuple(int(v) for v in weights)
        if len(self.w) != 4 or min(self.w) < 0:
            raise ValueError("weights must be 4 non-negative ints")
        # all four weights 0: the Random policy of fig:cache-policy-verify
        # (the normaliser of the policy comparison; R29)
        self.random = sum(self.w) == 0
        self.n_evict = 0
        self.hi_enc, self.lo_enc = hi_enc, lo_enc
        self.allow_upgrade = allow_upgrade
        # P:497 "we preload versions of the experts with different precision
        # levels" read as SPEC S:195: both versions, Low first (R30)
        self.prefetch_both = prefetch_both
        self.rank, self.world = rank, world
        self.R, self.F, self.H = {}, {}, {}
        self.T = 0
        self.mask = {}                 # key -> expiry layer
        self.cur_keys = set()          # non-skip selected keys of the last forward
        self.events = []

    # ------------------------------------------------------------ helpers
    def key(self, layer, expert):
        return layer * self.E + expert

    def owned(self, expert):
        return expert % self.world == self.rank

    def slot_of(self, pool, key):
        try:
            return self.pools[pool].index(key)
        except ValueError:
            return -1

    def priority(self, key, cur_layer):
        """Eq. 3 scaled by T*l_n*(a+b+c+d): an exact integer."""
        a, b, c, d = self.w
        lt = key // self.E
        ln = self.L
        return (ln * (a * self.R.get(key, 0) + b * self.F.get(key, 0) + c * self.H.get(key, 0))
                + d * self.T * (ln - ((lt - cur_layer + ln) % ln)))

    @staticmethod
    def _mix64(z):
        """splitmix64 finaliser (the counter-based generator the Random policy
        draws from; the library implements the same one)."""
        z &= (1 << 64) - 1
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & ((1 << 64) - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & ((1 << 64) - 1)
        return z ^ (z >> 31)

    def random_priority(self, key):
        """Random policy: a uniform draw per (eviction, member) --
        mix64(mix64(T * 2^32 + n_evict) + key); the argmin is the victim."""
        return self._mix64(self._mix64((self.T << 32) + self.n_evict) + key)

    def _use(self, key, high):
        self.R[key] = self.T
        self.F[key] = self.F.get(key, 0) + 1
        if high:
            self.H[key] = self.H.get(key, 0) + 1

    def _insert(self, pool, key, cur_layer, exclude):
        """Slot for key in pool: lowest free slot, else evict the Eq. 3 minimum."""
        slots = self.pools[pool]
        for i, k in enumerate(slots):
            if k is None:
                slots[i] = key
                return i, -1
        best = None
        for i, k in enumerate(slots):
            if k in self.mask or k in exclude:
                continue
            pr = self.random_priority(k) if self.random else self.priority(k, cur_layer)
            cand = (pr, k // self.E, k % self.E, i)
            if best is None or cand < best:
                best = cand
        if best is None:
            raise CapacityError(f"pool {pool} full and every member masked or in use")
        i = best[3]
        victim = slots[i]
        slots[i] = key
        self.n_evict += 1
        return i, victim

    # ------------------------------------------------------------ API
    def token_begin(self):
        """T += 1 (Eq. 3 'current token number').  Prefetch never wraps past
        the last layer, so every mask of the previous token has expired."""
        self.T += 1
        self.mask.clear()

    def reset_sequence(self):
        """zero R, F, H and T; pools and masks are kept."""
        self.R.clear()
        self.F.clear()
        self.H.clear()
        self.T = 0

    def _drop_masks(self, upto_layer):
        for k in [k for k, exp in self.mask.items() if exp <= upto_layer]:
            del self.mask[k]

    def forward(self, layer, route):
        """O9 for one token's route at `layer`.

        Returns served[i] per rank i: the encoding computed, or None (Skip or
        not owned).  Appends events.
        """
        self._drop_masks(layer - 1)
        picks = [(i, e, d) for i, (e, d) in enumerate(zip(route.experts, route.decisions))
                 if d != SKIP and self.owned(e)]
        self.cur_keys = {self.key(layer, e) for _, e, _ in picks}
        served = [None] * len(route.experts)
        for i, e, d in picks:
            key = self.key(layer, e)
            if d == HIGH:
                s = self.slot_of(POOL_HIGH, key)
                if s >= 0:
                    self._use(key, True)
                    self.events.append((EV_HIT, K_ONDEMAND, layer, e, self.hi_enc, s, -1))
                else:
                    s, v = self._insert(POOL_HIGH, key, layer, self.cur_keys)
                    self._use(key, True)
                    self.events.append((EV_LOAD, K_ONDEMAND, layer, e, self.hi_enc, s, v))
                served[i] = self.hi_enc
            else:  # LOW
                s = self.slot_of(POOL_LOW, key)
                sh = self.slot_of(POOL_HIGH, key)
                if s >= 0:
                    self._use(key, False)
                    self.events.append((EV_HIT, K_ONDEMAND, layer, e, self.lo_enc, s, -1))
                    served[i] = self.lo_enc
                elif self.allow_upgrade and sh >= 0:
                    self._use(key, True)
                    self.events.append((EV_HIT, K_ONDEMAND, layer, e, self.hi_enc, sh, -1))
                    served[i] = self.hi_enc
                else:
                    s, v = self._insert(POOL_LOW, key, layer, self.cur_keys)
                    self._use(key, False)
                    self.events.append((EV_LOAD, K_ONDEMAND, layer, e, self.lo_enc, s, v))
                    served[i] = self.lo_enc
        return served

    def present(self, layer, expert, decision):
        key = self.key(layer, expert)
        if decision == HIGH:
            return self.slot_of(POOL_HIGH, key) >= 0
        return (self.slot_of(POOL_LOW, key) >= 0
                or (self.allow_upgrade and self.slot_of(POOL_HIGH, key) >= 0))

    def prefetch(self, layer, predicted):
        """O10 after layer `layer`: predicted = {l': Route} for l' = layer+1..layer+p.

        Walks l' in increasing order; masks every predicted non-skip owned key
        with expiry l'; at the first l' with a key absent at its predicted
        precision inserts those keys (rank order, no record update) and stops.
        Returns the prefetched layer or -1.
        """
        self._drop_masks(layer)
        for lp in sorted(predicted):
            r = predicted[lp]
            picks = [(e, d) for e, d in zip(r.experts, r.decisions)
                     if d != SKIP and self.owned(e)]
            for e, _ in picks:
                k = self.key(lp, e)
                self.mask[k] = max(self.mask.get(k, lp), lp)
            missing = [(e, d) for e, d in picks if not self.present(lp, e, d)]
            if not missing:
                continue
            for e, d in missing:
                if self.prefetch_both:
                    # R30: the Low version, then the High one, each if its pool lacks the key
                    todo = [p_ for p_ in (POOL_LOW, POOL_HIGH)
                            if self.slot_of(p_, self.key(lp, e)) < 0]
                else:
                    todo = [POOL_HIGH if d == HIGH else POOL_LOW]
                for pool in todo:
                    enc = self.hi_enc if pool == POOL_HIGH else self.lo_enc
                    try:
                        s, v = self._insert(pool, self.key(lp, e), layer, self.cur_keys)
                    except CapacityError:
                        self.events.append((EV_DROP, K_PREFETCH, lp, e, enc, -1, -1))
                        continue
                    self.events.append((EV_LOAD, K_PREFETCH, lp, e, enc, s, v))
            return lp
        return -1

    def load(self, layer, expert, enc):
        """expert_cache_load: logical insert without a record update (idempotent)."""
        pool = POOL_HIGH if enc == self.hi_enc else POOL_LOW
        key = self.key(layer, expert)
        if self.slot_of(pool, key) >= 0:
            return
        s, v = self._insert(pool, key, layer, set())
        self.events.append((EV_LOAD, K_EXPLICIT, layer, expert, enc, s, v))
