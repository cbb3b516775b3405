// Two-pool Eq. 3 expert cache + Sec. 3.3 prefetch walk (see cache.h).
#include "cache.h"

#include <algorithm>
#include <new>

#include "hobbit.h"

namespace hb {

ExpertCache::ExpertCache(int n_layers, int n_experts, int top_k, int cap_high, int cap_low,
                         const int w[4], int hi_enc, int lo_enc, bool allow_upgrade,
                         int rank, int world, bool prefetch_both)
    : L_(n_layers), E_(n_experts), K_(top_k), hi_enc_(hi_enc), lo_enc_(lo_enc),
      upgrade_(allow_upgrade), both_(prefetch_both), rank_(rank), world_(world) {
  for (int i = 0; i < 4; ++i) w_[i] = w[i];
  random_ = w[0] + w[1] + w[2] + w[3] == 0;
  const int nkeys = L_ * E_;
  pool_[POOL_HIGH].assign(std::max(cap_high, 0), -1);
  pool_[POOL_LOW].assign(std::max(cap_low, 0), -1);
  where_[0].assign(nkeys, -1);
  where_[1].assign(nkeys, -1);
  R_.assign(nkeys, 0);
  F_.assign(nkeys, 0);
  H_.assign(nkeys, 0);
  mask_exp_.assign(nkeys, -1);
  cur_.assign(nkeys, 0);
}

// Eq. 3 scaled by T * l_n * (a+b+c+d), an exact integer:
//   P = l_n (a R + b F + c H) + d T (l_n - ((l_t - l_i + l_n) mod l_n))
int64_t ExpertCache::priority(int key, int cur_layer) const {
  const int64_t ln = L_;
  const int lt = key / E_;
  const int64_t dist = ((lt - cur_layer) % L_ + L_) % L_;
  return ln * (w_[0] * R_[key] + w_[1] * F_[key] + w_[2] * H_[key]) +
         (int64_t)w_[3] * T_ * (ln - dist);
}

void ExpertCache::token_begin() {
  ++T_;
  // prefetch never looks past the last layer: every mask has expired
  for (int k : masked_keys_) mask_exp_[k] = -1;
  masked_keys_.clear();
}

void ExpertCache::reset_sequence() {  // records and T only
  std::fill(R_.begin(), R_.end(), 0);
  std::fill(F_.begin(), F_.end(), 0);
  std::fill(H_.begin(), H_.end(), 0);
  T_ = 0;
}

void ExpertCache::drop_masks(int upto_layer) {
  std::vector<int> keep;
  for (int k : masked_keys_) {
    if (mask_exp_[k] <= upto_layer) mask_exp_[k] = -1;
    else keep.push_back(k);
  }
  masked_keys_.swap(keep);
}

void ExpertCache::use(int key, bool high) {  // R = T, F += 1, H += [High]
  R_[key] = T_;
  F_[key] += 1;
  if (high) H_[key] += 1;
}

int ExpertCache::insert(int pool, int key, int cur_layer, bool exclude_current) {
  std::vector<int>& slots = pool_[pool];
  int victim_slot = -1;
  for (size_t i = 0; i < slots.size(); ++i)
    if (slots[i] < 0) { victim_slot = (int)i; break; }
  int victim = -1;
  if (victim_slot < 0) {
    int64_t bp = 0;
    uint64_t br = 0;
    int bk = -1;
    for (size_t i = 0; i < slots.size(); ++i) {
      const int k = slots[i];
      if (masked(k) || (exclude_current && cur_[k])) continue;
      if (random_) {                     // Random policy (all-zero weights, R29)
        const uint64_t r = mix64(mix64(((uint64_t)T_ << 32) + (uint64_t)n_evict_) + (uint64_t)k);
        if (bk < 0 || r < br || (r == br && k < bk)) {
          br = r;
          bk = k;
          victim_slot = (int)i;
        }
        continue;
      }
      const int64_t p = priority(k, cur_layer);
      // argmin over (P, layer, expert); key = layer*E+expert orders (layer, expert)
      if (bk < 0 || p < bp || (p == bp && k < bk)) {
        bp = p;
        bk = k;
        victim_slot = (int)i;
      }
    }
    if (bk < 0) return -1;
    victim = bk;
    ++n_evict_;
    where_[pool][victim] = -1;
  }
  slots[victim_slot] = key;
  where_[pool][key] = victim_slot;
  last_victim_ = victim;
  return victim_slot;
}

int ExpertCache::forward(int layer, const int32_t* experts, const uint8_t* prec,
                         uint8_t* served, int* pool_out, int* slot_out, uint8_t* hit_out) {
  if (T_ == 0) {               // Eq. 3 divides by T: a forward needs token_begin first
    err = "forward before token_begin (T = 0)";
    return HB_ESTATE;
  }
  drop_masks(layer - 1);
  for (int k : cur_list_) cur_[k] = 0;
  cur_list_.clear();
  for (int i = 0; i < K_; ++i) {
    served[i] = HB_ENC_NONE;
    pool_out[i] = -1;
    slot_out[i] = -1;
    hit_out[i] = 0;
    if (prec[i] != HB_SKIP && owned(experts[i])) {
      const int k = key(layer, experts[i]);
      if (!cur_[k]) { cur_[k] = 1; cur_list_.push_back(k); }
    }
  }
  for (int i = 0; i < K_; ++i) {
    const int e = experts[i];
    if (prec[i] == HB_SKIP || !owned(e)) continue;
    const int k = key(layer, e);
    if (prec[i] == HB_HIGH) {
      int s = slot_of(POOL_HIGH, k);
      if (s >= 0) {
        use(k, true);
        events.push_back({EV_HIT, K_ONDEMAND, layer, e, hi_enc_, s, -1});
        hit_out[i] = 1;
      } else {
        s = insert(POOL_HIGH, k, layer, true);
        if (s < 0) { err = "high pool full and every member masked or in use"; return HB_ECAPACITY; }
        use(k, true);
        events.push_back({EV_LOAD, K_ONDEMAND, layer, e, hi_enc_, s, last_victim_});
      }
      served[i] = (uint8_t)hi_enc_;
      pool_out[i] = POOL_HIGH;
      slot_out[i] = s;
    } else {  // HB_LOW
      int s = slot_of(POOL_LOW, k);
      const int sh = slot_of(POOL_HIGH, k);
      if (s >= 0) {
        use(k, false);
        events.push_back({EV_HIT, K_ONDEMAND, layer, e, lo_enc_, s, -1});
        served[i] = (uint8_t)lo_enc_;
        pool_out[i] = POOL_LOW;
        slot_out[i] = s;
        hit_out[i] = 1;
      } else if (upgrade_ && sh >= 0) {  // Low served by the High copy
        use(k, true);
        events.push_back({EV_HIT, K_ONDEMAND, layer, e, hi_enc_, sh, -1});
        served[i] = (uint8_t)hi_enc_;
        pool_out[i] = POOL_HIGH;
        slot_out[i] = sh;
        hit_out[i] = 1;
      } else {
        s = insert(POOL_LOW, k, layer, true);
        if (s < 0) { err = "low pool full and every member masked or in use"; return HB_ECAPACITY; }
        use(k, false);
        events.push_back({EV_LOAD, K_ONDEMAND, layer, e, lo_enc_, s, last_victim_});
        served[i] = (uint8_t)lo_enc_;
        pool_out[i] = POOL_LOW;
        slot_out[i] = s;
      }
    }
  }
  return HB_OK;
}

bool ExpertCache::present(int layer, int expert, int prec) const {
  const int k = key(layer, expert);
  if (prec == HB_HIGH) return slot_of(POOL_HIGH, k) >= 0;
  return slot_of(POOL_LOW, k) >= 0 || (upgrade_ && slot_of(POOL_HIGH, k) >= 0);
}

int ExpertCache::prefetch(int layer, int n_pred, const int32_t* experts, const uint8_t* prec,
                          int* prefetched) {
  *prefetched = -1;
  drop_masks(layer);
  for (int j = 0; j < n_pred; ++j) {
    const int lp = layer + 1 + j;
    if (lp >= L_) break;
    const int32_t* ex = experts + (size_t)j * K_;
    const uint8_t* pr = prec + (size_t)j * K_;
    bool any_missing = false;
    for (int i = 0; i < K_; ++i) {
      if (pr[i] == HB_SKIP || !owned(ex[i])) continue;
      const int k = key(lp, ex[i]);
      if (mask_exp_[k] < 0) masked_keys_.push_back(k);
      mask_exp_[k] = std::max(mask_exp_[k], lp);
    }
    for (int i = 0; i < K_; ++i)
      if (pr[i] != HB_SKIP && owned(ex[i]) && !present(lp, ex[i], pr[i])) any_missing = true;
    if (!any_missing) continue;
    for (int i = 0; i < K_; ++i) {
      if (pr[i] == HB_SKIP || !owned(ex[i]) || present(lp, ex[i], pr[i])) continue;
      // R30 (prefetch_both): the Low version, then the High one, each if its
      // pool lacks the key; else the predicted precision only
      int pools[2], np = 0;
      if (both_) {
        for (int pl : {POOL_LOW, POOL_HIGH})
          if (slot_of(pl, key(lp, ex[i])) < 0) pools[np++] = pl;
      } else {
        pools[np++] = pr[i] == HB_HIGH ? POOL_HIGH : POOL_LOW;
      }
      for (int q = 0; q < np; ++q) {
        const int pool = pools[q];
        const int enc = pool == POOL_HIGH ? hi_enc_ : lo_enc_;
        const int s = insert(pool, key(lp, ex[i]), layer, true);
        if (s < 0) {
          events.push_back({EV_DROP, K_PREFETCH, lp, ex[i], enc, -1, -1});
          continue;
        }
        events.push_back({EV_LOAD, K_PREFETCH, lp, ex[i], enc, s, last_victim_});
      }
    }
    *prefetched = lp;
    return HB_OK;
  }
  return HB_OK;
}

int ExpertCache::load(int layer, int expert, int enc, bool* queued) {
  *queued = false;
  if (enc != hi_enc_ && enc != lo_enc_) { err = "encoding is neither hi_enc nor lo_enc"; return HB_EINVAL; }
  const int pool = pool_of_enc(enc);
  const int k = key(layer, expert);
  if (slot_of(pool, k) >= 0) return HB_OK;
  const int s = insert(pool, k, layer, false);
  if (s < 0) { err = "pool full and every member masked"; return HB_ECAPACITY; }
  events.push_back({EV_LOAD, K_EXPLICIT, layer, expert, enc, s, last_victim_});
  *queued = true;
  return HB_OK;
}

}  // namespace hb

// ------------------------------------------------------- C ABI (host only)
struct hb_cache {
  hb::ExpertCache* c;
  int top_k;
  int n_layers, n_experts, hi_enc, lo_enc;
  std::string err;
};

// argument validation of the host-only ABI (the device context checks the same)
static int bad(hb_cache* c, const char* why) {
  c->err = why;
  return HB_EINVAL;
}
static int check_layer(hb_cache* c, int layer) {
  return layer < 0 || layer >= c->n_layers ? bad(c, "bad layer") : HB_OK;
}
static int check_sel(hb_cache* c, int n, const int32_t* experts, const uint8_t* prec) {
  for (int i = 0; i < n; ++i) {
    if (experts[i] < 0 || experts[i] >= c->n_experts) return bad(c, "bad expert id");
    if (prec[i] > HB_SKIP) return bad(c, "bad precision code");
  }
  return HB_OK;
}

static int check_cfg_cache(const hb_config* cfg, std::string* err) {
  if (!cfg || cfg->n_layers <= 0 || cfg->n_experts <= 0 || cfg->top_k <= 0 ||
      cfg->top_k > cfg->n_experts) { *err = "bad dims"; return HB_EINVAL; }
  if (cfg->w_lru < 0 || cfg->w_lfu < 0 || cfg->w_lhu < 0 || cfg->w_fld < 0 ||
      false) { *err = "bad Eq. 3 weights"; return HB_EINVAL; }
  if (cfg->world <= 0 || cfg->rank < 0 || cfg->rank >= cfg->world) { *err = "bad rank/world"; return HB_EINVAL; }
  if (cfg->hi_enc == cfg->lo_enc) { *err = "hi_enc == lo_enc"; return HB_EINVAL; }
  return HB_OK;
}

extern "C" {

int hbc_create(const hb_config* cfg, hb_cache** out) {
  std::string err;
  if (!out) return HB_EINVAL;
  int rc = check_cfg_cache(cfg, &err);
  if (rc) return rc;
  const int w[4] = {cfg->w_lru, cfg->w_lfu, cfg->w_lhu, cfg->w_fld};
  hb_cache* c = new (std::nothrow) hb_cache;
  if (!c) return HB_ENOMEM;
  c->c = new (std::nothrow) hb::ExpertCache(cfg->n_layers, cfg->n_experts, cfg->top_k,
                                            cfg->cap_high, cfg->cap_low, w, cfg->hi_enc,
                                            cfg->lo_enc, cfg->allow_upgrade != 0, cfg->rank,
                                            cfg->world, cfg->prefetch_both != 0);
  if (!c->c) { delete c; return HB_ENOMEM; }
  c->top_k = cfg->top_k;
  c->n_layers = cfg->n_layers;
  c->n_experts = cfg->n_experts;
  c->hi_enc = cfg->hi_enc;
  c->lo_enc = cfg->lo_enc;
  *out = c;
  return HB_OK;
}

int hbc_destroy(hb_cache* c) {
  if (!c) return HB_EINVAL;
  delete c->c;
  delete c;
  return HB_OK;
}

int hbc_token_begin(hb_cache* c) { if (!c) return HB_EINVAL; c->c->token_begin(); return HB_OK; }
int hbc_reset_sequence(hb_cache* c) { if (!c) return HB_EINVAL; c->c->reset_sequence(); return HB_OK; }

int hbc_forward(hb_cache* c, int layer, const int32_t* experts, const uint8_t* prec,
                uint8_t* served) {
  if (!c || !experts || !prec || !served) return HB_EINVAL;
  if (int rc = check_layer(c, layer)) return rc;
  if (int rc = check_sel(c, c->top_k, experts, prec)) return rc;
  std::vector<int> pool(c->top_k), slot(c->top_k);
  std::vector<uint8_t> hit(c->top_k);
  int rc = c->c->forward(layer, experts, prec, served, pool.data(), slot.data(), hit.data());
  if (rc) c->err = c->c->err;
  return rc;
}

int hbc_prefetch(hb_cache* c, int layer, int n_pred, const int32_t* experts,
                 const uint8_t* prec, int* prefetched) {
  if (!c || !prefetched || n_pred < 0 || (n_pred > 0 && (!experts || !prec))) return HB_EINVAL;
  if (int rc = check_layer(c, layer)) return rc;
  const int np = std::min(n_pred, c->n_layers - 1 - layer);
  if (np > 0)
    if (int rc = check_sel(c, np * c->top_k, experts, prec)) return rc;
  const int rc = c->c->prefetch(layer, n_pred, experts, prec, prefetched);
  if (rc) c->err = c->c->err;
  return rc;
}

int hbc_load(hb_cache* c, int layer, int expert, int enc) {
  if (!c) return HB_EINVAL;
  if (int rc = check_layer(c, layer)) return rc;
  if (expert < 0 || expert >= c->n_experts) return bad(c, "bad expert id");
  if (enc != c->hi_enc && enc != c->lo_enc) return bad(c, "encoding is neither hi_enc nor lo_enc");
  bool q;
  int rc = c->c->load(layer, expert, enc, &q);
  if (rc) c->err = c->c->err;
  return rc;
}

int hbc_get_events(hb_cache* c, hb_event* out, int cap) {
  if (!c || (cap > 0 && !out)) return HB_EINVAL;
  const int n = std::min<int>(cap, (int)c->c->events.size());
  for (int i = 0; i < n; ++i) out[i] = c->c->events[i];
  c->c->events.erase(c->c->events.begin(), c->c->events.begin() + n);
  return n;
}

const char* hbc_last_error(const hb_cache* c) { return c ? c->err.c_str() : "null cache"; }

}  // extern "C"
