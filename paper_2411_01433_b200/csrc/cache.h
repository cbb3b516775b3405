// Two-pool expert cache with the Eq. 3 policy and the Sec. 3.3 prefetch walk
// (host state machine of the offload path).
//
// Paper: Sec. 3.4, P:619-633 (Eq. 3, separate high/low precision caches,
// record update on use, LHU only for High, per-sequence reset); Sec. 3.3,
// P:497 (predict next layers, walk while all cached, mask predictions,
// prefetch the first layer with a miss).  Readings: DESIGN.md R5, R6, R13-R20.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hobbit.h"

namespace hb {

enum { EV_HIT = 0, EV_LOAD = 1, EV_DROP = 2 };
enum { K_ONDEMAND = 0, K_PREFETCH = 1, K_EXPLICIT = 2 };
enum { POOL_HIGH = 0, POOL_LOW = 1 };

class ExpertCache {
 public:
  ExpertCache(int n_layers, int n_experts, int top_k, int cap_high, int cap_low,
              const int w[4], int hi_enc, int lo_enc, bool allow_upgrade, int rank,
              int world, bool prefetch_both = false);

  void token_begin();
  void reset_sequence();

  // O9 for one token at `layer`.  experts/prec: top_k in rank order.
  // served[i]: encoding computed or HB_ENC_NONE; pool_out/slot_out[i]: where
  // the served copy lives (-1 if none); hit_out[i]: 1 if resident before.
  // New load events are appended to `events` (and returned via first_new).
  int forward(int layer, const int32_t* experts, const uint8_t* prec, uint8_t* served,
              int* pool_out, int* slot_out, uint8_t* hit_out);

  // O10: n_pred lookahead layers [n_pred][top_k].  *prefetched = layer or -1.
  int prefetch(int layer, int n_pred, const int32_t* experts, const uint8_t* prec,
               int* prefetched);

  // expert_cache_load: logical insert without record update (idempotent).
  int load(int layer, int expert, int enc, bool* queued);

  int key(int layer, int expert) const { return layer * E_ + expert; }
  bool owned(int expert) const { return expert % world_ == rank_; }
  int slot_of(int pool, int key) const { return where_[pool][key]; }
  int pool_of_enc(int enc) const { return enc == hi_enc_ ? POOL_HIGH : POOL_LOW; }
  int64_t priority(int key, int cur_layer) const;
  static uint64_t mix64(uint64_t z) {              // splitmix64 finaliser (Random policy)
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }

  std::vector<hb_event> events;   // drained by the caller
  std::string err;

 private:
  bool masked(int key) const { return mask_exp_[key] >= 0; }
  void drop_masks(int upto_layer);
  void use(int key, bool high);
  // returns slot >= 0, sets *victim (key or -1); -1 if nothing is eligible
  int insert(int pool, int key, int cur_layer, bool exclude_current);
  bool present(int layer, int expert, int prec) const;

  int L_, E_, K_;
  int w_[4];
  int hi_enc_, lo_enc_;
  bool upgrade_;
  bool both_;                           // prefetch both versions, Low first (R30)
  int rank_, world_;
  int64_t T_ = 0;
  bool random_ = false;                            // all Eq. 3 weights 0: Random policy
  uint64_t n_evict_ = 0;
  std::vector<int> pool_[2];            // slot -> key or -1
  std::vector<int> where_[2];           // key -> slot or -1
  std::vector<int64_t> R_, F_, H_;      // per key records
  std::vector<int> mask_exp_;           // key -> expiry layer or -1
  std::vector<int> masked_keys_;        // keys with a live mask
  std::vector<char> cur_;               // key selected (non-skip) at the current layer
  std::vector<int> cur_list_;
  int last_victim_ = -1;                // victim of the last insert()
};

}  // namespace hb
