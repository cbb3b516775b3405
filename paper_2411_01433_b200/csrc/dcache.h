// Device-resident expert cache manager + GPU-initiated loads (dcache.cu).
#pragma once

#include "hb_internal.h"

namespace hb {

// One load task per (pool, slot): the blob of the key that slot holds.
struct DcTask {
  const uint8_t* src;           // blob in mapped pinned host memory (device address)
  uint8_t* dst;                 // the slot in HBM
  unsigned long long bytes;
  unsigned nchunks;
  unsigned gen;                 // bumped per new task of this slot
  unsigned long long ctl;       // (gen << 32) | next chunk to claim
  unsigned long long done;      // (gen << 32) | chunks copied
  unsigned rw;                  // bit 31: being replaced; low bits: copiers holding the slot
  int fg;                       // needed by the current forward
  unsigned long long seq;       // creation order (background: oldest first)
  int live;
  int layer;                    // the key's layer
  int bg;                       // 1: prefetch task (background until a forward needs it)
};

// Cache state in HBM (arrays allocated by the context; the struct itself too).
struct DcState {
  int L, E, K, cap[2], w[4], hi_enc, lo_enc, upgrade, rank, world, random;
  int both;                     // prefetch both versions, Low first (R30)
  long long T;
  unsigned long long n_evict;
  int* pool[2];                 // slot -> key or -1
  int* where[2];                // key -> slot or -1
  long long *R, *F, *H;         // per key records
  int* mask_exp;                // key -> expiry layer or -1
  int* masked_keys;             // keys with a live mask
  int n_masked;
  char* cur;                    // key selected (non-skip) at the current layer
  int* cur_list;
  int n_cur;
  hb_event* log;                // event log (drained by hb_get_events)
  int log_n, log_cap, log_overflow;
  int err;                      // sticky HB_E* code (pool full ...)
  uint8_t* pool_mem[2];
  unsigned long long slot_bytes[2];
  unsigned long long bbytes[4];
  unsigned long long chunk;     // bytes per copy chunk
  DcTask* task[2];              // [cap[pool]]
  unsigned long long seq;
  int need[kMaxTopK];           // pool * 65536 + slot of the current forward's served slots
  int n_need;
  int yield;                    // 1: background copiers stop claiming chunks
  int cur_layer;                // layer of the last forward (background skips stale prefetches)
  unsigned fg_exit;             // foreground CTAs done (self-resetting)
  unsigned long long bytes_fg, bytes_bg;   // bytes copied by the foreground / background copiers
};

enum { DC_FORWARD = 0, DC_PREFETCH = 1, DC_LOAD = 2 };

struct DcParams {
  int op;
  int layer;
  int n_pred;                   // prefetch: routed lookahead layers
  int expert, enc;              // load
  int do_reset, t_add, clear_masks;   // hb_reset_sequence / hb_token_begin since the last op
  hb_decision* dec;             // forward: [K] (served_enc / hit written); prefetch: [n_pred][K]
  const uint8_t* const* host_blob;   // [L][E][4] device addresses of the host blobs
  JobTable jt;                  // forward: the job table K2 reads
  int H, F;
  int* err_host;                // mapped pinned word: sticky error for the host
};

cudaError_t launch_dc_op(DcState* st, const DcParams& p, cudaStream_t s);
cudaError_t launch_dc_copy_fg(DcState* st, int ctas, cudaStream_t s);
cudaError_t launch_dc_copy_bg(DcState* st, int ctas, cudaStream_t s);

}  // namespace hb
