// Internal declarations shared by the library's translation units.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hobbit.h"

namespace hb {

constexpr int kMaxTopK = 8;
constexpr int kStampStride = 16;        // u64 per hb_stamps record
constexpr int kMaxRouteLayers = 5;      // max lookahead p (routers stacked in one launch)
constexpr int kNumSM = 148;             // B200
#ifndef HB_GEMV_WARPS
#define HB_GEMV_WARPS 12   // 12 x 168 registers: no spills (16 x 128 spilled 700 B; r01 sweep 8/10/12/14/16)
#endif
#ifndef HB_WARP_SMEM_KB
#define HB_WARP_SMEM_KB 13
#endif
constexpr int kGemvWarps = HB_GEMV_WARPS;   // warps per GEMV CTA (one CTA per SM)
constexpr int kRouterThreads = 512;

// Byte offsets of the sections of one matrix inside an expert blob.
// Tile-major layout: unit (tile of 16 rows, 64-byte group) = 1 KB of codes at
// q + 1024*unit, and 16 scale records of SB bytes at s + 16*SB*unit.
struct MatLayout {
  uint64_t q;        // code section (the permuted fp16 values for F16)
  uint64_t s;        // scale section: per (unit, row) d[BPG] (+ m[BPG] for Q2)
};
struct BlobLayout {
  MatLayout mat[3];  // W1 [F,H], W3 [F,H], W2 [H,F]
  uint64_t total;
};
int blob_layout(int enc, int hidden, int ffn, BlobLayout* out);   // host
// Canonical blob (include/hobbit.h): per matrix the code
// section q (row-major, LSB first), d [N][K/32] and (Q2) m, 256-byte aligned.
struct CanonLayout {
  uint64_t q[3], d[3], m[3];   // section offsets per matrix (0 when absent); Q2K: m = dmin
  uint64_t sc[3];              // Q2K: the sub-block bytes [N][K/16]
  uint64_t total;
};
int canonical_layout(int enc, int hidden, int ffn, CanonLayout* out);   // host
// canonical (device) -> device layout (device), stream-ordered
int launch_repack_canonical(int enc, int hidden, int ffn, const uint8_t* src, uint8_t* dst,
                            cudaStream_t s);

// One (expert, served encoding) group of a layer on this rank: the GEMV
// kernels stream its blob once for all of its token slots.
struct Job {
  const uint8_t* blob;
  int32_t enc;
  int32_t expert;
  int32_t n_tok;       // token slots of this job
  int32_t slot_off;    // first slot in slot_token / slot_gate / h
};

// Virtual job: <= kVSlots token slots of one job (one mma N tile), the unit
// of the GEMV kernels' work space.
constexpr int kVSlots = 8;
constexpr int kMaxVJobs = 256;         // per forward (checked at hb_create)
struct VJobD {
  const uint8_t* blob;
  int32_t enc;
  int32_t slot0;
  int32_t nslot;
  int32_t pad;
};

// Device job table of one forward: [hdr | jobs | slot_token | slot_gate | tok_slots |
// vjobs | vcum13 | vcum2]
struct JobTable {
  int32_t* hdr;        // [0] n_jobs, [1] n_slots, [2] n_vjobs
  Job* jobs;           // max_jobs
  int32_t* slot_token; // max_slots
  float* slot_gate;    // max_slots
  int32_t* tok_slots;  // [max_batch][top_k] slot of each (token, rank) or -1, rank order
  VJobD* vjobs;        // max_vjobs
  long long* vcum13;   // [max_vjobs + 1] K2a units before vjob v (last = total)
  long long* vcum2;    // [max_vjobs + 1] K2b units before vjob v
};

#if defined(__CUDACC__)
#define HB_HD __host__ __device__
#else
#define HB_HD
#endif
HB_HD inline int epg_of_enc(int enc) {
  return enc == HB_F16 ? 32 : enc == HB_Q8 ? 64 : enc == HB_Q4 ? 128 : 256;
}
// Split jobs into virtual jobs and lay out the unit spaces of K2a (tiles of
// F rows x groups of H) and K2b (tiles of H rows x groups of F).
HB_HD inline int build_vjobs(const Job* jobs, int nj, int H, int F, VJobD* vj, long long* c13,
                             long long* c2) {
  int nv = 0;
  long long u13 = 0, u2 = 0;
  for (int j = 0; j < nj; ++j) {
    for (int s = 0; s < jobs[j].n_tok; s += kVSlots) {
      VJobD d;
      d.blob = jobs[j].blob;
      d.enc = jobs[j].enc;
      d.slot0 = jobs[j].slot_off + s;
      d.nslot = jobs[j].n_tok - s < kVSlots ? jobs[j].n_tok - s : kVSlots;
      d.pad = 0;
      vj[nv] = d;
      c13[nv] = u13;
      c2[nv] = u2;
      u13 += (long long)(F / 16) * (H / epg_of_enc(d.enc));
      u2 += (long long)(H / 16) * (F / epg_of_enc(d.enc));
      ++nv;
    }
  }
  c13[nv] = u13;
  c2[nv] = u2;
  return nv;
}

struct RouterParams {
  const __half* x;                     // [B, H]
  const __half* wg[kMaxRouteLayers];   // router of each routed layer
  int n_route;                         // routed layers in this launch
  int B, E, H, F, k;
  int64_t theta1, theta2;              // k = 2 exact gap test
  int th1_kind, th2_kind;              // 0 finite, +1 always true, -1 never
  double t1, t2;                       // k > 2 fp64 test
  int rank, world;
  int strict;                          // 0: Low served by hi_enc when the expert is touched High (R27)
  int no_vjobs;                        // the forward runs K3 (own vjob3 table): skip the GEMV vjob table
  hb_decision* dec;                    // [n_route][B][k]
  long long* lbuf;                     // [n_route][B][E][2] exact logits (scratch)
  int* rowbad;                         // [n_route][B] non-finite x flags (scratch)
  int filtered;                        // decode (B = 1, k = 2, cluster): filtered router
  int filtered_batch;                  // batches (one CTA per row): filtered router
  const float* wnorm;                  // [E] ||W_e||_2 of route layer 0 (filtered router)
  __half* x_save;                      // [H] copy of x (filtered router: lazy exact logits)
  long long* logits;                   // [B][E][2] copy for route 0, or null
  uint4* x_perm;                       // [B][H/8] pair-permuted x, or null
  float* xsum;                         // [B][H/32], or null
  float* zero_buf[3];                  // zeroed by the router grid: K2a sums, y, the other sum buffer
  long long zero_n[3];                 // floats
  // resident job building (blob_table != null): last CTA builds the table
  const uint8_t* const* blob_table;    // [E][4] device blob of (expert, enc) for this layer
  int hi_enc, lo_enc;
  JobTable jt;
  unsigned* done;                      // grid completion counter (self-resetting)
  unsigned long long* stamps;          // hb_stamps records (diagnostic HB_LEGACY_TL build only)
  int stamp_cap;
  const unsigned* fwd_idx;
};

struct GemvParams {
  JobTable jt;
  BlobLayout lay[4];
  int H, F, B, k;
  const __half* x_raw;                 // [B][H] the caller's x (fused decode kernel)
  const uint4* x_perm;                 // [B][H/8]
  const float* xsum;                   // [B][H/32]
  float* au;                           // [slots][2][F] K2a sums W1 x | W3 x (zeroed by router)
  uint4* h_hi;                         // [slots][F/8]  pair-permuted fp16 hi part of h  (h_global)
  uint4* h_lo;                         // [slots][F/8]  fp16 residual h - hi             (h_global)
  float* hsum;                         // [slots][F/32] block sums of h                  (h_global)
  int h_global;                        // K2b reads h from h_hi/h_lo/hsum (built by launch_hfin)
                                       // instead of building it in shared memory per CTA
  float* y;                            // [B][H] (zeroed by router)
  const int* rowbad;                   // [B] router's non-finite x flags: NaN rows (R28)
  int hfin_tail;                       // K2a ends with a grid barrier + h (no hfin kernel)
  int kq;                              // the Q2 slot holds HB_Q2K blobs (R32)
  int det;                             // hb_config.deterministic: whole row tiles dealt statically
  int ctas;                            // K2a / K2b grid (<= kGemvCTAs)
  int clean;                           // hfin zeroes the K2a sums it read and the y rows (the
                                       // solo router zeroes nothing)
  int keep_y;                          // hfin leaves y alone (second chain of a split forward)
  unsigned* gbar;                      // that grid barrier [count, generation] (self-resetting)
  // work feed: a static share of the units, then dynamic chunks (K2)
  unsigned* ctr;                       // chunk counters: [0] K2a, [1] K2b, [2 + q] K2a group q, [2 + 148 + q] K2b group q
  int max_vjobs;                       // table entries to preload (>= n_vjobs + 1)
  float static_frac;                   // K2a: fraction of units dealt as static warp ranges
  float static_frac2;                  // K2b
  int chunk;                           // units per dynamic chunk
  float k2b_w[4];                      // K2b CTA split: cost of a unit per encoding (F16 = 1)
  // in-kernel %globaltimer records (hb_stamps), legacy chain: K2a start/end,
  // K2b h-staged/end; null = off
  unsigned long long* stamps;
  int stamp_cap;
  unsigned* fwd_idx;                   // [record index, exit counter]
};

// Fused decode kernel (batch 1, top-2, resident): router + K2a + K2b in one
// launch per layer (gemv.cu)
struct FusedParams {
  GemvParams g;                        // g.x_raw = x, g.au = this forward's sum buffer
  const __half* wg;                    // router rows of the layer [E][H]
  const uint8_t* const* blob_table;    // [E][4] device blob of (expert, enc)
  int E;
  const float* wnorm;                  // [E] ||W_e||_2 rounded up (hb_set_router)
  int64_t theta1, theta2;
  int th1_kind, th2_kind;
  int rank, world, hi_enc, lo_enc;
  hb_decision* dec;                    // [2] decision records (written by CTA 0)
  __half* x_save;                      // [H] copy of x for hb_get_logits, or null
  float* zero_other;                   // the other sum buffer, zeroed for the next forward
  long long zero_n;
  unsigned* gbar;                      // grid barrier [count, generation] (self-resetting)
  unsigned long long* stamps;          // profile records [cap][kStampStride] or null
  int stamp_cap;
  unsigned* fwd_idx;                   // [record index, exit counter]
  int router_only;                     // one CTA: decisions, job table, x_perm / xsum only
};
// split = false: router + K2a + grid barrier + K2b (one kernel); true:
// router + K2a only (writes the global job table), the caller follows with
// launch_hfin + launch_w2
void launch_fused(const FusedParams& p, bool split, cudaStream_t s);
bool fused_fits(int E, int H, int F, int hi_enc, int lo_enc);
void launch_router(const RouterParams& p, cudaStream_t s);

// Token-sharded expert parallelism (router.cu): the tokens of
// a layer are split over the ranks; each rank routes its own tokens, sends
// one row per (token, owner rank) -- x and the token's selections that rank
// owns -- computes the rows it received as one batch, and sends each row's
// gate-weighted expert sum back, where each token sums its rows.  Fixed
// capacity C = max_batch rows per (source, dest): no counts exchange, no host
// sync.
struct TsParams {
  const hb_decision* dec;      // local decisions [B][k] (the router's)
  const __half* x;             // local x [B][H]
  int B, k, H, R, C;
  int* pos;                    // [B][k] row dest * C + position of the selection's owner, or -1
  hb_ts_meta* meta_send;       // [R][C]
  __half* rows_send;           // [R][C][H]
  const float* ret;            // [R][C][H] gate-weighted expert outputs of this rank's rows
  float* y;                    // [B][H]
  const int* rowbad;           // [B] non-finite x (R28): NaN row
};
void launch_ts_pack(const TsParams& p, cudaStream_t s);
void launch_ts_combine(const TsParams& p, cudaStream_t s);
// decisions (one selection per received row, the rest Skip), pair-permuted x,
// zeroed rowbad and y, then the job table (p.blob_table) of the n = p.B rows
void launch_ts_jobs(const RouterParams& p, const hb_ts_meta* meta, const __half* rows, float* y,
                    cudaStream_t s);
// batch-1 decode router on one reserved SM (router.cu); the GEMV kernels then
// run on kNumSM - 1 CTAs and hfin cleans the sums / zeroes y (GemvParams::clean)
bool router_solo_fits(int E, int H, int k);
void launch_router_solo(const RouterParams& p, cudaStream_t s);
// kernel launch allowing programmatic dependent launch (the kernel overlaps
// the tail of its predecessor in the stream and orders itself with
// griddepcontrol.wait before touching the predecessor's outputs)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, int smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
// cudaFuncAttributeMaxDynamicSharedMemorySize is per device: set it once per
// (kernel, current device), thread-safe (a process may drive several GPUs)
cudaError_t set_max_dyn_smem_impl(const void* kernel, int bytes);
template <typename... KArgs>
inline cudaError_t set_max_dyn_smem(void (*kernel)(KArgs...), int bytes) {
  return set_max_dyn_smem_impl(reinterpret_cast<const void*>(kernel), bytes);
}
void launch_w13(const GemvParams& p, cudaStream_t s);
void launch_hfin(const GemvParams& p, int max_slots, cudaStream_t s);
void launch_w2(const GemvParams& p, cudaStream_t s);
int w2_stage_capacity();               // bytes of the K2b shared-memory stage of h
constexpr int kGemvCTAs = kNumSM;      // persistent grid: one CTA per SM
constexpr int kGemvTotalWarps = kGemvCTAs * kGemvWarps;
int launch_quantize_expert(int enc, int hidden, int ffn, const __half* w1, const __half* w3,
                           const __half* w2, uint8_t* blob, cudaStream_t s);
void launch_synth(__half* dst, size_t n, uint64_t key, float scale, uint64_t start,
                  cudaStream_t s);

}  // namespace hb
