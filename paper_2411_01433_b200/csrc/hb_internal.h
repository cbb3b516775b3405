// Internal declarations shared by the library's translation units.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hobbit.h"

namespace hb {

constexpr int kMaxTopK = 8;
constexpr int kMaxRouteLayers = 4;      // 1 + max lookahead p handled per launch
constexpr int kNumSM = 148;             // B200
#ifndef HB_GEMV_WARPS
#define HB_GEMV_WARPS 16
#endif
#ifndef HB_WARP_SMEM_KB
#define HB_WARP_SMEM_KB 13
#endif
constexpr int kGemvWarps = HB_GEMV_WARPS;   // warps per GEMV CTA (one CTA per SM)
constexpr int kRouterThreads = 128;

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

// One (expert, served encoding) group of a layer on this rank: the GEMV
// kernels stream its blob once for all of its token slots.
struct Job {
  const uint8_t* blob;
  int32_t enc;
  int32_t expert;
  int32_t n_tok;       // token slots of this job
  int32_t slot_off;    // first slot in slot_token / slot_gate / h
};

// Device job table of one forward: [hdr | jobs | slot_token | slot_gate]
struct JobTable {
  int32_t* hdr;        // [0] n_jobs, [1] n_slots
  Job* jobs;           // max_jobs
  int32_t* slot_token; // max_slots
  float* slot_gate;    // max_slots
  int32_t* tok_slots;  // [max_batch][top_k] slot of each (token, rank) or -1, rank order
};

struct RouterParams {
  const __half* x;                     // [B, H]
  const __half* wg[kMaxRouteLayers];   // router of each routed layer
  int n_route;                         // routed layers in this launch
  int B, E, H, k;
  int64_t theta1, theta2;              // k = 2 exact gap test
  int th1_kind, th2_kind;              // 0 finite, +1 always true, -1 never
  double t1, t2;                       // k > 2 fp64 test
  int rank, world;
  hb_decision* dec;                    // [n_route][B][k]
  long long* lbuf;                     // [n_route][B][E][2] exact logits (scratch)
  long long* logits;                   // [B][E][2] copy for route 0, or null
  uint4* x_perm;                       // [B][H/8] pair-permuted x, or null
  float* xsum;                         // [B][H/32], or null
  float* zero_buf;                     // zeroed by the router grid (h block sums)
  long long zero_n;
  // resident job building (blob_table != null): last CTA builds the table
  const uint8_t* const* blob_table;    // [E][4] device blob of (expert, enc) for this layer
  int hi_enc, lo_enc;
  JobTable jt;
  unsigned* done;                      // grid completion counter (self-resetting)
};

struct GemvParams {
  JobTable jt;
  BlobLayout lay[4];
  int H, F, B, k;
  const uint4* x_perm;                 // [B][H/8]
  const float* xsum;                   // [B][H/32]
  uint4* h_hi;                         // [slots][F/8]  pair-permuted fp16 hi part of h
  uint4* h_lo;                         // [slots][F/8]  fp16 residual h - hi
  float* hsum;                         // [slots][F/32] block sums of h (zeroed by router)
  float* part;                         // stream-K pieces [warps][2][32 lanes][8]
  float* ob;                           // [slots][H] per-slot W2 outputs
  unsigned* cnt13;                     // [max_vjobs][F/16] piece counters (self-resetting)
  unsigned* cnt2;                      // [max_vjobs][H/16]
  unsigned* cnty;                      // [H/16] job counters of the y combine
  float* y;                            // [B][H]
};

void launch_router(const RouterParams& p, cudaStream_t s);
void launch_w13(const GemvParams& p, cudaStream_t s);
void launch_w2(const GemvParams& p, cudaStream_t s);
constexpr int kVSlots = 8;             // token slots per virtual job (one mma N tile)
constexpr int kGemvCTAs = kNumSM;      // persistent grid: one CTA per SM
constexpr int kGemvTotalWarps = kGemvCTAs * kGemvWarps;
constexpr int kPartFloats = 8;         // per lane per piece
int launch_quantize_expert(int enc, int hidden, int ffn, const __half* w1, const __half* w3,
                           const __half* w2, uint8_t* blob, cudaStream_t s);
void launch_synth(__half* dst, size_t n, uint64_t key, float scale, uint64_t start,
                  cudaStream_t s);

}  // namespace hb
