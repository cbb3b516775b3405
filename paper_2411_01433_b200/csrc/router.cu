// K1: exact router + top-k + softmax gates + Eq. 2 scores + T1/T2 decision,
// plus the stacked next-layer prediction (the "Stacking Computer") and,
// in fully-resident mode, the per-layer job table for the GEMV kernels.
//
// Paper: gating = linear layer + top-k (Sec. 2.1); experts ranked by
// normalised ||G(x)_e|| and scored by Eq. 2; High if s <= T1,
// rank 0 always High; T2 bypasses.  Readings DESIGN.md R1-R3,
// R9: softmax over the selected logits; ties -> lower expert index; High
// s<=T1 / Low T1<s<=T2 / Skip s>T2; logits computed EXACTLY.
//
// Exact logits: every fp16 is m*2^e (m 11-bit signed, e in [-24, 5]), so a
// product is m_w*m_x * 2^(e_w+e_x) with e_w+e_x+48 in [0, 58].  Each thread
// splits its products into three int64 accumulators by shift range (see
// dot_exact) and the CTA combines them into one int128 L on a 2^-48 grid.
// The k = 2 decision is the integer test  L0 - L1 <= Theta  (hb_theta).
//
// Launch: one CTA per (route layer, token): n_route*B CTAs of 256 threads, a
// warp per expert row.  At batch-1 decode (one CTA) the same CTA decides and
// builds the job table from shared memory -- no grid-wide hand-off, no global
// read-backs (the router is on the critical path of every layer).  With
// several rows, the last CTA to finish (grid counter) decides for all of
// them.  Route-0 CTAs also write the pair-permuted copy of their token's x
// and its block sums for the GEMV kernels.  Static inputs (router rows, the
// blob table) are fetched before griddepcontrol.wait, i.e. while the previous
// kernel of the stream is still finishing.
#include <cuda_fp16.h>

#include <algorithm>

#include "hb_internal.h"
#include "exact_dot.cuh"
#include "tl_stamps.cuh"

namespace hb {

#ifdef HB_DBG_TIMELINE
__device__ unsigned long long g_rtl[16];
#define HB_RTL(i) do { if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_rtl[i] = t_; } } while (0)
#else
#define HB_RTL(i) do { } while (0)
#endif
// HB_LEGACY_TL == 2: router sub-steps of the leader CTA in hb_stamps fields 8..14
// (SM clock cycles after griddepcontrol.wait, kept in registers and written
// once at the end: no stamp overhead inside the measured steps)
#if HB_LEGACY_TL == 2
#define HB_RSUB(f) do { tl_sub[(f) - 8] = clock64(); } while (0)
#else
#define HB_RSUB(f) do { } while (0)
#endif

__device__ double i128_to_double(i128 v) {
  const bool neg = v < 0;
  unsigned __int128 a = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
  const u64 h = (u64)(a >> 64), l = (u64)a;
  double d = (double)h * 18446744073709551616.0 + (double)l;
  return neg ? -d : d;
}

__device__ __forceinline__ i128 load_logit(const long long* lb, size_t i) {
  const u64 lo = (u64)__ldcg(lb + 2 * i);
  const long long hi = __ldcg(lb + 2 * i + 1);
  return ((i128)hi << 64) | (i128)lo;
}


// O4-O6 for one (route layer, token) given its E exact logits L and the
// top-k selection sel (O3): gates, scores, decisions.  Writes the k records to
// `out` (and `out_s` if given).
__device__ void decide_sel(const RouterParams& p, const i128* L, const int* sel, int b,
                           hb_decision* out, hb_decision* out_s) {
  const double l0 = i128_to_double(L[sel[0]]) * 0x1p-48;
  double g[kMaxTopK], tot = 1.0;
  g[0] = 1.0;                                     // exp(l0 - l0)
  for (int i = 1; i < p.k; ++i) {                 // O4: softmax over the selected
    g[i] = exp(i128_to_double(L[sel[i]]) * 0x1p-48 - l0);
    tot += g[i];
  }
  uint8_t prec[kMaxTopK];
  prec[0] = HB_HIGH;                              // P:423 first expert always High
  if (p.k == 2) {                                 // O6 exact: gap vs Theta
    const i128 G = L[sel[0]] - L[sel[1]];
    prec[1] = gap_le(G, p.th1_kind, p.theta1) ? HB_HIGH
            : gap_le(G, p.th2_kind, p.theta2) ? HB_LOW : HB_SKIP;
  } else {                                        // O5/O6 in fp64
    double s = 0.0;
    for (int i = 1; i < p.k; ++i) {
      s += g[i - 1] / tot;
      prec[i] = s <= p.t1 ? HB_HIGH : s <= p.t2 ? HB_LOW : HB_SKIP;
    }
  }
  for (int i = 0; i < p.k; ++i) {
    hb_decision d;
    d.token = b;
    d.expert = sel[i];
    d.sel_rank = (uint8_t)i;
    d.prec = prec[i];
    d.served_enc = HB_ENC_NONE;
    d.hit = 0;
    d.gate = (float)(g[i] / tot);
    out[i] = d;
    if (out_s) out_s[i] = d;
  }
}

// A token with a non-finite x element: every selection Skip, expert -1, gate
// NaN (its y row is NaN, written by the zeroing CTAs); R28.
__device__ void decide_nonfinite(const RouterParams& p, int b, hb_decision* out, hb_decision* out_s) {
  for (int i = 0; i < p.k; ++i) {
    hb_decision d;
    d.token = b;
    d.expert = -1;
    d.sel_rank = (uint8_t)i;
    d.prec = HB_SKIP;
    d.served_enc = HB_ENC_NONE;
    d.hit = 0;
    d.gate = __int_as_float(0x7fc00000);
    out[i] = d;
    if (out_s) out_s[i] = d;
  }
}

// O3-O6, one thread: top-k by (L desc, index asc), then decide_sel
__device__ void decide(const RouterParams& p, const i128* L, int b, hb_decision* out,
                       hb_decision* out_s) {
  int sel[kMaxTopK];
  unsigned long long taken = 0ull;
  for (int i = 0; i < p.k; ++i) {
    int best = -1;
    for (int e = 0; e < p.E; ++e) {
      if (taken >> e & 1ull) continue;
      if (best < 0 || L[e] > L[best]) best = e;
    }
    sel[i] = best;
    taken |= 1ull << best;
  }
  decide_sel(p, L, sel, b, out, out_s);
}

// O3 by one warp: k rounds of a warp arg-max over (L desc, index asc).  The
// same selection as decide(), with a dependency chain of ~k*5 shuffle steps
// instead of E*k serial compares (the router is on every layer's critical path).
__device__ __forceinline__ void topk_warp(const RouterParams& p, const i128* L, int* sel) {
  const int lane = threadIdx.x & 31;
  unsigned long long taken = 0ull;
  for (int i = 0; i < p.k; ++i) {
    int be = -1;
    i128 bv = 0;
    for (int e = lane; e < p.E; e += 32)
      if (!(taken >> e & 1ull) && (be < 0 || L[e] > bv)) { bv = L[e]; be = e; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 olo = __shfl_xor_sync(0xffffffffu, (u64)bv, o);
      const u64 ohi = __shfl_xor_sync(0xffffffffu, (u64)(bv >> 64), o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      const i128 ov = (i128)(((unsigned __int128)ohi << 64) | olo);
      if (oe >= 0 && (be < 0 || ov > bv || (ov == bv && oe < be))) { bv = ov; be = oe; }
    }
    sel[i] = be;
    taken |= 1ull << be;
  }
}

// O3-O6 for top-2 routing (the paper's models) by one warp, shortest
// dependency chain: lane e ranks its logit against all E in parallel (same
// order as decide(): L desc, index asc), the two winners come from ballots,
// the decision is the exact integer gap test and the two gates follow from
// one exp: g0 = 1 / (1 + exp(l1 - l0)), g1 = exp(l1 - l0) g0 (fp32; the
// decision itself is the exact integer test).
__device__ __forceinline__ void decide_k2_warp(const RouterParams& p, const i128* L, int b, hb_decision* out,
                               hb_decision* out_s) {
  const int lane = threadIdx.x & 31;
  HB_RTL(13);
  int rank = 2;
  if (lane < p.E) {
    const i128 v = L[lane];
    rank = 0;
    for (int e = 0; e < p.E; ++e) {
      const i128 o = L[e];
      rank += (o > v) || (o == v && e < lane);
    }
  }
  HB_RTL(8);
  const unsigned m0 = __ballot_sync(0xffffffffu, rank == 0);
  const unsigned m1 = __ballot_sync(0xffffffffu, rank == 1);
  HB_RTL(9);
  if (lane == 0) {
    const int e0 = __ffs(m0) - 1, e1 = __ffs(m1) - 1;
    const i128 G = L[e0] - L[e1];                  // >= 0
    const uint8_t prec1 = gap_le(G, p.th1_kind, p.theta1) ? HB_HIGH
                        : gap_le(G, p.th2_kind, p.theta2) ? HB_LOW : HB_SKIP;
    // gates in fp32 (|error| ~1e-7, the records are fp32): the fp64 exp and
    // divisions cost ~1.5 us of single-thread latency on the critical path
    const float d = G >= ((i128)1 << 62) ? 1e30f : (float)(long long)G * 0x1p-48f;
    const float ex = expf(-d);
    const float g0 = 1.f / (1.f + ex), g1 = ex * g0;
    HB_RTL(10);
    hb_decision r0, r1;
    r0.token = b; r0.expert = e0; r0.sel_rank = 0; r0.prec = HB_HIGH;
    r0.served_enc = HB_ENC_NONE; r0.hit = 0; r0.gate = (float)g0;
    r1.token = b; r1.expert = e1; r1.sel_rank = 1; r1.prec = prec1;
    r1.served_enc = HB_ENC_NONE; r1.hit = 0; r1.gate = (float)g1;
    out[0] = r0; out[1] = r1;
    HB_RTL(11);
    out_s[0] = r0; out_s[1] = r1;
    HB_RTL(12);
  }
}

constexpr int kMaxDecSmem = 512;
#ifndef HB_ROUTER_CLUSTER
#define HB_ROUTER_CLUSTER 8
#endif
constexpr int kRouterCluster = HB_ROUTER_CLUSTER;   // CTAs (SMs) per (route layer, token) row (decode)

struct RouterSmem {
  i128 L[64];                          // this CTA's exact logits
#ifdef HB_PART16
  u64 part[kRouterThreads / 32][3];
#else
  u64 part[64 > kRouterThreads / 32 ? 64 : kRouterThreads / 32][3];  // per task (E*wpe <= max(64, NW))
#endif
  u64 cpart[64][3];                    // this CTA's partial per expert (read by the leader)
  hb_decision dec[kMaxDecSmem];        // route-0 decisions (single-CTA / last-CTA path)
  const uint8_t* blob[64 * 4];         // blob table of the layer
  Job jobs[2 * 64 + 1];
  int count[2 * 64], jobid[2 * 64], fill[2 * 64];
  unsigned long long hmask;            // experts with a High selection (non-strict upgrade)
  int bad;                             // this CTA's slice of x has a non-finite element
  u64 bad2;                            // the same as a u64 (read by the cluster leader)
  int last;
};

// Shared memory of the batch router kernel (router_batch_kernel): one CTA per
// token, the filtered router, the job table built by the last CTA.
struct BatchSmem {
  float red[kRouterThreads / 32][64];  // per warp fp32 partial logit per expert
  float xqw[kRouterThreads / 32];      // per warp sum of x^2
  double Lf[64];                       // filtered logits of the row
  u64 part[64][3];                     // exact fallback: per task partial
  i128 L[64];                          // exact fallback: logits
  const uint8_t* blob[64 * 4];         // blob table of the layer (last CTA)
  Job jobs[2 * 64 + 1];
  int count[2 * 64], jobid[2 * 64], fill[2 * 64];
  unsigned long long hmask;
  int ok, last;
};

// Shared memory of the decode router kernel (router_dec_kernel): one token,
// top-2, E <= 32 experts, the filtered router with its exact fallback.
struct DecSmem {
  i128 L[64];                          // exact logits (fallback, leader)
  u64 part[64][3];                     // exact partial per task (fallback)
  hb_decision dec[2];
  const uint8_t* blob[64 * 4];         // blob table of the layer
  Job jobs[33];
  float fpart[64];                     // per task fp32 partial logit
  double fcp[64];                      // this CTA's partial per expert (read by the leader)
  float xqw[kRouterThreads / 32];      // per warp sum of x^2 of the slice
  double cxq;                          // this CTA's sum of x^2
  double Lf[64];                       // filtered logits (leader)
  double xs;                           // ||x||^2 (leader)
  u64 bad2;                            // non-finite x flag (read by the leader)
  int bad, ok;
};

// Job key of a selection: expert * 2 + (served from lo_enc), or -1 (Skip /
// not owned).  Non-strict mode (R27): a Low selection of an expert
// that a High selection of the same forward also touches is served by the
// hi_enc copy (hmask bit e), so every touched expert is streamed once.
__device__ __forceinline__ int sel_key(const RouterParams& p, const hb_decision& d,
                                       unsigned long long hmask) {
  if (d.prec == HB_SKIP || d.expert < 0 || d.expert % p.world != p.rank) return -1;
  const bool hi = d.prec == HB_HIGH || (!p.strict && ((hmask >> d.expert) & 1ull));
  return d.expert * 2 + (hi ? 0 : 1);
}
__device__ __forceinline__ unsigned long long high_bit(const RouterParams& p, const hb_decision& d) {
  return (d.prec == HB_HIGH && d.expert >= 0 && d.expert % p.world == p.rank) ? 1ull << d.expert : 0ull;
}

// resident mode: group the non-skipped owned selections into (expert, enc)
// jobs, ordered by expert then High before Low; slots in token order.  All
// reads come from shared memory; the global table is written once.
__device__ void build_jobs(const RouterParams& p, RouterSmem& sm, const hb_decision* dec) {
  const int nkey = 2 * p.E;
  for (int i = 0; i < nkey; ++i) sm.count[i] = 0;
  const int nsel = p.B * p.k;
  unsigned long long hmask = 0ull;
  for (int i = 0; i < nsel; ++i) hmask |= high_bit(p, dec[i]);
  for (int i = 0; i < nsel; ++i) {
    const int key = sel_key(p, dec[i], hmask);
    if (key >= 0) sm.count[key]++;
  }
  int nj = 0, off = 0;
  for (int key = 0; key < nkey; ++key) {
    sm.jobid[key] = -1;
    sm.fill[key] = 0;
    if (!sm.count[key]) continue;
    const int e = key >> 1;
    const int enc = (key & 1) ? p.lo_enc : p.hi_enc;
    Job j;
    j.blob = sm.blob[e * 4 + enc];
    j.enc = enc;
    j.expert = e;
    j.n_tok = sm.count[key];
    j.slot_off = off;
    sm.jobs[nj] = j;
    p.jt.jobs[nj] = j;
    sm.jobid[key] = nj++;
    off += sm.count[key];
  }
  for (int i = 0; i < nsel; ++i) {
    hb_decision d = dec[i];
    p.jt.tok_slots[i] = -1;
    const int key = sel_key(p, d, hmask);
    if (key < 0) continue;
    const int slot = sm.jobs[sm.jobid[key]].slot_off + sm.fill[key]++;
    p.jt.slot_token[slot] = d.token;
    p.jt.slot_gate[slot] = d.gate;
    p.jt.tok_slots[i] = slot;
    d.served_enc = (uint8_t)((key & 1) ? p.lo_enc : p.hi_enc);
    d.hit = 1;
    p.dec[i] = d;
  }
  p.jt.hdr[0] = nj;
  p.jt.hdr[1] = off;
  p.jt.hdr[2] = p.no_vjobs ? 0 : build_vjobs(sm.jobs, nj, p.H, p.F, p.jt.vjobs, p.jt.vcum13, p.jt.vcum2);
}

// build_jobs for batches, by the whole (last) CTA: per-key counts with shared
// atomics, job offsets by one thread (<= 2E keys), then slots in token order
// by warp 0 (ballot ranks within each 32-selection chunk).  Same table as
// build_jobs; the serial version read the decisions from global memory one
// dependent load at a time (~0.5 us per selection at B = 512).
template <typename SmemT>
__device__ void build_jobs_cta(const RouterParams& p, SmemT& sm, const hb_decision* dec) {
  const int nkey = 2 * p.E, nsel = p.B * p.k, tid = threadIdx.x;
  for (int i = tid; i < nkey; i += blockDim.x) { sm.count[i] = 0; sm.fill[i] = 0; }
  if (tid == 0) sm.hmask = 0ull;
  __syncthreads();
  if (!p.strict) {
    unsigned long long hm = 0ull;
    for (int i = tid; i < nsel; i += blockDim.x) hm |= high_bit(p, dec[i]);
    if (hm) atomicOr(&sm.hmask, hm);
    __syncthreads();
  }
  const unsigned long long hmask = sm.hmask;
  for (int i = tid; i < nsel; i += blockDim.x) {
    const int key = sel_key(p, dec[i], hmask);
    if (key >= 0) atomicAdd(&sm.count[key], 1);
  }
  __syncthreads();
  if (tid == 0) {
    int nj = 0, off = 0;
    for (int key = 0; key < nkey; ++key) {
      sm.jobid[key] = -1;
      if (!sm.count[key]) continue;
      const int e = key >> 1;
      const int enc = (key & 1) ? p.lo_enc : p.hi_enc;
      Job j;
      j.blob = sm.blob[e * 4 + enc];
      j.enc = enc;
      j.expert = e;
      j.n_tok = sm.count[key];
      j.slot_off = off;
      sm.jobs[nj] = j;
      p.jt.jobs[nj] = j;
      sm.jobid[key] = nj++;
      off += sm.count[key];
    }
    p.jt.hdr[0] = nj;
    p.jt.hdr[1] = off;
    sm.last = nj;                                  // reused: number of jobs
  }
  __syncthreads();
  if (tid < 32) {
    const int lane = tid;
    for (int base = 0; base < nsel; base += 32) {
      const int i = base + lane;
      int key = -1;
      hb_decision d;
      if (i < nsel) {
        d = dec[i];
        key = sel_key(p, d, hmask);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      if (key >= 0) {
        const int slot = sm.jobs[sm.jobid[key]].slot_off + sm.fill[key] + rank;
        p.jt.slot_token[slot] = d.token;
        p.jt.slot_gate[slot] = d.gate;
        p.jt.tok_slots[i] = slot;
        d.served_enc = (uint8_t)((key & 1) ? p.lo_enc : p.hi_enc);
        d.hit = 1;
        p.dec[i] = d;
      } else if (i < nsel) {
        p.jt.tok_slots[i] = -1;
      }
      __syncwarp();
      if (key >= 0 && rank == __popc(peers) - 1) sm.fill[key] += __popc(peers);
      __syncwarp();
    }
    if (lane == 0)
      p.jt.hdr[2] = p.no_vjobs ? 0
                                : build_vjobs(sm.jobs, sm.last, p.H, p.F, p.jt.vjobs, p.jt.vcum13, p.jt.vcum2);
  }
}

// build_jobs by one warp when the forward has <= 32 selections (decode): the
// same table (jobs by key = expert*2 + Low, slots in selection order) from
// per-lane counts instead of serial loops.
template <typename SmemT>
__device__ __forceinline__ void build_jobs_warp_to(const RouterParams& p, SmemT& sm, const hb_decision* dec,
                                                   const JobTable& jt, hb_decision* dout) {
  const int lane = threadIdx.x & 31;
  const int nsel = p.B * p.k;
  constexpr int kNone = 0x7FFFFFFF;
  hb_decision d{};
  int key = kNone;
  if (lane < nsel) d = dec[lane];
  const unsigned long long hb = lane < nsel ? high_bit(p, d) : 0ull;
  const unsigned long long hmask =
      ((unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(hb >> 32)) << 32) |
      __reduce_or_sync(0xffffffffu, (unsigned)hb);
  if (lane < nsel) {
    const int k0 = sel_key(p, d, hmask);
    if (k0 >= 0) key = k0;
  }
  const bool valid = key != kNone;
  int less = 0, rank = 0, ntok = 0;
  for (int j = 0; j < nsel; ++j) {
    const int kj = __shfl_sync(0xffffffffu, key, j);
    less += kj != kNone && kj < key;
    ntok += kj == key;
    rank += kj == key && j < lane;
  }
  const bool first = valid && rank == 0;
  int jid = 0;
  for (int j = 0; j < nsel; ++j) {
    const int kj = __shfl_sync(0xffffffffu, key, j);
    const int fj = __shfl_sync(0xffffffffu, (int)first, j);
    jid += fj && kj < key;
  }
  const int nj = __popc(__ballot_sync(0xffffffffu, first));
  const int nslot = __popc(__ballot_sync(0xffffffffu, valid));
  if (lane < nsel) jt.tok_slots[lane] = -1;
  if (valid) {
    const int slot = less + rank;
    const int enc = (key & 1) ? p.lo_enc : p.hi_enc;
    jt.slot_token[slot] = d.token;
    jt.slot_gate[slot] = d.gate;
    jt.tok_slots[lane] = slot;
    d.served_enc = (uint8_t)enc;
    d.hit = 1;
    dout[lane] = d;
    if (first) {
      Job j;
      j.blob = sm.blob[(key >> 1) * 4 + enc];
      j.enc = enc;
      j.expert = key >> 1;
      j.n_tok = ntok;
      j.slot_off = less;
      sm.jobs[jid] = j;
      jt.jobs[jid] = j;
    }
  }
  __syncwarp();
  if (lane == 0) {
    jt.hdr[0] = nj;
    jt.hdr[1] = nslot;
    jt.hdr[2] = build_vjobs(sm.jobs, nj, p.H, p.F, jt.vjobs, jt.vcum13, jt.vcum2);
  }
}
template <typename SmemT>
__device__ __forceinline__ void build_jobs_warp(const RouterParams& p, SmemT& sm, const hb_decision* dec) {
  build_jobs_warp_to(p, sm, dec, p.jt, p.dec);
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ u64 ld_dsmem_u64(const void* local, int rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local), r;
  u64 v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(r) : "memory");
  return v;
}

// C = CTAs per (route layer, token) row: 8 (a cluster, decode: the token's
// logits in ~1/8 of the latency) or 1 (batches: one CTA per row, no cluster --
// 8-CTA clusters per token cost ~1 us per token at B = 512)

// fp16 x8 -> fp32 x8
__device__ __forceinline__ void r_h2f8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ double ld_dsmem_f64(const void* local, int rank) {
  return __longlong_as_double((long long)ld_dsmem_u64(local, rank));
}

// pair-permuted x and block sums of the slice [s0, s1) (uint4 chunks) for
// the GEMV kernels
__device__ __forceinline__ void write_xperm(const RouterParams& p, const __half* x, int s0, int s1,
                                            int b) {
  for (int blk = s0 / 4 + threadIdx.x; blk < s1 / 4; blk += blockDim.x) {
    const uint4* src = reinterpret_cast<const uint4*>(x + blk * 32);
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 t = src[i];
      v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
    }
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      sum += __half2float(__ushort_as_half((unsigned short)(v[i >> 1] >> (16 * (i & 1)))));
    p.xsum[(size_t)b * (p.H / 32) + blk] = sum;
#pragma unroll
    for (int t = 0; t < 4; ++t) {                  // uint4 t: Q_c = (x[8t+c], x[8t+c+4])
      uint32_t q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e0 = 8 * t + c, e1 = e0 + 4;
        const uint32_t lo16 = (v[e0 >> 1] >> (16 * (e0 & 1))) & 0xFFFF;
        const uint32_t hi16 = (v[e1 >> 1] >> (16 * (e1 & 1))) & 0xFFFF;
        q[c] = lo16 | (hi16 << 16);
      }
      p.x_perm[(size_t)b * (p.H / 8) + blk * 4 + t] = make_uint4(q[0], q[1], q[2], q[3]);
    }
  }
}

// Batch-1 decode, k = 2, one cluster: the FILTERED router.  Every CTA sums
// fp32 products (exact for fp16 x fp16) of its slice of H in FFMA chains and
// warp trees; the leader adds the CTA partials in fp64 and decides the top-2
// order and the T1/T2 tests from these when every comparison clears a
// rigorous bound on the rounding error (Cauchy-Schwarz: sum |w x| <= ||w_e||
// ||x||, R9'), else from the exact integer logits it computes itself
// (rare).  Either way the decisions are the exact ones.  The gates come from
// the filtered gap (R25).
// Zeroing CTAs of the router grids: the buffers the GEMV kernels accumulate
// into (K2a sums, y, ...); they belong to the previous kernels of the
// stream, so wait first.  CTA zc of nzc.
__device__ void zero_buffers(const RouterParams& p, int zc, int nzc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int tid = threadIdx.x;
  const long long t0 = (long long)zc * blockDim.x + tid;
  const long long stride = (long long)nzc * blockDim.x;
#pragma unroll
  for (int z = 0; z < 3; ++z) {
    float* zb = p.zero_buf[z];
    const long long n = p.zero_n[z];
    if ((reinterpret_cast<uintptr_t>(zb) & 15) == 0) {
      for (long long i = t0; i < n / 4; i += stride)
        reinterpret_cast<float4*>(zb)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (long long i = (n / 4) * 4 + t0; i < n; i += stride) zb[i] = 0.f;
    } else {
      for (long long i = t0; i < n; i += stride) zb[i] = 0.f;
    }
  }
}

template <int C>
__device__ __forceinline__ void route_filtered(const RouterParams& p, DecSmem& sm, int crank,
                                               int s0, int s1, int b, int rl) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kRouterThreads / 32;
  const __half* x = p.x + (size_t)b * p.H;
  const uint4* x4 = reinterpret_cast<const uint4*>(x);
  const int wpe = p.E >= NW ? 1 : NW / p.E;
  int xbad = 0;
  float xq = 0.f;
  for (int task = warp; task < p.E * wpe; task += NW) {
    const int e = task / wpe, part = task - e * wpe;
    const uint4* w4 = reinterpret_cast<const uint4*>(p.wg[rl] + (size_t)e * p.H);
    const int j0 = s0 + part * (s1 - s0) / wpe, j1 = s0 + (part + 1) * (s1 - s0) / wpe;
    float acc = 0.f;
    for (int j = j0 + lane; j < j1; j += 32) {
      const uint4 wv = w4[j];
      const uint4 xv = x4[j];
      float wf[8], xf[8];
      r_h2f8(wv, wf);
      r_h2f8(xv, xf);
      if (e == 0) {                               // every chunk of the slice once
        const uint32_t xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          xbad |= ((xa[q] & 0x7C00u) == 0x7C00u) | ((xa[q] & 0x7C000000u) == 0x7C000000u);
#pragma unroll
        for (int q = 0; q < 8; ++q) xq = fmaf(xf[q], xf[q], xq);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = fmaf(wf[q], xf[q], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sm.fpart[task] = acc;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) xq += __shfl_xor_sync(0xffffffffu, xq, o);
  if (lane == 0) sm.xqw[warp] = xq;
  const int bad = __syncthreads_or(xbad);
  if (tid < p.E) {
    double v = 0.0;
    for (int q = 0; q < wpe; ++q) v += (double)sm.fpart[tid * wpe + q];
    sm.fcp[tid] = v;
  }
  if (tid == kRouterThreads - 1) {
    double v = 0.0;
    for (int w = 0; w < NW; ++w) v += (double)sm.xqw[w];
    sm.cxq = v;
    sm.bad2 = (u64)bad;
  }
  if (rl == 0) {
    if (p.x_save)
      for (int j = s0 + tid; j < s1; j += blockDim.x) reinterpret_cast<uint4*>(p.x_save)[j] = x4[j];
    if (p.x_perm) write_xperm(p, x, s0, s1, b);
  }
  cluster_sync_all();
  if (crank == 0) {
    if (tid < p.E * C) {                        // e = tid / C, rank r = tid % C; C | 32
      const int e = tid / C, r = tid - e * C;
      double v = ld_dsmem_f64(&sm.fcp[e], r);
#pragma unroll
      for (int o = 1; o < C; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (r == 0) sm.Lf[e] = v;
    }
    if (tid == kRouterThreads - 1) {
      double xs = 0.0;
      int bd = 0;
      for (int r = 0; r < C; ++r) {
        xs += ld_dsmem_f64(&sm.cxq, r);
        bd |= (int)ld_dsmem_u64(&sm.bad2, r);
      }
      sm.xs = xs;
      sm.bad = bd;
    }
  }
  cluster_sync_all();                             // remote reads done: the other CTAs may exit
  if (crank != 0) return;
  if (tid == 0) p.rowbad[b] = sm.bad;             // the expert kernels write NaN rows (R28)
  if (warp == 0) {
    if (sm.bad) {
      if (lane == 0) { decide_nonfinite(p, b, p.dec, sm.dec); sm.ok = 1; }
    } else {
      // error of a logit: fp32 chains of m products per lane (gamma_{m-1}),
      // warp trees (gamma_5), fp64 sums (negligible): (m + 5) * 2^-24 *
      // sum|p| * (1 + 1e-6), with sum|p| <= ||w_e|| ||x|| (||x|| rounded up)
      const int chunks = (s1 - s0) / wpe;
      const int m = 8 * ((chunks + 31) / 32);
      const double xn = sqrt(sm.xs) * (1.0 + 1e-6) + 1e-30;
      const double c = (m + 6) * 0x1p-24 * 1.0001;
      const int e = lane;
      const double v = e < p.E ? sm.Lf[e] : -1e300;
      const double ep = e < p.E ? c * (double)p.wnorm[e] * xn : 0.0;
      int r = 0;
      if (e < p.E)
        for (int f = 0; f < p.E; ++f) { const double o = sm.Lf[f]; r += (o > v) || (o == v && f < e); }
      const unsigned m0 = __ballot_sync(0xffffffffu, e < p.E && r == 0);
      const unsigned m1 = __ballot_sync(0xffffffffu, e < p.E && r == 1);
      const int e0 = __ffs(m0) - 1, e1 = __ffs(m1) - 1;
      double rest = (e < p.E && r >= 2) ? v + ep : -1e300;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rest = fmax(rest, __shfl_xor_sync(0xffffffffu, rest, o));
      const double L0 = __shfl_sync(0xffffffffu, v, e0), L1 = __shfl_sync(0xffffffffu, v, e1);
      const double ep0 = __shfl_sync(0xffffffffu, ep, e0), ep1 = __shfl_sync(0xffffffffu, ep, e1);
      const double G = L0 - L1, mg = ep0 + ep1 + 1e-12 * (1.0 + fabs(L0) + fabs(L1));
      bool ok = (L0 - ep0 > L1 + ep1) && (L1 - ep1 > rest);
      if (p.th1_kind == 0) ok = ok && fabs(G - (double)p.theta1 * 0x1p-48) > mg;
      if (p.th2_kind == 0) ok = ok && fabs(G - (double)p.theta2 * 0x1p-48) > mg;
      if (ok && lane == 0) {
        const uint8_t prec1 = (p.th1_kind > 0 || (p.th1_kind == 0 && G <= (double)p.theta1 * 0x1p-48)) ? HB_HIGH
                            : (p.th2_kind > 0 || (p.th2_kind == 0 && G <= (double)p.theta2 * 0x1p-48)) ? HB_LOW
                                                                                                    : HB_SKIP;
        const float ex = expf(-(float)G);
        const float g0 = 1.f / (1.f + ex), g1 = ex * g0;
        hb_decision r0, r1;
        r0.token = b; r0.expert = e0; r0.sel_rank = 0; r0.prec = HB_HIGH;
        r0.served_enc = HB_ENC_NONE; r0.hit = 0; r0.gate = g0;
        r1.token = b; r1.expert = e1; r1.sel_rank = 1; r1.prec = prec1;
        r1.served_enc = HB_ENC_NONE; r1.hit = 0; r1.gate = g1;
        p.dec[0] = r0; p.dec[1] = r1;
        sm.dec[0] = r0; sm.dec[1] = r1;
      }
      if (lane == 0) sm.ok = ok;
    }
  }
  __syncthreads();
  if (!sm.ok) {
    // ---- exact fallback by the leader alone over the whole of H (rare)
    const int n8 = p.H / 8;
    for (int task = warp; task < p.E * wpe; task += NW) {
      const int e = task / wpe, part = task - e * wpe;
      const uint4* w4 = reinterpret_cast<const uint4*>(p.wg[rl] + (size_t)e * p.H);
      const int j0 = part * n8 / wpe, j1 = (part + 1) * n8 / wpe;
      u64 lo = 0, mid = 0, hi = 0;
      for (int j = j0 + lane; j < j1; j += 32) {
        const uint4 wv = w4[j];
        const uint4 xv = x4[j];
        const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
          accum_exact((wa[i >> 1] >> (16 * (i & 1))) & 0xFFFF, (xa[i >> 1] >> (16 * (i & 1))) & 0xFFFF,
                      lo, mid, hi);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        mid += __shfl_xor_sync(0xffffffffu, mid, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      if (lane == 0) { sm.part[task][0] = lo; sm.part[task][1] = mid; sm.part[task][2] = hi; }
    }
    __syncthreads();
    for (int e = tid; e < p.E; e += blockDim.x) {
      u64 lo = 0, mid = 0, hi = 0;
      for (int q = 0; q < wpe; ++q) {
        lo += sm.part[e * wpe + q][0]; mid += sm.part[e * wpe + q][1]; hi += sm.part[e * wpe + q][2];
      }
      sm.L[e] = (i128)(long long)lo + ((i128)(long long)mid << 20) + ((i128)(long long)hi << 40);
    }
    __syncthreads();
    if (warp == 0) decide_k2_warp(p, sm.L, b, p.dec, sm.dec);
    __syncthreads();
  }
  if (warp == 0 && p.blob_table) build_jobs_warp(p, sm, sm.dec);
}

template <int C>
__global__ void __launch_bounds__(kRouterThreads)
router_kernel(const __grid_constant__ RouterParams p) {
  __shared__ RouterSmem sm;
  HB_RTL(0);
#ifdef HB_LEGACY_TL
  const unsigned long long tl_entry = tl_now();
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kRouterThreads / 32;
  const int nrows = p.n_route * p.B;
  const int row = blockIdx.x / C, crank = blockIdx.x % C;   // cluster = one row
  if (row >= nrows) {
    zero_buffers(p, blockIdx.x - nrows * C, gridDim.x - nrows * C);
#if HB_LEGACY_TL == 1
    __syncthreads();
    if (tid == 0) tl_max(tl_rec(p.stamps, p.stamp_cap, p.fwd_idx), 13, tl_now());
#endif
    return;
  }
  const int b = row % p.B;
  const int rl = row / p.B;
  // this CTA's slice of the hidden dimension (in uint4 = 8 fp16)
  const int n8 = p.H / 8;
  const int s0 = crank * n8 / C, s1 = (crank + 1) * n8 / C;
  // ---- static inputs before waiting on the previous kernel: this CTA's
  // slice of the router rows into L2, the layer's blob table (leader)
  {
    const char* wb = reinterpret_cast<const char*>(p.wg[rl]);
    const int lpr = (s1 - s0) * 16 / 128;                  // 128-byte lines per row slice
    for (int i = tid; i < p.E * lpr; i += kRouterThreads) {
      const int e = i / lpr, l = i - e * lpr;
      asm volatile("prefetch.global.L2 [%0];" :: "l"(wb + ((size_t)e * n8 + s0) * 16 + (size_t)l * 128));
    }
    if (p.blob_table && crank == 0)
      for (int i = tid; i < 4 * p.E; i += kRouterThreads) sm.blob[i] = p.blob_table[i];
  }
  // programmatic dependent launch: x and the job table belong to the
  // previous kernels of the stream
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  HB_RTL(1);
#if HB_LEGACY_TL == 2
  long long tl_sub[7] = {0, 0, 0, 0, 0, 0, 0};
  const long long tl_c0 = clock64();
#endif
#ifdef HB_LEGACY_TL
  if (tid == 0) {
    unsigned long long* rec = tl_rec(p.stamps, p.stamp_cap, p.fwd_idx);
    tl_min(rec, 6, tl_now());
    tl_min(rec, 5, tl_entry);
  }
#endif

  // ---- O2: exact partial logits of token b over this CTA's slice, every
  // expert (a warp per expert, or several warps per expert when E < 8)
  const __half* x = p.x + (size_t)b * p.H;
  const uint4* x4 = reinterpret_cast<const uint4*>(x);
  const int wpe = p.E >= NW ? 1 : NW / p.E;
  int xbad = 0;                                 // non-finite x in the slice (R28)
  for (int task = warp; task < p.E * wpe; task += NW) {
    const int e = task / wpe, part = task - e * wpe;
    const uint4* w4 = reinterpret_cast<const uint4*>(p.wg[rl] + (size_t)e * p.H);
    const int j0 = s0 + part * (s1 - s0) / wpe, j1 = s0 + (part + 1) * (s1 - s0) / wpe;
    u64 lo = 0, mid = 0, hi = 0;
#pragma unroll 2
    for (int j = j0 + lane; j < j1; j += 32) {
      const uint4 wv = w4[j];
      const uint4 xv = x4[j];
      const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
      const uint32_t xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        xbad |= ((xa[q] & 0x7C00u) == 0x7C00u) | ((xa[q] & 0x7C000000u) == 0x7C000000u);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        accum_exact((wa[i >> 1] >> (16 * (i & 1))) & 0xFFFF, (xa[i >> 1] >> (16 * (i & 1))) & 0xFFFF,
                    lo, mid, hi);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo += __shfl_xor_sync(0xffffffffu, lo, o);
      mid += __shfl_xor_sync(0xffffffffu, mid, o);
      hi += __shfl_xor_sync(0xffffffffu, hi, o);
    }
    if (lane == 0) { sm.part[task][0] = lo; sm.part[task][1] = mid; sm.part[task][2] = hi; }
  }
  {
    // every x chunk of the slice was read by the expert-0 tasks above
    const int bad = __syncthreads_or(xbad);
    if (tid == 0) { sm.bad = bad; sm.bad2 = (u64)bad; }
  }
  for (int e = tid; e < p.E; e += blockDim.x) {            // CTA partial per expert
    u64 lo = 0, mid = 0, hi = 0;
    for (int q = 0; q < wpe; ++q) {
      lo += sm.part[e * wpe + q][0]; mid += sm.part[e * wpe + q][1]; hi += sm.part[e * wpe + q][2];
    }
    sm.cpart[e][0] = lo; sm.cpart[e][1] = mid; sm.cpart[e][2] = hi;
  }
  HB_RTL(2);
  HB_RSUB(8);
  // ---- pair-permuted x and block sums of this slice for the GEMV kernels
  if (p.x_perm && rl == 0) write_xperm(p, x, s0, s1, b);
  HB_RSUB(9);
  // ---- combine the cluster's partials in the leader (distributed shared memory)
  if (C > 1) cluster_sync_all();
  else __syncthreads();
  HB_RSUB(10);
  if (crank == 0) {
    if (C > 1 && tid == kRouterThreads - 1) {   // a thread the logit combine does not use
      int bad = 0;
      for (int r = 0; r < C; ++r) bad |= (int)ld_dsmem_u64(&sm.bad2, r);
      sm.bad = bad;
    }
    for (int e = tid; e < p.E; e += blockDim.x) {
      u64 lo = 0, mid = 0, hi = 0;
      for (int r = 0; r < C; ++r) {
        if (C > 1) {
          lo += ld_dsmem_u64(&sm.cpart[e][0], r);
          mid += ld_dsmem_u64(&sm.cpart[e][1], r);
          hi += ld_dsmem_u64(&sm.cpart[e][2], r);
        } else {
          lo += sm.cpart[e][0]; mid += sm.cpart[e][1]; hi += sm.cpart[e][2];
        }
      }
      sm.L[e] = (i128)(long long)lo + ((i128)(long long)mid << 20) + ((i128)(long long)hi << 40);
    }
  }
  HB_RSUB(11);
  if (C > 1) cluster_sync_all();             // remote reads done: the other CTAs may exit
  else __syncthreads();
  if (crank != 0) return;
  HB_RTL(3);
  HB_RSUB(12);
  HB_RTL(4);
  if (rl == 0 && p.logits)
    for (int e = tid; e < p.E; e += blockDim.x) {
      p.logits[((size_t)b * p.E + e) * 2 + 0] = (long long)(u64)sm.L[e];
      p.logits[((size_t)b * p.E + e) * 2 + 1] = (long long)(sm.L[e] >> 64);
    }

  // ---- single (route layer, token): decide and build the jobs right here
  if (nrows == 1) {
    if (tid == 0) p.rowbad[b] = sm.bad;       // the expert kernels write NaN rows (R28)
    if (warp == 0) {
      if (sm.bad) {
        if (lane == 0) decide_nonfinite(p, b, p.dec, sm.dec);
      } else if (p.k == 2 && p.E <= 32) {
        decide_k2_warp(p, sm.L, b, p.dec, sm.dec);
      } else {
        int sel[kMaxTopK];
        topk_warp(p, sm.L, sel);
        if (lane == 0) decide_sel(p, sm.L, sel, b, p.dec, sm.dec);
      }
      __syncwarp();
      HB_RTL(5);
      HB_RSUB(13);
      if (p.blob_table) {
        if (p.B * p.k <= 32) build_jobs_warp(p, sm, sm.dec);
        else if (lane == 0) build_jobs(p, sm, sm.dec);
      }
      HB_RTL(6);
      HB_RSUB(14);
      HB_RTL(7);                               // back-to-back: cost of one stamp
#ifdef HB_LEGACY_TL
      if (lane == 0) {
        unsigned long long* rec = tl_rec(p.stamps, p.stamp_cap, p.fwd_idx);
        tl_max(rec, 7, tl_now());
#if HB_LEGACY_TL == 2
        if (blockIdx.x == 0)
          for (int f = 0; f < 7; ++f) tl_max(rec, 8 + f, (unsigned long long)(tl_sub[f] - tl_c0));
#endif
      }
#endif
    }
    return;
  }

  // ---- several rows: publish the logits; the last leader decides for all
  if (tid == 0) p.rowbad[(size_t)rl * p.B + b] = sm.bad;
  for (int e = tid; e < p.E; e += blockDim.x) {
    const size_t idx = ((size_t)rl * p.B + b) * p.E + e;
    p.lbuf[2 * idx] = (long long)(u64)sm.L[e];
    p.lbuf[2 * idx + 1] = (long long)(sm.L[e] >> 64);
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(p.done, 1u);
    sm.last = (prev == (unsigned)nrows - 1);
  }
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  const bool dec_smem = p.B * p.k <= kMaxDecSmem;
  for (int i = tid; i < p.n_route * p.B; i += blockDim.x) {
    const int r = i / p.B, bb = i % p.B;
    i128 L[64];
    const size_t base = ((size_t)r * p.B + bb) * p.E;
    if (__ldcg(p.rowbad + (size_t)r * p.B + bb)) {
      decide_nonfinite(p, bb, p.dec + ((size_t)r * p.B + bb) * p.k,
                       r == 0 && dec_smem ? sm.dec + (size_t)bb * p.k : nullptr);
      continue;
    }
    for (int e = 0; e < p.E; ++e) L[e] = load_logit(p.lbuf, base + e);
    decide(p, L, bb, p.dec + ((size_t)r * p.B + bb) * p.k,
           r == 0 && dec_smem ? sm.dec + (size_t)bb * p.k : nullptr);
  }
  __syncthreads();
  if (p.blob_table) {
    __threadfence();
    build_jobs_cta(p, sm, dec_smem ? sm.dec : p.dec);
  }
  if (tid == 0) *p.done = 0u;
}


// Decode router (batch 1, top-2, E <= 32): one cluster of C CTAs runs the
// filtered router (route_filtered), extra CTAs zero the accumulation
// buffers.  A kernel of its own: small code and shared memory (the general
// router kernel is measurably slower when this path is compiled into it).
template <int C>
__global__ void __launch_bounds__(kRouterThreads)
router_dec_kernel(const __grid_constant__ RouterParams p) {
  __shared__ DecSmem sm;
  if ((int)blockIdx.x >= C) {
    zero_buffers(p, blockIdx.x - C, gridDim.x - C);
    return;
  }
  const int tid = threadIdx.x;
  const int crank = blockIdx.x;
  const int n8 = p.H / 8;
  const int s0 = crank * n8 / C, s1 = (crank + 1) * n8 / C;
  {
    const char* wb = reinterpret_cast<const char*>(p.wg[0]);
    const int lpr = (s1 - s0) * 16 / 128;
    for (int i = tid; i < p.E * lpr; i += kRouterThreads) {
      const int e = i / lpr, l = i - e * lpr;
      asm volatile("prefetch.global.L2 [%0];" :: "l"(wb + ((size_t)e * n8 + s0) * 16 + (size_t)l * 128));
    }
    if (p.blob_table && crank == 0)
      for (int i = tid; i < 4 * p.E; i += kRouterThreads) sm.blob[i] = p.blob_table[i];
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  route_filtered<C>(p, sm, crank, s0, s1, 0, 0);
}


// Decode router on a reserved SM (batch 1, one route layer, top-2, E <= 32;
// DESIGN.md section 5 "router").  One CTA of 1024 threads; the GEMV kernels of
// the chain run on the other 147 SMs, so this CTA is resident as soon as the
// previous K2b triggers its dependents, ~25 us before that K2b ends.  It uses
// the time for everything that does not depend on x:
//   * the layer's router rows W_g [E][H] into shared memory (bulk copies),
//     the blob table and the row norms;
//   * a complete dry run of the routing code on whatever x holds (results
//     into shared-memory sinks, global stores predicated off): the router
//     runs once per layer between much larger kernels, so otherwise every
//     step of it starts from a cold instruction cache (measured: ~7800 SM
//     cycles for the decide + job-table steps alone, tools/legacy_timeline.py).
// After griddepcontrol.wait only x (8 KB) is loaded; the logits are the
// filtered ones (R9': exact fp16 x fp16 products in fp32 FFMA chains of 8,
// warp trees, fp64 sums over warps, Cauchy-Schwarz bound), the exact integer
// path decides when a comparison does not clear the bound.  The accumulation
// buffers are not zeroed here: hfin leaves the K2a sums clean and zeroes y
// (GemvParams::clean).
constexpr int kSoloThreads = 1024;
constexpr int kSoloWarps = kSoloThreads / 32;
struct SoloSmem {
  float red[kSoloWarps][32];           // per warp fp32 partial logit per expert
  float xqw[kSoloWarps];               // per warp sum of x^2
  double Lf[32];                       // filtered logits
  double xsq;                          // ||x||^2
  u64 part[kSoloWarps][32][3];         // exact fallback: per warp partial per expert
  i128 L[32];                          // exact fallback: logits
  hb_decision dec[2];
  const uint8_t* blob[32 * 4];
  Job jobs[3];
  float wn[32];
  uint4 xs[1024];                      // x (H <= 8192)
  // pass-0 destinations
  hb_decision dry_dec[2];
  int32_t dry_hdr[3], dry_slot_token[2], dry_tok_slots[2], dry_rowbad;
  float dry_slot_gate[2];
  Job dry_jobs[2];
  VJobD dry_vjobs[2];
  long long dry_vcum13[3], dry_vcum2[3];
  uint64_t wbar;
  int ok, bad;
};
extern __shared__ __align__(128) uint8_t solo_dyn[];   // W_g [E][H] fp16

// The job table of one token's two selections (B = 1, k = 2) by lanes 0 and
// 1 of a warp: the table build_jobs_warp writes for nsel = 2 (jobs and slots
// by key = expert * 2 + served-from-lo_enc, one slot per job, vjob = job),
// without its loops (the router is on every layer's critical path).
__device__ __forceinline__ void build_jobs_k2(const RouterParams& p, const hb_decision* dec,
                                              const uint8_t* const* blob, const JobTable& jt,
                                              hb_decision* dout) {
  const int lane = threadIdx.x & 31;
  hb_decision d = dec[lane & 1];
  const unsigned long long hb = lane < 2 ? high_bit(p, d) : 0ull;
  const unsigned long long hmask = hb | __shfl_xor_sync(0xffffffffu, hb, 1);
  const int key = lane < 2 ? sel_key(p, d, hmask) : -1;
  const int ko = __shfl_xor_sync(0xffffffffu, key, 1);
  const bool valid = key >= 0;
  const int slot = valid ? (ko >= 0 && ko < key ? 1 : 0) : -1;
  const int nj = (key >= 0) + (ko >= 0);
  const int enc = (key & 1) ? p.lo_enc : p.hi_enc;
  const long long u13 = valid ? (long long)(p.F / 16) * (p.H / epg_of_enc(enc)) : 0;
  const long long u2 = valid ? (long long)(p.H / 16) * (p.F / epg_of_enc(enc)) : 0;
  const long long o13 = __shfl_xor_sync(0xffffffffu, u13, 1), o2 = __shfl_xor_sync(0xffffffffu, u2, 1);
  if (lane >= 2) return;
  jt.tok_slots[lane] = slot;
  if (valid) {
    const uint8_t* b = blob[(key >> 1) * 4 + enc];
    jt.slot_token[slot] = 0;
    jt.slot_gate[slot] = d.gate;
    Job j;
    j.blob = b; j.enc = enc; j.expert = key >> 1; j.n_tok = 1; j.slot_off = slot;
    jt.jobs[slot] = j;
    VJobD v;
    v.blob = b; v.enc = enc; v.slot0 = slot; v.nslot = 1; v.pad = 0;
    jt.vjobs[slot] = v;
    jt.vcum13[slot + 1] = slot ? u13 + o13 : u13;   // cumulative units, vjobs in slot order
    jt.vcum2[slot + 1] = slot ? u2 + o2 : u2;
    d.served_enc = (uint8_t)enc;
    d.hit = 1;
    dout[lane] = d;
  }
  if (lane == 0) {
    jt.vcum13[0] = 0;
    jt.vcum2[0] = 0;
    jt.hdr[0] = nj;
    jt.hdr[1] = nj;
    jt.hdr[2] = nj;
  }
}

__global__ void __launch_bounds__(kSoloThreads, 1)
router_solo_kernel(const __grid_constant__ RouterParams p) {
  __shared__ SoloSmem sm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int E = p.E, n8 = p.H / 8;
  const int G = kSoloThreads / n8;             // thread groups over the x chunks (n8 | 1024)
  const int wpg = n8 / 32;                     // warps per group
  const int c = tid % n8, g = tid / n8;        // this thread: chunk c, experts g, g + G, ...
  const uint4* w4 = reinterpret_cast<const uint4*>(solo_dyn);
  const uint32_t wbar = (uint32_t)__cvta_generic_to_shared(&sm.wbar);
#ifdef HB_LEGACY_TL
  const unsigned long long tl_entry = tl_now();
#endif
#if HB_LEGACY_TL == 2
  long long tl_sub[7] = {0, 0, 0, 0, 0, 0, 0};
  long long tl_c0 = 0;
#endif
  // ---- static inputs: router rows by bulk copies, blob table, row norms
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(wbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t total = (uint32_t)E * p.H * 2;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(wbar), "r"(total) : "memory");
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(solo_dyn);
    for (uint32_t off = 0; off < total; off += 16384) {
      const uint32_t len = total - off < 16384 ? total - off : 16384;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          :: "r"(dst + off), "l"(reinterpret_cast<const char*>(p.wg[0]) + off), "r"(len), "r"(wbar)
          : "memory");
    }
  }
  if (p.blob_table)
    for (int i = tid; i < 4 * E; i += kSoloThreads) sm.blob[i] = p.blob_table[i];
  for (int i = tid; i < E; i += kSoloThreads) sm.wn[i] = p.wnorm[i];
  JobTable dry_jt;
  dry_jt.hdr = sm.dry_hdr;
  dry_jt.jobs = sm.dry_jobs;
  dry_jt.slot_token = sm.dry_slot_token;
  dry_jt.slot_gate = sm.dry_slot_gate;
  dry_jt.tok_slots = sm.dry_tok_slots;
  dry_jt.vjobs = sm.dry_vjobs;
  dry_jt.vcum13 = sm.dry_vcum13;
  dry_jt.vcum2 = sm.dry_vcum2;
  __syncthreads();
  {                                            // router rows landed
    uint32_t done;
    do {
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0, 1, 0, P; }"
                   : "=r"(done) : "r"(wbar) : "memory");
    } while (!done);
  }
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    const bool live = pass == 1;
    if (live) {
      asm volatile("griddepcontrol.wait;" ::: "memory");       // x belongs to earlier work
      asm volatile("griddepcontrol.launch_dependents;");
#ifdef HB_LEGACY_TL
      if (tid == 0) {
        unsigned long long* rec = tl_rec(p.stamps, p.stamp_cap, p.fwd_idx);
        tl_min(rec, 6, tl_now());
        tl_min(rec, 5, tl_entry);
      }
#endif
#if HB_LEGACY_TL == 2
      tl_c0 = clock64();
#endif
    }
    // ---- x (L2 loads: the pass-0 x must never sit in L1), finiteness, ||x||^2
    int xbad = 0;
    float xq = 0.f;
    if (tid < n8) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p.x) + tid);
      sm.xs[tid] = v;
      const uint32_t xa[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        xbad |= ((xa[q] & 0x7C00u) == 0x7C00u) | ((xa[q] & 0x7C000000u) == 0x7C000000u);
      float xf[8];
      r_h2f8(v, xf);
#pragma unroll
      for (int q = 0; q < 8; ++q) xq = fmaf(xf[q], xf[q], xq);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xq += __shfl_xor_sync(0xffffffffu, xq, o);
    if (lane == 0) sm.xqw[warp] = xq;
    const int bad = __syncthreads_or(xbad);
    HB_RSUB(8);
    // ---- filtered partial logits: chunk c of x against experts g, g + G, ...
    {
      float xf[8];
      r_h2f8(sm.xs[c], xf);
      for (int e = g; e < E; e += G) {
        float wf[8];
        r_h2f8(w4[(size_t)e * n8 + c], wf);
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = fmaf(wf[q], xf[q], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) sm.red[warp][e] = acc;
      }
    }
    __syncthreads();
    // ---- fp64 sums: warp e < E sums expert e over the warps of its group,
    // the last warp sums ||x||^2 (fixed shuffle trees: deterministic)
    if (warp < E) {
      const int w0 = (warp % G) * wpg;
      double v = lane < wpg ? (double)sm.red[w0 + lane][warp] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sm.Lf[warp] = v;
    } else if (warp == kSoloWarps - 1) {
      double v = (double)sm.xqw[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sm.xsq = v;
    }
    __syncthreads();
    HB_RSUB(9);
    if (warp == 0) {
      // ---- warp 0: the certainty of every comparison, decisions, gates, jobs
      hb_decision* dout = live ? p.dec : sm.dry_dec;
      // error of a logit: fp32 chains of 8 products (gamma_7), warp trees
      // (gamma_5), fp64 sums over warps (negligible): (8 + 6) * 2^-24 *
      // sum|p| * (1 + 1e-4), with sum|p| <= ||w_e|| ||x|| (||x|| rounded up)
      const double xn = sqrt(sm.xsq) * (1.0 + 1e-6) + 1e-30;
      const double cb = 14.0 * 0x1p-24 * 1.0001;
      const int e = lane;
      const double v = e < E ? sm.Lf[e] : -1e300;
      const double ep = e < E ? cb * (double)sm.wn[e] * xn : 0.0;
      int r = 0;                                 // rank by (L desc, index asc); lanes >= E unused
      for (int f = 0; f < E; ++f) {
        const double o = sm.Lf[f];
        r += (o > v) || (o == v && f < e);
      }
      const unsigned m0 = __ballot_sync(0xffffffffu, e < E && r == 0);
      const unsigned m1 = __ballot_sync(0xffffffffu, e < E && r == 1);
      const int e0 = __ffs(m0) - 1, e1 = __ffs(m1) - 1;
      double rest = (e < E && r >= 2) ? v + ep : -1e300;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rest = fmax(rest, __shfl_xor_sync(0xffffffffu, rest, o));
      const double L0 = sm.Lf[e0], L1 = sm.Lf[e1];
      const double ep0 = __shfl_sync(0xffffffffu, ep, e0), ep1 = __shfl_sync(0xffffffffu, ep, e1);
      const double Gp = L0 - L1, mg = ep0 + ep1 + 1e-12 * (1.0 + fabs(L0) + fabs(L1));
      bool ok = !bad && (L0 - ep0 > L1 + ep1) && (L1 - ep1 > rest);
      if (p.th1_kind == 0) ok = ok && fabs(Gp - (double)p.theta1 * 0x1p-48) > mg;
      if (p.th2_kind == 0) ok = ok && fabs(Gp - (double)p.theta2 * 0x1p-48) > mg;
      if (lane < 2) {
        // lane 0 writes selection 0, lane 1 selection 1
        const uint8_t prec1 =
            (p.th1_kind > 0 || (p.th1_kind == 0 && Gp <= (double)p.theta1 * 0x1p-48)) ? HB_HIGH
            : (p.th2_kind > 0 || (p.th2_kind == 0 && Gp <= (double)p.theta2 * 0x1p-48)) ? HB_LOW
                                                                                        : HB_SKIP;
        const float ex = expf(-(float)Gp);
        const float g0 = 1.f / (1.f + ex);
        hb_decision d;
        d.token = 0; d.sel_rank = (uint8_t)lane; d.served_enc = HB_ENC_NONE; d.hit = 0;
        if (bad) {                               // R28: Skip, expert -1, gate NaN
          d.expert = -1; d.prec = HB_SKIP; d.gate = __int_as_float(0x7fc00000);
        } else {
          d.expert = lane ? e1 : e0; d.prec = lane ? prec1 : (uint8_t)HB_HIGH; d.gate = lane ? ex * g0 : g0;
        }
        if (ok || bad) { dout[lane] = d; sm.dec[lane] = d; }
        if (lane == 0) { *(live ? p.rowbad : &sm.dry_rowbad) = bad; sm.ok = ok || bad; }
      }
      __syncwarp();
      HB_RSUB(10);
      if ((ok || bad) && p.blob_table) build_jobs_k2(p, sm.dec, sm.blob, live ? p.jt : dry_jt, dout);
      HB_RSUB(11);
    } else if (live) {
      // ---- the other warps meanwhile: pair-permuted x + block sums (K2a) and
      // the copy for the lazy exact logits
      const int t2 = tid - 32;
      if (t2 < n8 / 4) {
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 t = sm.xs[4 * t2 + i];
          v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
        }
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          sum += __half2float(__ushort_as_half((unsigned short)(v[i >> 1] >> (16 * (i & 1)))));
        p.xsum[t2] = sum;
#pragma unroll
        for (int t = 0; t < 4; ++t) {            // uint4 t: Q_c = (x[8t+c], x[8t+c+4])
          uint32_t q[4];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int e0 = 8 * t + cc, e1 = e0 + 4;
            const uint32_t lo16 = (v[e0 >> 1] >> (16 * (e0 & 1))) & 0xFFFF;
            const uint32_t hi16 = (v[e1 >> 1] >> (16 * (e1 & 1))) & 0xFFFF;
            q[cc] = lo16 | (hi16 << 16);
          }
          p.x_perm[t2 * 4 + t] = make_uint4(q[0], q[1], q[2], q[3]);
        }
      }
      if (p.x_save && t2 < n8) reinterpret_cast<uint4*>(p.x_save)[t2] = sm.xs[t2];
    }
    __syncthreads();
    if (!sm.ok) {
      // ---- exact fallback (rare): integer logits from the same shared rows
      const uint4 xv = sm.xs[c];
      const uint32_t xa[4] = {xv.x, xv.y, xv.z, xv.w};
      for (int e = g; e < E; e += G) {
        const uint4 wv = w4[(size_t)e * n8 + c];
        const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
        u64 lo = 0, mid = 0, hi = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          accum_exact((wa[i >> 1] >> (16 * (i & 1))) & 0xFFFF, (xa[i >> 1] >> (16 * (i & 1))) & 0xFFFF,
                      lo, mid, hi);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo += __shfl_xor_sync(0xffffffffu, lo, o);
          mid += __shfl_xor_sync(0xffffffffu, mid, o);
          hi += __shfl_xor_sync(0xffffffffu, hi, o);
        }
        if (lane == 0) { sm.part[warp][e][0] = lo; sm.part[warp][e][1] = mid; sm.part[warp][e][2] = hi; }
      }
      __syncthreads();
      if (tid < E) {
        const int w0 = (tid % G) * wpg;
        u64 lo = 0, mid = 0, hi = 0;
        for (int w = 0; w < wpg; ++w) {
          lo += sm.part[w0 + w][tid][0]; mid += sm.part[w0 + w][tid][1]; hi += sm.part[w0 + w][tid][2];
        }
        sm.L[tid] = (i128)(long long)lo + ((i128)(long long)mid << 20) + ((i128)(long long)hi << 40);
      }
      __syncthreads();
      if (warp == 0) {
        hb_decision* dout = live ? p.dec : sm.dry_dec;
        decide_k2_warp(p, sm.L, 0, dout, sm.dec);
        __syncwarp();
        if (p.blob_table) build_jobs_k2(p, sm.dec, sm.blob, live ? p.jt : dry_jt, dout);
      }
    }
#ifdef HB_LEGACY_TL
    if (live && tid == 0) {
      unsigned long long* rec = tl_rec(p.stamps, p.stamp_cap, p.fwd_idx);
      tl_max(rec, 7, tl_now());
#if HB_LEGACY_TL == 2
      for (int f = 0; f < 4; ++f) tl_max(rec, 8 + f, (unsigned long long)(tl_sub[f] - tl_c0));
#endif
    }
#endif
    __syncthreads();
  }
}

bool router_solo_fits(int E, int H, int k) {
  const int n8 = H / 8;
  return k == 2 && E >= 2 && E <= 31 && n8 >= 32 && n8 <= kSoloThreads && kSoloThreads % n8 == 0 &&
         (long long)E * H * 2 + (long long)sizeof(SoloSmem) + 1024 <= 227 * 1024;
}

void launch_router_solo(const RouterParams& p, cudaStream_t s) {
  const int smem = p.E * p.H * 2;
  static int max_dyn = [] {                  // once: the largest the static part leaves
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, router_solo_kernel);
    return 227 * 1024 - (int)fa.sharedSizeBytes;
  }();
  set_max_dyn_smem(router_solo_kernel, max_dyn);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kSoloThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, router_solo_kernel, p);
}

// Router for batches (n_route = 1, top-2, E <= 64): one CTA per token row,
// the filtered router (fp32 products in FFMA chains, warp trees, fp64 sums
// over warps, Cauchy-Schwarz bound; the exact integer path for a row whose
// comparisons do not clear the bound), each row decided in its own CTA; the
// last CTA builds the job table.  Extra CTAs zero the accumulation buffers.
// Replaces the exact per-row partials of router_kernel<1> (R9').
__global__ void __launch_bounds__(kRouterThreads)
router_batch_kernel(const __grid_constant__ RouterParams p) {
  __shared__ BatchSmem sm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kRouterThreads / 32;
  if ((int)blockIdx.x >= p.B) {
    zero_buffers(p, blockIdx.x - p.B, gridDim.x - p.B);
    return;
  }
  const int b = blockIdx.x;
  const int E = p.E, n8 = p.H / 8;
  if (p.blob_table)
    for (int i = tid; i < 4 * E; i += kRouterThreads) sm.blob[i] = p.blob_table[i];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const __half* x = p.x + (size_t)b * p.H;
  const uint4* x4 = reinterpret_cast<const uint4*>(x);
  const uint4* w4 = reinterpret_cast<const uint4*>(p.wg[0]);
  int xbad = 0;
  float xq = 0.f;
  int nch = 0;
  for (int c = tid; c < n8; c += kRouterThreads) ++nch;
  for (int e0 = 0; e0 < E; e0 += 16) {
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.f;
    for (int c = tid; c < n8; c += kRouterThreads) {
      const uint4 xv = x4[c];
      float xf[8];
      r_h2f8(xv, xf);
      if (e0 == 0) {
        const uint32_t xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          xbad |= ((xa[q] & 0x7C00u) == 0x7C00u) | ((xa[q] & 0x7C000000u) == 0x7C000000u);
#pragma unroll
        for (int q = 0; q < 8; ++q) xq = fmaf(xf[q], xf[q], xq);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (e0 + j >= E) break;
        float wf[8];
        r_h2f8(w4[(size_t)(e0 + j) * n8 + c], wf);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[j] = fmaf(wf[q], xf[q], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float v = acc[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && e0 + j < E) sm.red[warp][e0 + j] = v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) xq += __shfl_xor_sync(0xffffffffu, xq, o);
  if (lane == 0) sm.xqw[warp] = xq;
  const int bad = __syncthreads_or(xbad);
  if (p.x_save)                                     // lazy exact logits (hb_get_logits)
    for (int c = tid; c < n8; c += kRouterThreads)
      reinterpret_cast<uint4*>(p.x_save + (size_t)b * p.H)[c] = x4[c];
  if (p.x_perm) write_xperm(p, x, 0, n8, b);
  if (tid < E) {
    double v = 0.0;
    for (int w = 0; w < NW; ++w) v += (double)sm.red[w][tid];
    sm.Lf[tid] = v;
  }
  __syncthreads();
  if (warp == 0) {
    if (bad) {
      if (lane == 0) { decide_nonfinite(p, b, p.dec + (size_t)b * 2, nullptr); sm.ok = 1; }
    } else {
      double xs = 0.0;
      for (int w = 0; w < NW; ++w) xs += (double)sm.xqw[w];
      // error of a logit: chains of m = 8 * nch products (gamma_{m-1}), warp
      // trees (gamma_5), fp64 sums over warps (negligible): (m + 6) 2^-24
      // (1 + 1e-4) sum|p|, sum|p| <= ||w_e|| ||x|| (||x|| rounded up)
      const int m = 8 * __shfl_sync(0xffffffffu, nch, 0);
      const double xn = sqrt(xs) * (1.0 + 1e-6) + 1e-30;
      const double cb = (m + 6) * 0x1p-24 * 1.0001;
      double vh[2] = {-1e300, -1e300}, eh[2] = {0.0, 0.0};
      int rk[2] = {64, 64};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h;
        if (e < E) {
          vh[h] = sm.Lf[e];
          eh[h] = cb * (double)p.wnorm[e] * xn;
          int r = 0;
          for (int f = 0; f < E; ++f) { const double o = sm.Lf[f]; r += (o > vh[h]) || (o == vh[h] && f < e); }
          rk[h] = r;
        }
      }
      const unsigned m0 = __ballot_sync(0xffffffffu, rk[0] == 0), m0b = __ballot_sync(0xffffffffu, rk[1] == 0);
      const unsigned m1 = __ballot_sync(0xffffffffu, rk[0] == 1), m1b = __ballot_sync(0xffffffffu, rk[1] == 1);
      const int e0 = m0 ? __ffs(m0) - 1 : 32 + __ffs(m0b) - 1;
      const int e1 = m1 ? __ffs(m1) - 1 : 32 + __ffs(m1b) - 1;
      double rest = -1e300;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (lane + 32 * h < E && rk[h] >= 2) rest = fmax(rest, vh[h] + eh[h]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rest = fmax(rest, __shfl_xor_sync(0xffffffffu, rest, o));
      if (lane == 0) {
        const double L0 = sm.Lf[e0], L1 = sm.Lf[e1];
        const double ep0 = cb * (double)p.wnorm[e0] * xn, ep1 = cb * (double)p.wnorm[e1] * xn;
        const double G = L0 - L1, mg = ep0 + ep1 + 1e-12 * (1.0 + fabs(L0) + fabs(L1));
        bool ok = (L0 - ep0 > L1 + ep1) && (L1 - ep1 > rest);
        if (p.th1_kind == 0) ok = ok && fabs(G - (double)p.theta1 * 0x1p-48) > mg;
        if (p.th2_kind == 0) ok = ok && fabs(G - (double)p.theta2 * 0x1p-48) > mg;
        if (ok) {
          const uint8_t prec1 = (p.th1_kind > 0 || (p.th1_kind == 0 && G <= (double)p.theta1 * 0x1p-48)) ? HB_HIGH
                              : (p.th2_kind > 0 || (p.th2_kind == 0 && G <= (double)p.theta2 * 0x1p-48)) ? HB_LOW
                                                                                                      : HB_SKIP;
          const float ex = expf(-(float)G);
          const float g0 = 1.f / (1.f + ex), g1 = ex * g0;
          hb_decision r0, r1;
          r0.token = b; r0.expert = e0; r0.sel_rank = 0; r0.prec = HB_HIGH;
          r0.served_enc = HB_ENC_NONE; r0.hit = 0; r0.gate = g0;
          r1.token = b; r1.expert = e1; r1.sel_rank = 1; r1.prec = prec1;
          r1.served_enc = HB_ENC_NONE; r1.hit = 0; r1.gate = g1;
          p.dec[(size_t)b * 2] = r0;
          p.dec[(size_t)b * 2 + 1] = r1;
        }
        sm.ok = ok;
      }
    }
  }
  __syncthreads();
  if (!sm.ok) {
    // ---- exact fallback for this row (rare): integer logits over all of H
    const int wpe = E >= NW ? 1 : NW / E;
    for (int task = warp; task < E * wpe; task += NW) {
      const int e = task / wpe, part = task - e * wpe;
      const uint4* we = w4 + (size_t)e * n8;
      const int j0 = part * n8 / wpe, j1 = (part + 1) * n8 / wpe;
      u64 lo = 0, mid = 0, hi = 0;
      for (int j = j0 + lane; j < j1; j += 32) {
        const uint4 wv = we[j];
        const uint4 xv = x4[j];
        const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
          accum_exact((wa[i >> 1] >> (16 * (i & 1))) & 0xFFFF, (xa[i >> 1] >> (16 * (i & 1))) & 0xFFFF,
                      lo, mid, hi);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        mid += __shfl_xor_sync(0xffffffffu, mid, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      if (lane == 0) { sm.part[task][0] = lo; sm.part[task][1] = mid; sm.part[task][2] = hi; }
    }
    __syncthreads();
    for (int e = tid; e < E; e += blockDim.x) {
      u64 lo = 0, mid = 0, hi = 0;
      for (int q = 0; q < wpe; ++q) {
        lo += sm.part[e * wpe + q][0]; mid += sm.part[e * wpe + q][1]; hi += sm.part[e * wpe + q][2];
      }
      sm.L[e] = (i128)(long long)lo + ((i128)(long long)mid << 20) + ((i128)(long long)hi << 40);
    }
    __syncthreads();
    if (warp == 0) {
      if (E <= 32) {
        decide_k2_warp(p, sm.L, b, p.dec + (size_t)b * 2, p.dec + (size_t)b * 2);
      } else {
        int sel[kMaxTopK];
        topk_warp(p, sm.L, sel);
        if (lane == 0) decide_sel(p, sm.L, sel, b, p.dec + (size_t)b * 2, nullptr);
      }
    }
  }
  if (tid == 0) p.rowbad[b] = bad;
  // ---- the last row CTA builds the job table from every row's decisions
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    sm.last = atomicAdd(p.done, 1u) == (unsigned)p.B - 1;
  }
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  if (p.blob_table) build_jobs_cta(p, sm, p.dec);
  if (tid == 0) *p.done = 0u;
}

void launch_router(const RouterParams& p, cudaStream_t s) {
  // one 8-CTA cluster per (route layer, token) row, plus clusters of CTAs that
  // zero the GEMV accumulation buffers in parallel
  const int C = p.n_route * p.B >= 16 ? 1 : kRouterCluster;
  const bool dec = p.filtered && p.n_route == 1 && p.B == 1 && p.k == 2 && p.E <= 32;
  const long long nz4 = (p.zero_n[0] + p.zero_n[1] + p.zero_n[2]) / 4;
  int zc = nz4 ? (int)std::min<long long>(32, (nz4 + 2 * kRouterThreads - 1) / (2 * kRouterThreads)) : 0;
  zc = (zc + C - 1) / C * C;
  const int grid = p.n_route * p.B * C + zc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRouterThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = kRouterCluster;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  const bool batch = p.filtered_batch && p.n_route == 1 && C == 1 && p.k == 2 && p.E <= 64;
  if (dec) {
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, router_dec_kernel<kRouterCluster>, p);
  } else if (batch) {
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, router_batch_kernel, p);
  } else if (C == 1) {
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, router_kernel<1>, p);
  } else {
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, router_kernel<kRouterCluster>, p);
  }
}

// ------------------------------------------------ token-sharded EP (f3)
// One CTA per local token b: one row per owner rank of its non-skipped
// selections (owners in the order of the token's selections).  The row of
// (b, owner d) is d * C + (number of tokens before b with a selection owned by
// d): a prefix count over the decisions, deterministic.  The row carries the
// token's selections owned by d (rank order) and its x.
__global__ void __launch_bounds__(128) ts_pack_kernel(const __grid_constant__ TsParams p) {
  const int b = blockIdx.x, tid = threadIdx.x;
  __shared__ int s_dest[kMaxTopK], s_cnt[kMaxTopK], s_row[kMaxTopK];
  __shared__ int s_nd;
  if (tid == 0) {                                // the token's owners, in selection order
    int nd = 0;
    for (int i = 0; i < p.k; ++i) {
      const hb_decision d = p.dec[b * p.k + i];
      if (d.prec == HB_SKIP || d.expert < 0) continue;
      const int dest = d.expert % p.R;
      bool seen = false;
      for (int q = 0; q < nd; ++q) seen |= s_dest[q] == dest;
      if (!seen) { s_cnt[nd] = 0; s_dest[nd++] = dest; }
    }
    s_nd = nd;
  }
  __syncthreads();
  const int nd = s_nd;
  // rows already taken in each owner's block: tokens before b with a selection it owns
  for (int bb = tid; bb < b; bb += blockDim.x) {
    unsigned mask = 0u;
    for (int i = 0; i < p.k; ++i) {
      const hb_decision o = p.dec[bb * p.k + i];
      if (o.prec == HB_SKIP || o.expert < 0) continue;
      for (int q = 0; q < nd; ++q) if (o.expert % p.R == s_dest[q]) mask |= 1u << q;
    }
    for (int q = 0; q < nd; ++q) if (mask >> q & 1u) atomicAdd(&s_cnt[q], 1);
  }
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < nd; ++q) {
      s_row[q] = s_dest[q] * p.C + s_cnt[q];
      hb_ts_meta m;
      m.token = b;
      m.n = 0;
      for (int z = 0; z < kMaxTopK; ++z) { m.expert[z] = -1; m.prec[z] = HB_SKIP; m.gate[z] = 0.f; }
      for (int i = 0; i < p.k; ++i) {
        const hb_decision d = p.dec[b * p.k + i];
        if (d.prec == HB_SKIP || d.expert < 0 || d.expert % p.R != s_dest[q]) continue;
        m.expert[m.n] = d.expert;
        m.prec[m.n] = d.prec;
        m.gate[m.n] = d.gate;
        m.n += 1;
      }
      p.meta_send[s_row[q]] = m;
    }
    for (int i = 0; i < p.k; ++i) {
      const hb_decision d = p.dec[b * p.k + i];
      int pos = -1;
      if (d.prec != HB_SKIP && d.expert >= 0)
        for (int q = 0; q < nd; ++q) if (d.expert % p.R == s_dest[q]) pos = s_row[q];
      p.pos[b * p.k + i] = pos;
    }
  }
  __syncthreads();
  const uint4* src = reinterpret_cast<const uint4*>(p.x + (size_t)b * p.H);
  for (int r = 0; r < nd; ++r) {
    uint4* dst = reinterpret_cast<uint4*>(p.rows_send + (size_t)s_row[r] * p.H);
    for (int i = tid; i < p.H / 8; i += blockDim.x) dst[i] = src[i];
  }
}

// y[b] = sum of the token's returned rows (one per owner, in the order of the
// token's selections); NaN for a token whose x was non-finite (R28)
__global__ void __launch_bounds__(256) ts_combine_kernel(const __grid_constant__ TsParams p) {
  const int b = blockIdx.x;
  const bool bad = p.rowbad && p.rowbad[b];
  int pos[kMaxTopK];
  for (int i = 0; i < p.k; ++i) {
    pos[i] = p.pos[b * p.k + i];
    for (int q = 0; q < i; ++q)
      if (pos[q] == pos[i]) pos[i] = -1;        // the owner's row counted once
  }
  for (int c = threadIdx.x * 4; c < p.H; c += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < p.k; ++i) {
      if (pos[i] < 0) continue;
      const float4 v = *reinterpret_cast<const float4*>(p.ret + (size_t)pos[i] * p.H + c);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (bad) acc = make_float4(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000),
                               __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    *reinterpret_cast<float4*>(p.y + (size_t)b * p.H + c) = acc;
  }
}

// Received rows -> the owner's batch: one CTA per row writes the row's k
// decision records (its n selections, then Skip), its pair-permuted x and
// block sums, zero rowbad and zero y; the last CTA builds the job table.
__global__ void __launch_bounds__(kRouterThreads)
ts_jobs_kernel(const __grid_constant__ RouterParams p, const hb_ts_meta* meta, const __half* rows,
               float* y) {
  __shared__ BatchSmem sm;
  const int j = blockIdx.x, tid = threadIdx.x;
  if (tid < p.k) {
    const hb_ts_meta& m = meta[j];
    hb_decision d;
    d.token = j;
    d.sel_rank = (uint8_t)tid;
    d.served_enc = HB_ENC_NONE;
    d.hit = 0;
    if (m.token >= 0 && tid < m.n) {             // the row's selections, then Skip
      d.expert = m.expert[tid];
      d.prec = m.prec[tid];
      d.gate = m.gate[tid];
    } else {
      d.expert = -1;
      d.prec = HB_SKIP;
      d.gate = 0.f;
    }
    p.dec[j * p.k + tid] = d;
  }
  if (tid == 0) p.rowbad[j] = 0;
  write_xperm(p, rows + (size_t)j * p.H, 0, p.H / 8, j);
  for (int c = tid * 4; c < p.H; c += blockDim.x * 4)
    *reinterpret_cast<float4*>(y + (size_t)j * p.H + c) = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = tid; i < 4 * p.E; i += blockDim.x) sm.blob[i] = p.blob_table[i];
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    sm.last = atomicAdd(p.done, 1u) == (unsigned)p.B - 1;
  }
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  build_jobs_cta(p, sm, p.dec);
  if (tid == 0) *p.done = 0u;
}

void launch_ts_pack(const TsParams& p, cudaStream_t s) {
  if (p.B > 0) ts_pack_kernel<<<p.B, 128, 0, s>>>(p);
}
void launch_ts_combine(const TsParams& p, cudaStream_t s) {
  if (p.B > 0) ts_combine_kernel<<<p.B, 256, 0, s>>>(p);
}
void launch_ts_jobs(const RouterParams& p, const hb_ts_meta* meta, const __half* rows, float* y,
                    cudaStream_t s) {
  ts_jobs_kernel<<<p.B, kRouterThreads, 0, s>>>(p, meta, rows, y);
}

}  // namespace hb

#ifdef HB_DBG_TIMELINE
extern "C" int hb_debug_router_timeline(void* host) {
  return (int)cudaMemcpyFromSymbol(host, hb::g_rtl, sizeof(hb::g_rtl));
}
#endif
