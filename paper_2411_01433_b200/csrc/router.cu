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
// Launch: one CTA per (route layer, token, expert) row: B*n_route*E CTAs of
// 128 threads (at B = 1 decode the 8 or 16 rows run in parallel instead of
// one CTA walking them).  The last CTA to finish (grid counter) selects the
// top-k of every (route layer, token), writes the decision records and, in
// resident mode, the job table.  The CTAs of expert 0 also write the
// pair-permuted copy of x and its block sums for the GEMV kernels.
#include <cuda_fp16.h>

#include "hb_internal.h"

namespace hb {

typedef __int128 i128;
typedef unsigned long long u64;

__device__ __forceinline__ void fp16_mant_exp(uint32_t bits, int& m, int& e) {
  const int ex = (bits >> 10) & 0x1F;
  const int man = bits & 0x3FF;
  m = ex ? (man | 0x400) : man;
  e = ex ? ex - 25 : -24;              // value = m * 2^e
  if (bits & 0x8000) m = -m;
}

// Products m_w*m_x (|.| < 2^22) shifted by s = e_w+e_x+48 in [0, 58] go to
// three int64 accumulators by s range: [0,20) -> lo, [20,40) -> mid (shifted
// by s-20), [40,58] -> hi (shifted by s-40).  Each term is < 2^41, so up to
// 2^20 terms cannot overflow; L = lo + mid*2^20 + hi*2^40 exactly.
__device__ __forceinline__ void accum_exact(uint32_t wbits, uint32_t xbits, u64& lo, u64& mid,
                                            u64& hi) {
  int mw, ew, mx, ex;
  fp16_mant_exp(wbits, mw, ew);
  fp16_mant_exp(xbits, mx, ex);
  const u64 p = (u64)(long long)(mw * mx);
  const int s = ew + ex + 48;
  if (s >= 40) hi += p << (s - 40);
  else if (s >= 20) mid += p << (s - 20);
  else lo += p << s;
}

__device__ __forceinline__ bool gap_le(i128 G, int kind, long long theta) {
  if (kind > 0) return true;
  if (kind < 0) return false;
  return G <= (i128)theta;
}

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

// O3-O6 for one (route layer, token): top-k, gates, scores, decisions
__device__ void decide(const RouterParams& p, int rl, int b) {
  const size_t base = ((size_t)rl * p.B + b) * p.E;
  i128 L[64];
  for (int e = 0; e < p.E; ++e) L[e] = load_logit(p.lbuf, base + e);
  int sel[kMaxTopK];
  unsigned long long taken = 0ull;
  for (int i = 0; i < p.k; ++i) {                 // O3: (L desc, index asc)
    int best = -1;
    for (int e = 0; e < p.E; ++e) {
      if (taken >> e & 1ull) continue;
      if (best < 0 || L[e] > L[best]) best = e;
    }
    sel[i] = best;
    taken |= 1ull << best;
  }
  const double l0 = i128_to_double(L[sel[0]]) * 0x1p-48;
  double g[kMaxTopK], tot = 0.0;
  for (int i = 0; i < p.k; ++i) {                 // O4: softmax over the selected
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
  hb_decision* out = p.dec + ((size_t)rl * p.B + b) * p.k;
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
  }
  if (rl == 0 && p.logits)
    for (int e = 0; e < p.E; ++e) {
      p.logits[((size_t)b * p.E + e) * 2 + 0] = (long long)(u64)L[e];
      p.logits[((size_t)b * p.E + e) * 2 + 1] = (long long)(L[e] >> 64);
    }
}

// resident mode: group the non-skipped owned selections into (expert, enc) jobs
__device__ void build_jobs(const RouterParams& p) {
  int count[2 * 64], jobid[2 * 64], fill[2 * 64];
  const int nkey = 2 * p.E;
  for (int i = 0; i < nkey; ++i) count[i] = 0;
  const int nsel = p.B * p.k;
  for (int i = 0; i < nsel; ++i) {
    const int4 raw = __ldcg(reinterpret_cast<const int4*>(p.dec) + i);
    const hb_decision& d = *reinterpret_cast<const hb_decision*>(&raw);
    if (d.prec == HB_SKIP || d.expert % p.world != p.rank) continue;
    count[d.expert * 2 + (d.prec == HB_HIGH ? 0 : 1)]++;
  }
  int nj = 0, off = 0;
  for (int key = 0; key < nkey; ++key) {     // jobs by expert, High before Low
    jobid[key] = -1;
    fill[key] = 0;
    if (!count[key]) continue;
    const int e = key >> 1;
    const int enc = (key & 1) ? p.lo_enc : p.hi_enc;
    Job j;
    j.blob = p.blob_table[e * 4 + enc];
    j.enc = enc;
    j.expert = e;
    j.n_tok = count[key];
    j.slot_off = off;
    p.jt.jobs[nj] = j;
    jobid[key] = nj++;
    off += count[key];
  }
  for (int i = 0; i < nsel; ++i) {           // slots in token order
    const int4 raw = __ldcg(reinterpret_cast<const int4*>(p.dec) + i);
    hb_decision d = *reinterpret_cast<const hb_decision*>(&raw);
    p.jt.tok_slots[i] = -1;
    if (d.prec == HB_SKIP || d.expert % p.world != p.rank) continue;
    const int key = d.expert * 2 + (d.prec == HB_HIGH ? 0 : 1);
    const int slot = p.jt.jobs[jobid[key]].slot_off + fill[key]++;
    p.jt.slot_token[slot] = d.token;
    p.jt.slot_gate[slot] = d.gate;
    p.jt.tok_slots[i] = slot;
    d.served_enc = (uint8_t)((key & 1) ? p.lo_enc : p.hi_enc);
    d.hit = 1;
    p.dec[i] = d;
  }
  p.jt.hdr[0] = nj;
  p.jt.hdr[1] = off;
}

__global__ void __launch_bounds__(kRouterThreads)
router_kernel(const __grid_constant__ RouterParams p) {
  __shared__ u64 red[3][kRouterThreads / 32];
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int e = blockIdx.x % p.E;
  const int b = (blockIdx.x / p.E) % p.B;
  const int rl = blockIdx.x / (p.E * p.B);

  // zero the GEMV h block-sum buffer (grid-stride)
  for (long long i = blockIdx.x * (long long)blockDim.x + tid; i < p.zero_n;
       i += (long long)gridDim.x * blockDim.x)
    p.zero_buf[i] = 0.f;

  // O2: exact logit of row e of layer rl for token b
  const __half* x = p.x + (size_t)b * p.H;
  const __half* w = p.wg[rl] + (size_t)e * p.H;
  u64 lo = 0, mid = 0, hi = 0;
  for (int h0 = tid * 8; h0 < p.H; h0 += 8 * kRouterThreads) {
    const uint4 wv = *reinterpret_cast<const uint4*>(w + h0);
    const uint4 xv = *reinterpret_cast<const uint4*>(x + h0);
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
  if (lane == 0) { red[0][warp] = lo; red[1][warp] = mid; red[2][warp] = hi; }

  // pair-permuted x and block sums for the GEMV kernels (route 0, expert 0 CTAs)
  if (p.x_perm && rl == 0 && e == 0) {
    for (int blk = tid; blk < p.H / 32; blk += blockDim.x) {
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
  __syncthreads();
  if (tid == 0) {
    u64 L0 = 0, L1 = 0, L2 = 0;
    for (int i = 0; i < kRouterThreads / 32; ++i) { L0 += red[0][i]; L1 += red[1][i]; L2 += red[2][i]; }
    const i128 L = (i128)(long long)L0 + ((i128)(long long)L1 << 20) + ((i128)(long long)L2 << 40);
    const size_t idx = ((size_t)rl * p.B + b) * p.E + e;
    p.lbuf[2 * idx] = (long long)(u64)L;
    p.lbuf[2 * idx + 1] = (long long)(L >> 64);
    __threadfence();
    const unsigned prev = atomicAdd(p.done, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  // ---- last CTA: decisions for every (route layer, token), then jobs ----
  __threadfence();
  for (int i = tid; i < p.n_route * p.B; i += blockDim.x) decide(p, i / p.B, i % p.B);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (p.blob_table) build_jobs(p);
    __threadfence();
    *p.done = 0u;
  }
}

void launch_router(const RouterParams& p, cudaStream_t s) {
  const int grid = p.n_route * p.B * p.E;
  router_kernel<<<grid, kRouterThreads, 0, s>>>(p);
}

}  // namespace hb
