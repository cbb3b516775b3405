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
// product is m_w*m_x * 2^(e_w+e_x) with e_w+e_x+48 in [0, 58].  Each lane
// splits its products into three int64 accumulators by shift range (see
// dot_exact) and the warp combines them into one int128 L on a 2^-48 grid.  The k = 2
// decision is then the integer test  L0 - L1 <= Theta  (Theta from hb_theta).
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

// lane-partial exact dot product of one router row with x (H elements, 8 per
// step).  Products m_w*m_x (|.| < 2^22) shifted by s = e_w+e_x+48 in [0, 58]
// go to three int64 accumulators by s range: [0,20) -> lo, [20,40) -> mid
// (shifted by s-20), [40,58] -> hi (shifted by s-40).  Each term is < 2^41,
// so H <= 2^20 terms cannot overflow; L = lo + mid*2^20 + hi*2^40 exactly.
__device__ __forceinline__ void dot_exact(const __half* __restrict__ w, const __half* __restrict__ x,
                                          int H, int lane, u64& lo, u64& mid, u64& hi) {
  for (int h0 = lane * 8; h0 < H; h0 += 256) {
    const uint4 wv = *reinterpret_cast<const uint4*>(w + h0);
    const uint4 xv = *reinterpret_cast<const uint4*>(x + h0);
    const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
    const uint32_t xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int mw, ew, mx, ex;
      fp16_mant_exp((wa[i >> 1] >> (16 * (i & 1))) & 0xFFFF, mw, ew);
      fp16_mant_exp((xa[i >> 1] >> (16 * (i & 1))) & 0xFFFF, mx, ex);
      const u64 p = (u64)(long long)(mw * mx);
      const int s = ew + ex + 48;
      if (s >= 40) hi += p << (s - 40);
      else if (s >= 20) mid += p << (s - 20);
      else lo += p << s;
    }
  }
}

__device__ __forceinline__ bool gap_le(i128 G, int kind, long long theta) {
  if (kind > 0) return true;
  if (kind < 0) return false;
  return G <= (i128)theta;
}

__device__ double i128_to_double(i128 v) {
  // v = hi*2^64 + lo; |v| < 2^93 here
  const bool neg = v < 0;
  unsigned __int128 a = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
  const u64 h = (u64)(a >> 64), l = (u64)a;
  double d = (double)h * 18446744073709551616.0 + (double)l;
  return neg ? -d : d;
}

__global__ void __launch_bounds__(kRouterThreads)
router_kernel(const RouterParams p) {
  extern __shared__ unsigned char smem_raw[];
  i128* logit = reinterpret_cast<i128*>(smem_raw);      // [n_route][E]
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int rows = p.n_route * p.E;

  // zero the GEMV h block-sum buffer (grid-stride)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.zero_n;
       i += (long long)gridDim.x * blockDim.x)
    p.zero_buf[i] = 0.f;

  for (int b = blockIdx.x; b < p.B; b += gridDim.x) {
    const __half* x = p.x + (size_t)b * p.H;
    for (int r = warp; r < rows; r += nwarps) {
      const int rl = r / p.E, e = r % p.E;
      u64 lo = 0, mid = 0, hi = 0;
      dot_exact(p.wg[rl] + (size_t)e * p.H, x, p.H, lane, lo, mid, hi);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        mid += __shfl_xor_sync(0xffffffffu, mid, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      if (lane == 0)
        logit[r] = (i128)(long long)lo + ((i128)(long long)mid << 20) + ((i128)(long long)hi << 40);
    }
    // pair-permuted x and block sums for the GEMV kernels (route 0 only)
    if (p.x_perm) {
      for (int blk = threadIdx.x; blk < p.H / 32; blk += blockDim.x) {
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
        // uint4 t holds Q_c = (x[8t+c], x[8t+c+4]), c = 0..3
#pragma unroll
        for (int t = 0; t < 4; ++t) {
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
    // top-k, gates, Eq. 2 scores, decisions: one thread per routed layer
    if (threadIdx.x < p.n_route) {
      const int rl = threadIdx.x;
      const i128* L = logit + rl * p.E;
      int sel[kMaxTopK];
      unsigned long long taken = 0ull;
      for (int i = 0; i < p.k; ++i) {         // O3: (L desc, index asc)
        int best = -1;
        for (int e = 0; e < p.E; ++e) {
          if (taken >> e & 1ull) continue;
          if (best < 0 || L[e] > L[best]) best = e;
        }
        sel[i] = best;
        taken |= 1ull << best;
      }
      double l0 = i128_to_double(L[sel[0]]) * 0x1p-48, g[kMaxTopK], tot = 0.0;
      for (int i = 0; i < p.k; ++i) {
        g[i] = exp(i128_to_double(L[sel[i]]) * 0x1p-48 - l0);
        tot += g[i];
      }
      uint8_t prec[kMaxTopK];
      prec[0] = HB_HIGH;                      // P:423 first expert always High
      if (p.k == 2) {
        const i128 G = L[sel[0]] - L[sel[1]];
        prec[1] = gap_le(G, p.th1_kind, p.theta1) ? HB_HIGH
                : gap_le(G, p.th2_kind, p.theta2) ? HB_LOW : HB_SKIP;
      } else {
        double s = 0.0;                       // Eq. 2 prefix sums of normalised gates
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
    }
    if (p.logits) {
      for (int e = threadIdx.x; e < p.E; e += blockDim.x) {
        const i128 v = logit[e];
        p.logits[((size_t)b * p.E + e) * 2 + 0] = (long long)(u64)v;
        p.logits[((size_t)b * p.E + e) * 2 + 1] = (long long)(v >> 64);
      }
    }
    __syncthreads();
  }

  if (!p.blob_table) return;
  // ---- last CTA builds the job table (fully resident mode, O7 strict) ----
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(p.done, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
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
  for (int key = 0; key < nkey; ++key) {
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
  for (int i = 0; i < nsel; ++i) {
    const int4 raw = __ldcg(reinterpret_cast<const int4*>(p.dec) + i);
    hb_decision d = *reinterpret_cast<const hb_decision*>(&raw);
    if (d.prec == HB_SKIP || d.expert % p.world != p.rank) continue;
    const int key = d.expert * 2 + (d.prec == HB_HIGH ? 0 : 1);
    const int slot = p.jt.jobs[jobid[key]].slot_off + fill[key]++;
    p.jt.slot_token[slot] = d.token;
    p.jt.slot_gate[slot] = d.gate;
    d.served_enc = (uint8_t)((key & 1) ? p.lo_enc : p.hi_enc);
    d.hit = 1;
    p.dec[i] = d;
  }
  p.jt.hdr[0] = nj;
  p.jt.hdr[1] = off;
  __threadfence();
  *p.done = 0u;
}

void launch_router(const RouterParams& p, int grid, cudaStream_t s) {
  const size_t smem = sizeof(i128) * (size_t)p.n_route * p.E;
  router_kernel<<<grid, kRouterThreads, smem, s>>>(p);
}

}  // namespace hb
