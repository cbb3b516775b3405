// Exact router arithmetic shared by the router kernel (router.cu) and the
// fused decode kernel's exact fallback (gemv.cu): every fp16 is m * 2^e
// (m 11-bit signed, e in [-24, 5]), so a product is m_w*m_x * 2^(e_w+e_x)
// with e_w+e_x+48 in [0, 58]; three int64 buckets by shift range hold the
// sum exactly (R9; P:216 gating linear layer).
#pragma once
#include <stdint.h>

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
  const long long p = (long long)(mw * mx);
  const int s = ew + ex + 48;
  // branch-free: the bucket of s and the term shifted into it (no divergence)
  const int r = (s >= 20) + (s >= 40);
  const u64 term = (u64)(p << (s - 20 * r));
  lo += r == 0 ? term : 0ull;
  mid += r == 1 ? term : 0ull;
  hi += r == 2 ? term : 0ull;
}

__device__ __forceinline__ bool gap_le(i128 G, int kind, long long theta) {
  if (kind > 0) return true;
  if (kind < 0) return false;
  return G <= (i128)theta;
}


}  // namespace hb
