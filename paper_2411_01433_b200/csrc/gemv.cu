// K2a / K2b: grouped mixed-precision dequant-GEMV of the selected experts.
//
//   K2a  a = W1 x, u = W3 x               per job (expert, served encoding)
//   K2b  h = silu(a) * u;  y = sum_jobs gate * (W2 h)     Eq. 1
//
// Paper: the layer output is the gate-weighted sum of the selected experts
// (Eq. 1); a Low expert is computed from its low-precision version;
// experts are SwiGLU FFNs (reading R10).  This is the B200 hot path: batch-1
// decode streams 66-352 MB of expert weights per token-layer, so the kernels
// are HBM-bound; their job is to keep ~100-200 KB of loads in flight per SM
// on every SM for the whole kernel while spending few instructions per weight.
//
// Structure:
//  * warp-level STREAM-K.  The work of a launch is a sequence of UNITS, one
//    unit = one 64-byte group of the 16 rows of a row tile (of W1 and W3
//    together for K2a), ordered (virtual job, tile, group).  Every unit moves
//    the same number of weight bytes whatever the encoding, so giving each of
//    the 148 x 16 warps an equal contiguous range of units balances HBM
//    traffic to within one unit.  A warp streams its range as ONE pipeline
//    (no drain at tile boundaries); at the end of each tile piece it adds its
//    partial sums into the output with fire-and-forget fp32 reductions
//    (red.global.add): K2a into a/u [slot][2][F], K2b (times the gate) into y.
//    No counters, fences or combine passes; the summation order of the <= 3
//    pieces of a row varies from run to run (reading R24);
//  * each warp owns a multi-stage shared-memory ring filled with cp.async
//    (L1 bypassed, L2 evict-first): per unit the 1 KB of codes of each matrix
//    and the 16 rows' block scales;
//  * the B operand (x for K2a; h = silu(a) * u as an fp16 hi/lo pair for
//    K2b, plus block sums for Q2) lives in ONE CTA-wide shared-memory stage,
//    built by all warps of the CTA right after they issued their first ring
//    loads (so the build overlaps the first HBM round trip) and published
//    through an mbarrier;
//  * the dot products run on the tensor cores as mma.sync.m16n8k16 with the
//    weights as A (16 rows x 16 k) and up to 8 token slots as B: dequantised
//    codes are EXACT in fp16 (q-8, q, int8 q), so every per-block partial sum
//    is an fp32 sum of exact products; the block scale is applied in fp32
//    after each 32-element block (acc += d*D_b (+ m*S_b for Q2));
//  * x and h are stored "pair-permuted" (Q_c = (v[8t+c], v[8t+c+4])) so that
//    the B fragment is one 16-byte load per block and lane, and the blob
//    layout puts lane t's share of every block of a group in bytes
//    [16t, 16t+16);
//  * K2b takes h as an fp16 hi/lo pair (h = hi + lo to ~2^-22) and issues two
//    MMAs per k-step, so W2 sees h at ~fp32 precision.
#include <cuda_fp16.h>

#include <algorithm>

#include "hb_internal.h"
#include "tl_stamps.cuh"
#include "exact_dot.cuh"

namespace hb {

// ------------------------------------------------------------ primitives
#ifdef HB_DBG_TIMELINE
// diagnostic build only: per-warp %globaltimer stamps of the last K2a / K2b launch
// [kernel][warp][0 entry, 1 stage done, 2 stream loop done, 3 publish done]
__device__ unsigned long long g_tl[2][kGemvCTAs * kGemvWarps][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HB_TL(W13, gw, i) do { if ((threadIdx.x & 31) == 0) g_tl[(W13) ? 0 : 1][gw][i] = gtimer(); } while (0)
#else
#define HB_TL(W13, gw, i) do { } while (0)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t smem_u32_(const void* p) { return smem_u32(p); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void cp_async16_ef(uint32_t dst, const void* src, uint64_t pol) {
#ifdef HB_NO_EVICT_HINT
  (void)pol;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
#else
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
               :: "r"(dst), "l"(src), "l"(pol));
#endif
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N)); }
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// fire-and-forget fp32 add into global memory (no generic-address fallback)
__device__ __forceinline__ void red_add(float* a, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" :: "l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ float lds_half(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return __half2float(__ushort_as_half(v));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t f2h2u(float v) {     // (rn(v), rn(v)) as a packed pair
  __half2 h = __float2half2_rn(v);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
#ifdef HB_DBG_NOMMA
  d[0] += __uint_as_float((a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1) & 0x3F800000u);
  return;
#endif
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// (a & MASK) | 0x64006400 : two fp16 values 1024 + field
template <uint32_t MASK>
__device__ __forceinline__ uint32_t lop_magic(uint32_t a) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "n"(MASK), "n"(0x64006400));
  return r;
}
__device__ __forceinline__ uint32_t hsub2u(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hfma2u(uint32_t a, uint32_t b, uint32_t c) {
  __half2 r = __hfma2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b),
                      *reinterpret_cast<__half2*>(&c));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t u4get(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

#ifdef HB_DBG_NOLO
constexpr bool kDbgNoLo = true;              // diagnostic: K2b without the h-lo MMAs
#else
constexpr bool kDbgNoLo = false;
#endif

// fp16 pair constants
constexpr uint32_t kH1032 = 0x64086408u;    // 1032 = 1024 + 8
constexpr uint32_t kH1152 = 0x64806480u;    // 1152 = 1024 + 128
constexpr uint32_t kH1024 = 0x64006400u;
constexpr uint32_t kHinv4 = 0x34003400u;    // 1/4
constexpr uint32_t kHinv16 = 0x2C002C00u;   // 1/16
constexpr uint32_t kHinv64 = 0x24002400u;   // 1/64
constexpr uint32_t kHm256 = 0xDC00DC00u;    // -256
constexpr uint32_t kHm72 = 0xD480D480u;     // -72
constexpr uint32_t kHm64 = 0xD400D400u;     // -64
constexpr uint32_t kHm16 = 0xCC00CC00u;     // -16

// ---------------------------------------------------- per-encoding traits
// A group is 64 bytes of one row: BPG blocks of 32 elements (EPG elements);
// SB = bytes of scales (d, then m for Q2) per row per group.
template <int ENC> struct Enc;
template <> struct Enc<HB_F16> { static constexpr int BPG = 1, EPG = 32,  SB = 0;  };
template <> struct Enc<HB_Q8>  { static constexpr int BPG = 2, EPG = 64,  SB = 4;  };
template <> struct Enc<HB_Q4>  { static constexpr int BPG = 4, EPG = 128, SB = 8;  };
template <> struct Enc<HB_Q2>  { static constexpr int BPG = 8, EPG = 256, SB = 32; };
// HB_Q2K (R32), kernel-internal template value (the context stores it in the
// Q2 slot): Q2's code layout, 20-byte records [d, dmin, sc[16]] (2.625 bpw)
constexpr int kEncQ2K = 4;
template <> struct Enc<kEncQ2K> { static constexpr int BPG = 8, EPG = 256, SB = 20; };

__host__ __device__ constexpr int epg_of(int enc) {
  return enc == HB_F16 ? 32 : enc == HB_Q8 ? 64 : enc == HB_Q4 ? 128 : 256;
}

// Shared memory of a GEMV CTA: kGemvWarps private cp.async rings (weights +
// scales) followed by ONE CTA-wide stage of the B operand (x for K2a, h hi/lo
// for K2b, and their block sums), built once per CTA, so the hot loop reads
// its B fragments with one shared-memory load per block instead of an L2
// round trip (K2b also computes h = silu(a) * u only here, not per unit).
template <bool W13> struct KCfg;
template <> struct KCfg<true> {        // K2a: x is small (8 KB per token at H=4096)
  static constexpr int RING = 16 * 12 * 1024 / kGemvWarps / 128 * 128;
  static constexpr int XSTAGE = 28 * 1024;  // 3 tokens at H = 4096
};
template <> struct KCfg<false> {       // K2b: h of one slot, half the columns: 29.6 KB at F=14336
  static constexpr int RING = 16 * 12288 / kGemvWarps / 128 * 128;
  static constexpr int XSTAGE = 30 * 1024;
};
template <bool W13>
constexpr int gemv_smem_bytes() { return kGemvWarps * KCfg<W13>::RING + KCfg<W13>::XSTAGE; }

// Ring stage layout of one unit: W codes | S scales
template <int ENC, int NMAT, int NU, int RINGB>
struct Ring {
  static constexpr int BPG = Enc<ENC>::BPG, SB = Enc<ENC>::SB;
  static constexpr int W = NMAT * NU * 1024;          // NU consecutive units per stage
  static constexpr int S = NMAT * NU * 16 * SB;
  static constexpr int STAGE = (W + S + 127) / 128 * 128;
#ifndef HB_MAX_DEPTH
#define HB_MAX_DEPTH 16
#endif
  static constexpr int DEPTH = RINGB / STAGE >= HB_MAX_DEPTH ? HB_MAX_DEPTH : RINGB / STAGE;
  static_assert(DEPTH >= 2, "ring too small");
};

// Dequantise block `blk` of the lane's 16-byte share into P0..P3, the fp16
// pairs (w[8t+c], w[8t+c+4]) with the codes' exact integer values (scale
// applied later), or the fp16 weights themselves for F16.
template <int ENC>
__device__ __forceinline__ void dequant(const uint4& v, int blk, uint32_t (&P)[4]) {
  if constexpr (ENC == HB_F16) {
    P[0] = prmt(v.x, v.z, 0x5410);
    P[1] = prmt(v.x, v.z, 0x7632);
    P[2] = prmt(v.y, v.w, 0x5410);
    P[3] = prmt(v.y, v.w, 0x7632);
  } else if constexpr (ENC == HB_Q8) {
    // block j holds r0..3 in word 2j, r4..7 in word 2j+1; q+128 via xor.
    // Interleave once (u = r0 r4 r1 r5, w = r2 r6 r3 r7), then one PRMT with
    // the 0x64 exponent bytes per pair: (1024 + q + 128) - 1152 = q exactly
    const uint32_t a = u4get(v, 2 * blk) ^ 0x80808080u;
    const uint32_t b = u4get(v, 2 * blk + 1) ^ 0x80808080u;
    const uint32_t u = prmt(a, b, 0x5140u), w = prmt(a, b, 0x7362u);
    P[0] = hsub2u(prmt(u, 0x64646464u, 0x4140u), kH1152);
    P[1] = hsub2u(prmt(u, 0x64646464u, 0x4342u), kH1152);
    P[2] = hsub2u(prmt(w, 0x64646464u, 0x4140u), kH1152);
    P[3] = hsub2u(prmt(w, 0x64646464u, 0x4342u), kH1152);
  } else if constexpr (ENC == HB_Q4) {
    const uint32_t w = u4get(v, blk);                     // nibble r = element 8t+r
    const uint32_t w8 = w >> 8;
    P[0] = hsub2u(lop_magic<0x000F000Fu>(w), kH1032);
    P[1] = hfma2u(lop_magic<0x00F000F0u>(w), kHinv16, kHm72);
    P[2] = hsub2u(lop_magic<0x000F000Fu>(w8), kH1032);
    P[3] = hfma2u(lop_magic<0x00F000F0u>(w8), kHinv16, kHm72);
  } else {  // Q2: word blk/2, fields of block blk at bits (8*(blk&1)) + {2c, 16+2c}
    const uint32_t w = u4get(v, blk >> 1) >> (8 * (blk & 1));
    P[0] = hsub2u(lop_magic<0x00030003u>(w), kH1024);
    P[1] = hfma2u(lop_magic<0x000C000Cu>(w), kHinv4, kHm256);
    P[2] = hfma2u(lop_magic<0x00300030u>(w), kHinv16, kHm64);
    P[3] = hfma2u(lop_magic<0x00C000C0u>(w), kHinv64, kHm16);
  }
}

// ------------------------------------------------------------ B operand of K2b
// h of slot s, block j (32 consecutive rows of F) from the K2a sums:
// h = silu(a) * u (reading R10), split into fp16 hi + lo (hi = rn(h),
// lo = rn(h - hi)) and pair-permuted; returns the fp32 block sum (Q2 term).
__device__ __forceinline__ float h_block(const float* au, int F, int s, int j, uint4 (&hi)[4],
                                         uint4 (&lo)[4]) {
  const float4* pa = reinterpret_cast<const float4*>(au + (size_t)s * 2 * F + (size_t)j * 32);
  const float4* pu = reinterpret_cast<const float4*>(au + (size_t)s * 2 * F + F + (size_t)j * 32);
  float h[32];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 va = __ldcg(pa + q), vu = __ldcg(pu + q);
    h[4 * q + 0] = va.x; h[4 * q + 1] = va.y; h[4 * q + 2] = va.z; h[4 * q + 3] = va.w;
    const float uu[4] = {vu.x, vu.y, vu.z, vu.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float a = h[4 * q + i];
      h[4 * q + i] = a / (1.f + expf(-a)) * uu[i];
    }
  }
  float hs = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) hs += h[i];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    uint32_t wh[4], wl[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float e0 = h[8 * t + c], e1 = h[8 * t + c + 4];
      const __half h0 = __float2half_rn(e0), h1 = __float2half_rn(e1);
      const __half l0 = __float2half_rn(e0 - __half2float(h0));
      const __half l1 = __float2half_rn(e1 - __half2float(h1));
      wh[c] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
      wl[c] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
    }
    hi[t] = make_uint4(wh[0], wh[1], wh[2], wh[3]);
    lo[t] = make_uint4(wl[0], wl[1], wl[2], wl[3]);
  }
  return hs;
}

// ------------------------------------------------------------ CTA stage
// Shared-memory layout of the B operand (nrows = tokens for K2a, slots for K2b;
// kcols = staged columns per row):
//   part 0 (x / h hi) [nrows][kcols/8] uint4 | part 1 (h lo, K2b) | sums [nrows][kcols/32] f32
// Warp `w` of the CTA builds its share (items w, w + kGemvWarps, ...).
// K2a, legacy chain: copy the router's pair-permuted x and block sums.
__device__ void stage_share_xperm(const GemvParams& p, int w, uint8_t* st, int row0, int nrows) {
  const int lane = threadIdx.x & 31;
  const int K = p.H;
  const int n16 = nrows * (K / 8);
  uint4* dst = reinterpret_cast<uint4*>(st);
  const uint4* xs = p.x_perm + (size_t)row0 * (K / 8);
  for (int i = w * 32 + lane; i < n16; i += kGemvWarps * 32) dst[i] = __ldcg(xs + i);
  const int nz = nrows * (K / 32);
  float* zd = reinterpret_cast<float*>(st + (size_t)n16 * 16);
  const float* zs = p.xsum + (size_t)row0 * (K / 32);
  for (int i = w * 32 + lane; i < nz; i += kGemvWarps * 32) zd[i] = __ldcg(zs + i);
}
// K2a, fused decode: pair-permute x (Q_c = (x[8t+c], x[8t+c+4])) and sum each
// 32-element block (the Q2 m-term) straight from the caller's fp16 x.
__device__ __noinline__ void stage_share_xraw(const GemvParams& p, int w, uint8_t* st, int row0, int nrows) {
  const int lane = threadIdx.x & 31;
  const int K = p.H, nb = K / 32;
  uint4* dst = reinterpret_cast<uint4*>(st);
  float* zd = reinterpret_cast<float*>(st + (size_t)nrows * K * 2);
  for (int i = w * 32 + lane; i < nrows * nb; i += kGemvWarps * 32) {
    const int r = i / nb, blk = i - r * nb;
    const uint4* src = reinterpret_cast<const uint4*>(p.x_raw + (size_t)(row0 + r) * K + blk * 32);
    uint32_t v[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 t = __ldcg(src + q);
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e)
      sum += __half2float(__ushort_as_half((unsigned short)(v[e >> 1] >> (16 * (e & 1)))));
    zd[i] = sum;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      uint32_t q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e0 = 8 * t + c, e1 = e0 + 4;
        q[c] = ((v[e0 >> 1] >> (16 * (e0 & 1))) & 0xFFFF) | (((v[e1 >> 1] >> (16 * (e1 & 1))) & 0xFFFF) << 16);
      }
      dst[(size_t)r * (K / 8) + blk * 4 + t] = make_uint4(q[0], q[1], q[2], q[3]);
    }
  }
}
// K2b, fused decode: this CTA's column slice [c0, c0 + kcols) of h for slots
// [row0, row0 + nrows), h = silu(a) * u from the K2a sums (fp16 hi/lo pair +
// block sums), computed redundantly by every CTA of the slice's group.  Four
// lanes per 32-row block (lane t of the quad owns rows 8t..8t+7, i.e. chunk t
// of the pair-permuted hi / lo rows), as in hfin: short dependency chains.
__device__ void stage_share_h(const GemvParams& p, int w, uint8_t* st, int row0, int nrows,
                              int c0, int kcols) {
  const int lane = threadIdx.x & 31;
  const int nb = kcols / 32, K = p.F;
  uint4* dhi = reinterpret_cast<uint4*>(st);
  uint4* dlo = dhi + (size_t)nrows * (kcols / 8);
  float* zd = reinterpret_cast<float*>(dlo + (size_t)nrows * (kcols / 8));
  const int n = nrows * nb * 4;
  for (int i0 = w * 32; i0 < n; i0 += kGemvWarps * 32) {
    const int i = i0 + lane;
    const bool act = i < n;
    const int q = act ? i : 0;
    const int item = q >> 2, t = q & 3;
    const int s = item / nb, j = item - s * nb;
    const float* pa = p.au + (size_t)(row0 + s) * 2 * K + (size_t)c0 + (size_t)j * 32 + 8 * t;
    const float* pu = pa + K;
    const float4 a0 = __ldcg(reinterpret_cast<const float4*>(pa));
    const float4 a1 = __ldcg(reinterpret_cast<const float4*>(pa) + 1);
    const float4 u0 = __ldcg(reinterpret_cast<const float4*>(pu));
    const float4 u1 = __ldcg(reinterpret_cast<const float4*>(pu) + 1);
    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float uv[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
    float h[8], hs = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      h[r] = av[r] / (1.f + expf(-av[r])) * uv[r];
      hs += h[r];
    }
    uint32_t wh[4], wl[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {              // Q_c = (h[8t+c], h[8t+c+4])
      const __half h0 = __float2half_rn(h[c]), h1 = __float2half_rn(h[c + 4]);
      const __half l0 = __float2half_rn(h[c] - __half2float(h0));
      const __half l1 = __float2half_rn(h[c + 4] - __half2float(h1));
      wh[c] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
      wl[c] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
    }
    hs += __shfl_xor_sync(0xffffffffu, hs, 1);
    hs += __shfl_xor_sync(0xffffffffu, hs, 2);
    if (act) {
      dhi[(size_t)s * (kcols / 8) + j * 4 + t] = make_uint4(wh[0], wh[1], wh[2], wh[3]);
      dlo[(size_t)s * (kcols / 8) + j * 4 + t] = make_uint4(wl[0], wl[1], wl[2], wl[3]);
      if (t == 0) zd[item] = hs;
    }
  }
}

__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}

// Stage hand-off of one launch: every thread of the CTA arrives once (after its
// share of the build); readers wait for phase 0.
struct Stage {
  uint8_t* ptr;      // generic pointer of the stage
  uint32_t xst;      // its shared address
  uint32_t bar;      // mbarrier (count = blockDim.x)
  int row0;          // first staged row (token for x, slot for h)
  int nrows;
  int kcols;         // columns staged per row (K2b: one column slice of h)
  int nh, hs;        // K2b: column slices of the vjob, this CTA's slice
  bool on;           // B operand read from the stage (else from global memory)
};

// Fused decode: every warp reports the end of its K2a work; the CTA's last warp
// takes part in the grid-wide barrier (all K2a sums complete), then releases
// the CTA's warps.
struct FusedSync {
  unsigned* gcount;          // global arrivals (self-resetting)
  unsigned* ggen;            // global generation
  uint64_t* warps_done;      // shared mbarrier (count = CTA threads): threads past K2a
  uint64_t* released;        // shared mbarrier (count 1): completes once the grid barrier passed
  unsigned long long* stamp; // per-forward profile record or null
};
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ void fused_grid_barrier(const FusedSync& fs) {
  __threadfence();                     // this thread's K2a reductions before the arrival
  const uint32_t done = smem_u32(fs.warps_done), rel = smem_u32(fs.released);
  mbar_arrive(done);                   // every thread: its K2a work is done
  if (threadIdx.x == 0) {
    // thread 0 meets the other CTAs once every thread of this CTA arrived
    mbar_wait(done, 0);
    __threadfence();
    if (fs.stamp) atomicMax(fs.stamp + 2, gtimer_ns());
    const unsigned g = ld_acquire_gpu(fs.ggen);
    if (atomicAdd(fs.gcount, 1u) == gridDim.x - 1) {
      *fs.gcount = 0u;
      st_release_gpu(fs.ggen, g + 1u);
    } else {
      while (ld_acquire_gpu(fs.ggen) == g) __nanosleep(64);
    }
    if (fs.stamp) atomicMax(fs.stamp + 3, ~gtimer_ns());   // min, stored complemented
    mbar_arrive(rel);                                     // release the CTA
  }
  mbar_wait(rel, 0);                   // every thread: ordered after the whole grid's K2a
}

// K2b: h rows [row0, row0 + nrows) of h_hi | h_lo | hsum (built by hfin) into
// the stage with three bulk (TMA) copies issued by thread 0; every thread
// waits on the mbarrier's transaction count.
__device__ __forceinline__ void stage_h_bulk_and_wait(const GemvParams& p, const Stage& S) {
  if (threadIdx.x == 0) {
    const uint32_t rh = (uint32_t)S.kcols * 2, rz = (uint32_t)(S.kcols / 32) * 4;
    const uint32_t nh = S.nrows * rh;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(S.bar), "r"(S.nrows * (2 * rh + rz)) : "memory");
    for (int r = 0; r < S.nrows; ++r) {
      const size_t row = (size_t)(S.row0 + r);
      const char* src[3] = {
          reinterpret_cast<const char*>(p.h_hi) + row * p.F * 2 + (size_t)S.hs * rh,
          reinterpret_cast<const char*>(p.h_lo) + row * p.F * 2 + (size_t)S.hs * rh,
          reinterpret_cast<const char*>(p.hsum) + row * (p.F / 32) * 4 + (size_t)S.hs * rz};
      const uint32_t dst[3] = {r * rh, nh + r * rh, 2 * nh + r * rz}, len[3] = {rh, rh, rz};
#pragma unroll
      for (int i = 0; i < 3; ++i)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            :: "r"(S.xst + dst[i]), "l"(src[i]), "r"(len[i]), "r"(S.bar) : "memory");
    }
  }
  mbar_wait(S.bar, 0);
}

// The fused decode kernel's own job table (built by every CTA, in shared
// memory; file-scope __shared__, so only that kernel allocates it) and the
// grid barrier it meets between K2a and K2b.
constexpr int kFusedMaxV = 4;
__shared__ VJobD fz_vj[kFusedMaxV];
__shared__ int32_t fz_stok[kFusedMaxV];
__shared__ float fz_sgate[kFusedMaxV];
__shared__ int fz_nv, fz_nslot;
__shared__ FusedSync fz_fs;

// Job table access: the router's global table (legacy chain, FUSED = false)
// or the fused kernel's shared copy.  Templated so that the legacy kernels
// keep these in the constant bank instead of registers.
template <bool FUSED> struct JT;
#if HB_LEGACY_TL == 1
__shared__ unsigned long long tl_k2b_entry;
#endif
__shared__ int lg_nv, lg_nslot;     // legacy kernels: the header, read once per launch
template <> struct JT<false> {
  static __device__ __forceinline__ int nv(const GemvParams&) { return lg_nv; }
  static __device__ __forceinline__ int nslots(const GemvParams&) { return lg_nslot; }
  static __device__ __forceinline__ VJobD vjob(const GemvParams& p, int v) { return p.jt.vjobs[v]; }
  static __device__ __forceinline__ int stok(const GemvParams& p, int s) { return p.jt.slot_token[s]; }
  static __device__ __forceinline__ float sgate(const GemvParams& p, int s) { return p.jt.slot_gate[s]; }
};
template <> struct JT<true> {
  static __device__ __forceinline__ int nv(const GemvParams&) { return fz_nv; }
  static __device__ __forceinline__ int nslots(const GemvParams&) { return fz_nslot; }
  static __device__ __forceinline__ VJobD vjob(const GemvParams&, int v) { return fz_vj[v]; }
  static __device__ __forceinline__ int stok(const GemvParams&, int s) { return fz_stok[s]; }
  static __device__ __forceinline__ float sgate(const GemvParams&, int s) { return fz_sgate[s]; }
};

// K2a's x stage: every thread builds its share, arrives, waits
template <bool FUSED>
__device__ __forceinline__ void stage_x_and_wait(const GemvParams& p, const Stage& S) {
  if (FUSED) stage_share_xraw(p, threadIdx.x >> 5, S.ptr, S.row0, S.nrows);
  else stage_share_xperm(p, threadIdx.x >> 5, S.ptr, S.row0, S.nrows);
  mbar_arrive(S.bar);
  mbar_wait(S.bar, 0);
}
// K2b's h stage once the K2a sums are complete: legacy chain = wait for the
// previous kernels (K2a, hfin) and bulk-copy h; fused kernel = grid barrier,
// then build h from the sums
template <bool FUSED>
__device__ __forceinline__ void stage_h_and_wait(const GemvParams& p, const Stage& S) {
  if (!FUSED) {
    pdl_wait();
#if HB_LEGACY_TL == 1
    if (p.stamps && threadIdx.x == 0) {
      unsigned long long* rec = tl_rec(p.stamps, p.stamp_cap, p.fwd_idx);
      tl_min(rec, 12, tl_now());
      tl_min(rec, 11, tl_k2b_entry);
    }
#endif
    if (S.on) stage_h_bulk_and_wait(p, S);
#ifdef HB_NO_STAMPS
    if (false) {
#else
    if (p.stamps && threadIdx.x == 0) {
#endif
      const unsigned idx = __ldcg(p.fwd_idx);
      if (idx < (unsigned)p.stamp_cap) atomicMax(p.stamps + (size_t)idx * kStampStride + 3, ~gtimer_ns());
    }
    return;
  }
  fused_grid_barrier(fz_fs);
  if (S.on) {
    stage_share_h(p, threadIdx.x >> 5, S.ptr, S.row0, S.nrows, S.hs * S.kcols, S.kcols);
    mbar_arrive(S.bar);
    mbar_wait(S.bar, 0);
  }
  if (fz_fs.stamp && threadIdx.x == 0) {
    atomicMax(fz_fs.stamp + 8, gtimer_ns());           // last CTA with h staged
    atomicMax(fz_fs.stamp + 9, ~gtimer_ns());          // first CTA with h staged
  }
}

// ---------------------------------------------------------- work feed
// Virtual job: one job's token slots [slot0, slot0 + nslot), nslot <= kVSlots.
struct VJob {
  const uint8_t* blob;
  int enc;
  int slot0;
  int nslot;
};


// The units of a launch (ordered vjob, tile, group; vjob v owns
// [cum[v], cum[v+1])) are dealt in two phases: the first S = static_frac * U
// units as equal contiguous warp ranges (dealt SM-interleaved), the rest as
// chunks of `chunk` units from a global counter.  SMs do not all get the same
// share of HBM bandwidth (measured: per-SM stream times differ by up to 30%,
// in GPC-sized groups), so warps on slow SMs simply take fewer chunks.  The
// next chunk index is fetched one chunk ahead, so the atomic's latency is
// hidden behind the current chunk's loads.
struct FeedConst {         // per launch, in shared memory (CTA-wide constants)
  int base;                // first unit of the space this CTA works in
  int S, U;                // static units, all units of the space (< 2^31: checked by the host)
  int nch;                 // dynamic chunks
  int chunk;
  int nwarps;              // warps taking part (each fetches until it sees >= nch)
  unsigned* ctr;
};
struct Feed {
  int a, b;                // pending segment [a, b) (global units); empty when a >= b
  unsigned pre;            // lane 0: the prefetched fetch index
  bool done;
  const FeedConst* k;
  __device__ __forceinline__ void start() {
    if ((threadIdx.x & 31) == 0) pre = atomicAdd(k->ctr, 1u);
  }
  // next chunk into [a, b); false when the launch's work is exhausted
  __device__ __forceinline__ bool refill() {
    if (done) return false;
    const int c = (int)__shfl_sync(0xffffffffu, pre, 0);
    if (c >= k->nch) {
      // every warp receives exactly one index >= nch; the warp that receives
      // the last one hands the counter back zeroed for the next launch
      if ((threadIdx.x & 31) == 0 && c == k->nch + k->nwarps - 1) *k->ctr = 0u;
      done = true;
      return false;
    }
    a = k->base + k->S + c * k->chunk;
    b = min(a + k->chunk, k->base + k->U);
    if ((threadIdx.x & 31) == 0) pre = atomicAdd(k->ctr, 1u);
    return true;
  }
};

// ------------------------------------------------------------ the run
// Stream the feed's segments that lie in virtual job vj (units [cum, cum+Uv),
// unit l = tile * G + grp of the vjob) through the warp's ring as one
// pipeline.  W13: K2a (W1 and W3 rows, x); else K2b (W2 rows, h hi/lo).  The
// producer runs DEPTH-1 units ahead and records each unit's (tile, group,
// end-of-piece) in `meta` next to its ring slot.  `first`: the warp's first
// run of the launch, which builds its share of the CTA stage between issuing
// the ring prologue and consuming the first unit.
#ifdef HB_RUN_NOINLINE
#define HB_RUN_ATTR __noinline__
#else
#define HB_RUN_ATTR
#endif
template <int ENC, bool W13, bool XR, bool FUSED>
__device__ HB_RUN_ATTR void run(const GemvParams& p, const VJob& vj, int cum, int Uv, Feed& fd,
                    uint32_t ring, uint2* meta, const Stage& S, bool first) {
  constexpr int NMAT = W13 ? 2 : 1;
  constexpr bool SPLIT = !W13;
  constexpr int XS = SPLIT ? 2 : 1;
  // K2b streams two units (2 KB) per ring stage: half the per-stage overhead
  // and two independent MMA chains per iteration (K2b is issue-bound); K2a's
  // 2-matrix units are already 2 KB
  constexpr int NU = (!W13 && XR) ? 2 : 1;
  using R = Ring<ENC, NMAT, NU, KCfg<W13>::RING>;
  constexpr int BPG = R::BPG, SB = R::SB, DEPTH = R::DEPTH;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const bool lane0 = lane == 0;
  const int K = W13 ? p.H : p.F;
  const int G = K / Enc<ENC>::EPG;
  // K2b with a staged column slice: the space covers groups [goff, goff + Gs)
  // of every tile (Gs even, so a stage's NU = 2 units never straddle tiles)
  const int Gs = (!W13 && XR) ? G / S.nh : G;
  const int goff = (!W13 && XR) ? S.hs * Gs : 0;
  const uint64_t pol = evict_first_policy();
  // tile-major blobs: unit l (tile l/G, group l%G) = 1 KB of codes at q + 1024*l,
  // its 16 scale records at s + 16*SB*l -- a segment is one contiguous span
  const int ns = vj.nslot;

  // ---- producer: weights + scales
  int pl = 0, pe = 0;                          // vjob-local next unit / end of its segment
  int ptile = 0, pgrp = 0, pslot = 0, iss = 0;
  bool pactive = true;
  const uint8_t* qp[NMAT];
  const uint8_t* sp_[NMAT];
  auto take = [&]() -> bool {                  // the feed's next segment, if it is in this vjob
    if (fd.a >= fd.b && !fd.refill()) return false;
    if (fd.a < cum || fd.a >= cum + Uv) return false;
    pl = fd.a - cum;
    pe = min(fd.b, cum + Uv) - cum;
    fd.a = cum + pe;                           // a remainder past the vjob stays in the feed
    ptile = pl / Gs;
    pgrp = pl - ptile * Gs;
    const size_t u = (size_t)ptile * G + goff + pgrp;      // unit in the blob
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      const MatLayout& L = p.lay[ENC == kEncQ2K ? HB_Q2 : ENC].mat[W13 ? m : 2];
      qp[m] = vj.blob + L.q + u * 1024 + 16 * lane;
      sp_[m] = vj.blob + L.s + u * 16 * SB + 16 * lane;
    }
    return true;
  };
  auto issue = [&]() {
    if (pactive && pl == pe) pactive = take();
    if (pactive) {
      const uint32_t st = ring + pslot * R::STAGE;
#pragma unroll
      for (int m = 0; m < NMAT; ++m) {                 // NU x 1 KB contiguous per matrix
#pragma unroll
        for (int i = 0; i < 2 * NU; ++i)
          cp_async16_ef(st + m * NU * 1024 + 512 * i + 16 * lane, qp[m] + 512 * i, pol);
        if constexpr (SB > 0) {
#pragma unroll
          for (int o = 0; o < NU * 16 * SB; o += 512)
            if (o + 16 * lane < NU * 16 * SB)
              cp_async16_ef(st + R::W + m * NU * 16 * SB + o + 16 * lane, sp_[m] + o, pol);
        }
      }
      // meta: tile / group of the stage's first unit; bit 30 + u: unit u ends a
      // tile piece (tile end, or segment end).  Segments and Gs are multiples
      // of NU, so only the stage's last unit can end a piece.
      pl += NU;
      pgrp += NU;
      const bool endp = pgrp == Gs || pl == pe;
      if (lane0) meta[pslot] = make_uint2((uint32_t)ptile, (uint32_t)(pgrp - NU) | (endp ? 1u << (29 + NU) : 0u));
      int skip = 0;
      if (pgrp == Gs) { pgrp = 0; ++ptile; skip = G - Gs; }  // next tile's slice
#pragma unroll
      for (int m = 0; m < NMAT; ++m) {
        qp[m] += (size_t)(NU + skip) * 1024;
        sp_[m] += (size_t)(NU + skip) * 16 * SB;
      }
      pslot = pslot + 1 == DEPTH ? 0 : pslot + 1;
      ++iss;
    }
    cp_commit();
  };

  // K2a: x is tiny and already in L2 -- stage it before the weight loads are
  // queued (behind ~24 MB of ring prologues it would wait microseconds).
  // K2b: the ring prologue (W2 is independent of K2a) goes out first, during
  // K2a's tail; then wait for K2a and build h.
  if (W13 && first && S.on) stage_x_and_wait<FUSED>(p, S);
  if constexpr (FUSED && !W13) {
    // fused kernel, first K2b run: before the grid barrier, pull the units of
    // the ring prologue into L2 (prefetch: keeps HBM busy during the barrier
    // without queueing ring loads in front of the h build's reads), then the
    // barrier and h, then the prologue (now L2 hits)
    if (first) {
      const int n = min((DEPTH - 1) * NU, fd.b - fd.a);
      const int l = fd.a - cum + lane;
      if (lane < n && l < Uv) {
        const int tl = l / Gs, gr = l - tl * Gs;
        const size_t u = (size_t)tl * G + goff + gr;
        const MatLayout& L = p.lay[ENC == kEncQ2K ? HB_Q2 : ENC].mat[2];
        const char* q = reinterpret_cast<const char*>(vj.blob + L.q + u * 1024);
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("prefetch.global.L2 [%0];" :: "l"(q + 128 * i));
        if constexpr (SB > 0) {
          const char* sc = reinterpret_cast<const char*>(vj.blob + L.s + u * 16 * SB);
          for (int i = 0; i < 16 * SB; i += 128) asm volatile("prefetch.global.L2 [%0];" :: "l"(sc + i));
        }
      }
      stage_h_and_wait<FUSED>(p, S);
    }
  }
#ifndef HB_K2B_PRE
#define HB_K2B_PRE 64
#endif
  // K2b: HB_K2B_PRE stages before waiting for h (diagnostic knob), the rest after
  constexpr int PRE = (!FUSED && !W13) ? (HB_K2B_PRE < DEPTH - 1 ? HB_K2B_PRE : DEPTH - 1) : DEPTH - 1;
#pragma unroll 1
  for (int s = 0; s < PRE; ++s) issue();
  if (!FUSED && !W13 && first) stage_h_and_wait<FUSED>(p, S);  // h after K2a (hfin)
#pragma unroll 1
  for (int s = PRE; s < DEPTH - 1; ++s) issue();
  if (first) HB_TL(W13, (threadIdx.x >> 5) * gridDim.x + blockIdx.x, 2);

  // ---- lane constants: B-operand rows, outputs of the lane's two slots
  const int xg = min(g, ns - 1);
  const int z0 = min(2 * t, ns - 1), z1 = min(2 * t + 1, ns - 1);
  auto row_of = [&](int s) -> int {          // token (x) or slot (h) of vjob slot s
    const int sl = vj.slot0 + s;
    return W13 ? JT<FUSED>::stok(p, sl) : sl;
  };
  const uint4* gx0 = nullptr;
  const uint4* gx1 = nullptr;
  const float* gz0 = nullptr;
  const float* gz1 = nullptr;
  if constexpr (!XR) {
    if constexpr (W13) {
      gx0 = gx1 = p.x_perm + (size_t)row_of(xg) * (K / 8);
      gz0 = p.xsum + (size_t)row_of(z0) * (K / 32);
      gz1 = p.xsum + (size_t)row_of(z1) * (K / 32);
    } else {
      gx0 = p.h_hi + (size_t)row_of(xg) * (K / 8);
      gx1 = p.h_lo + (size_t)row_of(xg) * (K / 8);
      gz0 = p.hsum + (size_t)row_of(z0) * (K / 32);
      gz1 = p.hsum + (size_t)row_of(z1) * (K / 32);
    }
  }
  const int KC = S.kcols;
  const uint32_t sxb = S.xst + (uint32_t)(row_of(xg) - S.row0) * KC * 2 + t * 16;
  const uint32_t sxl = sxb + (uint32_t)S.nrows * KC * 2;
  const uint32_t szb = S.xst + (uint32_t)XS * S.nrows * KC * 2;
  const uint32_t sz0 = szb + (uint32_t)(row_of(z0) - S.row0) * (KC / 32) * 4;
  const uint32_t sz1 = szb + (uint32_t)(row_of(z1) - S.row0) * (KC / 32) * 4;
  // output targets of the lane's slots 2t, 2t+1 (K2a: a/u rows; K2b: y rows, gate)
  const bool v0 = 2 * t < ns, v1 = 2 * t + 1 < ns;
  float* out0;
  float* out1;
  float gate0 = 0.f, gate1 = 0.f;
  if constexpr (W13) {
    out0 = p.au + (size_t)(vj.slot0 + z0) * 2 * p.F;
    out1 = p.au + (size_t)(vj.slot0 + z1) * 2 * p.F;
  } else {
    out0 = p.y + (size_t)JT<FUSED>::stok(p, vj.slot0 + z0) * p.H;
    out1 = p.y + (size_t)JT<FUSED>::stok(p, vj.slot0 + z1) * p.H;
    gate0 = JT<FUSED>::sgate(p, vj.slot0 + z0);
    gate1 = JT<FUSED>::sgate(p, vj.slot0 + z1);
  }

  float acc[NMAT][4];
#pragma unroll
  for (int m = 0; m < NMAT; ++m)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;
  int cslot = 0;

  // dot products of one unit (codes at wst, scales at sst, group c_grp) into r
  auto unit_dot = [&](uint32_t wst, uint32_t sst, int c_grp, float (&r)[NMAT][4]) {
    uint4 w[NMAT][2];
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      w[m][0] = lds128(wst + m * NU * 1024 + g * 64 + 16 * t);
      w[m][1] = lds128(wst + m * NU * 1024 + (g + 8) * 64 + 16 * t);
    }
#ifdef HB_DBG_NOCOMPUTE
    r[0][0] += __uint_as_float((w[0][0].x ^ w[0][1].y) & 0x3F800000u);
    return;
#endif
    // Q2K: the records of rows g and g + 8 once per unit (d, dmin, 16 sub-block bytes)
    float q2d[NMAT][2], q2m[NMAT][2];
    uint32_t q2s[NMAT][2][4];
    if constexpr (ENC == kEncQ2K) {
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const uint32_t rec = sst + m * NU * 16 * SB + (g + 8 * h2) * SB;
          q2d[m][h2] = lds_half(rec);
          q2m[m][h2] = lds_half(rec + 2);
#pragma unroll
          for (int wv = 0; wv < 4; ++wv) q2s[m][h2][wv] = lds_u32(rec + 4 + 4 * wv);
        }
    }
#pragma unroll
    for (int blk = 0; blk < BPG; ++blk) {
      uint4 xb, xl;
      float s0 = 0.f, s1 = 0.f;
      if constexpr (XR) {
        const uint32_t gb = (uint32_t)(c_grp * BPG + blk);
#ifdef HB_DBG_NOBLDS
        xb = make_uint4(gb, gb + 1, gb + 2, gb + 3);
        xl = xb;
#else
        xb = lds128(sxb + gb * 64);
        if constexpr (SPLIT) xl = lds128(sxl + gb * 64);
#endif
        if constexpr (ENC == HB_Q2) {
          s0 = lds_f32(sz0 + gb * 4);
          s1 = lds_f32(sz1 + gb * 4);
        }
      } else {
        const size_t gb = (size_t)(c_grp * BPG + blk);
        xb = __ldg(gx0 + gb * 4 + t);
        if constexpr (SPLIT) xl = __ldg(gx1 + gb * 4 + t);
        if constexpr (ENC == HB_Q2) { s0 = __ldg(gz0 + gb); s1 = __ldg(gz1 + gb); }
      }
#pragma unroll
      for (int m = 0; m < NMAT; ++m) {
        uint32_t Pg[4], Ph[4];
        dequant<ENC>(w[m][0], blk, Pg);
        dequant<ENC>(w[m][1], blk, Ph);
        if constexpr (ENC == HB_F16) {
          mma16816(r[m], Pg[0], Ph[0], Pg[1], Ph[1], xb.x, xb.y);
          mma16816(r[m], Pg[2], Ph[2], Pg[3], Ph[3], xb.z, xb.w);
          if constexpr (SPLIT && !kDbgNoLo) {
            mma16816(r[m], Pg[0], Ph[0], Pg[1], Ph[1], xl.x, xl.y);
            mma16816(r[m], Pg[2], Ph[2], Pg[3], Ph[3], xl.z, xl.w);
          }
        } else if constexpr (ENC == kEncQ2K) {
          // Q2K (R32): lane t's pairs lie in sub-block 2 blk + t / 2 of rows g,
          // g + 8; w = d (sc & 15) q - dmin (sc >> 4) is formed in fp16 (scale
          // products rounded once, then one fma) and fed to the MMA directly
          // sub-block 2 blk + t / 2: byte 2 (blk % 2) + t / 2 of word blk / 2
          const int sh = 8 * (2 * (blk & 1) + (t >> 1));
          const uint32_t cg = (q2s[m][0][blk >> 1] >> sh) & 0xFFu;
          const uint32_t ch = (q2s[m][1][blk >> 1] >> sh) & 0xFFu;
          const uint32_t Dg = f2h2u(q2d[m][0] * (float)(cg & 15u));
          const uint32_t Mg = f2h2u(-q2m[m][0] * (float)(cg >> 4));
          const uint32_t Dh = f2h2u(q2d[m][1] * (float)(ch & 15u));
          const uint32_t Mh = f2h2u(-q2m[m][1] * (float)(ch >> 4));
          uint32_t Ag[4], Ah[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            Ag[c] = hfma2u(Pg[c], Dg, Mg);
            Ah[c] = hfma2u(Ph[c], Dh, Mh);
          }
          mma16816(r[m], Ag[0], Ah[0], Ag[1], Ah[1], xb.x, xb.y);
          mma16816(r[m], Ag[2], Ah[2], Ag[3], Ah[3], xb.z, xb.w);
          if constexpr (SPLIT && !kDbgNoLo) {
            mma16816(r[m], Ag[0], Ah[0], Ag[1], Ah[1], xl.x, xl.y);
            mma16816(r[m], Ag[2], Ah[2], Ag[3], Ah[3], xl.z, xl.w);
          }
        } else {
          const uint32_t sd = sst + m * NU * 16 * SB;
          const float dg = lds_half(sd + g * SB + 2 * blk);
          const float dh = lds_half(sd + (g + 8) * SB + 2 * blk);
          float D[4] = {0.f, 0.f, 0.f, 0.f};
          mma16816(D, Pg[0], Ph[0], Pg[1], Ph[1], xb.x, xb.y);
          mma16816(D, Pg[2], Ph[2], Pg[3], Ph[3], xb.z, xb.w);
          if constexpr (SPLIT && !kDbgNoLo) {
            mma16816(D, Pg[0], Ph[0], Pg[1], Ph[1], xl.x, xl.y);
            mma16816(D, Pg[2], Ph[2], Pg[3], Ph[3], xl.z, xl.w);
          }
          r[m][0] = fmaf(dg, D[0], r[m][0]);
          r[m][1] = fmaf(dg, D[1], r[m][1]);
          r[m][2] = fmaf(dh, D[2], r[m][2]);
          r[m][3] = fmaf(dh, D[3], r[m][3]);
          if constexpr (ENC == HB_Q2) {               // + m_row * sum_block(x)
            const float mg = lds_half(sd + g * SB + 16 + 2 * blk);
            const float mh = lds_half(sd + (g + 8) * SB + 16 + 2 * blk);
            r[m][0] = fmaf(mg, s0, r[m][0]);
            r[m][1] = fmaf(mg, s1, r[m][1]);
            r[m][2] = fmaf(mh, s0, r[m][2]);
            r[m][3] = fmaf(mh, s1, r[m][3]);
          }
        }
      }
    }
  };
  // end of a tile piece: add it into the output (fire-and-forget reductions)
  auto flush = [&](int c_tile) {
    const int r0 = c_tile * 16 + g;
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      const int off = W13 ? m * p.F + r0 : r0;
      if (v0) {
        red_add(out0 + off, W13 ? acc[m][0] : gate0 * acc[m][0]);
        red_add(out0 + off + 8, W13 ? acc[m][2] : gate0 * acc[m][2]);
      }
      if (v1) {
        red_add(out1 + off, W13 ? acc[m][1] : gate1 * acc[m][1]);
        red_add(out1 + off + 8, W13 ? acc[m][3] : gate1 * acc[m][3]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;
    }
  };

  for (int con = 0; con < iss; ++con) {            // iss grows while the producer runs
    __syncwarp();                                  // slot being refilled is consumed
    issue();
    cp_wait<DEPTH - 1>();
    __syncwarp();                                  // everyone's copies of stage con visible
    const uint2 md = meta[cslot];
    const uint32_t st = ring + cslot * R::STAGE;
    if (++cslot == DEPTH) cslot = 0;
    if constexpr (NU == 1) {
      unit_dot(st, st + R::W, (int)(md.y & 0x3FFFFFFFu), acc);
      if (md.y & 0x40000000u) flush((int)md.x);
    } else {
      // two units: independent partial sums, then in order into acc with the
      // piece boundaries between them
      const int tile0 = (int)md.x, grp0 = (int)(md.y & 0x3FFFFFFFu);
      const bool e0 = (md.y >> 30) & 1u, e1 = md.y >> 31;
      float r0[NMAT][4], r1[NMAT][4];
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) { r0[m][i] = 0.f; r1[m][i] = 0.f; }
      unit_dot(st, st + R::W, grp0, r0);
      unit_dot(st + 1024, st + R::W + 16 * SB, e0 ? 0 : grp0 + 1, r1);
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[m][i] += r0[m][i];
      if (e0) flush(tile0);
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[m][i] += r1[m][i];
      if (e1) flush(e0 ? tile0 + 1 : tile0);
    }
  }
  cp_wait<0>();
  __syncwarp();
}

extern __shared__ __align__(128) uint8_t gemv_smem[];


// What phase_setup decides for this CTA (every thread holds a copy).
struct PhaseCtx {
  bool part;               // K2b: CTA groups per sub-space (staged h slices)
  int base, Usp, vsp;      // sub-space of this CTA: first unit, units, index (-1: all)
  int ncta, cta;           // CTAs sharing the space, this CTA's index among them
  int KNU;                 // units per ring stage
};

// ---- the space this CTA works in.  K2a: all units (every SM gets the same
// mix of fp16 = HBM-heavy and low-bit = ALU-heavy units; measured: splitting
// K2a's CTAs per job leaves the low-bit group compute-bound and late).  K2b
// with h in shared memory: the CTAs are split into groups, one per sub-space
// (a vjob's column slice of h), sizes proportional to its cost (>= 1 CTA
// each), so a CTA stages only its slice of h and keeps a deep ring; its
// warps' feed covers that slice alone.  Contains __syncthreads.
#ifdef HB_PHASE_FI
#define HB_PHASE_ATTR __forceinline__
#else
#define HB_PHASE_ATTR
#endif
template <bool W13, bool FUSED>
__device__ HB_PHASE_ATTR void phase_setup(const GemvParams& p, const int* s_cum, FeedConst* s_fk, int* s_subb,
                            float* s_subc, int* s_subvh, int* s_nsub, uint32_t bar,
                            bool h_global, Stage& S, PhaseCtx& pc) {
  const int nv = JT<FUSED>::nv(p);
  const int U = s_cum[nv];
  constexpr int XS = W13 ? 1 : 2;
  const int K = W13 ? p.H : p.F;
  pc.part = !W13 && !h_global;
  S.ptr = gemv_smem + kGemvWarps * KCfg<W13>::RING;
  S.xst = smem_u32(S.ptr);
  S.bar = bar;
  pc.base = 0;
  pc.Usp = U;
  pc.ncta = gridDim.x;
  pc.cta = blockIdx.x;
  pc.vsp = -1;
  S.nh = 1;
  S.hs = 0;
  S.row0 = 0;
  S.nrows = W13 ? p.B : JT<FUSED>::nslots(p);
  S.kcols = K;
  S.on = W13 && (size_t)S.nrows * (XS * K * 2 + (K / 32) * 4) <= (size_t)KCfg<W13>::XSTAGE;
  if (pc.part) {
    // sub-spaces (vjob v, column slice h < nh(v)); nh = 2 when the slice has
    // an even number of groups.  CTAs [c0(q), c0(q+1)) work on sub-space q,
    // c0(q) = q + floor(cost before q * (n - nsub) / total cost)
    if (threadIdx.x == 0) {
      int q = 0;
      float cc = 0.f;
      for (int v = 0; v < nv; ++v) {
        const int enc = JT<FUSED>::vjob(p, v).enc;
        const int G = K / epg_of(enc);
        const int nh = G % 4 == 0 ? 2 : 1;
        const int uq = (s_cum[v + 1] - s_cum[v]) / nh;
        const float w = p.k2b_w[enc & 3];   // quantised units are ALU-heavier (HB_K2B_W)
        for (int h = 0; h < nh; ++h, ++q) {
          s_subvh[q] = v | (h << 16) | (nh << 24);
          s_subb[q] = s_cum[v] + h * uq;
          s_subc[q] = cc;
          cc += w * (h + 1 < nh ? uq : (s_cum[v + 1] - s_cum[v]) - h * uq);
        }
      }
      s_subb[q] = U;
      s_subc[q] = cc;
      *s_nsub = q;
    }
    __syncthreads();
    const int nsub = *s_nsub;
    const int spare = (int)gridDim.x - nsub;
    const float ctot = s_subc[nsub];
    auto c0 = [&](int q) { return q + (int)((double)s_subc[q] * spare / ctot); };
    int lo = 0, hi = nsub - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (c0(mid) <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    pc.vsp = lo;
    pc.base = s_subb[lo];
    pc.Usp = s_subb[lo + 1] - pc.base;
    pc.cta = blockIdx.x - c0(lo);
    pc.ncta = (lo + 1 < nsub ? c0(lo + 1) : (int)gridDim.x) - c0(lo);
    const VJobD d = JT<FUSED>::vjob(p, s_subvh[lo] & 0xFFFF);
    S.row0 = d.slot0;
    S.nrows = d.nslot;
    S.nh = s_subvh[lo] >> 24;
    S.hs = (s_subvh[lo] >> 16) & 0xFF;
    S.kcols = K / S.nh;
    // staged (2 units per ring stage) when the slice has an even number of
    // groups; otherwise this group reads h from global memory
    S.on = (K / epg_of(d.enc) / S.nh) % 2 == 0;
  }
  pc.KNU = (!W13 && S.on) ? 2 : 1;
  if (threadIdx.x == 0) {
    s_fk->base = pc.base;
    s_fk->U = pc.Usp;
    s_fk->S = min(pc.Usp, (int)((double)pc.Usp * (W13 ? p.static_frac : p.static_frac2))) & ~(pc.KNU - 1);
    s_fk->chunk = p.chunk;
    s_fk->nch = (pc.Usp - s_fk->S + p.chunk - 1) / p.chunk;
    s_fk->nwarps = pc.ncta * kGemvWarps;
    // counters: [0] K2a all units, [1] K2b all units, [2 + q] K2a group q,
    // [2 + kGemvCTAs + q] K2b group q (K2b fetches while K2a still runs)
    s_fk->ctr = p.ctr + (pc.vsp < 0 ? (W13 ? 0 : 1) : 2 + (W13 ? 0 : kGemvCTAs) + pc.vsp);
  }
  __syncthreads();
}

// Every warp streams its static range, then dynamic chunks, through its ring
// (no CTA-wide synchronisation: warps leave at different times).
template <bool W13, bool FUSED, bool KQ = false>
__device__ HB_PHASE_ATTR void phase_run(const GemvParams& p, const int* s_cum, const FeedConst* s_fk,
                          const int* s_subvh, const PhaseCtx& pc, const Stage& S, uint2* meta) {
  const int warp = threadIdx.x >> 5;
  Feed fd;
  fd.k = s_fk;
  fd.done = false;
  // static ranges are dealt SM-interleaved (warp * #CTAs + CTA): consecutive
  // ranges (same job, same encoding) land on different SMs
  const int gwl = warp * pc.ncta + pc.cta;
  fd.a = pc.base + ((int)((long long)s_fk->S * gwl / s_fk->nwarps) & ~(pc.KNU - 1));
  fd.b = pc.base + ((int)((long long)s_fk->S * (gwl + 1) / s_fk->nwarps) & ~(pc.KNU - 1));
  if (p.det && !pc.part) {
    // deterministic mode: every warp gets whole row tiles (every vjob has the
    // same number of tiles), so each output row of a vjob is one reduction
    const int nvj = JT<FUSED>::nv(p);
    const int tpv = (W13 ? p.F : p.H) / 16, T = nvj * tpv;
    auto unit_of = [&](int tau) -> int {
      if (tau >= T) return s_cum[nvj];
      const int v = tau / tpv;
      return s_cum[v] + (tau - v * tpv) * ((s_cum[v + 1] - s_cum[v]) / tpv);
    };
    fd.a = pc.base + unit_of((int)((long long)T * gwl / s_fk->nwarps));
    fd.b = pc.base + unit_of((int)((long long)T * (gwl + 1) / s_fk->nwarps));
  }
  fd.start();
  const uint32_t ring = smem_u32(gemv_smem) + warp * KCfg<W13>::RING;
  bool first = true;
  const int nv = JT<FUSED>::nv(p);
  while (fd.a < fd.b || fd.refill()) {
    int lo = 0, cv, Uv;
    if (pc.part) {                             // the CTA's sub-space (one vjob slice)
      lo = s_subvh[pc.vsp] & 0xFFFF;
      cv = pc.base;
      Uv = pc.Usp;
    } else {
      int hi = nv - 1;                         // vjob containing unit fd.a
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_cum[mid] <= fd.a) lo = mid; else hi = mid - 1;
      }
      cv = s_cum[lo];
      Uv = s_cum[lo + 1] - cv;
    }
    const VJobD d = JT<FUSED>::vjob(p, lo);
    const VJob vj{d.blob, d.enc, d.slot0, d.nslot};
#define HB_RUN(E, X) run<E, W13, X, FUSED>(p, vj, cv, Uv, fd, ring, meta, S, first)
    switch (vj.enc * 2 + (S.on ? 1 : 0)) {
      case 2 * HB_F16 + 1: HB_RUN(HB_F16, true); break;
      case 2 * HB_F16 + 0: HB_RUN(HB_F16, false); break;
      case 2 * HB_Q8 + 1: HB_RUN(HB_Q8, true); break;
      case 2 * HB_Q8 + 0: HB_RUN(HB_Q8, false); break;
      case 2 * HB_Q4 + 1: HB_RUN(HB_Q4, true); break;
      case 2 * HB_Q4 + 0: HB_RUN(HB_Q4, false); break;
      // the Q2 slot: HB_Q2K in the KQ kernels (their own instantiation, so the
      // default kernels' register allocation is not touched)
      case 2 * HB_Q2 + 1:
        if constexpr (KQ) HB_RUN(kEncQ2K, true); else HB_RUN(HB_Q2, true);
        break;
      default:
        if constexpr (KQ) HB_RUN(kEncQ2K, false); else HB_RUN(HB_Q2, false);
        break;
    }
#undef HB_RUN
    first = false;
  }
  if (first) {                               // no units at all: still take part in the stage
    if constexpr (W13) {
      if (S.on) stage_x_and_wait<FUSED>(p, S);
    } else {
      stage_h_and_wait<FUSED>(p, S);
    }
  }
}

// hb_stamps records of the legacy chain: K2a end (last CTA); K2b end (last
// CTA), and K2b's last CTA moves the record index on
template <bool W13>
__device__ __noinline__ void legacy_stamp_end_(const GemvParams& p) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned idx = __ldcg(p.fwd_idx);
  if (idx < (unsigned)p.stamp_cap) atomicMax(p.stamps + (size_t)idx * kStampStride + (W13 ? 2 : 4), gtimer_ns());
  if (!W13) {
    if (atomicAdd(p.fwd_idx + 1, 1u) == gridDim.x - 1) {
      p.fwd_idx[1] = 0u;
      p.fwd_idx[0] += 1u;
    }
  }
}

template <bool W13>
__device__ __forceinline__ void legacy_stamp_end(const GemvParams& p) {
#ifndef HB_NO_STAMPS
  if (p.stamps) legacy_stamp_end_<W13>(p);
#endif
}
__device__ __noinline__ void legacy_stamp_start(const GemvParams& p) {
  const unsigned idx = __ldcg(p.fwd_idx);
  if (idx < (unsigned)p.stamp_cap) {
    atomicMax(p.stamps + (size_t)idx * kStampStride + 0, ~gtimer_ns());
    atomicMax(p.stamps + (size_t)idx * kStampStride + 1, gtimer_ns());
  }
}

// hfin folded into the end of K2a (p.hfin_tail): the CTAs meet at a grid
// barrier once every K2a sum is complete, then each computes its share of
// h = silu(a) * u as the fp16 hi/lo rows + block sums K2b bulk-copies, and
// CTA b writes the NaN y row of token b (R28).  Saves the hfin launch and its
// hand-offs; K2b waits on K2a directly.  Cold code, not inlined.
__device__ __noinline__ void k2a_hfin_tail(const GemvParams& p, bool any) {
  if (any) {
    __syncthreads();                           // every warp of the CTA is past its K2a work
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned g = ld_acquire_gpu(p.gbar + 1);
      if (atomicAdd(p.gbar, 1u) == gridDim.x - 1) {
        p.gbar[0] = 0u;
        st_release_gpu(p.gbar + 1, g + 1u);
      } else {
        while (ld_acquire_gpu(p.gbar + 1) == g) __nanosleep(64);
      }
    }
    __syncthreads();
    const int nb = p.F / 32;
    const int n = lg_nslot * nb * 4;             // four threads per (slot, 32-row block)
    const int lane = threadIdx.x & 31;
    const int nthr = gridDim.x * blockDim.x;
    for (int i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += nthr) {
      const int i = i0 + lane;
      const bool act = i < n;
      const int q = act ? i : 0;
      const int item = q >> 2, t = q & 3;
      const int sl = item / nb, j = item - sl * nb;
      const float* pa = p.au + (size_t)sl * 2 * p.F + (size_t)j * 32 + 8 * t;
      const float* pu = pa + p.F;
      const float4 a0 = __ldcg(reinterpret_cast<const float4*>(pa));
      const float4 a1 = __ldcg(reinterpret_cast<const float4*>(pa) + 1);
      const float4 u0 = __ldcg(reinterpret_cast<const float4*>(pu));
      const float4 u1 = __ldcg(reinterpret_cast<const float4*>(pu) + 1);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float uv[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
      float h[8], hs = 0.f;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        h[r] = av[r] / (1.f + expf(-av[r])) * uv[r];
        hs += h[r];
      }
      uint32_t wh[4], wl[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {            // Q_c = (h[8t+c], h[8t+c+4])
        const __half h0 = __float2half_rn(h[c]), h1 = __float2half_rn(h[c + 4]);
        const __half l0 = __float2half_rn(h[c] - __half2float(h0));
        const __half l1 = __float2half_rn(h[c + 4] - __half2float(h1));
        wh[c] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
        wl[c] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
      }
      hs += __shfl_xor_sync(0xffffffffu, hs, 1);
      hs += __shfl_xor_sync(0xffffffffu, hs, 2);
      if (act) {
        p.h_hi[(size_t)sl * (p.F / 8) + j * 4 + t] = make_uint4(wh[0], wh[1], wh[2], wh[3]);
        p.h_lo[(size_t)sl * (p.F / 8) + j * 4 + t] = make_uint4(wl[0], wl[1], wl[2], wl[3]);
        if (t == 0) p.hsum[item] = hs;
      }
    }
  }
  if (p.rowbad)
    for (int b = blockIdx.x; b < p.B; b += gridDim.x)
      if (__ldcg(p.rowbad + b))
        for (int c = threadIdx.x; c < p.H; c += blockDim.x)
          p.y[(size_t)b * p.H + c] = __int_as_float(0x7fc00000);
}

// Legacy chain (router kernel -> K2a -> hfin -> K2b): batches, the offload
// path and configurations the fused kernel does not cover.  KQ: the Q2 slot
// holds HB_Q2K blobs (a separate instantiation).
template <bool W13, bool KQ>
__global__ void __launch_bounds__(kGemvWarps * 32, 1)
gemv_kernel(const __grid_constant__ GemvParams p) {
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_cum[kMaxVJobs + 1];
  __shared__ uint2 s_meta[kGemvWarps][16];
  __shared__ FeedConst s_fk;
  __shared__ int s_subb[kGemvCTAs + 1];         // K2b sub-space first units (+ total)
  __shared__ float s_subc[kGemvCTAs + 1];       // K2b sub-space cumulative cost (+ total)
  __shared__ int s_subvh[kGemvCTAs];            // vjob | slice << 16 | slices << 24
  __shared__ int s_nsub;
  const int warp = threadIdx.x >> 5;
  HB_TL(W13, warp * gridDim.x + blockIdx.x, 0);
#if HB_LEGACY_TL == 1
  const unsigned long long tl_entry = tl_now();
  if (!W13 && threadIdx.x == 0) tl_k2b_entry = tl_entry;
#endif
  // K2a needs the router's job table and x; K2b may read the table before
  // waiting (K2a triggers its dependents only after its own wait, i.e. after
  // the router completed) and waits for K2a's sums inside its first run
  if constexpr (W13) pdl_wait();
  pdl_trigger();
#if HB_LEGACY_TL == 1
  if (W13 && threadIdx.x == 0) tl_min(tl_rec(p.stamps, p.stamp_cap, p.fwd_idx), 8, tl_entry);
#endif
  const long long* cum = W13 ? p.jt.vcum13 : p.jt.vcum2;
  for (int i = threadIdx.x; i <= p.max_vjobs; i += blockDim.x) s_cum[i] = (int)__ldcg(cum + i);
  if (threadIdx.x == 0) {
    lg_nv = __ldcg(p.jt.hdr + 2);
    lg_nslot = __ldcg(p.jt.hdr + 1);
  }
  // stage hand-off: K2a every thread arrives after its share of the x copy;
  // K2b thread 0 arrives once with the bulk copies' transaction count
  if (threadIdx.x == 0) mbar_init(smem_u32(&s_bar), W13 ? blockDim.x : 1);
  __syncthreads();
#ifndef HB_NO_STAMPS
  if (W13 && p.stamps && threadIdx.x == 0) legacy_stamp_start(p);
#endif
  if (JT<false>::nv(p) == 0) {               // nothing owned: y stays zero (router)
    if (W13 && p.hfin_tail) k2a_hfin_tail(p, false);
    legacy_stamp_end<W13>(p);
    return;
  }
  Stage S;
  PhaseCtx pc;
  phase_setup<W13, false>(p, s_cum, &s_fk, s_subb, s_subc, s_subvh, &s_nsub, smem_u32(&s_bar),
                          p.h_global, S, pc);
  phase_run<W13, false, KQ>(p, s_cum, &s_fk, s_subvh, pc, S, s_meta[warp]);
  HB_TL(W13, warp * gridDim.x + blockIdx.x, 3);
  if (W13 && p.hfin_tail) k2a_hfin_tail(p, true);
#if HB_LEGACY_TL == 1
  if (W13) {
    __syncthreads();
    if (threadIdx.x == 0) tl_min(tl_rec(p.stamps, p.stamp_cap, p.fwd_idx), 14, tl_now());
  }
#endif
  legacy_stamp_end<W13>(p);
}

// ------------------------------------------------------------ fused decode
// One kernel per layer for batch-1 decode in resident mode (DESIGN.md "fused
// decode kernel"): every CTA
//   1. (before griddepcontrol.wait) bulk-copies the layer's router rows into
//      its shared memory;
//   2. routes the token itself: fp32 products (exact for fp16 x fp16) summed
//      in runs of 8 with FFMA, runs summed in fp64, together with a rigorous
//      bound on the rounding error; the top-2 order and the T1/T2 tests are
//      decided from these when every comparison clears the bound, else from
//      the exact integer logits (the same exact arithmetic as the router
//      kernel) -- so the decisions are the exact ones either way, and every
//      CTA derives the same decisions from the same operations (no hand-off);
//   3. builds the job table in shared memory;
//   4. runs K2a (W1/W3 + sums into au), then, per warp as soon as its K2a
//      work is done, issues the first W2 ring stages, meets the other CTAs
//      at a grid barrier (K2a sums complete), builds its slice of h from the
//      sums and runs K2b.
// Replaces router kernel + K2a + hfin + K2b and their three hand-offs.
constexpr int kFusedScratch = 160 * 1024;   // router scratch offset in dynamic smem (W_g below)
// |sum of 8 products in fp32 FFMA - exact| <= gamma_7 sum|p| (gamma_7 =
// 7u/(1-7u), u = 2^-24); the fp64 sums over runs add < 1e-13 relative; the
// bound sum itself is an fp32/fp64 sum of |p| (relative error <= gamma_7).
// 4.6e-7 * A >= (gamma_7 + 1e-13) (1 + gamma_7) (1 + 1e-13) * A.
constexpr double kEpsRel = 4.6e-7;

// The fused kernel runs each phase in a non-inlined function whose code is
// the legacy kernel's (run<> inlined into phase_run): a separate register
// allocation, so the router's state never competes with the streaming loops.
// p lives in shared memory (fz_p) so the functions address it cheaply.
__shared__ GemvParams fz_p;
__device__ __noinline__ void fused_k2a(const GemvParams& p, int* s_cum, FeedConst* s_fk,
                                       int* s_subb, float* s_subc, int* s_subvh, int* s_nsub,
                                       uint32_t bar, uint2* meta) {
  Stage S;
  PhaseCtx pc;
  phase_setup<true, true>(p, s_cum, s_fk, s_subb, s_subc, s_subvh, s_nsub, bar, false, S, pc);
  phase_run<true, true>(p, s_cum, s_fk, s_subvh, pc, S, meta);
}
__device__ __noinline__ void fused_k2b(const GemvParams& p, const int* s_cum, const FeedConst* s_fk,
                                       const int* s_subvh, const Stage* sS, const PhaseCtx* spc,
                                       uint2* meta) {
  const Stage S = *sS;
  const PhaseCtx pc = *spc;
  phase_run<false, true>(p, s_cum, s_fk, s_subvh, pc, S, meta);
}

// Decision records and the job table of the token (B = 1, top-2), by lane 0
// of warp 0 from the decided experts: gates g0 = 1/(1+e), g1 = e*g0 with
// e = exp(-gap) (reading R25); jobs by key (expert, High before Low), one
// slot each; shared copies for this CTA, and (CTA 0) the decision records
// and, in split mode, the global job table the K2b kernel reads.
// What the fused kernel's router needs, passed BY VALUE to the non-inlined
// router function (no generic accesses to the kernel parameter space there)
struct RouteArgs {
  const __half* x;
  __half* x_save;
  int E, H, F;
  int64_t theta1, theta2;
  int th1_kind, th2_kind;
  int rank, world, hi_enc, lo_enc;
  hb_decision* dec;
  JobTable jt;
};

template <bool K2B>
__device__ __forceinline__ void fused_jobs(const RouteArgs& fp, const uint8_t* const* s_blob,
                                           int e0, int e1,
                                           uint8_t prec1, float gd, int nonfinite, int* s_cum13,
                                           int* s_cum2) {
  if ((threadIdx.x & 31) != 0) return;
  const bool cta0 = blockIdx.x == 0;
  hb_decision r0, r1;
  s_cum13[0] = 0;
  s_cum2[0] = 0;
  if (!K2B && cta0) {
    fp.jt.vcum13[0] = 0;
    fp.jt.vcum2[0] = 0;
    fp.jt.tok_slots[0] = -1;
    fp.jt.tok_slots[1] = -1;
  }
  int nj = 0;
  if (nonfinite) {
    const float nan = __int_as_float(0x7fc00000);
    r0 = hb_decision{0, -1, 0, HB_SKIP, HB_ENC_NONE, 0, nan};
    r1 = hb_decision{0, -1, 1, HB_SKIP, HB_ENC_NONE, 0, nan};
  } else {
    const float ex = expf(-gd);
    const float g0 = 1.f / (1.f + ex), g1 = ex * g0;
    r0 = hb_decision{0, e0, 0, HB_HIGH, HB_ENC_NONE, 0, g0};
    r1 = hb_decision{0, e1, 1, prec1, HB_ENC_NONE, 0, g1};
    const bool v0 = e0 % fp.world == fp.rank;
    const bool v1 = prec1 != HB_SKIP && e1 % fp.world == fp.rank;
    const int enc1 = prec1 == HB_HIGH ? fp.hi_enc : fp.lo_enc;
    const bool swap = v0 && v1 && (e1 * 2 + (prec1 == HB_HIGH ? 0 : 1)) < e0 * 2;
    auto put = [&](int sel, int e, int enc, float g) {
      VJobD d;
      d.blob = s_blob[e * 4 + enc];
      d.enc = enc;
      d.slot0 = nj;
      d.nslot = 1;
      d.pad = 0;
      fz_vj[nj] = d;
      fz_stok[nj] = 0;
      fz_sgate[nj] = g;
      const int epg = epg_of_enc(enc);
      s_cum13[nj + 1] = s_cum13[nj] + (fp.F / 16) * (fp.H / epg);
      s_cum2[nj + 1] = s_cum2[nj] + (fp.H / 16) * (fp.F / epg);
      if (!K2B && cta0) {
        Job j;
        j.blob = d.blob;
        j.enc = enc;
        j.expert = e;
        j.n_tok = 1;
        j.slot_off = nj;
        fp.jt.jobs[nj] = j;
        fp.jt.slot_token[nj] = 0;
        fp.jt.slot_gate[nj] = g;
        fp.jt.vjobs[nj] = d;
        fp.jt.vcum13[nj + 1] = s_cum13[nj + 1];
        fp.jt.vcum2[nj + 1] = s_cum2[nj + 1];
        fp.jt.tok_slots[sel] = nj;
      }
      hb_decision& r = sel ? r1 : r0;
      r.served_enc = (uint8_t)enc;
      r.hit = 1;
      ++nj;
    };
    if (swap) {
      put(1, e1, enc1, g1);
      put(0, e0, fp.hi_enc, g0);
    } else {
      if (v0) put(0, e0, fp.hi_enc, g0);
      if (v1) put(1, e1, enc1, g1);
    }
  }
  fz_nv = nj;
  fz_nslot = nj;
  if (!K2B && cta0) {
    fp.jt.hdr[0] = nj;
    fp.jt.hdr[1] = nj;
    fp.jt.hdr[2] = nj;
  }
  if (cta0) {
    fp.dec[0] = r0;
    fp.dec[1] = r1;
  }
}

__device__ __forceinline__ void h2f8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Steps 2-3 of the fused kernel (route the token, decide, build the job
// table).  Returns the non-finite flag.
template <bool K2B>
__device__ __noinline__ int fused_route(const RouteArgs fp, int* s_cum13, int* s_cum2, int* s_ok,
                                       uint32_t wbar, unsigned long long* rec) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int E = fp.E, H = fp.H, n8 = H / 8;
  uint8_t* dyn = gemv_smem;
  double* red = reinterpret_cast<double*>(dyn + kFusedScratch);          // [12 warps][64] partial logits
  float* s_xq = reinterpret_cast<float*>(dyn + kFusedScratch + 12 * 64 * 8);              // [12] sum x^2
  float* s_wn = s_xq + 16;                                                                // [64] ||W_e||_2
  const uint8_t** s_blob = reinterpret_cast<const uint8_t**>(dyn + kFusedScratch + 8192);  // [E][4]
  u64* xpart = reinterpret_cast<u64*>(dyn + kFusedScratch + 12288);                       // [12][64][3]
  i128* s_Lx = reinterpret_cast<i128*>(dyn + kFusedScratch + 12288 + 12 * 64 * 24);       // [64]
  double* s_Lf = reinterpret_cast<double*>(dyn + kFusedScratch + 12288 + 12 * 64 * 24 + 1024);  // [64]
  double* s_ep = s_Lf + 64;                                                                     // [64]
  // ---- 2. route the token (B = 1).  x chunks of this thread in registers;
  // CTA 0 keeps a copy for the lazy exact logits (hb_get_logits)
  constexpr int kXC = 3;                       // H <= 9216
  uint4 xr[kXC];
  float xf[kXC][8];
  bool bad = false;
  float xq = 0.f;
#pragma unroll
  for (int i = 0; i < kXC; ++i) {
    const int c = tid + i * kGemvWarps * 32;
    xr[i] = c < n8 ? __ldcg(reinterpret_cast<const uint4*>(fp.x) + c) : make_uint4(0, 0, 0, 0);
    if (blockIdx.x == 0 && c < n8 && fp.x_save) reinterpret_cast<uint4*>(fp.x_save)[c] = xr[i];
    h2f8(xr[i], xf[i]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      bad |= !isfinite(xf[i][j]);
      xq = fmaf(xf[i][j], xf[i][j], xq);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) xq += __shfl_xor_sync(0xffffffffu, xq, o);
  if (lane == 0) s_xq[warp] = xq;
  const int nonfinite = __syncthreads_or(bad);
  mbar_wait(wbar, 0);                          // router rows landed
  if (rec && tid == 0) atomicMax(rec + 5, gtimer_ns());
  // filtered logits: per thread an fp32 FFMA chain over its <= 24 products
  // (fp16 x fp16 products are exact in fp32), warp sums in fp32 (5 levels),
  // the 12 warp partials summed in fp64 by warp 0 in a fixed order (every CTA
  // performs the same operations, so every CTA gets bit-identical values)
  const uint4* w4 = reinterpret_cast<const uint4*>(dyn);
  for (int e0 = 0; e0 < E; e0 += 8) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
    for (int i = 0; i < kXC; ++i) {
      const int c = tid + i * kGemvWarps * 32;
      if (c >= n8) break;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (e0 + j >= E) break;
        float wf[8];
        h2f8(w4[(size_t)(e0 + j) * n8 + c], wf);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[j] = fmaf(wf[q], xf[i][q], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float d = acc[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (lane == 0 && e0 + j < E) red[warp * 64 + e0 + j] = (double)d;
    }
  }
  __syncthreads();
  if (rec && tid == 0) atomicMax(rec + 6, gtimer_ns());
  // ---- 3. warp 0: top-2 by (L desc, index asc), the certainty of every
  // comparison, decisions, gates and (lanes 0/1) the job table
  if (warp == 0) {
    // lane l handles experts l and l + 32; the logits go through shared
    // memory (broadcast reads) for the ranking
    double xs = 0.0;
    for (int w = 0; w < kGemvWarps; ++w) xs += (double)s_xq[w];
    // Cauchy-Schwarz: sum |w_h x_h| <= ||w_e|| ||x||; ||x|| rounded up (the
    // fp32 squares carry a relative error < 1e-5).  Error of a logit: the fp32
    // chains (<= 24 products, gamma_23) and warp trees (gamma_5) plus the
    // fp64 sum over warps: <= 29.1 * 2^-24 * sum|p| < 1.74e-6 * sum|p|, so
    // 2.2e-6 * ||w_e|| ||x|| bounds it
    const double xn = (double)sqrtf((float)xs * 1.00002f) * 1.000001;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      if (e < E) {
        double l = 0.0;
#pragma unroll
        for (int w = 0; w < kGemvWarps; ++w) l += red[w * 64 + e];
        s_Lf[e] = l;
        s_ep[e] = 2.2e-6 * (double)s_wn[e] * xn;
      }
    }
    __syncwarp();
    if (rec && lane == 0) atomicMax(rec + 10, gtimer_ns());
    int rk[2] = {64, 64};
    double rest = -1e300;                      // max over ranks >= 2 of L + eps
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      if (e < E) {
        const double v = s_Lf[e];
        int r = 0;
        for (int f = 0; f < E; ++f) {
          const double o = s_Lf[f];
          r += (o > v) || (o == v && f < e);
        }
        rk[h] = r;
        if (r >= 2) rest = fmax(rest, v + s_ep[e]);
      }
    }
    const unsigned m0 = __ballot_sync(0xffffffffu, rk[0] == 0), m0b = __ballot_sync(0xffffffffu, rk[1] == 0);
    const unsigned m1 = __ballot_sync(0xffffffffu, rk[0] == 1), m1b = __ballot_sync(0xffffffffu, rk[1] == 1);
    const int e0 = m0 ? __ffs(m0) - 1 : 32 + __ffs(m0b) - 1;
    const int e1 = m1 ? __ffs(m1) - 1 : 32 + __ffs(m1b) - 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rest = fmax(rest, __shfl_xor_sync(0xffffffffu, rest, o));
    if (rec && lane == 0) atomicMax(rec + 11, gtimer_ns());
    const double L0 = s_Lf[e0], L1 = s_Lf[e1], ep0 = s_ep[e0], ep1 = s_ep[e1];
    const double G = L0 - L1, m = ep0 + ep1 + 1e-12 * (1.0 + fabs(L0) + fabs(L1));
    bool ok = !nonfinite && (L0 - ep0 > L1 + ep1) && (L1 - ep1 > rest);
    if (fp.th1_kind == 0) ok = ok && fabs(G - (double)fp.theta1 * 0x1p-48) > m;
    if (fp.th2_kind == 0) ok = ok && fabs(G - (double)fp.theta2 * 0x1p-48) > m;
    uint8_t prec1 = (fp.th1_kind > 0 || (fp.th1_kind == 0 && G <= (double)fp.theta1 * 0x1p-48)) ? HB_HIGH
                  : (fp.th2_kind > 0 || (fp.th2_kind == 0 && G <= (double)fp.theta2 * 0x1p-48)) ? HB_LOW
                                                                                                 : HB_SKIP;
    float gd = (float)G;
    if (rec && lane == 0) {
      atomicMax(rec + 12, gtimer_ns());
      if (!(ok || nonfinite) && blockIdx.x == 0) atomicAdd(rec + 14, 1ull);   // exact fallbacks
    }
    if (ok || nonfinite) {
      fused_jobs<K2B>(fp, s_blob, e0, e1, prec1, gd, nonfinite, s_cum13, s_cum2);
      if (lane == 0) (*s_ok) = 1;
    } else if (lane == 0) {
      (*s_ok) = 0;
    }
    if (rec && lane == 0) atomicMax(rec + 13, gtimer_ns());
  }
  __syncthreads();
  if (!(*s_ok)) {
    // ---- exact fallback: integer logits (every CTA takes this branch alike)
    for (int e = 0; e < E; ++e) {
      u64 lo = 0, mid = 0, hi = 0;
#pragma unroll
      for (int i = 0; i < kXC; ++i) {
        const int c = tid + i * kGemvWarps * 32;
        if (c >= n8) break;
        const uint4 wv = w4[(size_t)e * n8 + c];
        const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t xa[4] = {xr[i].x, xr[i].y, xr[i].z, xr[i].w};
#pragma unroll
        for (int q = 0; q < 8; ++q)
          accum_exact((wa[q >> 1] >> (16 * (q & 1))) & 0xFFFF, (xa[q >> 1] >> (16 * (q & 1))) & 0xFFFF,
                      lo, mid, hi);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        mid += __shfl_xor_sync(0xffffffffu, mid, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      if (lane == 0) {
        u64* d = xpart + ((size_t)warp * 64 + e) * 3;
        d[0] = lo; d[1] = mid; d[2] = hi;
      }
    }
    __syncthreads();
    if (tid < E) {
      u64 lo = 0, mid = 0, hi = 0;
      for (int w = 0; w < kGemvWarps; ++w) {
        const u64* d = xpart + ((size_t)w * 64 + tid) * 3;
        lo += d[0]; mid += d[1]; hi += d[2];
      }
      s_Lx[tid] = (i128)(long long)lo + ((i128)(long long)mid << 20) + ((i128)(long long)hi << 40);
    }
    __syncthreads();
    if (warp == 0) {
      int rk[2] = {64, 64};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h;
        if (e < E) {
          const i128 v = s_Lx[e];
          int r = 0;
          for (int f = 0; f < E; ++f) { const i128 o = s_Lx[f]; r += (o > v) || (o == v && f < e); }
          rk[h] = r;
        }
      }
      const unsigned m0 = __ballot_sync(0xffffffffu, rk[0] == 0), m0b = __ballot_sync(0xffffffffu, rk[1] == 0);
      const unsigned m1 = __ballot_sync(0xffffffffu, rk[0] == 1), m1b = __ballot_sync(0xffffffffu, rk[1] == 1);
      const int e0 = m0 ? __ffs(m0) - 1 : 32 + __ffs(m0b) - 1;
      const int e1 = m1 ? __ffs(m1) - 1 : 32 + __ffs(m1b) - 1;
      const i128 G = s_Lx[e0] - s_Lx[e1];      // >= 0
      const uint8_t prec1 = gap_le(G, fp.th1_kind, fp.theta1) ? HB_HIGH
                          : gap_le(G, fp.th2_kind, fp.theta2) ? HB_LOW : HB_SKIP;
      const float gd = G >= ((i128)1 << 62) ? 1e30f : (float)(long long)G * 0x1p-48f;
      fused_jobs<K2B>(fp, s_blob, e0, e1, prec1, gd, 0, s_cum13, s_cum2);
    }
    __syncthreads();
  }
  return nonfinite;
}

template <bool K2B>
__global__ void __launch_bounds__(kGemvWarps * 32, 1)
fused_decode_kernel(const __grid_constant__ FusedParams fp) {
  const GemvParams& p = fp.g;
  __shared__ __align__(8) uint64_t s_wbar, s_bar13, s_bar2;
  __shared__ int s_cum13[kFusedMaxV + 1], s_cum2[kFusedMaxV + 1];
  __shared__ uint2 s_meta[kGemvWarps][16];
  __shared__ FeedConst s_fk13, s_fk2;
  __shared__ int s_subb[kGemvCTAs + 1];
  __shared__ float s_subc[kGemvCTAs + 1];
  __shared__ int s_subvh[kGemvCTAs];
  __shared__ int s_nsub, s_nsub13;
  __shared__ int s_ok;
  __shared__ __align__(8) uint64_t s_released, s_warps_done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int E = fp.E, H = p.H, n8 = H / 8;
  uint8_t* dyn = gemv_smem;
  // router scratch above the router rows (W_g takes E*H*2 <= kFusedScratch)
  double* red = reinterpret_cast<double*>(dyn + kFusedScratch);          // [12 warps][64] partial logits
  float* s_xq = reinterpret_cast<float*>(dyn + kFusedScratch + 12 * 64 * 8);              // [12] sum x^2
  float* s_wn = s_xq + 16;                                                                // [64] ||W_e||_2
  const uint8_t** s_blob = reinterpret_cast<const uint8_t**>(dyn + kFusedScratch + 8192);  // [E][4]
  u64* xpart = reinterpret_cast<u64*>(dyn + kFusedScratch + 12288);                       // [12][64][3]
  i128* s_Lx = reinterpret_cast<i128*>(dyn + kFusedScratch + 12288 + 12 * 64 * 24);       // [64]
  double* s_Lf = reinterpret_cast<double*>(dyn + kFusedScratch + 12288 + 12 * 64 * 24 + 1024);  // [64]
  double* s_ep = s_Lf + 64;                                                                     // [64]

  // ---- 1. before waiting on the previous kernel: router rows (static) into
  // shared memory with bulk copies, blob table and row norms of the layer
  const uint32_t wbar = smem_u32(&s_wbar);
  if (tid == 0) {
    mbar_init(wbar, 1);
    mbar_init(smem_u32(&s_bar13), blockDim.x);
    mbar_init(smem_u32(&s_bar2), blockDim.x);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t total = (uint32_t)E * H * 2;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(wbar), "r"(total) : "memory");
    for (uint32_t off = 0; off < total; off += 16384) {
      const uint32_t len = total - off < 16384 ? total - off : 16384;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          :: "r"(smem_u32(dyn) + off), "l"(reinterpret_cast<const char*>(fp.wg) + off), "r"(len),
             "r"(wbar) : "memory");
    }
  }
  for (int i = tid; i < 4 * E; i += blockDim.x) s_blob[i] = fp.blob_table[i];
  for (int i = tid; i < E; i += blockDim.x) s_wn[i] = fp.wnorm[i];
  if (tid == 0) {
    mbar_init(smem_u32(&s_warps_done), blockDim.x);
    mbar_init(smem_u32(&s_released), 1);
  }
  __syncthreads();
  pdl_wait();                                  // x (and y, the sums) belong to earlier work
  if (K2B) pdl_trigger();
  unsigned long long* rec = nullptr;
  if (fp.stamps) {
    const unsigned idx = __ldcg(fp.fwd_idx);
    if (idx < (unsigned)fp.stamp_cap) rec = fp.stamps + (size_t)idx * kStampStride;
    if (rec && tid == 0) atomicMax(rec + 0, ~gtimer_ns());
  }

  const RouteArgs ra{p.x_raw, fp.x_save, fp.E, p.H, p.F, fp.theta1, fp.theta2, fp.th1_kind,
                     fp.th2_kind, fp.rank, fp.world, fp.hi_enc, fp.lo_enc, fp.dec, p.jt};
  const int nonfinite = fused_route<K2B>(ra, s_cum13, s_cum2, &s_ok, wbar, rec);
  const int nonfinite_tok = nonfinite;
  if (rec && tid == 0) atomicMax(rec + 7, gtimer_ns());

  // y row: 0 (the expert kernels add into it), NaN for a non-finite input
  {
    const float yv = nonfinite_tok ? __int_as_float(0x7fc00000) : 0.f;
    for (int i = blockIdx.x * blockDim.x + tid; i < H; i += gridDim.x * blockDim.x) p.y[i] = yv;
    // the other K2a-sum buffer, for the next forward (not touched by this one)
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < fp.zero_n;
         i += (long long)gridDim.x * blockDim.x)
      fp.zero_other[i] = 0.f;
  }
  // split mode: CTA 0 wrote the global job table; it becomes visible before
  // this CTA's trigger (the K2b kernel launches after every CTA triggered)
  if (!K2B && blockIdx.x == 0 && tid == 0) __threadfence();
  __syncthreads();
  if (!K2B) pdl_trigger();
  if (tid == 0) fz_fs = FusedSync{fp.gbar, fp.gbar + 1, &s_warps_done, &s_released, rec};
  if (rec && tid == 0) atomicMax(rec + 1, gtimer_ns());
  if (!K2B && fp.router_only) {
    // router kernel (one CTA): the pair-permuted x and its block sums for the
    // K2a kernel that follows (stage_share_xperm reads them)
    const int nb = H / 32;
    for (int i = tid; i < nb; i += blockDim.x) {
      const uint4* src = reinterpret_cast<const uint4*>(p.x_raw + (size_t)i * 32);
      uint32_t v[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 t = __ldcg(src + q);
        v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
      }
      float sum = 0.f;
#pragma unroll
      for (int e = 0; e < 32; ++e)
        sum += __half2float(__ushort_as_half((unsigned short)(v[e >> 1] >> (16 * (e & 1)))));
      const_cast<float*>(p.xsum)[i] = sum;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint32_t q[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int e0 = 8 * t + c, e1 = e0 + 4;
          q[c] = ((v[e0 >> 1] >> (16 * (e0 & 1))) & 0xFFFF) | (((v[e1 >> 1] >> (16 * (e1 & 1))) & 0xFFFF) << 16);
        }
        const_cast<uint4*>(p.x_perm)[i * 4 + t] = make_uint4(q[0], q[1], q[2], q[3]);
      }
    }
    if (fp.stamps) {
      __syncthreads();
      if (tid == 0 && rec) atomicMax(rec + 2, gtimer_ns());   // router kernel end
    }
    return;
  }
  if (!K2B) {
    // split mode: K2a only; hfin and the K2b kernel follow
    if (fz_nv > 0) {
      Stage S;
      PhaseCtx pc;
      phase_setup<true, true>(p, s_cum13, &s_fk13, s_subb, s_subc, s_subvh, &s_nsub13,
                              smem_u32(&s_bar13), false, S, pc);
      phase_run<true, true>(p, s_cum13, &s_fk13, s_subvh, pc, S, s_meta[warp]);
    }
    if (fp.stamps) {
      __syncthreads();
      if (tid == 0 && fz_fs.stamp) atomicMax(fz_fs.stamp + 2, gtimer_ns());
    }
    return;
  }
  if (fz_nv > 0) {
    // ---- 4. K2a, then K2b (the grid barrier sits in K2b's first run)
    // K2b's setup first (it has CTA-wide barriers; K2b's ring prologue is
    // issued per warp as soon as the warp's K2a work is done), stashed in
    // shared memory while K2a runs
    __shared__ Stage s_S2;
    __shared__ PhaseCtx s_pc2;
    if (tid == 0) fz_p = p;
    {
      Stage S2;
      PhaseCtx pc2;
      phase_setup<false, true>(p, s_cum2, &s_fk2, s_subb, s_subc, s_subvh, &s_nsub,
                               smem_u32(&s_bar2), false, S2, pc2);
      if (tid == 0) { s_S2 = S2; s_pc2 = pc2; }
    }
    __syncthreads();
    fused_k2a(fz_p, s_cum13, &s_fk13, s_subb, s_subc, s_subvh, &s_nsub13, smem_u32(&s_bar13),
              s_meta[warp]);
    fused_k2b(fz_p, s_cum2, &s_fk2, s_subvh, &s_S2, &s_pc2, s_meta[warp]);
  }
  if (fp.stamps) {
    __syncthreads();
    if (tid == 0) {
      unsigned long long* rec_end = fz_fs.stamp;
      if (rec_end) atomicMax(rec_end + 4, gtimer_ns());
      if (atomicAdd(fp.fwd_idx + 1, 1u) == gridDim.x - 1) {   // last CTA: next record
        fp.fwd_idx[1] = 0u;
        fp.fwd_idx[0] += 1u;
      }
    }
  }
}

// hfin: h = silu(a) * u of every slot from the K2a sums, as the fp16 hi/lo
// pair-permuted rows + block sums K2b reads (staged per CTA group by bulk
// copies, or straight from global memory at large batch).  Four threads per
// (slot, 32-row block): thread t owns the 16-byte chunk t of hi and lo, i.e.
// rows 8t..8t+7 (short dependency chains: this kernel sits between K2a and
// K2b on every layer's critical path).
__global__ void __launch_bounds__(256) hfin_kernel(const __grid_constant__ GemvParams p) {
#ifndef HB_HFIN_LATE
  pdl_trigger();                             // K2b may launch and prefetch its weights
#endif
  pdl_wait();                                // the K2a sums
#if HB_LEGACY_TL == 1
  if (threadIdx.x == 0) tl_min(tl_rec(p.stamps, p.stamp_cap, p.fwd_idx), 9, tl_now());
#endif
  // R28: CTA b writes the NaN y row of token b if its x had a non-finite
  // element (the router zeroed y; K2b adds after this kernel).  The flag is
  // loaded here, next to the sums, and used at the end.
  const int rowbad = (p.rowbad && (int)blockIdx.x < p.B) ? __ldcg(p.rowbad + blockIdx.x) : 0;
  const int nb = p.F / 32;
  const int n = __ldcg(p.jt.hdr + 1) * nb * 4;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (rowbad || (p.clean && !p.keep_y && (int)blockIdx.x < p.B)) {
    const float v = rowbad ? __int_as_float(0x7fc00000) : 0.f;
    for (int c = threadIdx.x; c < p.H; c += blockDim.x) p.y[(size_t)blockIdx.x * p.H + c] = v;
  }
  if (i >= ((n + 31) & ~31)) return;
  const bool act = i < n;
  const int q = act ? i : 0;
  const int item = q >> 2, t = q & 3;
  const int s = item / nb, j = item - s * nb;
  const float* pa = p.au + (size_t)s * 2 * p.F + (size_t)j * 32 + 8 * t;
  const float* pu = pa + p.F;
  const float4 a0 = __ldcg(reinterpret_cast<const float4*>(pa));
  const float4 a1 = __ldcg(reinterpret_cast<const float4*>(pa) + 1);
  const float4 u0 = __ldcg(reinterpret_cast<const float4*>(pu));
  const float4 u1 = __ldcg(reinterpret_cast<const float4*>(pu) + 1);
  if (p.clean && act) {                      // leave the sums clean for the next forward
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    float4* wa = const_cast<float4*>(reinterpret_cast<const float4*>(pa));
    float4* wu = const_cast<float4*>(reinterpret_cast<const float4*>(pu));
    wa[0] = z; wa[1] = z; wu[0] = z; wu[1] = z;
  }
  const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
  const float uv[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
  float h[8], hs = 0.f;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    // silu(a) u with the SFU exp and reciprocal (~2 ulp; h feeds W2 at ~fp32 precision)
    h[r] = av[r] * __frcp_rn(1.f + __expf(-av[r])) * uv[r];
    hs += h[r];
  }
  uint32_t wh[4], wl[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {              // Q_c = (h[8t+c], h[8t+c+4])
    const __half h0 = __float2half_rn(h[c]), h1 = __float2half_rn(h[c + 4]);
    const __half l0 = __float2half_rn(h[c] - __half2float(h0));
    const __half l1 = __float2half_rn(h[c + 4] - __half2float(h1));
    wh[c] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
    wl[c] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
  }
  hs += __shfl_xor_sync(0xffffffffu, hs, 1);
  hs += __shfl_xor_sync(0xffffffffu, hs, 2);
  if (act) {
    p.h_hi[(size_t)s * (p.F / 8) + j * 4 + t] = make_uint4(wh[0], wh[1], wh[2], wh[3]);
    p.h_lo[(size_t)s * (p.F / 8) + j * 4 + t] = make_uint4(wl[0], wl[1], wl[2], wl[3]);
    if (t == 0) p.hsum[item] = hs;
  }
#if HB_LEGACY_TL == 1
  if ((threadIdx.x & 31) == 0) tl_max(tl_rec(p.stamps, p.stamp_cap, p.fwd_idx), 10, tl_now());
#endif
#ifdef HB_HFIN_LATE
  pdl_trigger();                             // diagnostic: K2b launches once h is written
#endif
}

void launch_w13(const GemvParams& p, cudaStream_t s) {
  constexpr int smem = gemv_smem_bytes<true>();
  if (p.kq) {
    set_max_dyn_smem(gemv_kernel<true, true>, smem);
    launch_pdl(gemv_kernel<true, true>, p.ctas, kGemvWarps * 32, smem, s, p);
    return;
  }
  set_max_dyn_smem(gemv_kernel<true, false>, smem);
  launch_pdl(gemv_kernel<true, false>, p.ctas, kGemvWarps * 32, smem, s, p);
}
void launch_fused(const FusedParams& p, bool split, cudaStream_t s) {
  constexpr int smem = gemv_smem_bytes<false>() > gemv_smem_bytes<true>() ? gemv_smem_bytes<false>()
                                                                          : gemv_smem_bytes<true>();
  if (split || p.router_only) {
    set_max_dyn_smem(fused_decode_kernel<false>, smem);
    launch_pdl(fused_decode_kernel<false>, p.router_only ? 1 : kGemvCTAs, kGemvWarps * 32, smem, s, p);
  } else {
    set_max_dyn_smem(fused_decode_kernel<true>, smem);
    launch_pdl(fused_decode_kernel<true>, kGemvCTAs, kGemvWarps * 32, smem, s, p);
  }
}
bool fused_fits(int E, int H, int F, int hi_enc, int lo_enc) {
  if (E > 64 || (long long)E * H * 2 > kFusedScratch || H / 8 > 3 * kGemvWarps * 32) return false;
  if ((size_t)(2 * H + (H / 32) * 4) > (size_t)KCfg<true>::XSTAGE) return false;
  for (int enc : {hi_enc, lo_enc}) {          // every K2b sub-space stages its slice of h
    const int G = F / epg_of(enc), nh = G % 4 == 0 ? 2 : 1;
    if ((G / nh) % 2) return false;
    const size_t slice = (size_t)(F / nh) * 4 + (size_t)(F / nh / 32) * 4;
    if (slice > (size_t)KCfg<false>::XSTAGE) return false;
  }
  return true;
}
// hfin's CTAs are launched while K2a still holds every SM but the router's:
// a large (unused) shared-memory request keeps them one per SM, so they do
// not pile onto the first free SM and run serially there (measured: 8 CTAs
// on one SM, ~6 us; HB_HFIN_SMEM_KB, 0 = no request)
#ifndef HB_HFIN_SMEM_KB
#define HB_HFIN_SMEM_KB 120
#endif
void launch_hfin(const GemvParams& p, int max_slots, cudaStream_t s) {
  const int n = max_slots * (p.F / 32) * 4;
  constexpr int smem = HB_HFIN_SMEM_KB * 1024;
  if (smem > 48 * 1024) set_max_dyn_smem(hfin_kernel, smem);
  launch_pdl(hfin_kernel, std::max((n + 255) / 256, p.B), 256, smem, s, p);   // >= one CTA per token (R28)
}
void launch_w2(const GemvParams& p, cudaStream_t s) {
  constexpr int smem = gemv_smem_bytes<false>();
  if (p.kq) {
    set_max_dyn_smem(gemv_kernel<false, true>, smem);
    launch_pdl(gemv_kernel<false, true>, p.ctas, kGemvWarps * 32, smem, s, p);
    return;
  }
  set_max_dyn_smem(gemv_kernel<false, false>, smem);
  launch_pdl(gemv_kernel<false, false>, p.ctas, kGemvWarps * 32, smem, s, p);
}
int w2_stage_capacity() { return KCfg<false>::XSTAGE; }

}  // namespace hb

#ifdef HB_DBG_TIMELINE
extern "C" int hb_debug_timeline(void* host, int which) {
  return (int)cudaMemcpyFromSymbol(host, hb::g_tl, sizeof(hb::g_tl[0]),
                                   (size_t)which * sizeof(hb::g_tl[0]));
}
#endif
