// K2a / K2b: grouped mixed-precision dequant-GEMV of the selected experts.
//
//   K2a  h = silu(W1 x) * (W3 x)          per job (expert, served encoding)
//   K2b  y = sum_jobs gate * (W2 h)        Eq. 1, Skip = no job
//
// Paper: the layer output is the gate-weighted sum of the selected experts
// (Eq. 1); a Low expert is computed from its low-precision version;
// experts are SwiGLU FFNs (reading R10).  This is the B200 hot path: batch-1
// decode streams 66-352 MB of expert weights per token-layer, so the kernels
// are HBM-bound; their job is to keep ~6 MB of loads in flight while spending
// ~2 or fewer thread-instructions per weight on dequantisation.
//
// Structure:
//  * persistent grid, one 512-thread CTA per SM; work items are 16-row tiles
//    (K2a: of W1 and W3 together; K2b: of W2 x a split-K chunk of F), dealt
//    round-robin over CTAs first so every SM gets the same number of tiles;
//  * each warp streams its tile through a private multi-stage shared-memory
//    ring with cp.async.cg (16 B per lane per row, L1 bypassed, L2
//    evict-first), so ~96 KB per SM are in flight without holding registers;
//    a "group" is 64 bytes of one row, and lane t's 16 bytes of it hold its
//    share of every block of the group;
//  * the dot products run on the tensor cores as mma.sync.m16n8k16 with the
//    weights as A (16 rows x 16 k) and up to 8 token slots as B: dequantised
//    codes are EXACT in fp16 (q-8, q, int8 q), so every per-block partial sum
//    is an fp32 sum of exact products; the block scale is applied in fp32
//    after each 32-element block (acc += d*D_b (+ m*S_b for Q2));
//  * x and h are stored "pair-permuted" (Q_c = (v[8t+c], v[8t+c+4])) so that
//    the B fragment is one 16-byte load per block and lane;
//  * K2b takes h as an fp16 hi/lo pair (h = hi + lo to ~2^-22) and issues two
//    MMAs per k-step, so W2 sees h at ~fp32 precision.
#include <cuda_fp16.h>

#include "hb_internal.h"

namespace hb {

// ------------------------------------------------------------ primitives
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
               :: "r"(dst), "l"(src), "l"(pol));
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

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
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

constexpr int kWarpSmem = 12 * 1024;                    // per-warp cp.async ring
constexpr int kXStage = 24 * 1024;                      // CTA-shared copy of x / h chunk
constexpr int kGemvSmem = kGemvWarps * kWarpSmem + kXStage;   // 216 KB per CTA

// B-operand load: a generic 16-byte load (the source is either the CTA's
// shared-memory stage of x / h or, when it does not fit, global memory).
__device__ __forceinline__ uint4 ldx(const uint4* p) { return *p; }
__device__ __forceinline__ float ldxf(const float* p) { return *p; }

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
    // block j holds r0..3 in word 2j, r4..7 in word 2j+1; q+128 via xor
    const uint32_t a = u4get(v, 2 * blk) ^ 0x80808080u;
    const uint32_t b = u4get(v, 2 * blk + 1) ^ 0x80808080u;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t t = prmt(a, b, (uint32_t)(c | ((4 + c) << 8)));
      P[c] = hsub2u(lop_magic<0x00FF00FFu>(t), kH1152);
    }
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

// One matrix of an expert blob.
struct MatPtr {
  const uint8_t* q;      // codes
  const __half* d;       // scales [N][K/32]
  const __half* m;       // mins   [N][K/32]
};

// Token-slot sources of the B fragment (x or h) for NT 8-slot tiles.
template <int NT, bool SPLIT>
struct XSrc {
  const uint4* b[NT];      // row of slot (tile*8 + g): pair-permuted, uint4 per (block, t)
  const uint4* blo[NT];    // SPLIT: residual part
  const float* s0[NT];     // block sums of slots tile*8 + 2t and +1 (Q2 only)
  const float* s1[NT];
};

// Stream groups [g0, g1) of NMAT matrices (same rows, same K) against the
// slots in X; accumulate acc[m][n][4] (rows g,g+8 x slots 2t,2t+1).
// wsm: shared address of this warp's kWarpSmem-byte ring.
template <int ENC, int NMAT, int NT, bool SPLIT>
__device__ __forceinline__ void mainloop(uint32_t wsm, const MatPtr (&M)[NMAT], int K, int row0,
                                         int g0, int g1, const XSrc<NT, SPLIT>& X,
                                         float (&acc)[NMAT][NT][4]) {
  constexpr int BPG = Enc<ENC>::BPG, SB = Enc<ENC>::SB;
  constexpr int CODE = 16 * 64;                         // 16 rows x 64 B per matrix
  constexpr int SCALE = 16 * SB;
  constexpr int STAGE = NMAT * (CODE + SCALE);
  constexpr int DEPTH = kWarpSmem / STAGE >= 8 ? 8 : kWarpSmem / STAGE;
  static_assert(DEPTH >= 2, "ring too small");
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const size_t rowbytes = ENC == HB_F16 ? (size_t)K * 2 : ENC == HB_Q8 ? (size_t)K
                        : ENC == HB_Q4 ? (size_t)K / 2 : (size_t)K / 4;
  const int nb = K / 32;                                 // blocks (scales) per row
  const uint64_t pol = evict_first_policy();
  // producer: the lane copies rows g and g+8, bytes [16t, 16t+16) of each
  // group (exactly the bytes it consumes); scales: one lane per (row, part).
  const uint8_t* src[NMAT];
#pragma unroll
  for (int m = 0; m < NMAT; ++m) src[m] = M[m].q + (size_t)(row0 + g) * rowbytes + 16 * t;
  const size_t src8 = 8 * rowbytes;
  const int srow = lane & 15;                            // scale row of this lane
  const bool sact = ENC == HB_Q2 ? true : lane < 16;
  const __half* ssrc[NMAT];
#pragma unroll
  for (int m = 0; m < NMAT; ++m) {
    const __half* base = (ENC == HB_Q2 && lane >= 16) ? M[m].m : M[m].d;
    ssrc[m] = base + (size_t)(row0 + srow) * nb;
  }

  auto issue = [&](int grp) {
    if (grp < g1) {
      const uint32_t st = wsm + (grp % DEPTH) * STAGE;
#pragma unroll
      for (int m = 0; m < NMAT; ++m) {
        const uint8_t* s = src[m] + (size_t)grp * 64;
        cp_async16(st + m * CODE + g * 64 + 16 * t, s, pol);
        cp_async16(st + m * CODE + (g + 8) * 64 + 16 * t, s + src8, pol);
        if constexpr (SB > 0) {
          const uint32_t sd = st + NMAT * CODE + m * SCALE;
          if (sact) {
            if constexpr (ENC == HB_Q8) cp_async4(sd + srow * SB, ssrc[m] + grp * BPG);
            else if constexpr (ENC == HB_Q4) cp_async8(sd + srow * SB, ssrc[m] + grp * BPG);
            else cp_async16(sd + srow * SB + (lane >> 4) * 16, ssrc[m] + grp * BPG, pol);
          }
        }
      }
    }
    cp_commit();
  };

#pragma unroll
  for (int s = 0; s < DEPTH - 1; ++s) issue(g0 + s);

  for (int grp = g0; grp < g1; ++grp) {
    __syncwarp();                                  // slot (grp-1)%DEPTH fully consumed
    issue(grp + DEPTH - 1);
    cp_wait<DEPTH - 1>();
    __syncwarp();                                  // everyone's copies of grp visible
    const uint32_t st = wsm + (grp % DEPTH) * STAGE;
    uint4 w[NMAT][2];
#pragma unroll
    for (int m = 0; m < NMAT; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) w[m][h] = lds128(st + m * CODE + (g + 8 * h) * 64 + 16 * t);
#pragma unroll
    for (int blk = 0; blk < BPG; ++blk) {
      const int gblk = grp * BPG + blk;            // block index along K
      uint4 xb[NT], xl[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        xb[n] = ldx(X.b[n] + gblk * 4 + t);
        if constexpr (SPLIT) xl[n] = ldx(X.blo[n] + gblk * 4 + t);
      }
      float s0[NT], s1[NT];
      if constexpr (ENC == HB_Q2) {
#pragma unroll
        for (int n = 0; n < NT; ++n) { s0[n] = ldxf(X.s0[n] + gblk); s1[n] = ldxf(X.s1[n] + gblk); }
      }
#pragma unroll
      for (int m = 0; m < NMAT; ++m) {
        uint32_t Pg[4], Ph[4];
        dequant<ENC>(w[m][0], blk, Pg);
        dequant<ENC>(w[m][1], blk, Ph);
        float dg = 1.f, dh = 1.f, mg = 0.f, mh = 0.f;
        if constexpr (SB > 0) {
          const uint32_t sd = st + NMAT * CODE + m * SCALE;
          dg = lds_half(sd + g * SB + 2 * blk);
          dh = lds_half(sd + (g + 8) * SB + 2 * blk);
          if constexpr (ENC == HB_Q2) {
            mg = lds_half(sd + g * SB + 16 + 2 * blk);
            mh = lds_half(sd + (g + 8) * SB + 16 + 2 * blk);
          }
        }
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          if constexpr (ENC == HB_F16) {
            mma16816(acc[m][n], Pg[0], Ph[0], Pg[1], Ph[1], xb[n].x, xb[n].y);
            mma16816(acc[m][n], Pg[2], Ph[2], Pg[3], Ph[3], xb[n].z, xb[n].w);
            if constexpr (SPLIT) {
              mma16816(acc[m][n], Pg[0], Ph[0], Pg[1], Ph[1], xl[n].x, xl[n].y);
              mma16816(acc[m][n], Pg[2], Ph[2], Pg[3], Ph[3], xl[n].z, xl[n].w);
            }
          } else {
            float D[4] = {0.f, 0.f, 0.f, 0.f};
            mma16816(D, Pg[0], Ph[0], Pg[1], Ph[1], xb[n].x, xb[n].y);
            mma16816(D, Pg[2], Ph[2], Pg[3], Ph[3], xb[n].z, xb[n].w);
            if constexpr (SPLIT) {
              mma16816(D, Pg[0], Ph[0], Pg[1], Ph[1], xl[n].x, xl[n].y);
              mma16816(D, Pg[2], Ph[2], Pg[3], Ph[3], xl[n].z, xl[n].w);
            }
            acc[m][n][0] = fmaf(dg, D[0], acc[m][n][0]);
            acc[m][n][1] = fmaf(dg, D[1], acc[m][n][1]);
            acc[m][n][2] = fmaf(dh, D[2], acc[m][n][2]);
            acc[m][n][3] = fmaf(dh, D[3], acc[m][n][3]);
            if constexpr (ENC == HB_Q2) {               // + m_row * sum_block(x)
              acc[m][n][0] = fmaf(mg, s0[n], acc[m][n][0]);
              acc[m][n][1] = fmaf(mg, s1[n], acc[m][n][1]);
              acc[m][n][2] = fmaf(mh, s0[n], acc[m][n][2]);
              acc[m][n][3] = fmaf(mh, s1[n], acc[m][n][3]);
            }
          }
        }
      }
    }
  }
  cp_wait<0>();
  __syncwarp();
}

// position of element f of a row in the pair-permuted layout (in halves)
__device__ __forceinline__ int perm_pos(int f) {
  const int r8 = f & 31, t = r8 >> 3, r = r8 & 7;
  return (f & ~31) + 8 * t + 2 * (r & 3) + (r >> 2);
}

__device__ __forceinline__ int item_for(int it) {
  // item index of iteration `it` of this warp: CTAs first, then warps, so that
  // consecutive items land on different SMs.
  const int warp = threadIdx.x >> 5;
  return blockIdx.x + gridDim.x * (warp + kGemvWarps * it);
}

extern __shared__ __align__(128) uint8_t gemv_smem[];

__device__ __forceinline__ uint32_t warp_smem() {
  return smem_u32(gemv_smem) + (threadIdx.x >> 5) * kWarpSmem;
}
// the CTA-shared stage of the B operand (after the warps' rings)
__device__ __forceinline__ uint8_t* x_stage() { return gemv_smem + kGemvWarps * kWarpSmem; }

// CTA-wide copy of n16 16-byte words (global -> shared)
__device__ __forceinline__ void stage_copy(uint4* dst, const uint4* src, int n16) {
  for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldcg(src + i);
}

template <int ENC>
__device__ __forceinline__ MatPtr mat_ptr(const GemvParams& p, const Job& j, int mat) {
  const MatLayout& L = p.lay[ENC].mat[mat];
  MatPtr r;
  r.q = j.blob + L.q;
  r.d = reinterpret_cast<const __half*>(j.blob + L.d);
  r.m = reinterpret_cast<const __half*>(j.blob + L.m);
  return r;
}

// ------------------------------------------------------------------ K2a
template <int ENC, int NT>
__device__ __forceinline__ void w13_tile(const GemvParams& p, const Job& j, int row0,
                                         const uint4* xp, const float* xs) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const MatPtr M[2] = {mat_ptr<ENC>(p, j, 0), mat_ptr<ENC>(p, j, 1)};
  const int ngrp = p.H / Enc<ENC>::EPG;
  for (int t0 = 0; t0 < j.n_tok; t0 += 8 * NT) {
    XSrc<NT, false> X;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int sb = j.slot_off + min(t0 + 8 * n + g, j.n_tok - 1);
      const int s0 = j.slot_off + min(t0 + 8 * n + 2 * t, j.n_tok - 1);
      const int s1 = j.slot_off + min(t0 + 8 * n + 2 * t + 1, j.n_tok - 1);
      X.b[n] = xp + (size_t)p.jt.slot_token[sb] * (p.H / 8);
      X.s0[n] = xs + (size_t)p.jt.slot_token[s0] * (p.H / 32);
      X.s1[n] = xs + (size_t)p.jt.slot_token[s1] * (p.H / 32);
    }
    float acc[2][NT][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[m][n][i] = 0.f;
    mainloop<ENC, 2, NT, false>(warp_smem(), M, p.H, row0, 0, ngrp, X, acc);
    // epilogue: h = silu(a) * u, stored as pair-permuted fp16 hi + lo; block sums
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      float hs[2] = {0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int slot_rel = t0 + 8 * n + 2 * t + (i & 1);
        const int f = row0 + g + 8 * (i >> 1);
        const float a = acc[0][n][i], u = acc[1][n][i];
        const float h = a / (1.f + expf(-a)) * u;
        if (slot_rel < j.n_tok) {
          const int slot = j.slot_off + slot_rel;
          const __half hh = __float2half_rn(h);
          const __half hl = __float2half_rn(h - __half2float(hh));
          __half* hi = reinterpret_cast<__half*>(p.h_hi) + (size_t)slot * p.F;
          __half* lo = reinterpret_cast<__half*>(p.h_lo) + (size_t)slot * p.F;
          hi[perm_pos(f)] = hh;
          lo[perm_pos(f)] = hl;
          hs[i & 1] += h;
        }
      }
      // reduce the 16 rows of this tile (lanes with equal t) -> 2 slots per t
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        hs[0] += __shfl_xor_sync(0xffffffffu, hs[0], o);
        hs[1] += __shfl_xor_sync(0xffffffffu, hs[1], o);
      }
      if (g == 0) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int slot_rel = t0 + 8 * n + 2 * t + c;
          if (slot_rel < j.n_tok)
            atomicAdd(p.hsum + (size_t)(j.slot_off + slot_rel) * (p.F / 32) + row0 / 32, hs[c]);
        }
      }
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(kGemvWarps * 32, 1)
w13_kernel(const __grid_constant__ GemvParams p) {
  // zero the W2 split-K partials (consumed by the next kernel)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.partial_n;
       i += (long long)gridDim.x * blockDim.x)
    p.partial[i] = 0.f;
  const int n_jobs = p.jt.hdr[0];
  const int tiles = p.F / 16;
  const int n_items = n_jobs * tiles;
  if (blockIdx.x >= n_items) return;
  // stage x (pair-permuted) and its block sums in shared memory when they fit
  const uint4* xp = p.x_perm;
  const float* xs = p.xsum;
  const int nx16 = p.B * (p.H / 8), ns16 = p.B * (p.H / 32) / 4;
  if ((nx16 + ns16) * 16 <= kXStage) {
    uint4* st = reinterpret_cast<uint4*>(x_stage());
    stage_copy(st, p.x_perm, nx16);
    stage_copy(st + nx16, reinterpret_cast<const uint4*>(p.xsum), ns16);
    __syncthreads();
    xp = st;
    xs = reinterpret_cast<const float*>(st + nx16);
  }
  for (int it = 0;; ++it) {
    const int item = item_for(it);
    if (item >= n_items) break;
    const Job j = p.jt.jobs[item / tiles];
    const int row0 = (item % tiles) * 16;
    switch (j.enc) {
      case HB_F16: w13_tile<HB_F16, NT>(p, j, row0, xp, xs); break;
      case HB_Q8: w13_tile<HB_Q8, NT>(p, j, row0, xp, xs); break;
      case HB_Q4: w13_tile<HB_Q4, NT>(p, j, row0, xp, xs); break;
      default: w13_tile<HB_Q2, NT>(p, j, row0, xp, xs); break;
    }
  }
}

// ------------------------------------------------------------------ K2b
// B-operand view of h for one W2 chunk: element k of slot s is at
// hi[s*stride + k/8 ...] (stride in uint4), sums at sum[s*sstride + k/32].
struct HView {
  const uint4* hi;
  const uint4* lo;
  const float* sum;
  size_t stride, sstride;
};

template <int ENC, int NT>
__device__ __forceinline__ void w2_chunk(const GemvParams& p, const Job& j, int row0, int kbeg,
                                         int kend, int s, const HView& hv) {
  constexpr int EPG = Enc<ENC>::EPG;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const MatPtr M[1] = {mat_ptr<ENC>(p, j, 2)};
  for (int t0 = 0; t0 < j.n_tok; t0 += 8 * NT) {
    XSrc<NT, true> X;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int sb = j.slot_off + min(t0 + 8 * n + g, j.n_tok - 1);
      const int s0 = j.slot_off + min(t0 + 8 * n + 2 * t, j.n_tok - 1);
      const int s1 = j.slot_off + min(t0 + 8 * n + 2 * t + 1, j.n_tok - 1);
      X.b[n] = hv.hi + (size_t)sb * hv.stride;
      X.blo[n] = hv.lo + (size_t)sb * hv.stride;
      X.s0[n] = hv.sum + (size_t)s0 * hv.sstride;
      X.s1[n] = hv.sum + (size_t)s1 * hv.sstride;
    }
    float acc[1][NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[0][n][i] = 0.f;
    mainloop<ENC, 1, NT, true>(warp_smem(), M, p.F, row0, kbeg / EPG, kend / EPG, X, acc);
    // partial[s][token][row] += gate * o   (this warp owns (s, row tile))
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int slot_rel = t0 + 8 * n + 2 * t + (i & 1);
        if (slot_rel < j.n_tok) {
          const int slot = j.slot_off + slot_rel;
          const int tok = p.jt.slot_token[slot];
          const float gate = p.jt.slot_gate[slot];
          float* dst = p.partial + ((size_t)s * p.B + tok) * p.H + row0 + g + 8 * (i >> 1);
          *dst = fmaf(gate, acc[0][n][i], *dst);
        }
      }
  }
}

template <int NT>
__global__ void __launch_bounds__(kGemvWarps * 32, 1)
w2_kernel(const __grid_constant__ GemvParams p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_jobs = p.jt.hdr[0];
  const int n_slots = p.jt.hdr[1];
  const int tiles = p.H / 16;
  // every CTA works on ONE split-K chunk s (so its warps share the h chunk);
  // the row tiles of chunk s are dealt over the CTAs with blockIdx % S == s
  const int s = blockIdx.x % p.S;
  const int nS = (gridDim.x - s + p.S - 1) / p.S;
  const int cidx = blockIdx.x / p.S;
  const int kbeg = s * p.chunk, kend = min(p.F, kbeg + p.chunk);
  if (cidx >= tiles) return;
  // stage the chunk of h (hi, lo, block sums) of every slot when it fits
  HView hv{p.h_hi, p.h_lo, p.hsum, (size_t)p.F / 8, (size_t)p.F / 32};
  const int clen = kend - kbeg;
  const int nh16 = n_slots * (clen / 8), ns16 = n_slots * (clen / 32) / 4;
  if (n_jobs > 0 && (2 * nh16 + ns16) * 16 <= kXStage) {
    uint4* st = reinterpret_cast<uint4*>(x_stage());
    for (int sl = 0; sl < n_slots; ++sl) {
      stage_copy(st + sl * (clen / 8), p.h_hi + (size_t)sl * (p.F / 8) + kbeg / 8, clen / 8);
      stage_copy(st + nh16 + sl * (clen / 8), p.h_lo + (size_t)sl * (p.F / 8) + kbeg / 8, clen / 8);
      stage_copy(st + 2 * nh16 + sl * (clen / 32) / 4,
                 reinterpret_cast<const uint4*>(p.hsum + (size_t)sl * (p.F / 32) + kbeg / 32),
                 (clen / 32) / 4);
    }
    __syncthreads();
    // views indexed by global k: shift the bases back by the chunk start
    hv.hi = st - kbeg / 8;
    hv.lo = st + nh16 - kbeg / 8;
    hv.sum = reinterpret_cast<const float*>(st + 2 * nh16) - kbeg / 32;
    hv.stride = clen / 8;
    hv.sstride = clen / 32;
  }
  for (int it = 0;; ++it) {
    const int tile = cidx + nS * (warp + kGemvWarps * it);
    if (tile >= tiles) break;
    const int row0 = tile * 16;
    for (int jj = 0; jj < n_jobs; ++jj) {
      const Job j = p.jt.jobs[jj];
      switch (j.enc) {
        case HB_F16: w2_chunk<HB_F16, NT>(p, j, row0, kbeg, kend, s, hv); break;
        case HB_Q8: w2_chunk<HB_Q8, NT>(p, j, row0, kbeg, kend, s, hv); break;
        case HB_Q4: w2_chunk<HB_Q4, NT>(p, j, row0, kbeg, kend, s, hv); break;
        default: w2_chunk<HB_Q2, NT>(p, j, row0, kbeg, kend, s, hv); break;
      }
    }
    // the last chunk of this row tile reduces the S partials in order -> y
    __syncwarp();
    __threadfence();
    unsigned prev = 0;
    if (lane == 0) prev = atomicAdd(p.tile_count + tile, 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev == (unsigned)(p.S - 1)) {
      __threadfence();
      for (int e = lane; e < 16 * p.B; e += 32) {
        const int tok = e >> 4, r = row0 + (e & 15);
        float v = 0.f;
        for (int ss = 0; ss < p.S; ++ss)
          v += __ldcg(p.partial + ((size_t)ss * p.B + tok) * p.H + r);
        p.y[(size_t)tok * p.H + r] = v;
      }
      if (lane == 0) p.tile_count[tile] = 0u;
    }
  }
}

template <typename Kern>
static void set_smem(Kern kernel, bool& done) {
  if (!done) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvSmem);
    done = true;
  }
}

void launch_w13(const GemvParams& p, int nt, cudaStream_t s) {
  static bool d1 = false, d2 = false;
  if (nt <= 1) {
    set_smem(w13_kernel<1>, d1);
    w13_kernel<1><<<kNumSM, kGemvWarps * 32, kGemvSmem, s>>>(p);
  } else {
    set_smem(w13_kernel<2>, d2);
    w13_kernel<2><<<kNumSM, kGemvWarps * 32, kGemvSmem, s>>>(p);
  }
}
void launch_w2(const GemvParams& p, int nt, cudaStream_t s) {
  static bool d1 = false, d2 = false;
  if (nt <= 1) {
    set_smem(w2_kernel<1>, d1);
    w2_kernel<1><<<kNumSM, kGemvWarps * 32, kGemvSmem, s>>>(p);
  } else {
    set_smem(w2_kernel<2>, d2);
    w2_kernel<2><<<kNumSM, kGemvWarps * 32, kGemvSmem, s>>>(p);
  }
}

}  // namespace hb
