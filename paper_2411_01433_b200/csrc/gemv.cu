// K2a / K2b: grouped mixed-precision dequant-GEMV of the selected experts.
//
//   K2a  h = silu(W1 x) * (W3 x)          per job (expert, served encoding)
//   K2b  y = sum_jobs gate * (W2 h)        Eq. 1, Skip = no job
//
// Paper: the layer output is the gate-weighted sum of the selected experts
// (Eq. 1); a Low expert is computed from its low-precision version;
// experts are SwiGLU FFNs (reading R10).  This is the B200 hot path: batch-1
// decode streams 66-352 MB of expert weights per token-layer, so the kernels
// are HBM-bound; their job is to keep ~100 KB of loads in flight per SM on
// every SM for the whole kernel while spending few instructions per weight.
//
// Structure:
//  * warp-level STREAM-K.  The work of a launch is a sequence of UNITS, one
//    unit = one 64-byte group of the 16 rows of a row tile (of W1 and W3
//    together for K2a), ordered (virtual job, tile, group).  Every unit moves
//    the same number of weight bytes whatever the encoding, so giving each of
//    the 148 x 16 warps an equal contiguous range of units balances HBM
//    traffic to within one unit.  A warp streams its range as ONE pipeline
//    (no drain at tile boundaries); a tile split between warps leaves
//    "pieces" that the last-arriving warp adds up in warp order
//    (deterministic), then applies the epilogue;
//  * each warp owns a multi-stage shared-memory ring filled with cp.async:
//    its 16 bytes of the two rows g, g+8 of each unit (L1 bypassed, L2
//    evict-first), the block scales, and the B fragments (x or h, at most two
//    token slots at batch 1);
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

#include "hb_internal.h"

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
__device__ __forceinline__ void cp_async16_ef(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
               :: "r"(dst), "l"(src), "l"(pol));
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
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
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

__host__ __device__ constexpr int epg_of(int enc) {
  return enc == HB_F16 ? 32 : enc == HB_Q8 ? 64 : enc == HB_Q4 ? 128 : 256;
}

// Shared memory of a GEMV CTA: kGemvWarps private cp.async rings (weights +
// scales) followed by ONE CTA-wide stage of the B operand (x for K2a, h hi/lo
// for K2b, and their block sums), loaded once per CTA.  Reading B from a
// CTA copy instead of per unit from L2 avoids hammering the same few L2 lines
// from every warp of the GPU (measured: it capped the kernels at ~4.5 TB/s).
template <bool W13> struct KCfg;
template <> struct KCfg<true> {        // K2a: x is small (8 KB per token at H=4096)
  static constexpr int RING = 12 * 1024;
  static constexpr int XSTAGE = 32 * 1024;
};
template <> struct KCfg<false> {       // K2b: h of two slots is 118 KB at F=14336
  static constexpr int RING = 6656;
  static constexpr int XSTAGE = 120 * 1024;
};
template <bool W13>
constexpr int gemv_smem_bytes() { return kGemvWarps * KCfg<W13>::RING + KCfg<W13>::XSTAGE; }

// Ring stage layout of one unit: W codes | S scales
template <int ENC, int NMAT, int RINGB>
struct Ring {
  static constexpr int BPG = Enc<ENC>::BPG, SB = Enc<ENC>::SB;
  static constexpr int W = NMAT * 1024;
  static constexpr int S = NMAT * 16 * SB;
  static constexpr int STAGE = (W + S + 127) / 128 * 128;
  static constexpr int DEPTH = RINGB / STAGE >= 16 ? 16 : RINGB / STAGE;
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

// ---------------------------------------------------------- work space
// Virtual job: one job's token slots [slot0, slot0 + nslot), nslot <= kVSlots.
struct VJob {
  const uint8_t* blob;
  int enc;
  int slot0;
  int nslot;
};

__device__ __forceinline__ int n_vjobs(const GemvParams& p) {
  const int nj = p.jt.hdr[0];
  int nv = 0;
  for (int j = 0; j < nj; ++j) nv += (p.jt.jobs[j].n_tok + kVSlots - 1) / kVSlots;
  return nv;
}
__device__ __forceinline__ VJob get_vjob(const GemvParams& p, int v) {
  const int nj = p.jt.hdr[0];
  for (int j = 0; j < nj; ++j) {
    const Job& J = p.jt.jobs[j];
    const int np = (J.n_tok + kVSlots - 1) / kVSlots;
    if (v < np) {
      VJob r;
      r.blob = J.blob;
      r.enc = J.enc;
      r.slot0 = J.slot_off + v * kVSlots;
      r.nslot = min(kVSlots, J.n_tok - v * kVSlots);
      return r;
    }
    v -= np;
  }
  return VJob{nullptr, 0, 0, 0};
}

// Warp ranges: warp w owns units [b(w), b(w+1)), b(w) = floor(w*U/NW).
struct Space {
  long long U;
  int NW;
  __device__ __forceinline__ long long b(int w) const { return (long long)w * U / NW; }
  __device__ __forceinline__ int owner(long long u) const {
    int w = (int)((u * NW) / U);
    while (w + 1 < NW && b(w + 1) <= u) ++w;
    while (w > 0 && b(w) > u) --w;
    return w;
  }
};

// ------------------------------------------------------------ epilogues
// position of element f of a row in the pair-permuted layout (in halves)
__device__ __forceinline__ int perm_pos(int f) {
  const int r8 = f & 31, t = r8 >> 3, r = r8 & 7;
  return (f & ~31) + 8 * t + 2 * (r & 3) + (r >> 2);
}

// K2a: h = silu(a) * u for rows row0+g(+8), slots 2t, 2t+1 of the vjob
__device__ void finalize13(const GemvParams& p, const VJob& vj, int row0, const float (&acc)[2][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  float hs[2] = {0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int sl = 2 * t + (i & 1);
    const int f = row0 + g + 8 * (i >> 1);
    const float a = acc[0][i], u = acc[1][i];
    const float h = a / (1.f + expf(-a)) * u;
    if (sl < vj.nslot) {
      const int slot = vj.slot0 + sl;
      const __half hh = __float2half_rn(h);
      const __half hl = __float2half_rn(h - __half2float(hh));
      reinterpret_cast<__half*>(p.h_hi)[(size_t)slot * p.F + perm_pos(f)] = hh;
      reinterpret_cast<__half*>(p.h_lo)[(size_t)slot * p.F + perm_pos(f)] = hl;
      hs[i & 1] += h;
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {          // 16 rows of the tile, per slot
    hs[0] += __shfl_xor_sync(0xffffffffu, hs[0], o);
    hs[1] += __shfl_xor_sync(0xffffffffu, hs[1], o);
  }
  if (g == 0) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
      if (2 * t + c < vj.nslot)     // two tiles per 32-row block: fl(fl(0+a)+b) is order-free
        atomicAdd(p.hsum + (size_t)(vj.slot0 + 2 * t + c) * (p.F / 32) + row0 / 32, hs[c]);
  }
}

// K2b: o -> ob[slot][rows] of a finished (job, H tile)
__device__ void store_ob(const GemvParams& p, const VJob& vj, int tile, const float (&acc)[1][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int row0 = tile * 16;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int sl = 2 * t + (i & 1);
    if (sl < vj.nslot)
      p.ob[(size_t)(vj.slot0 + sl) * p.H + row0 + g + 8 * (i >> 1)] = acc[0][i];
  }
}

// after a fence: count this job as done for H tile `tile`; the last job of the
// tile writes y = Eq. 1 in fixed (token, rank) order
__device__ void publish_y(const GemvParams& p, int tile, int nv) {
  const int lane = threadIdx.x & 31;
  const int row0 = tile * 16;
  unsigned prev = 0;
  if (lane == 0) prev = atomicAdd(p.cnty + tile, 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != (unsigned)(nv - 1)) return;
  __threadfence();
  for (int e = lane; e < 16 * p.B; e += 32) {            // Eq. 1, ranks in order
    const int tok = e >> 4, r = row0 + (e & 15);
    float v = 0.f;
    for (int i = 0; i < p.k; ++i) {
      const int s = p.jt.tok_slots[tok * p.k + i];
      if (s >= 0) v = fmaf(p.jt.slot_gate[s], __ldcg(p.ob + (size_t)s * p.H + r), v);
    }
    p.y[(size_t)tok * p.H + r] = v;
  }
  if (lane == 0) p.cnty[tile] = 0u;
}

struct Pend {
  int tile;
  int kind;          // 0 partial piece stored in part[], 1 finished W2 tile (ob stored)
};
constexpr int kMaxPend = 4;

// ------------------------------------------------------------ the run
// Stream units [a, b) of virtual job v (unit l = tile * G + grp) through the
// warp's ring.  W13: K2a (W1 and W3 rows, x); else K2b (W2 rows, h hi/lo).
// XR: the B operand of every slot is in the CTA stage at shared address xst
// (W13: x_perm [B][H/8] uint4 | xsum [B][H/32]; W2: h_hi [S][F/8] | h_lo
// [S][F/8] | hsum [S][F/32]); otherwise it is read from global memory.
template <int ENC, bool W13, bool XR>
__device__ void run(const GemvParams& p, const VJob& vj, int v, int nv, long long cum,
                    long long a, long long b, const Space& sp, int gw, uint32_t ring,
                    uint32_t xst, int nrows_x) {
  constexpr int NMAT = W13 ? 2 : 1;
  constexpr bool SPLIT = !W13;
  constexpr int XS = SPLIT ? 2 : 1;
  using R = Ring<ENC, NMAT, KCfg<W13>::RING>;
  constexpr int BPG = R::BPG, SB = R::SB, DEPTH = R::DEPTH;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int K = W13 ? p.H : p.F;
  const int G = K / Enc<ENC>::EPG;
  const int nb = K / 32;
  const size_t rowbytes = ENC == HB_F16 ? (size_t)K * 2 : ENC == HB_Q8 ? (size_t)K
                        : ENC == HB_Q4 ? (size_t)K / 2 : (size_t)K / 4;
  const uint64_t pol = evict_first_policy();
  // matrices
  // tile-major blobs: unit l (tile l/G, group l%G) = 1 KB of codes at q + 1024*l,
  // its 16 scale records at s + 16*SB*l -- a warp's range is one contiguous span
  const uint8_t* qp[NMAT];
  const uint8_t* sp_[NMAT];
#pragma unroll
  for (int m = 0; m < NMAT; ++m) {
    const MatLayout& L = p.lay[ENC].mat[W13 ? m : 2];
    qp[m] = vj.blob + L.q + (size_t)a * 1024 + 16 * lane;
    sp_[m] = vj.blob + L.s + (size_t)a * 16 * SB + 16 * lane;
  }
  (void)rowbytes;
  (void)nb;
  const bool s_act = lane < SB;               // 16*SB bytes of scales per unit = SB lanes x 16 B
  const int ns = vj.nslot;
  // B-operand source of slot s (x or h hi/lo) and of its block sums
  auto xsrc_of = [&](int part, int s) -> const uint4* {
    const int sl = vj.slot0 + min(s, ns - 1);
    if constexpr (W13) return p.x_perm + (size_t)p.jt.slot_token[sl] * (p.H / 8);
    else return (part ? p.h_lo : p.h_hi) + (size_t)sl * (p.F / 8);
  };
  auto zsrc_of = [&](int s) -> const float* {
    const int sl = vj.slot0 + min(s, ns - 1);
    if constexpr (W13) return p.xsum + (size_t)p.jt.slot_token[sl] * (p.H / 32);
    else return p.hsum + (size_t)sl * (p.F / 32);
  };

  // ---- producer: weights + scales only (B operand is in the CTA stage)
  long long pl = a;
  int pslot = 0;
  auto issue = [&]() {
    if (pl < b) {
      const uint32_t st = ring + pslot * R::STAGE;
#pragma unroll
      for (int m = 0; m < NMAT; ++m) {                 // 2 x 512 contiguous bytes
        cp_async16_ef(st + m * 1024 + 16 * lane, qp[m], pol);
        cp_async16_ef(st + m * 1024 + 512 + 16 * lane, qp[m] + 512, pol);
        if constexpr (SB > 0)
          if (s_act) cp_async16_ef(st + R::W + m * 16 * SB + 16 * lane, sp_[m], pol);
      }
      ++pl;
#pragma unroll
      for (int m = 0; m < NMAT; ++m) { qp[m] += 1024; sp_[m] += 16 * SB; }
      if (++pslot == DEPTH) pslot = 0;
    }
    cp_commit();
  };

#pragma unroll 1
  for (int s = 0; s < DEPTH - 1; ++s) issue();

  float acc[NMAT][4];
#pragma unroll
  for (int m = 0; m < NMAT; ++m)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;
  int c_tile = (int)(a / G), c_grp = (int)(a % G), piece0 = c_grp;
  int cslot = 0;
  const int xg = min(g, ns - 1), z0 = min(2 * t, ns - 1), z1 = min(2 * t + 1, ns - 1);
  // deferred publications: partial pieces (kind 0) and finished W2 tiles (kind 1)
  Pend pend[kMaxPend];
  int npend = 0;
  auto publish = [&](const Pend* pd, int n) {
    if (n == 0) return;
    __syncwarp();
    __threadfence();
    int ytile[kMaxPend];
    int ny = 0;
    for (int i = 0; i < n; ++i) {
      const int tile = pd[i].tile;
      if (pd[i].kind == 1) { ytile[ny++] = tile; continue; }
      const long long gu0 = cum + (long long)tile * G, gu1 = gu0 + G;
      const int wa = sp.owner(gu0), wb = sp.owner(gu1 - 1);
      unsigned* cnt = (W13 ? p.cnt13 + (size_t)v * (p.F / 16) : p.cnt2 + (size_t)v * (p.H / 16)) + tile;
      unsigned prev = 0;
      if (lane == 0) prev = atomicAdd(cnt, 1u);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev != (unsigned)(wb - wa)) continue;
      // last piece of the tile: add all pieces in warp order (deterministic)
      __threadfence();
      float sum[NMAT][4];
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q) sum[m][q] = 0.f;
      for (int w2 = wa; w2 <= wb; ++w2) {
        const int ks = sp.b(w2) >= gu0 ? 0 : 1;
        const float* src = p.part + (((size_t)w2 * 2 + ks) * 32 + lane) * kPartFloats;
#pragma unroll
        for (int m = 0; m < NMAT; ++m) {
          const float4 q = __ldcg(reinterpret_cast<const float4*>(src + 4 * m));
          sum[m][0] += q.x; sum[m][1] += q.y; sum[m][2] += q.z; sum[m][3] += q.w;
        }
      }
      if (lane == 0) *cnt = 0u;
      if constexpr (W13) {
        finalize13(p, vj, tile * 16, sum);
      } else {
        store_ob(p, vj, tile, sum);
        ytile[ny++] = tile;
      }
    }
    if (ny) {
      __syncwarp();
      __threadfence();
      for (int i = 0; i < ny; ++i) publish_y(p, ytile[i], nv);
    }
  };
  // B-operand sources: rows (token for x, slot for h) of the lane's fragment slots
  auto row_of = [&](int s) -> int {
    const int sl = vj.slot0 + min(s, ns - 1);
    return W13 ? p.jt.slot_token[sl] : sl;
  };
  const uint4* gx0 = XR ? nullptr : xsrc_of(0, xg);
  const uint4* gx1 = XR ? nullptr : xsrc_of(XS - 1, xg);
  const float* gz0 = XR ? nullptr : zsrc_of(z0);
  const float* gz1 = XR ? nullptr : zsrc_of(z1);
  // stage addresses (XR): part p of row r at xst + (p*nrows + r)*K*2, sums after
  const uint32_t sxb = xst + (uint32_t)row_of(xg) * K * 2 + t * 16;
  const uint32_t sxl = sxb + (uint32_t)nrows_x * K * 2;
  const uint32_t szb = xst + (uint32_t)XS * nrows_x * K * 2;
  const uint32_t sz0 = szb + (uint32_t)row_of(z0) * (K / 32) * 4;
  const uint32_t sz1 = szb + (uint32_t)row_of(z1) * (K / 32) * 4;

  for (long long l = a; l < b; ++l) {
    __syncwarp();                                  // slot being refilled is consumed
    issue();
    cp_wait<DEPTH - 1>();
    __syncwarp();                                  // everyone's copies of unit l visible
    const uint32_t st = ring + cslot * R::STAGE;
    if (++cslot == DEPTH) cslot = 0;
    uint4 w[NMAT][2];
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      w[m][0] = lds128(st + m * 1024 + g * 64 + 16 * t);
      w[m][1] = lds128(st + m * 1024 + (g + 8) * 64 + 16 * t);
    }
#ifdef HB_DBG_NOCOMPUTE
    acc[0][0] += __uint_as_float((w[0][0].x ^ w[0][1].y) & 0x3F800000u);
    if (false)
#endif
#pragma unroll
    for (int blk = 0; blk < BPG; ++blk) {
      uint4 xb, xl;
      float s0 = 0.f, s1 = 0.f;
      if constexpr (XR) {
        const uint32_t gb = (uint32_t)(c_grp * BPG + blk);
        xb = lds128(sxb + gb * 64);
        if constexpr (SPLIT) xl = lds128(sxl + gb * 64);
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
          mma16816(acc[m], Pg[0], Ph[0], Pg[1], Ph[1], xb.x, xb.y);
          mma16816(acc[m], Pg[2], Ph[2], Pg[3], Ph[3], xb.z, xb.w);
          if constexpr (SPLIT) {
            mma16816(acc[m], Pg[0], Ph[0], Pg[1], Ph[1], xl.x, xl.y);
            mma16816(acc[m], Pg[2], Ph[2], Pg[3], Ph[3], xl.z, xl.w);
          }
        } else {
          const uint32_t sd = st + R::W + m * 16 * SB;
          const float dg = lds_half(sd + g * SB + 2 * blk);
          const float dh = lds_half(sd + (g + 8) * SB + 2 * blk);
          float D[4] = {0.f, 0.f, 0.f, 0.f};
          mma16816(D, Pg[0], Ph[0], Pg[1], Ph[1], xb.x, xb.y);
          mma16816(D, Pg[2], Ph[2], Pg[3], Ph[3], xb.z, xb.w);
          if constexpr (SPLIT) {
            mma16816(D, Pg[0], Ph[0], Pg[1], Ph[1], xl.x, xl.y);
            mma16816(D, Pg[2], Ph[2], Pg[3], Ph[3], xl.z, xl.w);
          }
          acc[m][0] = fmaf(dg, D[0], acc[m][0]);
          acc[m][1] = fmaf(dg, D[1], acc[m][1]);
          acc[m][2] = fmaf(dh, D[2], acc[m][2]);
          acc[m][3] = fmaf(dh, D[3], acc[m][3]);
          if constexpr (ENC == HB_Q2) {               // + m_row * sum_block(x)
            const float mg = lds_half(sd + g * SB + 16 + 2 * blk);
            const float mh = lds_half(sd + (g + 8) * SB + 16 + 2 * blk);
            acc[m][0] = fmaf(mg, s0, acc[m][0]);
            acc[m][1] = fmaf(mg, s1, acc[m][1]);
            acc[m][2] = fmaf(mh, s0, acc[m][2]);
            acc[m][3] = fmaf(mh, s1, acc[m][3]);
          }
        }
      }
    }
    // ---- end of a tile piece?  (anything that needs a fence is deferred to the
    // end of the run, so the cp.async pipeline never drains mid-stream)
#ifdef HB_DBG_NOEPI
    if (false) {
#else
    if (c_grp == G - 1 || l == b - 1) {
#endif
      if (npend == kMaxPend) {                 // cannot happen at production sizes
        cp_wait<0>();
        publish(pend, npend);
        npend = 0;
      }
      if (piece0 == 0 && c_grp == G - 1) {
        if constexpr (W13) {
          finalize13(p, vj, c_tile * 16, acc);
        } else {
          store_ob(p, vj, c_tile, acc);
          pend[npend++] = Pend{c_tile, 1};
        }
      } else {
        // partial piece: store it; counting / combining happens in publish()
        const long long gu0 = cum + (long long)c_tile * G;
        const int pslot_k = sp.b(gw) >= gu0 ? 0 : 1;
        float* dst = p.part + (((size_t)gw * 2 + pslot_k) * 32 + lane) * kPartFloats;
#pragma unroll
        for (int m = 0; m < NMAT; ++m)
          *reinterpret_cast<float4*>(dst + 4 * m) = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
        pend[npend++] = Pend{c_tile, 0};
      }
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;
      piece0 = 0;
    }
    if (++c_grp == G) { c_grp = 0; ++c_tile; }
  }
  cp_wait<0>();
  __syncwarp();
  HB_TL(W13, gw, 2);
  publish(pend, npend);
  HB_TL(W13, gw, 3);
}

extern __shared__ __align__(128) uint8_t gemv_smem[];

template <bool W13>
__global__ void __launch_bounds__(kGemvWarps * 32, 1)
gemv_kernel(const __grid_constant__ GemvParams p) {
  const int warp = threadIdx.x >> 5;
#ifdef HB_DBG_TIMELINE
  HB_TL(W13, warp * gridDim.x + blockIdx.x, 0);
#endif
  const int nv = n_vjobs(p);
  if (!W13 && nv == 0) {                                     // nothing owned: y = 0
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)p.B * p.H;
         i += (long long)gridDim.x * blockDim.x)
      p.y[i] = 0.f;
    return;
  }
  const int T = W13 ? p.F / 16 : p.H / 16;
  const int K = W13 ? p.H : p.F;
  constexpr int XS = W13 ? 1 : 2;
  // ---- CTA stage of the B operand (all rows: tokens for x, slots for h)
  const uint32_t xst = smem_u32(gemv_smem) + kGemvWarps * KCfg<W13>::RING;
  const int nrows = W13 ? p.B : p.jt.hdr[1];
  const size_t stage_bytes = (size_t)nrows * (XS * K * 2 + (K / 32) * 4);
  const bool xr = stage_bytes <= (size_t)KCfg<W13>::XSTAGE;
  if (xr) {
    uint4* dst = reinterpret_cast<uint4*>(gemv_smem + kGemvWarps * KCfg<W13>::RING);
    const int n16 = nrows * (K / 8);                          // one part, all rows
    const uint4* src0 = W13 ? p.x_perm : p.h_hi;
    for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldcg(src0 + i);
    if (!W13)
      for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[n16 + i] = __ldcg(p.h_lo + i);
    const uint4* zs = reinterpret_cast<const uint4*>(W13 ? p.xsum : p.hsum);
    const int nz16 = nrows * (K / 32) / 4;
    for (int i = threadIdx.x; i < nz16; i += blockDim.x) dst[XS * n16 + i] = __ldcg(zs + i);
  }
  __syncthreads();
  HB_TL(W13, warp * gridDim.x + blockIdx.x, 1);
  long long U = 0;
  for (int v = 0; v < nv; ++v) U += (long long)T * (K / epg_of(get_vjob(p, v).enc));
  // at most U warps take part, so every participating warp owns >= 1 unit
  Space sp{U, (int)min((long long)gridDim.x * kGemvWarps, U)};
  // warp ranges are dealt SM-interleaved: consecutive ranges (same job, same
  // encoding) land on different SMs, so every SM gets the same mix of
  // fp16 (HBM-heavy) and low-bit (ALU-heavy) units
  const int gw = warp * gridDim.x + blockIdx.x;
  if (gw >= sp.NW) return;
  const long long u0 = sp.b(gw), u1 = sp.b(gw + 1);
  const uint32_t ring = smem_u32(gemv_smem) + warp * KCfg<W13>::RING;
  long long cum = 0;
  int v = 0;
  for (; v < nv; ++v) {                                       // vjob containing u0
    const long long Uv = (long long)T * (K / epg_of(get_vjob(p, v).enc));
    if (u0 < cum + Uv) break;
    cum += Uv;
  }
  long long u = u0;
  while (u < u1 && v < nv) {
    const VJob vj = get_vjob(p, v);
    const long long Uv = (long long)T * (K / epg_of(vj.enc));
    const long long a = u - cum, b = min(u1, cum + Uv) - cum;
#define HB_RUN(E, X) run<E, W13, X>(p, vj, v, nv, cum, a, b, sp, gw, ring, xst, nrows)
    switch (vj.enc * 2 + (xr ? 1 : 0)) {
      case 2 * HB_F16 + 1: HB_RUN(HB_F16, true); break;
      case 2 * HB_F16 + 0: HB_RUN(HB_F16, false); break;
      case 2 * HB_Q8 + 1: HB_RUN(HB_Q8, true); break;
      case 2 * HB_Q8 + 0: HB_RUN(HB_Q8, false); break;
      case 2 * HB_Q4 + 1: HB_RUN(HB_Q4, true); break;
      case 2 * HB_Q4 + 0: HB_RUN(HB_Q4, false); break;
      case 2 * HB_Q2 + 1: HB_RUN(HB_Q2, true); break;
      default: HB_RUN(HB_Q2, false); break;
    }
#undef HB_RUN
    u = cum + b;
    cum += Uv;
    ++v;
  }
}

template <typename Kern>
static void set_smem(Kern kernel, int bytes, bool& done) {
  if (!done) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done = true;
  }
}

void launch_w13(const GemvParams& p, cudaStream_t s) {
  static bool d = false;
  constexpr int smem = gemv_smem_bytes<true>();
  set_smem(gemv_kernel<true>, smem, d);
  gemv_kernel<true><<<kGemvCTAs, kGemvWarps * 32, smem, s>>>(p);
}
void launch_w2(const GemvParams& p, cudaStream_t s) {
  static bool d = false;
  constexpr int smem = gemv_smem_bytes<false>();
  set_smem(gemv_kernel<false>, smem, d);
  gemv_kernel<false><<<kGemvCTAs, kGemvWarps * 32, smem, s>>>(p);
}

}  // namespace hb

#ifdef HB_DBG_TIMELINE
extern "C" int hb_debug_timeline(void* host, int which) {
  return (int)cudaMemcpyFromSymbol(host, hb::g_tl, sizeof(hb::g_tl[0]),
                                   (size_t)which * sizeof(hb::g_tl[0]));
}
#endif
