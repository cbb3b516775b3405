// K3: batched-decode / prefill expert FFN as a grouped
// mixed-precision GEMM on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Eq. 1 for a batch: for every (expert, served encoding) job the
// tokens routed to it form the N side of two GEMMs,
//     K3a:  a = W1 X^T, u = W3 X^T  -> h = silu(a) * u        (SwiGLU epilogue)
//     K3b:  o = W2 h^T              -> y[token] += g * o       (Eq. 1 epilogue)
// P:820 / P:1018: the paper runs batch 1 only and notes that prefill touches
// nearly every expert; at B >= 32 tokens per layer the per-expert token count
// M_e = B*k/E makes these real dense contractions.
//
// Design ("K3"):
//  * vjob3 = <= 128 tokens of one job (F16: <= 256; MMA N = np = round-up-16 of the count).
//    k3_prep (one launch) builds the vjob3 table from the router's job table
//    and gathers X of every vjob3 into xg in the UMMA canonical K-major layout
//    (8x8 core matrices, 16-byte rows), so each K3a stage gets X with ONE bulk
//    copy; K3a's epilogue writes h straight into the same layout for K3b.
//  * Item = (vjob3, 128-row weight tile[, K split]); persistent grid, one CTA
//    per SM, items dealt round-robin.  Warp roles:
//      warp 13  producer: TMA bulk copies (cp.async.bulk) of the raw units of
//               the tile (codes + scales, our tile-major blob layout) into a
//               3-slot raw ring (mbarrier complete_tx);
//      warps 0-7 converters: raw units -> fp16 canonical A tiles (F16 is a
//               relayout, Q8/Q4/Q2 dequantise with half2 magic numbers) in a
//               2-slot canonical ring; thread 0 also bulk-copies the B tile;
//      warp 12  MMA issuer: one thread issues tcgen05.mma.kind::f16 (M=128,
//               N=np, K=16) into a TMEM accumulator, tcgen05.commit frees the
//               canonical slot / signals the epilogue;
//      warps 8-11 epilogue: tcgen05.ld the accumulator (warp w%4 owns TMEM
//               lanes 32(w%4)..+31 = tile rows), SwiGLU -> h (K3a) or
//               g-weighted red.add into y (K3b).  Two TMEM accumulator buffers
//               let the epilogue of item i overlap the main loop of item i+1.
//  * Weights are dequantised to fp16 (one rounding of d*q, d*q+m) because the
//    tensor core accumulates across blocks; h is rounded to fp16 for K3b
//    (R26).  Accumulation is fp32 in TMEM.
#include <type_traits>

#include "hb_internal.h"
#include "k3.h"

namespace hb {

namespace {

constexpr int kRows = 128;                 // weight rows per tile = MMA M
constexpr int kBK = 64;                    // K elements per canonical stage
constexpr int kRawSlots = 4;
constexpr int kCanSlots = 3;
constexpr int kMaxBSlots = 12;
constexpr int kConvWarps = 16;             // warps 0..15 dequantise (all on one step)
constexpr int kConvThreads = kConvWarps * 32;
constexpr int kEpiWarp0 = kConvWarps;      // 4 epilogue warps (warp % 4 = TMEM lane quarter)
constexpr int kMmaWarp = kConvWarps + 4;
constexpr int kProdWarp = kConvWarps + 5;  // raw codes + scales
constexpr int kBProdWarp = kConvWarps + 6; // B tiles
constexpr int kThreads = (kConvWarps + 7) * 32;
constexpr int kRawCode = 16384;            // NMAT x 8 tiles x ru units of 1 KB
constexpr int kRawScale = 8192;
constexpr int kRawBytes = kRawCode + kRawScale;
constexpr int kAMat = kRows * kBK * 2;     // 16 KB fp16 A tile per matrix
constexpr int kABytes = 2 * kAMat;
constexpr int kBBytes = kK3MaxN * kBK * 2; // 16 KB: largest B tile (np = 128)
constexpr int kBRing = 32768;
constexpr int kBarOff = kRawSlots * kRawBytes + kCanSlots * kABytes + kBRing;
constexpr int kSmem = kBarOff + 512 + 1024;   // + alignment slack (swizzle atoms: 1 KB)
// TS variant (K3Params::ts): no fp16 A stages in shared memory -- the
// converters dequantise into TMEM (columns 256..511: 4 two-matrix or 8
// one-matrix stages of 64 K) and the MMA reads A from there, so the raw ring
// gets the shared memory the A stages held
// (measured: 5/6/7 raw slots, 32-80 KB of B tiles, 4-6 A stages and one or
// two accumulator buffers all within 1 %; the A stage in TMEM is the gain)
constexpr int kRawSlotsTS = 7;
constexpr int kBRingTS = 56 * 1024;            // B tiles in flight (np = 64: 7 slots)
constexpr int kBarOffTS = kRawSlotsTS * kRawBytes + kBRingTS;
constexpr int kSmemTS = kBarOffTS + 1024 + 1024;   // barriers: up to 66 x 8 B

#ifdef HB_K3_TRACE
// diagnostic timeline (tools/k3_trace.py): CTA 0 stamps %globaltimer per event
__device__ unsigned long long g_k3_trace[4][4096];
__device__ __forceinline__ void k3_stamp(int ch, int i) {
  if (blockIdx.x == 0 && i < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k3_trace[ch][i] = t;
  }
}
#define K3_STAMP(ch, i) k3_stamp(ch, i)
#else
#define K3_STAMP(ch, i)
#endif
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint32_t b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(b), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(b) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_add_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" :: "r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
        : "=r"(done) : "r"(b), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma4(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3,
                                     uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];"
      :: "r"(dst), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const void* tmap, int c0, int c1, int c2,
                                     uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(dst), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// K-major, no swizzle: 8x(16 B) core matrices; K-adjacent core matrices 128 B
// apart (LBO), 8-row groups 1024 B apart (SBO); version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46);
}
// K-major SWIZZLE_64B: LBO field 1 (unused), SBO = 8 rows x 64 B = 512 B
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) |
         ((uint64_t)(512 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

// kind::f16 instruction descriptor: D f32, A/B f16, both K-major, N, M=128
__device__ __forceinline__ uint32_t idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                     uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
      :: "r"(tmem_d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
}
// A from TMEM (K-major: lane = row, column c holds K elements 2c, 2c + 1)
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bd, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
      :: "r"(tmem_d), "r"(tmem_a), "l"(bd), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
               :: "r"(taddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t and_or(uint32_t x, uint32_t m, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(x), "r"(m), "r"(c));   // (a & b) | c
  return r;
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint16_t lds16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ __half2 bcast(uint16_t h) {
  return u2h((uint32_t)h | ((uint32_t)h << 16));
}


// Q4 K chunks are consumed in the pair-permuted K order (0 4 1 5 2 6 3 7)
// within each 8-element chunk; the B operand of Q4 vjob3 (X gather, K3a's h
// epilogue) is stored in the same order, so the dot products are unchanged.
// Nibble r = element r: (e0, e4) and (e2, e6) are the low nibbles of the
// half-words of v and v >> 8, (e1, e5) and (e3, e7) the high ones (x16).
__device__ __forceinline__ uint4 q4_chunk_perm(uint32_t v, __half2 d) {
  const uint32_t v8 = v >> 8;
  const __half2 off = u2h(0x64086408u), inv16 = u2h(0x2C002C00u), m72 = u2h(0xD480D480u);
  uint4 o;
  o.x = h2u(__hmul2(__hsub2(u2h(and_or(v, 0x000F000Fu, 0x64006400u)), off), d));
  o.y = h2u(__hmul2(__hfma2(u2h(and_or(v, 0x00F000F0u, 0x64006400u)), inv16, m72), d));
  o.z = h2u(__hmul2(__hsub2(u2h(and_or(v8, 0x000F000Fu, 0x64006400u)), off), d));
  o.w = h2u(__hmul2(__hfma2(u2h(and_or(v8, 0x00F000F0u, 0x64006400u)), inv16, m72), d));
  return o;
}
// position of element j (0..7) of a chunk in that order
__device__ __forceinline__ int q4_perm_pos(int j) { return ((j & 3) << 1) | (j >> 2); }
__device__ __forceinline__ uint4 q8_chunk(uint32_t a, uint32_t b, __half2 d) {
  a ^= 0x80808080u;
  b ^= 0x80808080u;
  const uint32_t M = 0x64646464u;
  const __half2 off = u2h(0x64806480u);                    // (1152, 1152)
  uint4 o;
  o.x = h2u(__hmul2(__hsub2(u2h(prmt(a, M, 0x5150)), off), d));
  o.y = h2u(__hmul2(__hsub2(u2h(prmt(a, M, 0x5352)), off), d));
  o.z = h2u(__hmul2(__hsub2(u2h(prmt(b, M, 0x5150)), off), d));
  o.w = h2u(__hmul2(__hsub2(u2h(prmt(b, M, 0x5352)), off), d));
  return o;
}
// c0 = [byte(q0..3), 0, byte(q0..3), 0], c1 likewise for q4..7
__device__ __forceinline__ uint4 q2_chunk(uint32_t c0, uint32_t c1, __half2 d, __half2 m) {
  const __half2 n01 = u2h(0x34003C00u), b01 = u2h(0xDC00E400u);  // (1, 1/4), (-1024, -256)
  const __half2 n23 = u2h(0x24002C00u), b23 = u2h(0xCC00D400u);  // (1/16, 1/64), (-64, -16)
  uint4 o;
  o.x = h2u(__hfma2(__hfma2(u2h(and_or(c0, 0x000C0003u, 0x64006400u)), n01, b01), d, m));
  o.y = h2u(__hfma2(__hfma2(u2h(and_or(c0, 0x00C00030u, 0x64006400u)), n23, b23), d, m));
  o.z = h2u(__hfma2(__hfma2(u2h(and_or(c1, 0x000C0003u, 0x64006400u)), n01, b01), d, m));
  o.w = h2u(__hfma2(__hfma2(u2h(and_or(c1, 0x00C00030u, 0x64006400u)), n23, b23), d, m));
  return o;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
// Two consecutive 8-element K chunks (blocks j0, j0 + 1, same 8-element
// position t) of one row: code/sc point at this step's bytes of the row.
__device__ __forceinline__ void dequant16(int enc, uint32_t code, uint32_t sc, uint4& w0, uint4& w1) {
  const uint32_t dd = lds32(sc);                           // d[j0] | d[j0 + 1] << 16
  const __half2 d0 = u2h(prmt(dd, 0, 0x1010)), d1 = u2h(prmt(dd, 0, 0x3232));
  if (enc == HB_Q4) {
    const uint2 v = lds64(code);
    w0 = q4_chunk_perm(v.x, d0);
    w1 = q4_chunk_perm(v.y, d1);
  } else if (enc == HB_Q8) {
    const uint4 v = lds128(code);
    w0 = q8_chunk(v.x, v.y, d0);
    w1 = q8_chunk(v.z, v.w, d1);
  } else {
    const uint32_t mm = lds32(sc + 16);
    const __half2 m0 = u2h(prmt(mm, 0, 0x1010)), m1 = u2h(prmt(mm, 0, 0x3232));
    const uint32_t v = lds32(code);
    w0 = q2_chunk(prmt(v, 0, 0x4040), prmt(v, 0, 0x4242), d0, m0);
    w1 = q2_chunk(prmt(v, 0, 0x4141), prmt(v, 0, 0x4343), d1, m1);
  }
}

__device__ __forceinline__ int scale_rec(int enc) {   // SB, bytes per (unit, row)
  return enc == HB_Q8 ? 4 : enc == HB_Q4 ? 8 : enc == HB_Q2 ? 32 : 0;
}
// HB_Q2K (R32) in the Q2 slot: Q2's codes, 20-byte records
// [d, dmin, sc16]; chunk t of blocks j0, j0 + 1 lies in sub-blocks
// 2 j + t / 2.  w = q (d sc_lo) - dmin sc_hi with both scales rounded once
// to fp16 (R34), then the one fp16 fma of q2_chunk.
__device__ __forceinline__ void dequant16_q2k(uint32_t code, uint32_t rec, int j0, int t, uint4& w0,
                                              uint4& w1) {
  const float d = __half2float(__ushort_as_half(lds16(rec)));
  const float dm = __half2float(__ushort_as_half(lds16(rec + 2)));
  const uint32_t c0 = lds8(rec + 4 + 2 * j0 + (t >> 1));
  const uint32_t c1 = lds8(rec + 4 + 2 * j0 + 2 + (t >> 1));
  const __half2 d0 = __float2half2_rn(d * (float)(c0 & 15u)), m0 = __float2half2_rn(-dm * (float)(c0 >> 4));
  const __half2 d1 = __float2half2_rn(d * (float)(c1 & 15u)), m1 = __float2half2_rn(-dm * (float)(c1 >> 4));
  const uint32_t v = lds32(code);
  w0 = q2_chunk(prmt(v, 0, 0x4040), prmt(v, 0, 0x4242), d0, m0);
  w1 = q2_chunk(prmt(v, 0, 0x4141), prmt(v, 0, 0x4343), d1, m1);
}
// raw units per (matrix, 16-row tile) in one raw slot: 16 KB of codes per slot
template <int NMAT>
__device__ __forceinline__ int raw_units(int enc, int kitem) {
  return NMAT == 2 ? 1 : (kitem % (2 * epg_of_enc(enc)) == 0 ? 2 : 1);
}

struct Item {
  const V3* v;
  int tile;      // 128-row tile of the weight matrix
  int ks;        // K split index (K3b)
};

template <int NMAT>
__device__ __forceinline__ Item item_of(const K3Params& p, int it, int v0) {
  Item r;
  if (NMAT == 2) {
    const int tpv = p.F / kRows;
    r.v = p.tab->v + v0 + it / tpv;
    r.tile = it % tpv;
    r.ks = 0;
  } else {
    const int tpv = (p.H / kRows) * p.ks;
    r.v = p.tab->v + v0 + it / tpv;
    r.tile = (it % tpv) / p.ks;
    r.ks = (it % tpv) % p.ks;
  }
  return r;
}

// Epilogue of one item: warp quarter q4 holds TMEM lanes (= tile rows)
// 32*q4 .. +31.  K3a: h = silu(a) * u to hB (K3b's canonical B layout);
// K3b: y[token] += g * o (Eq. 1) with fp32 reductions.
template <int NMAT>
__device__ __forceinline__ void epilogue_item(const K3Params& p, const Item& I, uint32_t tacc,
                                              int q4, int lane, int ms = 128) {
  const int np = I.v->np, n_real = I.v->n;
  const int row = I.tile * kRows + q4 * 32 + lane;   // weight row of this thread
  for (int n0 = 0; n0 < np; n0 += 16) {
    if (NMAT == 2) {
      float a[16], uu[16];
      tmem_ld16(tacc + n0, a);
      tmem_ld16(tacc + ms + n0, uu);
      // h (fp16) into hB in K3b's canonical B layout: K index = row (of F)
      const int j = I.v->enc == HB_Q4 ? q4_perm_pos(row & 7) : (row & 7);
      __half* hb = p.hB + I.v->hoff + (size_t)(row >> 6) * np * kBK +
                   ((row & 63) >> 3) * 64 + j;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int n = n0 + i;
        const float s = a[i] / (1.0f + __expf(-a[i]));
        const float hv = n < n_real ? s * uu[i] : 0.0f;
        hb[(n >> 3) * 512 + (n & 7) * 8] = __float2half_rn(hv);
      }
    } else {
      float o[16];
      tmem_ld16(tacc + n0, o);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int n = n0 + i;
        if (n < n_real) {
          const int slot = I.v->slot0 + n;
          const int tok = p.jt.slot_token[slot];
          const float g = p.jt.slot_gate[slot];
          atomicAdd(p.y + (size_t)tok * p.H + row, g * o[i]);
        }
      }
    }
  }
}

// Quantised items (Q8/Q4/Q2): persistent tcgen05 GEMM.  NMAT = 2: K3a (W1, W3
// over K = H; SwiGLU epilogue); NMAT = 1: K3b (W2 over K = F / ks; Eq. 1).
// Rings: raw codes + scales (bulk copies) -> 16 converter warps -> fp16 A
// stages; B tiles (X or h, np x 64) in their own ring fed by a second
// producer, so their L2 latency is hidden.  TS = true (default, K3Params::ts):
// the converters write A into TMEM with tcgen05.st (warp w: lanes 32 (w % 4)..,
// K chunks w / 4) and the MMA reads A from TMEM (kind::f16, A-from-TMEM form),
// so no fp16 A tile goes through shared memory and the raw ring gets 7 x 24 KB
// (K3a Q4 at B = 256: 338 -> 308 us; profiles/r02_k3_ts.md).  TS = false: A
// stages in shared memory (4 raw slots, 3 x 32 KB SW64 A stages).
template <int NMAT, bool TS>
__global__ void __launch_bounds__(kThreads, 1) k3_kernel(K3Params p) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t sbase = (su32(sm) + 1023) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bars = sbase + (TS ? kBarOffTS : kBarOff);
  constexpr int R = TS ? kRawSlotsTS : kRawSlots, BS = kMaxBSlots;
  constexpr int CS = TS ? 12 : kCanSlots;        // barriers for up to CS A stages
  auto raw_full = [&](int i) { return bars + 8 * i; };
  auto raw_empty = [&](int i) { return bars + 8 * (R + i); };
  auto can_full = [&](int i) { return bars + 8 * (2 * R + i); };
  auto can_empty = [&](int i) { return bars + 8 * (2 * R + CS + i); };
  auto b_full = [&](int i) { return bars + 8 * (2 * R + 2 * CS + i); };
  auto b_empty = [&](int i) { return bars + 8 * (2 * R + 2 * CS + BS + i); };
  auto tm_full = [&](int i) { return bars + 8 * (2 * R + 2 * CS + 2 * BS + i); };
  auto tm_empty = [&](int i) { return bars + 8 * (2 * R + 2 * CS + 2 * BS + 2 + i); };
  const uint32_t tslot = bars + 8 * (2 * R + 2 * CS + 2 * BS + 4);
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) {
      bar_init(raw_full(i), 1);
      bar_init(raw_empty(i), kConvWarps);
    }
    for (int i = 0; i < CS; ++i) {
      bar_init(can_full(i), kConvWarps);
      bar_init(can_empty(i), 1);
    }
    for (int i = 0; i < BS; ++i) {
      bar_init(b_full(i), 1);
      bar_init(b_empty(i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(tm_full(i), 1);
      bar_init(tm_empty(i), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"(tslot) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tbase) : "r"(tslot));

  const int v0 = p.tab->n16;                      // F16 vjob3 go to k3d_kernel
  const int nv = p.tab->n - v0;
  const int per_v = NMAT == 2 ? p.F / kRows : (p.H / kRows) * p.ks;
  const int n_items = nv * per_v;
  const int Kdim = NMAT == 2 ? p.H : p.F;          // reduction length of the matrix
  const int Kitem = NMAT == 2 ? p.H : p.F / p.ks;  // K per item
  const int nsteps = Kitem / kBK;
  // B ring geometry from the largest np of this launch's vjob3
  int npmax = 16;
  for (int v = v0; v < p.tab->n; ++v) npmax = max(npmax, p.tab->v[v].np);
  const int bslot = npmax * kBK * 2;
  const int nb = min(BS, (TS ? kBRingTS : kBRing) / bslot);
  const uint32_t bring = sbase + R * kRawBytes + (TS ? 0 : kCanSlots * kABytes);
  // TMEM accumulators: TS keeps columns 0..255 for them (per matrix MS columns,
  // two buffers when they fit, else one); the smem variant uses 2 x 256
  // TS: accumulators first (MS columns per matrix, two buffers when they fit
  // in 256 columns), the A stages of NMAT x 32 columns after them
  const int MS = TS ? (npmax <= 64 ? 64 : 128) : 128;
  const int nbuf = TS ? (NMAT * MS * 2 > 256 ? 1 : 2) : 2;
  const uint32_t bufc = TS ? (uint32_t)(NMAT * MS) : 256u;
  const uint32_t abase = TS ? (uint32_t)(nbuf * NMAT * MS) : 0u;
  const int nst = TS ? min(CS, (int)((512u - abase) / (NMAT * 32))) : CS;

  if (warp == kProdWarp) {
    if (lane == 0) {                               // raw codes + scales
      int rs = 0, ntp = 0;
      uint32_t rph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item I = item_of<NMAT>(p, it, v0);
        const int enc = I.v->enc;
        const int epg = epg_of_enc(enc), ru = raw_units<NMAT>(enc, Kitem);
        const int sb = (p.kq && enc == HB_Q2) ? 20 : scale_rec(enc);
        const int G = Kdim / epg;
        const int nraw = Kitem / (ru * epg);
        const int g0 = I.ks * (Kitem / epg);
        const uint32_t cbytes = 8 * ru * 1024, sbytes = 8 * ru * 16 * sb;   // per matrix
        const uint32_t tx = NMAT * (cbytes + sbytes);
        const CUtensorMap* tm = p.tmap + (I.v->expert * 4 + enc) * 6;
        (void)G;
        for (int r = 0; r < nraw; ++r) {
          bar_wait(raw_empty(rs), rph ^ 1);
          if (NMAT == 2) K3_STAMP(1, ntp++);
          bar_expect_tx(raw_full(rs), tx);
          const uint32_t dst = sbase + rs * kRawBytes;
          // one tensor copy per (matrix, unit column): 8 tiles x 16 rows x 64 B
          // of codes, 8 tiles x 16 scale records; raw slot [m][u][tile][...]
#pragma unroll
          for (int m = 0; m < NMAT; ++m) {
            const int mi = NMAT == 2 ? m : 2;
            for (int u = 0; u < ru; ++u) {
              const int g = g0 + r * ru + u;
              tma4(dst + m * cbytes + u * 8192, tm + mi, 0, 0, I.tile * 8, g, raw_full(rs));
              tma3(dst + kRawCode + m * sbytes + u * 128 * sb, tm + 3 + mi, 0, I.tile * 8, g,
                   raw_full(rs));
            }
          }
          if (++rs == R) { rs = 0; rph ^= 1; }
        }
      }
    }
  } else if (warp == kBProdWarp) {
    if (lane == 0) {                               // B tiles, one per canonical step
      int bs = 0, ntb = 0;
      uint32_t bph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item I = item_of<NMAT>(p, it, v0);
        const int np = I.v->np;
        const __half* bsrc = (NMAT == 2 ? p.xg + I.v->xoff : p.hB + I.v->hoff) +
                             (size_t)I.ks * nsteps * np * kBK;
        for (int s = 0; s < nsteps; ++s) {
          bar_wait(b_empty(bs), bph ^ 1);
          if (NMAT == 2) K3_STAMP(0, ntb++);
          bar_expect_tx(b_full(bs), np * kBK * 2);
          bulk_g2s(bring + bs * bslot, bsrc + (size_t)s * np * kBK, np * kBK * 2, b_full(bs));
          if (++bs == nb) { bs = 0; bph ^= 1; }
        }
      }
    }
  } else if (warp < kConvWarps) {
    const int tid = threadIdx.x;
    // thread = (row, t): its share of the row's raw piece for one 64-K step
    // -> K chunks kc = t and 4 + t (blocks j0, j0 + 1).  Quarter-warps store
    // 8 rows of one chunk: conflict-free 16-byte stores.
    // TS: warp w writes TMEM lanes 32 (w % 4) .. +31 (its rows), K chunks t = w / 4
    const int t = TS ? warp >> 2 : (tid >> 3) & 3;
    const int row = TS ? 32 * (warp & 3) + lane : (tid & 7) + 8 * (tid >> 5);
    const int tl = row >> 4, rr = row & 15;
    int rs = 0, cs = 0, ntc = 0, ntr = 0;
    uint32_t rph = 0, cph = 0;
    // one item's raw slots, the encoding a compile-time constant (EK: 4 = Q2K)
    auto conv_item = [&](auto ek) {
      constexpr int EK = decltype(ek)::value;
      constexpr int ENC = EK == 4 ? HB_Q2 : EK;
      constexpr int epg = ENC == HB_Q8 ? 64 : ENC == HB_Q4 ? 128 : 256;
      constexpr int sb = EK == 4 ? 20 : ENC == HB_Q8 ? 4 : ENC == HB_Q4 ? 8 : 32;
      const int ru = raw_units<NMAT>(ENC, Kitem);
      const int nraw = Kitem / (ru * epg);
      const int cpr = ru * epg / kBK;               // canonical stages per raw slot
      for (int r = 0; r < nraw; ++r) {
        if (lane == 0) bar_wait(raw_full(rs), rph);     // one poller per warp
        __syncwarp();
        if (NMAT == 2 && tid == 0) K3_STAMP(1, ntr++);
        const uint32_t raw = sbase + rs * kRawBytes;
        for (int c = 0; c < cpr; ++c) {
          // step-uniform offsets inside the raw slot (oracle/formats.py layout)
          const int u = ENC == HB_Q8 ? c : ENC == HB_Q4 ? (c >> 1) : (c >> 2);
          const int coff = ENC == HB_Q8 ? 0 : ENC == HB_Q4 ? 8 * (c & 1) : 4 * (c & 3);
          const int soff = ENC == HB_Q8 ? 0 : ENC == HB_Q4 ? 4 * (c & 1) : 4 * (c & 3);
          // dequantise into registers first (the raw slot is ready), then wait
          // for the A stage: the ALU chain overlaps the MMA of older stages
          uint4 w[NMAT][2];
#pragma unroll
          for (int m = 0; m < NMAT; ++m) {
            const int su = u * 8 + tl;                // raw slot [m][u][tile]
            const uint32_t code = raw + m * (8 * ru * 1024) + su * 1024 + rr * 64 + 16 * t + coff;
            const uint32_t sc = raw + kRawCode + m * (8 * ru * 16 * sb) + su * 16 * sb + rr * sb;
            if constexpr (EK == 4) dequant16_q2k(code, sc, 2 * (c & 3), t, w[m][0], w[m][1]);
            else dequant16(ENC, code, sc + soff, w[m][0], w[m][1]);
          }
          if (lane == 0) bar_wait(can_empty(cs), cph ^ 1);
          __syncwarp();
          if constexpr (TS) {
            tc_fence_after();
            // chunk kc (8 fp16) of the row -> columns 4 kc .. 4 kc + 3 of the stage
#pragma unroll
            for (int m = 0; m < NMAT; ++m) {
              const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + abase +
                                  (uint32_t)(cs * NMAT * 32 + m * 32);
              tmem_st4(ta + 4 * t, w[m][0]);
              tmem_st4(ta + 16 + 4 * t, w[m][1]);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
          } else {
            const uint32_t can = sbase + kRawSlots * kRawBytes + cs * kABytes;
#pragma unroll
            for (int m = 0; m < NMAT; ++m) {
              // UMMA K-major SWIZZLE_64B (as the TMA path): K chunk kc of a row in
              // block kc / 4 (8 KB = 128 rows x 64 B), 16-byte slot (kc % 4) ^ ((row / 2) % 4)
              const uint32_t dst = can + m * kAMat + row * 64 + ((t ^ ((row >> 1) & 3)) << 4);
              sts128(dst, w[m][0]);
              sts128(dst + 8192, w[m][1]);
            }
#ifndef HB_K3_NOFENCE
            fence_async_smem();
#endif
          }
          __syncwarp();
          if (lane == 0) bar_arrive(can_full(cs));
          if (NMAT == 2 && tid == 0) K3_STAMP(2, ntc++);
          if (++cs == nst) { cs = 0; cph ^= 1; }
        }
        __syncwarp();
        if (lane == 0) bar_arrive(raw_empty(rs));
        if (++rs == R) { rs = 0; rph ^= 1; }
      }
    };
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item I = item_of<NMAT>(p, it, v0);
      const int enc = I.v->enc;
      if (enc == HB_Q4) conv_item(std::integral_constant<int, HB_Q4>{});
      else if (enc == HB_Q8) conv_item(std::integral_constant<int, HB_Q8>{});
      else if (p.kq) conv_item(std::integral_constant<int, 4>{});
      else conv_item(std::integral_constant<int, HB_Q2>{});
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      int cs = 0, bs = 0, ab = 0, ntm = 0;
      uint32_t cph = 0, bph = 0, abph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item I = item_of<NMAT>(p, it, v0);
        const uint32_t idesc = idesc_f16(I.v->np);
        bar_wait(tm_empty(ab), abph ^ 1);
        tc_fence_after();
        const uint32_t tacc = tbase + ab * bufc;
        for (int s = 0; s < nsteps; ++s) {
          bar_wait(can_full(cs), cph);
          bar_wait(b_full(bs), bph);
          if (NMAT == 2) K3_STAMP(3, ntm++);
          tc_fence_after();
          const uint32_t bt = bring + bs * bslot;
          if constexpr (TS) {
#pragma unroll
            for (int m = 0; m < NMAT; ++m)
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)
                umma_ts(tacc + m * MS, tbase + abase + (uint32_t)(cs * NMAT * 32 + m * 32 + kk * 8),
                        sdesc(bt + kk * 256), idesc, (s | kk) ? 1u : 0u);
          } else {
            const uint32_t can = sbase + kRawSlots * kRawBytes + cs * kABytes;
#pragma unroll
            for (int m = 0; m < NMAT; ++m)
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)
                umma(tacc + m * 128, sdesc_sw64(can + m * kAMat + (kk >> 1) * 8192 + (kk & 1) * 32),
                     sdesc(bt + kk * 256), idesc, (s | kk) ? 1u : 0u);
          }
          umma_commit(can_empty(cs));
          umma_commit(b_empty(bs));
          if (++cs == nst) { cs = 0; cph ^= 1; }
          if (++bs == nb) { bs = 0; bph ^= 1; }
        }
        umma_commit(tm_full(ab));
        if (++ab == nbuf) { ab = 0; abph ^= 1; }
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
    const int q4 = warp & 3;
    int ab = 0;
    uint32_t abph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item I = item_of<NMAT>(p, it, v0);
      bar_wait(tm_full(ab), abph);
      tc_fence_after();
      epilogue_item<NMAT>(p, I, tbase + ((uint32_t)(q4 * 32) << 16) + ab * bufc, q4, lane, MS);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(tm_empty(ab));
      if (++ab == nbuf) { ab = 0; abph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase) : "memory");
  }
}

// ---------------------------------------------------------------- F16 direct
// F16 items: the fp16 weights need no conversion, so the producer moves them
// with 4-D TMA tensor copies (tensor map per matrix over our unit layout:
// dims k%32 | row-in-tile | tile | group, box 32 x 16 x 8 x 2 = 128 rows x 64 K)
// straight into shared memory in the UMMA K-major SWIZZLE_64B layout (8-row x
// 64 B atoms, 16-byte chunks XOR (row/2)%4).  No converter warps; the ring
// holds 4 (K3a) / 6 (K3b) stages.
constexpr int kDThreads = 256;            // warp 0 producer, 1 MMA, 4..7 epilogue
template <int NMAT>
constexpr int d_slots() { return NMAT == 2 ? 4 : 6; }
template <int NMAT>
constexpr int d_slot_bytes() { return NMAT * kAMat + kBBytes; }
template <int NMAT>
constexpr int d_smem() { return d_slots<NMAT>() * d_slot_bytes<NMAT>() + 1024 + 256; }

template <int NMAT>
__global__ void __launch_bounds__(kDThreads, 1) k3d_kernel(K3Params p) {
  constexpr int SMAX = d_slots<NMAT>(), RING = SMAX * d_slot_bytes<NMAT>();
  extern __shared__ uint8_t smd[];
  const uint32_t raw0 = su32(smd);
  const uint32_t sbase = (raw0 + 1023) & ~1023u;            // swizzle atoms: 1 KB aligned
  const uint32_t bars = sbase + RING;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto full = [&](int i) { return bars + 8 * i; };
  auto empty = [&](int i) { return bars + 8 * (SMAX + i); };
  auto tm_full = [&](int i) { return bars + 8 * (2 * SMAX + i); };
  auto tm_empty = [&](int i) { return bars + 8 * (2 * SMAX + 2 + i); };
  const uint32_t tslot = bars + 8 * (2 * SMAX + 4);
  // geometry from the largest F16 vjob3 of this launch (np <= 256): stage =
  // A tiles + that B tile; accumulators of MSd columns per matrix, two
  // buffers when they fit in TMEM (np > 128 at NMAT = 2: one buffer)
  const int nv = p.tab->n16;
  int npmax = 16;
  for (int v = 0; v < nv; ++v) npmax = max(npmax, p.tab->v[v].np);
  const int MSd = npmax <= 128 ? 128 : 256;
  const uint32_t bufc = (uint32_t)(NMAT * MSd);
  const int nbuf = 2 * bufc <= 512 ? 2 : 1;
  const int SB = NMAT * kAMat + npmax * kBK * 2;
  const int S = min(SMAX, RING / SB);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      bar_init(full(i), 1);
      bar_init(empty(i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(tm_full(i), 1);
      bar_init(tm_empty(i), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"(tslot) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tbase) : "r"(tslot));

  const int per_v = NMAT == 2 ? p.F / kRows : (p.H / kRows) * p.ks;
  const int n_items = nv * per_v;
  const int Kitem = NMAT == 2 ? p.H : p.F / p.ks;
  const int nsteps = Kitem / kBK;

  if (warp == 0) {
    if (lane == 0) {
      int cs = 0;
      uint32_t cph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item I = item_of<NMAT>(p, it, 0);
        const int np = I.v->np;
        const CUtensorMap* tm = p.tmap + (I.v->expert * 4 + HB_F16) * 6;
        const __half* bsrc = (NMAT == 2 ? p.xg + I.v->xoff : p.hB + I.v->hoff) +
                             (size_t)I.ks * nsteps * np * kBK;
        const int g0 = I.ks * (Kitem / 32);
        for (int s = 0; s < nsteps; ++s) {
          bar_wait(empty(cs), cph ^ 1);
          const uint32_t dst = sbase + cs * SB;
          bar_expect_tx(full(cs), NMAT * kAMat + np * kBK * 2);
#pragma unroll
          for (int m = 0; m < NMAT; ++m)
            tma4(dst + m * kAMat, tm + (NMAT == 2 ? m : 2), 0, 0, I.tile * 8, g0 + 2 * s, full(cs));
          bulk_g2s(dst + NMAT * kAMat, bsrc + (size_t)s * np * kBK, np * kBK * 2, full(cs));
          if (++cs == S) { cs = 0; cph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int cs = 0, ab = 0;
      uint32_t cph = 0, abph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item I = item_of<NMAT>(p, it, 0);
        const uint32_t idesc = idesc_f16(I.v->np);
        bar_wait(tm_empty(ab), abph ^ 1);
        tc_fence_after();
        const uint32_t tacc = tbase + ab * bufc;
        for (int s = 0; s < nsteps; ++s) {
          bar_wait(full(cs), cph);
          tc_fence_after();
          const uint32_t st = sbase + cs * SB;
#pragma unroll
          for (int m = 0; m < NMAT; ++m)
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma(tacc + m * MSd, sdesc_sw64(st + m * kAMat + (kk >> 1) * 8192 + (kk & 1) * 32),
                   sdesc(st + NMAT * kAMat + kk * 256), idesc, (s | kk) ? 1u : 0u);
          umma_commit(empty(cs));
          if (++cs == S) { cs = 0; cph ^= 1; }
        }
        umma_commit(tm_full(ab));
        if (++ab == nbuf) { ab = 0; abph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    int ab = 0;
    uint32_t abph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item I = item_of<NMAT>(p, it, 0);
      bar_wait(tm_full(ab), abph);
      tc_fence_after();
      epilogue_item<NMAT>(p, I, tbase + ((uint32_t)(q4 * 32) << 16) + ab * bufc, q4, lane, MSd);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(tm_empty(ab));
      if (++ab == nbuf) { ab = 0; abph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase) : "memory");
  }
}

// vjob3 table from the router's job table (every CTA rebuilds it in shared
// memory; CTA 0 publishes it) + gather of X into xg (canonical B layout).
__global__ void __launch_bounds__(256) k3_prep_kernel(K3Params p, const __half* __restrict__ x) {
  __shared__ V3 tab[kK3MaxV3];
  __shared__ Job sjobs[2 * 64 + 1];
  __shared__ int s_n;
  // R28: NaN rows of y for tokens whose x had a non-finite element
  for (int b = blockIdx.x; b < p.B; b += gridDim.x)
    if (__ldcg(p.rowbad + b))
      for (int i = threadIdx.x; i < p.H; i += blockDim.x) p.y[(size_t)b * p.H + i] = __int_as_float(0x7fc00000);
  // the router's jobs into shared memory once (the serial table walk below
  // then reads no global memory)
  const int nj = min(__ldcg(p.jt.hdr), 2 * 64 + 1);
  for (int j = threadIdx.x; j < nj; j += blockDim.x) sjobs[j] = p.jt.jobs[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0, n16 = 0;
    long long xo = 0, ho = 0;
    // F16 jobs first (k3d_kernel: TMA straight into the MMA layout), then the rest
    for (int pass = 0; pass < 2; ++pass)
    for (int j = 0; j < nj; ++j) {
      const Job J = sjobs[j];
      if ((J.enc == HB_F16) != (pass == 0)) continue;
      const int cap = J.enc == HB_F16 ? kK3MaxNF16 : kK3MaxN;
      for (int s = 0; s < J.n_tok && n < kK3MaxV3; s += cap) {
        V3 v;
        v.blob = J.blob;
        v.enc = J.enc;
        v.expert = J.expert;
        n16 += pass == 0;
        v.slot0 = J.slot_off + s;
        v.n = J.n_tok - s < cap ? J.n_tok - s : cap;
        v.np = (v.n + 15) & ~15;
        v.xoff = xo;
        v.hoff = ho;
        xo += (long long)v.np * p.H;
        ho += (long long)v.np * p.F;
        tab[n++] = v;
      }
    }
    s_n = n;
    if (blockIdx.x == 0) {
      p.tab->n = n;
      p.tab->n16 = n16;
    }
  }
  __syncthreads();
  const int nv = s_n;
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < nv; i += blockDim.x) p.tab->v[i] = tab[i];
  // gather: block (v, kstep) = np rows x 64 K in canonical order; chunk c of
  // 16 B sits at byte 16c: row n = (c/64)*8 + c%8, K chunk kc = (c/8)%8
  const int steps = p.H / kBK;
  for (int w = blockIdx.x; w < nv * steps; w += gridDim.x) {
    const V3& v = tab[w / steps];
    const int ks = w % steps;
    uint4* dst = reinterpret_cast<uint4*>(p.xg + v.xoff + (size_t)ks * v.np * kBK);
    for (int c = threadIdx.x; c < v.np * 8; c += blockDim.x) {
      const int n = (c >> 6) * 8 + (c & 7), kc = (c >> 3) & 7;
      uint4 val = make_uint4(0, 0, 0, 0);
      if (n < v.n) {
        const int tok = p.jt.slot_token[v.slot0 + n];
        val = *reinterpret_cast<const uint4*>(x + (size_t)tok * p.H + ks * kBK + kc * 8);
        if (v.enc == HB_Q4)                          // the Q4 converters' K order
          val = make_uint4(prmt(val.x, val.z, 0x5410), prmt(val.x, val.z, 0x7632),
                           prmt(val.y, val.w, 0x5410), prmt(val.y, val.w, 0x7632));
      }
      dst[c] = val;
    }
  }
}

}  // namespace

int k3_smem_bytes() { return kSmem; }

// Tensor map of an F16 matrix [n, k] stored as units (oracle/formats.py):
// element (row, kk) at byte 1024*(G*(row/16) + kk/32) + 64*(row%16) + 2*(kk%32).
static int encode_tiled(CUtensorMap* out, CUtensorMapDataType dt, int rank, const void* base,
                        const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                        CUtensorMapSwizzle sw);
int k3_encode_f16_map(CUtensorMap* out, const void* q, int n, int k) {
  const cuuint64_t G = (cuuint64_t)k / 32;
  const cuuint64_t dims[4] = {32, 16, (cuuint64_t)n / 16, G};
  const cuuint64_t strides[3] = {64, G * 1024, 1024};          // bytes, dims 1..3
  const cuuint32_t box[4] = {32, 16, 8, 2};
  return encode_tiled(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, q, dims, strides, box,
                      CU_TENSOR_MAP_SWIZZLE_64B);
}
// Quantised matrix [n, k] of encoding enc: codes as 4-D u8 (64 B | row | tile
// | group), box = 8 tiles x 1 unit; scales as 3-D u16 (unit record block |
// tile | group), box = 8 tiles x 1 unit.
int k3_encode_q_maps(CUtensorMap* code, CUtensorMap* scale, int enc, const void* q, const void* s,
                     int n, int k) {
  const bool q2k = enc == HB_Q2K;
  if (q2k) enc = HB_Q2;                       // Q2's codes, 20-byte records
  const cuuint64_t G = (cuuint64_t)k / epg_of_enc(enc);
  const cuuint64_t sb = q2k ? 20 : enc == HB_Q8 ? 4 : enc == HB_Q4 ? 8 : 32;
  const cuuint64_t cd[4] = {64, 16, (cuuint64_t)n / 16, G};
  const cuuint64_t cs[3] = {64, G * 1024, 1024};
  const cuuint32_t cb[4] = {64, 16, 8, 1};
  if (encode_tiled(code, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, q, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE))
    return -1;
  const cuuint64_t sd[3] = {8 * sb, (cuuint64_t)n / 16, G};
  const cuuint64_t ss[2] = {G * 16 * sb, 16 * sb};
  const cuuint32_t sbx[3] = {(cuuint32_t)(8 * sb), 8, 1};
  return encode_tiled(scale, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, s, sd, ss, sbx,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
}
static int encode_tiled(CUtensorMap* out, CUtensorMapDataType dt, int rank, const void* base,
                        const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                        CUtensorMapSwizzle sw) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !f)
      return -1;
    fn = reinterpret_cast<Fn>(f);
  }
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(out, dt, rank, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

}  // namespace hb
#ifdef HB_K3_TRACE
extern "C" int hb_k3_trace(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, hb::g_k3_trace, bytes) == cudaSuccess ? 0 : -4;
}
#endif
namespace hb {

void launch_k3_prep(const K3Params& p, const __half* x, cudaStream_t s) {
  k3_prep_kernel<<<2 * kNumSM, 256, 0, s>>>(p, x);
}
template <int NMAT>
static void launch_q(const K3Params& p, cudaStream_t s) {
  if (p.ts) {
    set_max_dyn_smem(k3_kernel<NMAT, true>, kSmemTS);
    k3_kernel<NMAT, true><<<kNumSM, kThreads, kSmemTS, s>>>(p);
  } else {
    set_max_dyn_smem(k3_kernel<NMAT, false>, kSmem);
    k3_kernel<NMAT, false><<<kNumSM, kThreads, kSmem, s>>>(p);
  }
}
void launch_k3a(const K3Params& p, cudaStream_t s) {
  set_max_dyn_smem(k3d_kernel<2>, d_smem<2>());
  if (p.has_f16) k3d_kernel<2><<<kNumSM, kDThreads, d_smem<2>(), s>>>(p);
  if (p.has_q) launch_q<2>(p, s);
}
void launch_k3b(const K3Params& p, cudaStream_t s) {
  set_max_dyn_smem(k3d_kernel<1>, d_smem<1>());
  if (p.has_f16) k3d_kernel<1><<<kNumSM, kDThreads, d_smem<1>(), s>>>(p);
  if (p.has_q) launch_q<1>(p, s);
}

}  // namespace hb
