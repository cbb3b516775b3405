// Canonical expert blob (row-major, LSB-first codes, then d,
// then m, sections 256-byte aligned) -> the library's tile-major device
// layout.  Registration-time only: the oracle and any
// external producer write the canonical blob; the GEMV/GEMM kernels stream
// the device layout.
//
// One thread per (matrix row n, 32-element block blk).  Every device byte of
// a unit row holds elements of a single block, so a thread assembles whole
// bytes: with t = (k%32)/8, q = k%8, j = block within the 64-byte group,
//   F16  o = 2*(k%32)                   -> the block's 64 bytes in order
//   Q8   o = 16t + 8j + q               -> 8 canonical bytes per t
//   Q4   o = 16t + 4j + q/2 (nibble q%2) -> canonical bytes 4t..4t+3 (same nibble order)
//   Q2   o = 16t + 4(j/2) + 2(q/4) + (j%2), bits 2(q%4)
//                                        -> canonical byte 2t+h to 16t + 4(j/2) + 2h + (j%2)
// and the scale record of (n, group) at 16*SB*(G*tile + grp) + SB*r holds d
// of block j at +2j and (Q2) m at +2*BPG + 2j.
#include <cuda_fp16.h>

#include <algorithm>

#include "hb_internal.h"

namespace hb {

struct RepackMat {
  const uint8_t* sc;    // Q2K: canonical sub-block bytes [N][K/16]
  const uint8_t* q;     // canonical code section (fp16 values for F16)
  const uint16_t* d;    // canonical d [N][K/32] (quantised)
  const uint16_t* m;    // canonical m [N][K/32] (Q2)
  uint8_t* dq;          // device code section
  uint8_t* ds;          // device scale section
  int N, K;
};
struct RepackParams {
  RepackMat mat[3];
  int enc;
};

__global__ void repack_kernel(const __grid_constant__ RepackParams p) {
  const int mi = blockIdx.y;
  const RepackMat& M = p.mat[mi];
  const int nblk = M.K / 32;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)M.N * nblk) return;
  const int n = (int)(i / nblk), blk = (int)(i - (long long)n * nblk);
  const int enc = p.enc == HB_Q2K ? HB_Q2 : p.enc;   // Q2K codes are Q2's
  const int epg = epg_of_enc(enc), bpg = epg / 32;
  const int G = M.K / epg, tile = n / 16, r = n % 16, grp = blk / bpg, j = blk % bpg;
  uint8_t* base = M.dq + 1024ull * ((size_t)G * tile + grp) + 64 * r;
  if (enc == HB_F16) {
    const uint4* src = reinterpret_cast<const uint4*>(M.q + ((size_t)n * M.K + 32 * blk) * 2);
    uint4* dst = reinterpret_cast<uint4*>(base);
#pragma unroll
    for (int c = 0; c < 4; ++c) dst[c] = src[c];
    return;
  }
  if (enc == HB_Q8) {
    const uint2* src = reinterpret_cast<const uint2*>(M.q + (size_t)n * M.K + 32 * blk);
#pragma unroll
    for (int t = 0; t < 4; ++t) *reinterpret_cast<uint2*>(base + 16 * t + 8 * j) = src[t];
  } else if (enc == HB_Q4) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(M.q + (size_t)n * M.K / 2 + 16 * blk);
#pragma unroll
    for (int t = 0; t < 4; ++t) *reinterpret_cast<uint32_t*>(base + 16 * t + 4 * j) = src[t];
  } else {
    const uint8_t* src = M.q + (size_t)n * M.K / 4 + 8 * blk;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) base[16 * t + 4 * (j / 2) + 2 * h + (j % 2)] = src[2 * t + h];
  }
  const int sb = p.enc == HB_Q2K ? 20 : 2 * bpg * (enc == HB_Q2 ? 2 : 1);
  uint16_t* rec = reinterpret_cast<uint16_t*>(M.ds + 16ull * sb * ((size_t)G * tile + grp) + sb * r);
  if (p.enc == HB_Q2K) {            // 20-byte record: d, dmin, sc[16] of the super-block (R32)
    uint8_t* rb = reinterpret_cast<uint8_t*>(rec);
    rb[4 + 2 * j] = M.sc[(size_t)n * (M.K / 16) + 2 * blk];
    rb[4 + 2 * j + 1] = M.sc[(size_t)n * (M.K / 16) + 2 * blk + 1];
    if (j == 0) {
      rec[0] = M.d[(size_t)n * G + grp];
      rec[1] = M.m[(size_t)n * G + grp];
    }
    return;
  }
  rec[j] = M.d[(size_t)n * nblk + blk];
  if (enc == HB_Q2) rec[bpg + j] = M.m[(size_t)n * nblk + blk];
}

int canonical_layout(int enc, int hidden, int ffn, CanonLayout* out) {
  if (enc < HB_F16 || enc > HB_Q2K || hidden <= 0 || ffn <= 0 || hidden % 256 || ffn % 256)
    return HB_EINVAL;
  if (enc == HB_Q2K) {              // q, sc [N][K/16], d [N][K/256], dmin [N][K/256]
    const int N[3] = {ffn, ffn, hidden}, K[3] = {hidden, hidden, ffn};
    auto align = [](uint64_t v) { return (v + 255) / 256 * 256; };
    uint64_t off = 0;
    for (int m = 0; m < 3; ++m) {
      out->q[m] = off;
      off = align(off + (uint64_t)N[m] * K[m] / 4);
      out->sc[m] = off;
      off = align(off + (uint64_t)N[m] * (K[m] / 16));
      out->d[m] = off;
      off = align(off + (uint64_t)N[m] * (K[m] / 256) * 2);
      out->m[m] = off;
      off = align(off + (uint64_t)N[m] * (K[m] / 256) * 2);
    }
    out->total = off;
    return HB_OK;
  }
  for (int m = 0; m < 3; ++m) out->sc[m] = 0;
  const int N[3] = {ffn, ffn, hidden}, K[3] = {hidden, hidden, ffn};
  const int bits = enc == HB_F16 ? 16 : enc == HB_Q8 ? 8 : enc == HB_Q4 ? 4 : 2;
  auto align = [](uint64_t v) { return (v + 255) / 256 * 256; };
  uint64_t off = 0;
  for (int m = 0; m < 3; ++m) {
    out->q[m] = off;
    off = align(off + (uint64_t)N[m] * K[m] * bits / 8);
    out->d[m] = out->m[m] = 0;
    if (enc != HB_F16) {
      out->d[m] = off;
      off = align(off + (uint64_t)N[m] * (K[m] / 32) * 2);
    }
    if (enc == HB_Q2) {
      out->m[m] = off;
      off = align(off + (uint64_t)N[m] * (K[m] / 32) * 2);
    }
  }
  out->total = off;
  return HB_OK;
}

int launch_repack_canonical(int enc, int hidden, int ffn, const uint8_t* src, uint8_t* dst,
                            cudaStream_t s) {
  CanonLayout C;
  BlobLayout D;
  if (canonical_layout(enc, hidden, ffn, &C) || blob_layout(enc, hidden, ffn, &D)) return HB_EINVAL;
  RepackParams p{};
  p.enc = enc;
  const int N[3] = {ffn, ffn, hidden}, K[3] = {hidden, hidden, ffn};
  long long most = 0;
  for (int m = 0; m < 3; ++m) {
    p.mat[m].q = src + C.q[m];
    p.mat[m].sc = src + C.sc[m];
    p.mat[m].d = reinterpret_cast<const uint16_t*>(src + C.d[m]);
    p.mat[m].m = reinterpret_cast<const uint16_t*>(src + C.m[m]);
    p.mat[m].dq = dst + D.mat[m].q;
    p.mat[m].ds = dst + D.mat[m].s;
    p.mat[m].N = N[m];
    p.mat[m].K = K[m];
    most = std::max(most, (long long)N[m] * (K[m] / 32));
  }
  repack_kernel<<<dim3((unsigned)((most + 255) / 256), 3), 256, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? HB_OK : HB_ECUDA;
}

}  // namespace hb
