// Offline quantiser (reading R8, off the hot path) and the seeded synthetic
// generator (the counter-based generator of synthgen/, reproduced bit for bit).
//
// Paper: HOBBIT keeps int4 / int2 versions of fp16 / int8 experts (P:294,
// P:801) but does not define the bit formats; ours are block-32 formats in
// the style of Llama.cpp's legacy quants (Q8_0 / Q4_0) plus an affine 2-bit
// format (R7, R8).  All arithmetic is IEEE fp32 in a fixed order
// (no fast-math in this translation unit), so the bytes are a deterministic
// function of the fp16 input.
#include <cuda_fp16.h>

#include <algorithm>

#include "hb_internal.h"

namespace hb {

__device__ __forceinline__ float f16(const __half* p, size_t i) { return __half2float(p[i]); }

// F16 "codes": the fp16 values permuted into tile-major units
__global__ void f16_tile_kernel(const __half* __restrict__ w, int n, int k, uint8_t* __restrict__ q) {
  const int groups = k / 32;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)n * groups) return;
  const int row = (int)(gid / groups), grp = (int)(gid % groups);
  const uint4* src = reinterpret_cast<const uint4*>(w + (size_t)row * k + (size_t)grp * 32);
  const size_t unit = (size_t)(row / 16) * groups + grp;
  uint4* dst = reinterpret_cast<uint4*>(q + unit * 1024 + (row % 16) * 64);
#pragma unroll
  for (int i = 0; i < 4; ++i) dst[i] = src[i];
}

// one thread per (row, 64-byte group); writes the row's 64 bytes of the unit
// (tile-major layout) and its scale record
template <int ENC>
__global__ void quant_kernel(const __half* __restrict__ w, int n, int k, uint8_t* __restrict__ q,
                             uint8_t* __restrict__ ssec) {
  constexpr int EPG = ENC == HB_Q8 ? 64 : ENC == HB_Q4 ? 128 : 256;
  constexpr int BPG = EPG / 32;
  constexpr int SB = 2 * BPG * (ENC == HB_Q2 ? 2 : 1);
  const int groups = k / EPG;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)n * groups) return;
  const int row = (int)(gid / groups), grp = (int)(gid % groups);
  const size_t unit = (size_t)(row / 16) * groups + grp;
  __half* rec = reinterpret_cast<__half*>(ssec + (unit * 16 + row % 16) * SB);
  const __half* src = w + (size_t)row * k + (size_t)grp * EPG;
  uint32_t words[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) words[i] = 0u;
  for (int j = 0; j < BPG; ++j) {
    const __half* x = src + 32 * j;
    int code[32];
    float dval = 0.f, mval = 0.f;
    if (ENC == HB_Q8) {
      float amax = 0.f;
      for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(f16(x, i)));
      const __half d16 = __float2half_rn(__fdiv_rn(amax, 127.0f));
      const float d = __half2float(d16);
      dval = d;
      for (int i = 0; i < 32; ++i) {
        if (d == 0.f) { code[i] = 0; continue; }
        const float v = __fdiv_rn(f16(x, i), d);
        float r = copysignf(floorf(__fadd_rn(fabsf(v), 0.5f)), v);   // round half away
        r = fminf(fmaxf(r, -127.f), 127.f);
        code[i] = (int)r;
      }
      rec[j] = d16;
    } else if (ENC == HB_Q4) {
      float m = 0.f;                                  // signed value of max |x|, first on ties
      for (int i = 0; i < 32; ++i) {
        const float v = f16(x, i);
        if (fabsf(v) > fabsf(m)) m = v;
      }
      const __half d16 = __float2half_rn(__fdiv_rn(m, -8.0f));
      const float d = __half2float(d16);
      dval = d;
      for (int i = 0; i < 32; ++i) {
        if (d == 0.f) { code[i] = 8; continue; }
        float r = floorf(__fadd_rn(__fdiv_rn(f16(x, i), d), 8.5f));
        r = fminf(fmaxf(r, 0.f), 15.f);
        code[i] = (int)r;
      }
      rec[j] = d16;
    } else {
      float mn = f16(x, 0), mx = f16(x, 0);
      for (int i = 1; i < 32; ++i) {
        mn = fminf(mn, f16(x, i));
        mx = fmaxf(mx, f16(x, i));
      }
      const __half d16 = __float2half_rn(__fdiv_rn(__fsub_rn(mx, mn), 3.0f));
      const __half m16 = __float2half_rn(mn);
      const float d = __half2float(d16), m = __half2float(m16);
      dval = d;
      mval = m;
      for (int i = 0; i < 32; ++i) {
        if (d == 0.f) { code[i] = 0; continue; }
        float r = rintf(__fdiv_rn(__fsub_rn(f16(x, i), m), d));   // half-even
        r = fminf(fmaxf(r, 0.f), 3.f);
        code[i] = (int)r;
      }
      rec[j] = d16;
      rec[BPG + j] = m16;
    }
    (void)dval;
    (void)mval;
    // place codes: element 32j + 8t + r of the group
    for (int t = 0; t < 4; ++t)
      for (int r = 0; r < 8; ++r) {
        const uint32_t c = (uint32_t)code[8 * t + r];
        if (ENC == HB_Q8) {                 // byte 16t + 8j + r
          const int byte = 16 * t + 8 * j + r;
          words[byte >> 2] |= (c & 0xFFu) << (8 * (byte & 3));
        } else if (ENC == HB_Q4) {          // byte 16t + 4j + r/2, nibble r%2
          const int byte = 16 * t + 4 * j + (r >> 1);
          words[byte >> 2] |= (c & 0xFu) << (8 * (byte & 3) + 4 * (r & 1));
        } else {                            // byte 16t + 4(j/2) + 2(r/4) + j%2, bits 2(r%4)
          const int byte = 16 * t + 4 * (j >> 1) + 2 * (r >> 2) + (j & 1);
          words[byte >> 2] |= (c & 0x3u) << (8 * (byte & 3) + 2 * (r & 3));
        }
      }
  }
  uint4* dst = reinterpret_cast<uint4*>(q + unit * 1024 + (row % 16) * 64);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    dst[i] = make_uint4(words[4 * i], words[4 * i + 1], words[4 * i + 2], words[4 * i + 3]);
}

// Q2K (R33; oracle/formats.quantize_q2k): one thread per (row,
// super-block of 256); the codes go where Q2's go, the record holds d, dmin
// and the 16 sub-block bytes.  IEEE fp32 in the oracle's order.
__global__ void quant_q2k_kernel(const __half* __restrict__ w, int n, int k, uint8_t* __restrict__ q,
                                 uint8_t* __restrict__ ssec) {
  const int groups = k / 256;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)n * groups) return;
  const int row = (int)(gid / groups), grp = (int)(gid % groups);
  const size_t unit = (size_t)(row / 16) * groups + grp;
  const __half* src = w + (size_t)row * k + (size_t)grp * 256;
  float s_j[16], mm_j[16];
  float smax = 0.f, mmax = 0.f;
  for (int j = 0; j < 16; ++j) {
    float mn = 0.f, mx = f16(src, 16 * j);
    for (int l = 0; l < 16; ++l) {
      const float v = f16(src, 16 * j + l);
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    s_j[j] = __fdiv_rn(__fsub_rn(mx, mn), 3.0f);
    mm_j[j] = -mn;
    smax = fmaxf(smax, s_j[j]);
    mmax = fmaxf(mmax, mm_j[j]);
  }
  const __half d16 = __float2half_rn(__fdiv_rn(smax, 15.0f));
  const __half dm16 = __float2half_rn(__fdiv_rn(mmax, 15.0f));
  const float d = __half2float(d16), dm = __half2float(dm16);
  uint8_t* rec = ssec + (unit * 16 + row % 16) * 20;        // 20-byte record
  reinterpret_cast<__half*>(rec)[0] = d16;
  reinterpret_cast<__half*>(rec)[1] = dm16;
  uint32_t words[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) words[i] = 0u;
  for (int j = 0; j < 16; ++j) {
    const float lo = d == 0.f ? 0.f : fminf(fmaxf(rintf(__fdiv_rn(s_j[j], d)), 0.f), 15.f);
    const float hi = dm == 0.f ? 0.f : fminf(fmaxf(rintf(__fdiv_rn(mm_j[j], dm)), 0.f), 15.f);
    rec[4 + j] = (uint8_t)((int)lo | ((int)hi << 4));
    const float dl = __fmul_rn(d, lo), ml = __fmul_rn(dm, hi);
    for (int l = 0; l < 16; ++l) {
      const int e = 16 * j + l;                      // element of the super-block
      uint32_t c = 0;
      if (dl != 0.f) c = (uint32_t)fminf(fmaxf(rintf(__fdiv_rn(__fadd_rn(f16(src, e), ml), dl)), 0.f), 3.f);
      // Q2 placement: element 32 jb + 8 t + r -> byte 16t + 4(jb/2) + 2(r/4) + jb%2, bits 2(r%4)
      const int jb = e >> 5, t = (e & 31) >> 3, r = e & 7;
      const int byte = 16 * t + 4 * (jb >> 1) + 2 * (r >> 2) + (jb & 1);
      words[byte >> 2] |= c << (8 * (byte & 3) + 2 * (r & 3));
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(q + unit * 1024 + (row % 16) * 64);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    dst[i] = make_uint4(words[4 * i], words[4 * i + 1], words[4 * i + 2], words[4 * i + 3]);
}

int launch_quantize_expert(int enc, int hidden, int ffn, const __half* w1, const __half* w3,
                           const __half* w2, uint8_t* blob, cudaStream_t s) {
  BlobLayout L;
  int rc = blob_layout(enc, hidden, ffn, &L);
  if (rc) return rc;
  const __half* src[3] = {w1, w3, w2};
  const int N[3] = {ffn, ffn, hidden}, K[3] = {hidden, hidden, ffn};
  for (int m = 0; m < 3; ++m) {
    if (enc == HB_F16) {
      const long long threads = (long long)N[m] * (K[m] / 32);
      f16_tile_kernel<<<(int)((threads + 127) / 128), 128, 0, s>>>(src[m], N[m], K[m],
                                                                     blob + L.mat[m].q);
      continue;
    }
    const int epg = enc == HB_Q8 ? 64 : enc == HB_Q4 ? 128 : 256;
    const long long threads = (long long)N[m] * (K[m] / epg);
    const int grid = (int)((threads + 127) / 128);
    uint8_t* q = blob + L.mat[m].q;
    uint8_t* sc = blob + L.mat[m].s;
    if (enc == HB_Q2K) quant_q2k_kernel<<<grid, 128, 0, s>>>(src[m], N[m], K[m], q, sc);
    else if (enc == HB_Q8) quant_kernel<HB_Q8><<<grid, 128, 0, s>>>(src[m], N[m], K[m], q, sc);
    else if (enc == HB_Q4) quant_kernel<HB_Q4><<<grid, 128, 0, s>>>(src[m], N[m], K[m], q, sc);
    else quant_kernel<HB_Q2><<<grid, 128, 0, s>>>(src[m], N[m], K[m], q, sc);
  }
  return cudaGetLastError() == cudaSuccess ? HB_OK : HB_ECUDA;
}

// ---------------------------------------------------------------- synth
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_kernel(__half* __restrict__ dst, size_t n, unsigned long long key,
                             float scale, unsigned long long start) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long u = mix64(key + (start + i + 1ull) * 0x9E3779B97F4A7C15ull);
    const int s = (int)(u & 0xFFFF) + (int)((u >> 16) & 0xFFFF) + (int)((u >> 32) & 0xFFFF) +
                  (int)(u >> 48) - 131070;
    dst[i] = __float2half_rn(__fmul_rn((float)s, scale));
  }
}

void launch_synth(__half* dst, size_t n, uint64_t key, float scale, uint64_t start,
                  cudaStream_t s) {
  const int grid = (int)std::min<size_t>((n + 255) / 256, (size_t)kNumSM * 16);
  synth_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(dst, n, key, scale, start);
}

}  // namespace hb
