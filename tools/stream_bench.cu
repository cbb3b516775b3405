// Read-bandwidth microbenchmark for the GEMV memory pipeline design choices.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
// Each warp streams a contiguous range of 1 KB units (as the K2 kernels do)
// with one of: (A) cp.async 16 B x 2 per lane into a smem ring of DEPTH
// stages, (B) one TMA bulk copy of CHUNK units per stage, (C) plain
// ld.global.nc.v4 with UNROLL loads in flight per lane.  The consumer reads
// its 32 bytes back (A/B) and folds them into a checksum.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;"); }
template <int N> __device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;" :: "n"(N)); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar)); }
__device__ __forceinline__ void mbar_tx(uint32_t bar, unsigned b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned ph) {
  asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" :: "r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, unsigned n, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}

extern __shared__ __align__(1024) uint8_t smem[];

template <int DEPTH>
__global__ void k_cpasync(const uint8_t* buf, size_t units, int warps_per_cta, unsigned long long* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = warp * gridDim.x + blockIdx.x, nw = gridDim.x * warps_per_cta;
  const size_t u0 = units * gw / nw, u1 = units * (gw + 1) / nw;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + warp * DEPTH * 1024;
  uint32_t acc = 0;
  size_t pu = u0;
  auto issue = [&]() {
    if (pu < u1) {
      const uint32_t st = ring + (pu % DEPTH) * 1024;
      cp16(st + 16 * lane, buf + pu * 1024 + 16 * lane);
      cp16(st + 512 + 16 * lane, buf + pu * 1024 + 512 + 16 * lane);
      ++pu;
    }
    commit();
  };
  for (int s = 0; s < DEPTH - 1; ++s) issue();
  for (size_t u = u0; u < u1; ++u) {
    __syncwarp();
    issue();
    waitg<DEPTH - 1>();
    const uint32_t st = ring + (u % DEPTH) * 1024;
    uint4 a = lds128(st + 16 * lane), b = lds128(st + 512 + 16 * lane);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

template <int DEPTH, int CHUNK>
__global__ void k_bulk(const uint8_t* buf, size_t units, int warps_per_cta, unsigned long long* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = warp * gridDim.x + blockIdx.x, nw = gridDim.x * warps_per_cta;
  size_t u0 = units * gw / nw, u1 = units * (gw + 1) / nw;
  u0 = u0 / CHUNK * CHUNK;
  u1 = u1 / CHUNK * CHUNK;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + warp * (DEPTH * CHUNK * 1024 + 128);
  const uint32_t bars = ring + DEPTH * CHUNK * 1024;
  if (lane == 0) { for (int s = 0; s < DEPTH; ++s) mbar_init(bars + 8 * s); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  uint32_t acc = 0, phases = 0;
  size_t pu = u0;
  int ps = 0, cs = 0;
  auto issue = [&]() {
    if (pu < u1) {
      if (lane == 0) {
        mbar_tx(bars + 8 * ps, CHUNK * 1024);
        bulk(ring + ps * CHUNK * 1024, buf + pu * 1024, CHUNK * 1024, bars + 8 * ps);
      }
      pu += CHUNK;
      if (++ps == DEPTH) ps = 0;
    }
  };
  for (int s = 0; s < DEPTH - 1; ++s) issue();
  for (size_t u = u0; u < u1; u += CHUNK) {
    __syncwarp();
    issue();
    mbar_wait(bars + 8 * cs, (phases >> cs) & 1);
    phases ^= 1u << cs;
    const uint32_t st = ring + cs * CHUNK * 1024;
    if (++cs == DEPTH) cs = 0;
#pragma unroll
    for (int c = 0; c < CHUNK; ++c) {
      uint4 a = lds128(st + c * 1024 + 16 * lane), b = lds128(st + c * 1024 + 512 + 16 * lane);
      acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
    }
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
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
template <uint32_t MASK>
__device__ __forceinline__ uint32_t lop_magic(uint32_t a) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "n"(MASK), "n"(0x64006400));
  return r;
}

// The K2a consumer emulated on the same stream: 2 matrices per 2 KB unit.
// MODE 0: F16 (PRMT + 2 chained HMMA per matrix); 1: F16 with a fresh D per
// unit (chain broken); 2: Q4 (4 blocks: LOP3 dequant + 2 HMMA + 4 FFMA each).
template <int DEPTH, int MODE>
__global__ void k_mma(const uint8_t* buf, size_t units, int warps_per_cta, unsigned long long* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = warp * gridDim.x + blockIdx.x, nw = gridDim.x * warps_per_cta;
  const size_t u0 = (units / 2) * gw / nw * 2, u1 = (units / 2) * (gw + 1) / nw * 2;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + warp * DEPTH * 2048;
  float acc[2][4] = {};
  const uint32_t xb0 = 0x3c003c00u, xb1 = 0x3c003c00u;
  size_t pu = u0;
  auto issue = [&]() {
    if (pu < u1) {
      const uint32_t st = ring + ((pu - u0) / 2 % DEPTH) * 2048;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        cp16(st + m * 1024 + 16 * lane, buf + (pu + m) * 1024 + 16 * lane);
        cp16(st + m * 1024 + 512 + 16 * lane, buf + (pu + m) * 1024 + 512 + 16 * lane);
      }
      pu += 2;
    }
    commit();
  };
  for (int s = 0; s < DEPTH - 1; ++s) issue();
  const int g = lane >> 2, t = lane & 3;
  for (size_t u = u0; u < u1; u += 2) {
    __syncwarp();
    issue();
    waitg<DEPTH - 1>();
    __syncwarp();
    const uint32_t st = ring + ((u - u0) / 2 % DEPTH) * 2048;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const uint4 a = lds128(st + m * 1024 + g * 64 + 16 * t);
      const uint4 b = lds128(st + m * 1024 + (g + 8) * 64 + 16 * t);
      if (MODE <= 1) {
        float D[4] = {0.f, 0.f, 0.f, 0.f};
        float (&tgt)[4] = MODE == 0 ? acc[m] : D;
        mma16816(tgt, prmt(a.x, a.z, 0x5410), prmt(b.x, b.z, 0x5410), prmt(a.x, a.z, 0x7632),
                 prmt(b.x, b.z, 0x7632), xb0, xb1);
        mma16816(tgt, prmt(a.y, a.w, 0x5410), prmt(b.y, b.w, 0x5410), prmt(a.y, a.w, 0x7632),
                 prmt(b.y, b.w, 0x7632), xb0, xb1);
        if (MODE == 1)
          for (int i = 0; i < 4; ++i) acc[m][i] += D[i];
      } else {
        const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int blk = 0; blk < 4; ++blk) {
          const uint32_t w = wa[blk], w8 = w >> 8, v = wb[blk], v8 = v >> 8;
          float D[4] = {0.f, 0.f, 0.f, 0.f};
          mma16816(D, lop_magic<0x000F000Fu>(w), lop_magic<0x000F000Fu>(v),
                   lop_magic<0x00F000F0u>(w), lop_magic<0x00F000F0u>(v), xb0, xb1);
          mma16816(D, lop_magic<0x000F000Fu>(w8), lop_magic<0x000F000Fu>(v8),
                   lop_magic<0x00F000F0u>(w8), lop_magic<0x00F000F0u>(v8), xb0, xb1);
          const float d = 0.5f + blk;
          for (int i = 0; i < 4; ++i) acc[m][i] = fmaf(d, D[i], acc[m][i]);
        }
      }
    }
  }
  float s = 0.f;
  for (int m = 0; m < 2; ++m)
    for (int i = 0; i < 4; ++i) s += acc[m][i];
  if (s == 1234.5f) atomicAdd(out, 1ull);
}

// NS separate streams per warp (matrix m of unit u at buf + m*span + u*1024),
// like K2a's W1 / W3 code sections (+ scale sections) far apart in a blob
template <int DEPTH, int NS>
__global__ void k_streams(const uint8_t* buf, size_t units, int warps_per_cta, unsigned long long* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = warp * gridDim.x + blockIdx.x, nw = gridDim.x * warps_per_cta;
  const size_t span = units / NS;                     // units per stream region
  const size_t u0 = span * gw / nw, u1 = span * (gw + 1) / nw;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + warp * DEPTH * NS * 1024;
  uint32_t acc = 0;
  size_t pu = u0;
  auto issue = [&]() {
    if (pu < u1) {
      const uint32_t st = ring + ((pu - u0) % DEPTH) * NS * 1024;
#pragma unroll
      for (int m = 0; m < NS; ++m) {
        const uint8_t* src = buf + ((size_t)m * span + pu) * 1024;
        cp16(st + m * 1024 + 16 * lane, src + 16 * lane);
        cp16(st + m * 1024 + 512 + 16 * lane, src + 512 + 16 * lane);
      }
      ++pu;
    }
    commit();
  };
  for (int s = 0; s < DEPTH - 1; ++s) issue();
  for (size_t u = u0; u < u1; ++u) {
    __syncwarp();
    issue();
    waitg<DEPTH - 1>();
    const uint32_t st = ring + ((u - u0) % DEPTH) * NS * 1024;
#pragma unroll
    for (int m = 0; m < NS; ++m) {
      uint4 a = lds128(st + m * 1024 + 16 * lane), b = lds128(st + m * 1024 + 512 + 16 * lane);
      acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
    }
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

template <int UNROLL>
__global__ void k_ldg(const uint8_t* buf, size_t units, int warps_per_cta, unsigned long long* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = warp * gridDim.x + blockIdx.x, nw = gridDim.x * warps_per_cta;
  size_t u0 = units * gw / nw, u1 = units * (gw + 1) / nw;
  uint32_t acc = 0;
  size_t u = u0;
  for (; u + UNROLL / 2 <= u1; u += UNROLL / 2) {
    uint4 r[UNROLL];
#pragma unroll
    for (int i = 0; i < UNROLL; ++i) r[i] = ldg_nc(buf + (u + i / 2) * 1024 + (i & 1) * 512 + 16 * lane);
#pragma unroll
    for (int i = 0; i < UNROLL; ++i) acc ^= r[i].x ^ r[i].y ^ r[i].z ^ r[i].w;
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

template <typename K>
float run(K kern, int ctas, int warps, size_t smem_bytes, const uint8_t* buf, size_t units,
          unsigned long long* out) {
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) kern<<<ctas, warps * 32, smem_bytes>>>(buf, units, warps, out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  const int iters = 5;
  for (int i = 0; i < iters; ++i) kern<<<ctas, warps * 32, smem_bytes>>>(buf, units, warps, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return units * 1024.0 * iters / (ms * 1e-3) / 1e9;
}

int main() {
  const size_t bytes = 4ull << 30;
  uint8_t* buf;
  unsigned long long* out;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(buf, 1, bytes));
  const size_t units = bytes / 1024;
  const int ctas = 148;
  if (getenv("STREAMS")) {               // separate streams per warp
    for (size_t mb : {4096, 300}) {
      const size_t u = mb * 1024;
      printf("streams=1 W=16 D=4 %5zu MB %7.0f GB/s\n", mb, run(k_streams<4, 1>, ctas, 16, 16 * 4 * 1024, buf, u, out));
      printf("streams=2 W=16 D=4 %5zu MB %7.0f GB/s\n", mb, run(k_streams<4, 2>, ctas, 16, 16 * 4 * 2048, buf, u, out));
      printf("streams=2 W=16 D=6 %5zu MB %7.0f GB/s\n", mb, run(k_streams<6, 2>, ctas, 16, 16 * 6 * 2048, buf, u, out));
      printf("streams=2 W=8  D=6 %5zu MB %7.0f GB/s\n", mb, run(k_streams<6, 2>, ctas, 8, 8 * 6 * 2048, buf, u, out));
      printf("streams=4 W=16 D=3 %5zu MB %7.0f GB/s\n", mb, run(k_streams<3, 4>, ctas, 16, 16 * 3 * 4096, buf, u, out));
      printf("streams=4 W=8  D=4 %5zu MB %7.0f GB/s\n", mb, run(k_streams<4, 4>, ctas, 8, 8 * 4 * 4096, buf, u, out));
    }
    return 0;
  }
  if (getenv("SIZE_SWEEP")) {            // fixed per-launch cost: bytes per launch sweep
    for (size_t mb : {4096, 1024, 300, 150, 66, 33}) {
      const size_t u = mb * 1024;
      printf("cp.async W=16 D=4 %5zu MB/launch %7.0f GB/s\n", mb, run(k_cpasync<4>, ctas, 16, 16 * 4 * 1024, buf, u, out));
      printf("mma Q4   W=12 D=4 %5zu MB/launch %7.0f GB/s\n", mb, run(k_mma<4, 2>, ctas, 12, 12 * 4 * 2048, buf, u, out));
    }
    return 0;
  }
  if (getenv("MMA_ONLY")) {
    for (int w : {8, 12, 16}) {
      printf("mma F16 chain   W=%2d D=4 %7.0f GB/s\n", w, run(k_mma<4, 0>, ctas, w, w * 4 * 2048, buf, units, out));
      printf("mma F16 chain   W=%2d D=6 %7.0f GB/s\n", w, run(k_mma<6, 0>, ctas, w, w * 6 * 2048, buf, units, out));
      printf("mma F16 fresh   W=%2d D=4 %7.0f GB/s\n", w, run(k_mma<4, 1>, ctas, w, w * 4 * 2048, buf, units, out));
      printf("mma F16 fresh   W=%2d D=6 %7.0f GB/s\n", w, run(k_mma<6, 1>, ctas, w, w * 6 * 2048, buf, units, out));
      printf("mma Q4          W=%2d D=4 %7.0f GB/s\n", w, run(k_mma<4, 2>, ctas, w, w * 4 * 2048, buf, units, out));
      printf("mma Q4          W=%2d D=6 %7.0f GB/s\n", w, run(k_mma<6, 2>, ctas, w, w * 6 * 2048, buf, units, out));
    }
    return 0;
  }
  for (int w : {8, 12, 16}) {
    printf("cp.async W=%2d D=4  %7.0f GB/s\n", w, run(k_cpasync<4>, ctas, w, w * 4 * 1024, buf, units, out));
    printf("cp.async W=%2d D=8  %7.0f GB/s\n", w, run(k_cpasync<8>, ctas, w, w * 8 * 1024, buf, units, out));
    if (w <= 12) printf("cp.async W=%2d D=16 %7.0f GB/s\n", w, run(k_cpasync<16>, ctas, w, w * 16 * 1024, buf, units, out));
    printf("bulk     W=%2d D=4 C=1 %7.0f GB/s\n", w, run(k_bulk<4, 1>, ctas, w, w * (4 * 1024 + 128), buf, units, out));
    printf("bulk     W=%2d D=8 C=1 %7.0f GB/s\n", w, run(k_bulk<8, 1>, ctas, w, w * (8 * 1024 + 128), buf, units, out));
    printf("bulk     W=%2d D=3 C=4 %7.0f GB/s\n", w, run(k_bulk<3, 4>, ctas, w, w * (12 * 1024 + 128), buf, units, out));
    if (w <= 8) printf("bulk     W=%2d D=4 C=6 %7.0f GB/s\n", w, run(k_bulk<4, 6>, ctas, w, w * (24 * 1024 + 128), buf, units, out));
    printf("ldg      W=%2d U=8  %7.0f GB/s\n", w, run(k_ldg<8>, ctas, w, 0, buf, units, out));
    printf("ldg      W=%2d U=16 %7.0f GB/s\n", w, run(k_ldg<16>, ctas, w, 0, buf, units, out));
  }
  for (int w : {16, 32}) {
    printf("ldg 2CTA W=%2d U=8  %7.0f GB/s\n", w, run(k_ldg<8>, 2 * ctas, w, 0, buf, units, out));
  }
  return 0;
}
