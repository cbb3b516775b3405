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
