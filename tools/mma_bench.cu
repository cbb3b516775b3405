// Legacy tensor-core (mma.sync.m16n8k16 f16 -> f32) throughput / latency on
// this GPU: the K2 GEMV kernels issue one HMMA.16816 per 16x8x16 tile, so
// this bounds how many weight bytes per second their inner loops can consume.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void k_mma(int iters, float* out) {
  float acc[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[c][i] = 0.f;
  uint32_t a0 = threadIdx.x * 0x00010001u, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a1 + 9;
  uint32_t b0 = 0x3c003c00u ^ threadIdx.x, b1 = b0 + 3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int CHAINS>
void run(int warps, int ctas_per_sm) {
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 4096, grid = 148 * ctas_per_sm;
  k_mma<CHAINS><<<grid, warps * 32>>>(16, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mma<CHAINS><<<grid, warps * 32>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)grid * warps * iters * CHAINS;
  printf("chains=%d warps/CTA=%2d CTAs/SM=%d: %8.1f G HMMA/s  (%6.1f TFLOP/s, %5.2f cycles/HMMA/SMSP @1.965GHz)\n",
         CHAINS, warps, ctas_per_sm, n / ms / 1e6, n * 4096 / ms / 1e9,
         1.965e9 * 148 * 4 / (n / ms * 1e3));
  cudaFree(out);
}

int main() {
  run<1>(16, 1);
  run<2>(16, 1);
  run<4>(16, 1);
  run<8>(16, 1);
  run<4>(32, 1);
  run<8>(32, 1);
  run<1>(4, 1);
  return 0;
}
