// K3: tcgen05 grouped GEMM for batched decode / prefill.
#pragma once

#include <cuda.h>

#include "hb_internal.h"

namespace hb {

constexpr int kK3MaxN = 128;    // tokens per vjob3 (MMA N, two TMEM accumulators per buffer)
constexpr int kK3MaxNF16 = 256; // F16 vjob3 (k3d_kernel): up to MMA N = 256, so an expert's weights
                                // stream once for up to 256 tokens
constexpr int kK3MaxV3 = 64;    // vjob3 entries per forward

// <= 128 token slots of one job; np = count rounded up to 16 (MMA N)
struct V3 {
  const uint8_t* blob;
  int32_t enc;
  int32_t slot0;
  int32_t n;
  int32_t np;
  int32_t expert;
  int32_t pad;
  long long xoff;                // fp16 elements: this vjob3's X in xg (np * H)
  long long hoff;                // fp16 elements: its h in hB (np * F)
};
struct K3Table {
  int32_t n;
  int32_t n16;                   // entries [0, n16) are F16 (k3d_kernel), the rest quantised
  int32_t pad[2];
  V3 v[kK3MaxV3];
};

struct K3Params {
  JobTable jt;
  BlobLayout lay[4];
  int H, F;
  int ks;                        // K3b K split (F / ks multiple of 256)
  __half* xg;                    // gathered X, canonical UMMA K-major blocks [v][H/64][np x 64]
  __half* hB;                    // h, same layout [v][F/64][np x 64]
  float* y;                      // [B][H] fp32, zeroed by the router
  const int* rowbad;             // [B] non-finite x flags (router): prep writes NaN rows (R28)
  int B;
  K3Table* tab;
  const CUtensorMap* tmap;       // [E][4 enc][6] tensor maps of this layer's blobs:
                                 //   F16: [0..2] W1, W3, W2; Q: [0..2] codes, [3..5] scales
  int has_f16, has_q;            // encodings in the pair (launch k3d_kernel / k3_kernel)
  int kq;                        // the Q2 slot holds HB_Q2K blobs (20-byte records, R32)
  int ts;                        // quantised items: A operand dequantised into TMEM (tcgen05.st,
                                 // A-from-TMEM MMA) instead of shared memory (HB_K3_TS)
};
// 4-D tensor map of one F16 matrix [n rows, k] in the unit layout (host)
int k3_encode_f16_map(CUtensorMap* out, const void* q, int n, int k);
int k3_encode_q_maps(CUtensorMap* code, CUtensorMap* scale, int enc, const void* q, const void* s,
                     int n, int k);

int k3_smem_bytes();
void launch_k3_prep(const K3Params& p, const __half* x, cudaStream_t s);
void launch_k3a(const K3Params& p, cudaStream_t s);
void launch_k3b(const K3Params& p, cudaStream_t s);

}  // namespace hb
