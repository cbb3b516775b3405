// C ABI of libhobbit (include/hobbit.h): context, expert registry, HBM slot
// pools, pinned next-level storage, copy stream + events (the Dynamic Expert
// Loader, P:349 / fig:handler), and the three calls of the paper's problem:
// moe_layer_forward, expert_cache_load, prefetch_next_layer.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <dlfcn.h>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <mutex>
#include <new>
#include <set>
#include <string>
#include <vector>

#include "cache.h"
#include "dcache.h"
#include "hb_internal.h"
#include "k3.h"
#include "hobbit.h"

namespace hb {

cudaError_t set_max_dyn_smem_impl(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({kernel, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kernel, dev});
  return e;
}

int blob_layout(int enc, int hidden, int ffn, BlobLayout* out) {
  if (enc < HB_F16 || enc > HB_Q2K || hidden <= 0 || ffn <= 0 || hidden % 256 || ffn % 256)
    return HB_EINVAL;
  if (enc == HB_Q2K) {                       // Q2's codes, 20-byte records [d, dmin, sc16] (R32)
    const int N[3] = {ffn, ffn, hidden}, K[3] = {hidden, hidden, ffn};
    auto align = [](uint64_t v) { return (v + 255) / 256 * 256; };
    uint64_t off = 0;
    for (int m = 0; m < 3; ++m) {
      out->mat[m].q = off;
      off = align(off + (uint64_t)N[m] * K[m] / 4);
      out->mat[m].s = off;
      off = align(off + (uint64_t)N[m] * (K[m] / 256) * 20);
    }
    CanonLayout C;
    canonical_layout(HB_Q2K, hidden, ffn, &C);
    out->total = std::max(off, C.total);       // the canonical blob's size
    return HB_OK;
  }
  // code section + one scale section per matrix (tile-major units, DESIGN.md
  // "Blob layout"); every section 256-byte aligned
  const int N[3] = {ffn, ffn, hidden}, K[3] = {hidden, hidden, ffn};
  const int bits = enc == HB_F16 ? 16 : enc == HB_Q8 ? 8 : enc == HB_Q4 ? 4 : 2;
  auto align = [](uint64_t v) { return (v + 255) / 256 * 256; };
  uint64_t off = 0;
  for (int m = 0; m < 3; ++m) {
    const uint64_t qbytes = (uint64_t)N[m] * K[m] * bits / 8;
    const uint64_t sbytes = (uint64_t)N[m] * (K[m] / 32) * 2 * (enc == HB_Q2 ? 2 : 1);
    out->mat[m].q = off;
    off = align(off + qbytes);
    out->mat[m].s = off;
    if (enc != HB_F16) off = align(off + sbytes);
  }
  out->total = off;
  return HB_OK;
}

}  // namespace hb

using namespace hb;

static thread_local std::string g_err;

struct hb_ctx {
  hb_config cfg{};
  int device = 0;
  bool resident = true;
  BlobLayout lay[4]{};
  size_t bbytes[4]{};
  // router weights [L][E][H]
  __half* wg = nullptr;
  float* wnorm = nullptr;                 // [L][E] ||W_e||_2 rounded up (fused router's error bound)
  std::vector<char> router_set;
  // resident registry: device blobs [L][E][4]
  std::vector<const uint8_t*> dev_blob;
  const uint8_t** dev_blob_table = nullptr;
  // offload registry: host blobs [L][E][4]
  std::vector<const uint8_t*> host_blob;
  std::vector<void*> arena;               // pinned copies owned by the library
  std::vector<void*> dev_owned;           // resident blobs copied into library HBM
  uint8_t* pool_mem[2] = {nullptr, nullptr};
  size_t slot_bytes[2] = {0, 0};
  std::vector<cudaEvent_t> slot_ready[2], slot_free[2];
  cudaStream_t copy_stream = nullptr;
  // chunked, cancellable prefetch: prefetch copies are
  // queued on the host and issued in chunks within a window of bytes in
  // flight; on-demand copies are issued at once (ahead of the unissued
  // chunks); a prefetch whose slot is reused before it was issued is dropped;
  // a hit on a slot whose prefetch is still queued issues the rest first.
  struct PfLoad { int pool, slot; const uint8_t* src; uint8_t* dst; size_t total, issued; };
  std::vector<PfLoad> pf_queue;
  std::vector<std::pair<cudaEvent_t, size_t>> pf_inflight;   // issued chunks (event, bytes)
  std::vector<cudaEvent_t> pf_event_pool;
  size_t pf_window = 64ull << 20, pf_chunk = 16ull << 20;     // HB_PREFETCH_WINDOW_MB / _CHUNK_MB
  ExpertCache* cache = nullptr;
  std::vector<hb_event> log;
  // device-resident cache manager (hb_config.device_cache):
  // state in HBM, SM copies from the mapped host blobs (dcache.cu)
  DcState* dc = nullptr;                  // device copy of the state
  DcState dc_h{};                         // host mirror (array pointers)
  const uint8_t** host_blob_dev = nullptr;   // [L][E][4] device addresses of the host blobs
  int* err_host = nullptr;                // mapped pinned sticky error word
  int* err_dev = nullptr;                 // its device address
  cudaEvent_t ev_fork = nullptr, ev_side = nullptr;
  bool side_pending = false;              // background copier not yet joined
  int dc_reset = 0, dc_tadd = 0, dc_clear = 0;   // token_begin / reset since the last cache op
  int dc_fg_ctas = 32, dc_bg_ctas = 16;   // HB_DC_FG_CTAS / HB_DC_BG_CTAS
  size_t dc_chunk = 256u << 10;           // HB_DC_CHUNK_KB
  uint64_t copied[2] = {0, 0};            // host path: bytes issued on demand / prefetch+explicit
  bool kq = false;                        // the Q2 slot holds HB_Q2K blobs (R32)
  // token-sharded EP (hb_config.token_sharded)
  bool ts = false;
  int ts_C = 0;                           // rows per (source, destination) = max_batch
  hb_decision* ts_dec = nullptr;          // local decisions [max_batch][k]
  int* ts_pos = nullptr;                  // [max_batch][k] dest * C + position or -1
  int* ts_rowbad = nullptr;               // [max_batch]
  int ts_batch = 0;                       // batch of the last dispatch
  hb_ts_meta* ts_meta[2] = {nullptr, nullptr};   // one-shot forward: send / recv
  __half* ts_rows[2] = {nullptr, nullptr};
  float* ts_ret[2] = {nullptr, nullptr};
  // scratch
  hb_decision* dec = nullptr;             // [B][k]
  hb_decision* dec_pred = nullptr;        // [p][B][k]
  hb_decision* dec_host = nullptr;        // pinned [(1+p)][B][k]
  long long* logits = nullptr;            // [B][E][2]
  long long* lbuf = nullptr;              // [P][B][E][2] router scratch
  int* rowbad = nullptr;                  // [P][B] non-finite flags (router scratch)
  uint4* x_perm = nullptr;
  float* xsum = nullptr;
  float* au = nullptr;                    // 2 x [slots][2][F] K2a sums (double-buffered)
  int au_cur = 0;                         // buffer of the last GEMV forward
  long long au_dirty[2] = {0, 0};         // floats of each buffer not yet zeroed again
  bool fused_ok = false;                  // fused decode kernel usable (B = 1, top-2, fits)
  unsigned* gbar = nullptr;               // fused kernel grid barrier [count, generation]
  unsigned* fwd_idx = nullptr;            // profile record index, exit counter
  unsigned long long* stamps = nullptr;   // [stamp_cap][8] per-forward %globaltimer records
  int stamp_cap = 0;
  bool stamps_on = false;
  __half* x_save = nullptr;               // x of the last fused forward (lazy exact logits)
  bool last_fused = false;
  bool last_filtered = false;             // last forward's router kept no exact logits
  bool hfin_tail = false;                 // HB_HFIN_TAIL=1: h at the end of K2a (grid barrier), no hfin kernel
  bool router_filtered = false;           // HB_ROUTER=filtered: batch-1 decode router kernel (diagnostic)
  bool router_solo = true;                // batch-1 decode: router_solo_kernel on a reserved SM (HB_ROUTER_SOLO=0: off)
  bool router_batch = true;               // filtered router for batches (HB_ROUTER=exact: off)
  bool fused_split = false;               // HB_FUSED_SPLIT=1: router+K2a kernel, then hfin + K2b
  bool fused_router = false;              // HB_FUSED_ROUTER=1: one-CTA router kernel + legacy K2a/hfin/K2b
  uint4* h_hi = nullptr;                  // h in global memory (large batches only)
  uint4* h_lo = nullptr;
  float* hsum = nullptr;
  bool force_h_global = false;            // HB_FORCE_H_GLOBAL=1 (tests of that path)
  unsigned* done = nullptr;
  unsigned* gctr = nullptr;               // GEMV chunk counters [2 + 2 * kGemvCTAs] (self-resetting)
  JobTable jt{};
  void* jt_dev = nullptr;
  void* jt_host = nullptr;                // pinned staging
  // offload path, hits first: the misses' job table (same layout as jt)
  JobTable jt2{};
  void* jt2_dev = nullptr;
  void* jt2_host = nullptr;
  bool hit_first = true;                  // HB_HIT_FIRST=0: one K2 chain after every load
  uint64_t split_fwds = 0;
  size_t jt_bytes = 0;
  int max_jobs = 0, max_slots = 0, max_vjobs = 0;
  float static_frac = 0.8f;               // GEMV work feed K2a (HB_STATIC_FRAC, HB_CHUNK)
  float static_frac2 = 0.8f;              // K2b (HB_STATIC_FRAC2)
  int chunk = 8;
  float k2b_w[4] = {1.f, 2.f, 3.f, 8.f};  // HB_K2B_W: K2b CTA-split cost per unit (~ weights per KB)
  // K3: tcgen05 grouped GEMM for batches >= k3_min_batch (A9); buffers exist
  // when max_batch > 1 and the vjob3 table bound fits
  int k3_min_batch = 4;                   // HB_K3_MIN_BATCH / hb_set_batched_min (K3 wins from B = 4, profiles/r01_batched.md)
  bool k3_ok = false;
  int k3_ks = 1;
  int k3_ts = 1;                          // quantised K3 items: A dequantised into TMEM (HB_K3_TS=0: smem)
  __half* k3_xg = nullptr;
  __half* k3_hB = nullptr;
  K3Table* k3_tab = nullptr;
  // EP exchange (A10) inside the library: NCCL all-reduce of y after the
  // expert kernels (hb_nccl_init); NCCL is dlopen'ed (the process's copy)
  void* nccl_comm = nullptr;
  CUtensorMap* k3_tmap = nullptr;         // [L][E][4][6] device tensor maps of the blobs (K3)
  cudaEvent_t dec_ready = nullptr;
  // kernel timing (hb_profile)
  std::vector<cudaEvent_t> prof_ev;       // 3 per recorded forward
  int prof_max = 0, prof_n = 0;
  // bookkeeping
  int last_batch = 0, last_layer = -1;
  bool last_host_decisions = false;
  bool token_started = false;
  uint64_t launches = 0;
  std::string err;
};

#define CUDA_TRY(ctx, call)                                                   \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(_e);        \
      return HB_ECUDA;                                                        \
    }                                                                         \
  } while (0)

static int fail(hb_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  else g_err = msg;
  return code;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
static int dc_create(hb_ctx* c);

// ---- NCCL, resolved at run time (libnccl.so.2 already loaded by the process,
// e.g. torch's, or found on the library path; HB_NCCL_LIB overrides)
struct NcclId { char internal[128]; };
struct NcclApi {
  int (*get_unique_id)(NcclId*) = nullptr;
  int (*comm_init_rank)(void**, int, NcclId, int) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  bool ok = false;
};
static NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* env = std::getenv("HB_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_unique_id = (int (*)(NcclId*))dlsym(h, "ncclGetUniqueId");
      api.comm_init_rank = (int (*)(void**, int, NcclId, int))dlsym(h, "ncclCommInitRank");
      api.all_reduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
          h, "ncclAllReduce");
      api.comm_destroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
      api.broadcast = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
          h, "ncclBroadcast");
      api.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
      api.send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclSend");
      api.recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclRecv");
      api.group_start = (int (*)())dlsym(h, "ncclGroupStart");
      api.group_end = (int (*)())dlsym(h, "ncclGroupEnd");
      api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy &&
               api.broadcast;
    }
  }
  return api;
}
constexpr int kNcclInt8 = 0, kNcclFloat16 = 6, kNcclFloat32 = 7, kNcclSum = 0;

extern "C" {

void hb_config_default(hb_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->n_layers = 32;
  c->n_experts = 8;
  c->top_k = 2;
  c->hidden = 4096;
  c->ffn = 14336;
  c->hi_enc = HB_F16;
  c->lo_enc = HB_Q4;
  c->t1 = 0.6;
  c->t2 = 0.9;
  c->lookahead_p = 1;
  c->w_lru = c->w_lfu = c->w_lhu = c->w_fld = 1;
  c->cap_high = c->cap_low = -1;
  c->allow_upgrade = 1;
  c->rank = 0;
  c->world = 1;
  c->max_batch = 1;
  c->strict = 1;
}

size_t hb_blob_bytes(int enc, int hidden, int ffn) {
  BlobLayout L;
  return blob_layout(enc, hidden, ffn, &L) ? 0 : (size_t)L.total;
}

int hb_blob_section(int enc, int hidden, int ffn, int mat, int sec, size_t* offset,
                    size_t* nbytes) {
  BlobLayout L;
  if (blob_layout(enc, hidden, ffn, &L) || mat < 0 || mat > 2 || sec < 0 || sec > 2 || !offset ||
      !nbytes)
    return fail(nullptr, HB_EINVAL, "bad blob section query");
  const int N = mat < 2 ? ffn : hidden, K = mat < 2 ? hidden : ffn;
  const int bits = enc == HB_F16 ? 16 : enc == HB_Q8 ? 8 : enc == HB_Q4 ? 4 : 2;
  if (sec == 0) { *offset = L.mat[mat].q; *nbytes = (size_t)N * K * bits / 8; return HB_OK; }
  if (enc == HB_F16 || sec == 2) return fail(nullptr, HB_EINVAL, "section does not exist");
  *offset = L.mat[mat].s;
  *nbytes = enc == HB_Q2K ? (size_t)N * (K / 256) * 20 : (size_t)N * (K / 32) * 2 * (enc == HB_Q2 ? 2 : 1);
  return HB_OK;
}

int hb_canonical_section(int enc, int hidden, int ffn, int mat, int sec, size_t* offset,
                         size_t* nbytes) {
  CanonLayout C;
  if (canonical_layout(enc, hidden, ffn, &C) || mat < 0 || mat > 2 || sec < 0 || sec > 3 ||
      !offset || !nbytes)
    return fail(nullptr, HB_EINVAL, "bad canonical section query");
  const int N = mat < 2 ? ffn : hidden, K = mat < 2 ? hidden : ffn;
  const int bits = enc == HB_F16 ? 16 : enc == HB_Q8 ? 8 : enc == HB_Q4 ? 4 : 2;
  if (sec == 0) { *offset = C.q[mat]; *nbytes = (size_t)N * K * bits / 8; return HB_OK; }
  if (enc == HB_Q2K) {
    if (sec == 1) { *offset = C.sc[mat]; *nbytes = (size_t)N * (K / 16); return HB_OK; }
    *offset = sec == 2 ? C.d[mat] : C.m[mat];
    *nbytes = (size_t)N * (K / 256) * 2;
    return HB_OK;
  }
  if (sec == 3 || enc == HB_F16 || (sec == 2 && enc != HB_Q2))
    return fail(nullptr, HB_EINVAL, "section does not exist");
  *offset = sec == 1 ? C.d[mat] : C.m[mat];
  *nbytes = (size_t)N * (K / 32) * 2;
  return HB_OK;
}

int hb_repack_canonical(int enc, int hidden, int ffn, const void* src, void* dst, void* stream) {
  if (!src || !dst) return fail(nullptr, HB_EINVAL, "null argument");
  const int rc = launch_repack_canonical(enc, hidden, ffn, (const uint8_t*)src, (uint8_t*)dst,
                                         (cudaStream_t)stream);
  if (rc) return fail(nullptr, rc, rc == HB_EINVAL ? "bad enc / dims" : "repack launch failed");
  return HB_OK;
}

int64_t hb_theta(double t, int* kind) {
  // floor(ln(T/(1-T)) * 2^48) in 80-bit long double (R9)
  if (t >= 1.0) { if (kind) *kind = 1; return 0; }
  if (t <= 0.0) { if (kind) *kind = -1; return 0; }
  if (kind) *kind = 0;
  const long double T = (long double)t;
  const long double v = logl(T / (1.0L - T)) * 281474976710656.0L;   // 2^48
  return (int64_t)floorl(v);
}

const char* hb_last_error(const hb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }
const char* hb_version(void) { return "hobbit-b200 0.1 (sm_100a)"; }

static void free_ctx(hb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  void* dptrs[] = {c->wg, c->dev_blob_table, c->pool_mem[0], c->pool_mem[1], c->dec, c->dec_pred,
                   c->logits, c->lbuf, c->x_perm, c->xsum, c->au, c->h_hi, c->h_lo,
                   c->hsum, c->done, c->gctr, c->jt_dev, c->jt2_dev, c->k3_xg, c->k3_hB, c->k3_tab, c->k3_tmap,
                   c->gbar, c->fwd_idx, c->stamps, c->x_save, c->wnorm, c->rowbad,
                   c->dc, c->host_blob_dev, c->dc_h.pool[0], c->dc_h.pool[1], c->dc_h.where[0],
                   c->dc_h.where[1], c->dc_h.R, c->dc_h.F, c->dc_h.H, c->dc_h.mask_exp,
                   c->dc_h.masked_keys, c->dc_h.cur, c->dc_h.cur_list, c->dc_h.log,
                   c->dc_h.task[0], c->dc_h.task[1], c->ts_dec, c->ts_pos, c->ts_rowbad,
                   c->ts_meta[0], c->ts_meta[1], c->ts_rows[0], c->ts_rows[1], c->ts_ret[0],
                   c->ts_ret[1]};
  for (void* p : dptrs)
    if (p) cudaFree(p);
  if (c->dec_host) cudaFreeHost(c->dec_host);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_side) cudaEventDestroy(c->ev_side);
  if (c->jt_host) cudaFreeHost(c->jt_host);
  if (c->jt2_host) cudaFreeHost(c->jt2_host);
  for (void* p : c->arena) cudaFreeHost(p);
  for (void* p : c->dev_owned) cudaFree(p);
  for (int i = 0; i < 2; ++i) {
    for (cudaEvent_t e : c->slot_ready[i]) cudaEventDestroy(e);
    for (cudaEvent_t e : c->slot_free[i]) cudaEventDestroy(e);
  }
  if (c->dec_ready) cudaEventDestroy(c->dec_ready);
  for (auto& pe : c->pf_inflight) cudaEventDestroy(pe.first);
  for (cudaEvent_t e : c->pf_event_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->nccl_comm) nccl_api().comm_destroy(c->nccl_comm);
  delete c->cache;
  delete c;
}

int hb_create(const hb_config* cfg, int device, hb_ctx** out) {
  if (!cfg || !out) return fail(nullptr, HB_EINVAL, "null argument");
  // HB_Q2K lives in the Q2 slot of every per-encoding table (same device
  // layout size); the context remembers the format (hb_ctx::kq) and maps the
  // encoding at the boundary (registration, loads, events, decisions)
  hb_config kin = *cfg;
  const bool kq = kin.hi_enc == HB_Q2K || kin.lo_enc == HB_Q2K;
  if (kq && (kin.hi_enc == HB_Q2 || kin.lo_enc == HB_Q2))
    return fail(nullptr, HB_EINVAL, "a pair may use HB_Q2K or HB_Q2, not both");
  if (kin.hi_enc == HB_Q2K) kin.hi_enc = HB_Q2;
  if (kin.lo_enc == HB_Q2K) kin.lo_enc = HB_Q2;
  const hb_config& k = kin;
  if (k.n_layers <= 0 || k.n_experts <= 0 || k.n_experts > 64 || k.top_k <= 0 ||
      k.top_k > k.n_experts || k.top_k > kMaxTopK)
    return fail(nullptr, HB_EINVAL, "bad n_layers / n_experts (<=64) / top_k (<=8)");
  if (k.hidden <= 0 || k.ffn <= 0 || k.hidden % 256 || k.ffn % 256)
    return fail(nullptr, HB_EINVAL, "hidden and ffn must be positive multiples of 256");
  if (!(k.t1 <= k.t2)) return fail(nullptr, HB_EINVAL, "t1 > t2 (S:131)");
  if (k.hi_enc < 0 || k.hi_enc > 3 || k.lo_enc < 0 || k.lo_enc > 3 || k.hi_enc == k.lo_enc)
    return fail(nullptr, HB_EINVAL, "bad encoding pair");
  if (k.world <= 0 || k.rank < 0 || k.rank >= k.world) return fail(nullptr, HB_EINVAL, "bad rank/world");
  if (k.max_batch <= 0) return fail(nullptr, HB_EINVAL, "max_batch must be > 0");
  if (k.lookahead_p < 0 || k.lookahead_p > kMaxRouteLayers - 1)
    return fail(nullptr, HB_EINVAL, "lookahead_p must be in [0, 4]");
  if (k.w_lru < 0 || k.w_lfu < 0 || k.w_lhu < 0 || k.w_fld < 0)
    return fail(nullptr, HB_EINVAL, "Eq. 3 weights must be >= 0 (all 0: Random policy)");
  const bool resident = k.cap_high < 0 && k.cap_low < 0;
  if (!resident && (k.cap_high < 0 || k.cap_low < 0))
    return fail(nullptr, HB_EINVAL, "cap_high and cap_low must both be -1 or both >= 0");

  hb_ctx* c = new (std::nothrow) hb_ctx;
  if (!c) return fail(nullptr, HB_ENOMEM, "out of host memory");
  c->cfg = k;
  c->kq = kq;
  c->device = device;
  c->resident = resident;
  for (int e = 0; e < 4; ++e) {
    blob_layout(kq && e == HB_Q2 ? HB_Q2K : e, k.hidden, k.ffn, &c->lay[e]);   // the Q2 slot
    c->bbytes[e] = c->lay[e].total;
  }
  auto bail = [&](int code, const std::string& m) {
    g_err = m;
    free_ctx(c);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(HB_ECUDA, "cudaSetDevice failed");
  if (k.token_sharded && (!resident || !k.strict))
    return fail(nullptr, HB_EINVAL, "token_sharded needs resident mode and strict = 1");
  // token-sharded: the owner computes up to world * max_batch * top_k received
  // rows per forward -- the batch every buffer below is sized for
  const int L = k.n_layers, E = k.n_experts,
            B = k.token_sharded ? k.world * k.max_batch * k.top_k : k.max_batch, K = k.top_k,
            H = k.hidden, F = k.ffn;
  const int P = std::max(1, k.lookahead_p);
  c->max_slots = B * K;
  c->max_jobs = std::min(2 * E, B * K) + 1;
  c->max_vjobs = c->max_jobs + (c->max_slots + kVSlots - 1) / kVSlots;
  if (c->max_vjobs + 1 > kMaxVJobs)
    return bail(HB_EUNSUPPORTED, "max_batch * top_k too large for one forward's job table");
  if ((long long)c->max_vjobs * (F / 16) * (H / 32) >= (1LL << 31))
    return bail(HB_EUNSUPPORTED, "GEMV unit space of one forward exceeds 2^31 units");
  auto dm = [&](void** p, size_t n) { return cudaMalloc(p, std::max<size_t>(n, 16)) == cudaSuccess; };
  bool ok = dm((void**)&c->wg, (size_t)L * E * H * 2) &&
            dm((void**)&c->dec, sizeof(hb_decision) * B * K) &&
            dm((void**)&c->dec_pred, sizeof(hb_decision) * P * B * K) &&
            dm((void**)&c->logits, sizeof(long long) * B * E * 2) &&
            dm((void**)&c->lbuf, sizeof(long long) * P * B * E * 2) &&
            dm((void**)&c->rowbad, sizeof(int) * P * B) &&
            dm((void**)&c->x_perm, (size_t)B * H * 2) && dm((void**)&c->xsum, (size_t)B * (H / 32) * 4) &&
            dm((void**)&c->au, 2 * (size_t)c->max_slots * 2 * F * 4) &&
            dm((void**)&c->gbar, 16) && dm((void**)&c->fwd_idx, 16) &&
            dm((void**)&c->wnorm, (size_t)L * E * 4) &&
            dm((void**)&c->x_save, (size_t)B * H * 2) &&
            dm((void**)&c->h_hi, (size_t)c->max_slots * F * 2) &&
            dm((void**)&c->h_lo, (size_t)c->max_slots * F * 2) &&
            dm((void**)&c->hsum, (size_t)c->max_slots * (F / 32) * 4) &&
            dm((void**)&c->done, 16) && dm((void**)&c->gctr, sizeof(unsigned) * (2 + 2 * kGemvCTAs));
  if (!ok) return bail(HB_ENOMEM, "device allocation of scratch failed");
  {
    const char* fh = std::getenv("HB_FORCE_H_GLOBAL");
    c->force_h_global = fh && fh[0] == '1';
    const char* sf = std::getenv("HB_STATIC_FRAC");
    if (sf) c->static_frac = std::min(1.0f, std::max(0.0f, (float)std::atof(sf)));
    const char* sf2 = std::getenv("HB_STATIC_FRAC2");
    if (sf2) c->static_frac2 = std::min(1.0f, std::max(0.0f, (float)std::atof(sf2)));
    const char* kw = std::getenv("HB_K2B_W");        // "f16,q8,q4,q2"
    if (kw) {
      float w[4];
      if (std::sscanf(kw, "%f,%f,%f,%f", &w[0], &w[1], &w[2], &w[3]) == 4)
        for (int e = 0; e < 4; ++e) c->k2b_w[e] = std::max(0.05f, w[e]);
    }
    const char* ch = std::getenv("HB_CHUNK");
    if (ch) c->chunk = (std::max(2, std::atoi(ch)) + 1) & ~1;   // even: K2b stages hold 2 units
  }
  {
    // K3 scratch: X and h of every vjob3 in canonical blocks (rows padded to 16)
    const int max_v3 = c->max_jobs + (c->max_slots + kK3MaxN - 1) / kK3MaxN;
    const size_t rows = (size_t)c->max_slots + 16 * (size_t)max_v3;
    if (B > 1 && max_v3 <= kK3MaxV3) {
      if (!dm((void**)&c->k3_xg, rows * H * 2) || !dm((void**)&c->k3_hB, rows * F * 2) ||
          !dm((void**)&c->k3_tab, sizeof(K3Table)) ||
          (resident && !dm((void**)&c->k3_tmap, sizeof(CUtensorMap) * (size_t)L * E * 24)))
        return bail(HB_ENOMEM, "K3 scratch allocation failed");
      c->k3_ok = true;
      c->k3_ks = (F / 2) % 256 == 0 && !k.deterministic ? 2 : 1;   // deterministic: no K split
      cudaMemset(c->k3_tab, 0, sizeof(K3Table));
    }
    const char* kt = std::getenv("HB_K3_TS");
    if (kt) c->k3_ts = kt[0] == '1';
    const char* km = std::getenv("HB_K3_MIN_BATCH");
    if (km) c->k3_min_batch = std::atoi(km);
  }
  cudaMemset(c->done, 0, 16);
  cudaMemset(c->au, 0, 2 * (size_t)c->max_slots * 2 * F * 4);
  cudaMemset(c->gbar, 0, 16);
  cudaMemset(c->fwd_idx, 0, 16);
  {
    // batch-1 decode chain: HB_DECODE = legacy (router
    // kernel, K2a, hfin, K2b: the default, fastest measured), fused (one
    // kernel per layer), split (router+K2a kernel, hfin, K2b) or router
    // (one-CTA filtered router kernel, K2a, hfin, K2b)
    const char* dm_ = std::getenv("HB_DECODE");
    const std::string mode = dm_ ? dm_ : "legacy";
    c->fused_ok = resident && K == 2 && mode != "legacy" && !kq &&
                  fused_fits(E, H, F, k.hi_enc, k.lo_enc);
    c->fused_split = mode == "split";
    c->fused_router = mode == "router";
    // measured slower (K2a CTAs held at the barrier: K2b's prologue cannot
    // overlap the K2a tail), kept as a diagnostic variant
    const char* pw = std::getenv("HB_PREFETCH_WINDOW_MB");
    if (pw) c->pf_window = (size_t)std::max(0, std::atoi(pw)) << 20;
    const char* pc = std::getenv("HB_PREFETCH_CHUNK_MB");
    if (pc) c->pf_chunk = (size_t)std::max(1, std::atoi(pc)) << 20;
    const char* hk = std::getenv("HB_HFIN_TAIL");
    c->hfin_tail = hk && hk[0] == '1';
    const char* re = std::getenv("HB_ROUTER");
    c->router_filtered = re && std::string(re) == "filtered";
    c->router_batch = !(re && std::string(re) == "exact");
    const char* rs = std::getenv("HB_ROUTER_SOLO");
    c->router_solo = !(rs && std::string(rs) == "0");
  }
  cudaMemset(c->gctr, 0, sizeof(unsigned) * (2 + 2 * kGemvCTAs));
  cudaMemset(c->wg, 0, (size_t)L * E * H * 2);
  // job table: hdr | jobs | slot_token | slot_gate | tok_slots
  const size_t o_jobs = 64, o_tok = align_up(o_jobs + sizeof(Job) * c->max_jobs, 64),
               o_gate = align_up(o_tok + 4 * (size_t)c->max_slots, 64),
               o_ts = align_up(o_gate + 4 * (size_t)c->max_slots, 64),
               o_vj = align_up(o_ts + 4 * (size_t)c->max_slots, 64),
               o_c13 = align_up(o_vj + sizeof(VJobD) * (c->max_vjobs + 1), 64),
               o_c2 = align_up(o_c13 + 8 * (size_t)(c->max_vjobs + 1), 64),
               total = align_up(o_c2 + 8 * (size_t)(c->max_vjobs + 1), 64);
  c->jt_bytes = total;
  if (!dm(&c->jt_dev, total) || cudaHostAlloc(&c->jt_host, total, cudaHostAllocDefault) != cudaSuccess)
    return bail(HB_ENOMEM, "job table allocation failed");
  cudaMemset(c->jt_dev, 0, total);
  uint8_t* jb = (uint8_t*)c->jt_dev;
  c->jt.hdr = (int32_t*)jb;
  c->jt.jobs = (Job*)(jb + o_jobs);
  c->jt.slot_token = (int32_t*)(jb + o_tok);
  c->jt.slot_gate = (float*)(jb + o_gate);
  c->jt.tok_slots = (int32_t*)(jb + o_ts);
  c->jt.vjobs = (VJobD*)(jb + o_vj);
  c->jt.vcum13 = (long long*)(jb + o_c13);
  c->jt.vcum2 = (long long*)(jb + o_c2);
  if (!resident) {                           // the misses' table of a split offload forward
    if (!dm(&c->jt2_dev, total) || cudaHostAlloc(&c->jt2_host, total, cudaHostAllocDefault) != cudaSuccess)
      return bail(HB_ENOMEM, "job table allocation failed");
    cudaMemset(c->jt2_dev, 0, total);
    uint8_t* j2 = (uint8_t*)c->jt2_dev;
    c->jt2.hdr = (int32_t*)j2;
    c->jt2.jobs = (Job*)(j2 + o_jobs);
    c->jt2.slot_token = (int32_t*)(j2 + o_tok);
    c->jt2.slot_gate = (float*)(j2 + o_gate);
    c->jt2.tok_slots = (int32_t*)(j2 + o_ts);
    c->jt2.vjobs = (VJobD*)(j2 + o_vj);
    c->jt2.vcum13 = (long long*)(j2 + o_c13);
    c->jt2.vcum2 = (long long*)(j2 + o_c2);
    const char* hf = std::getenv("HB_HIT_FIRST");
    c->hit_first = !(hf && hf[0] == '0');
  }
  if (cudaHostAlloc((void**)&c->dec_host, sizeof(hb_decision) * (1 + P) * B * K,
                    cudaHostAllocDefault) != cudaSuccess)
    return bail(HB_ENOMEM, "pinned decision buffer allocation failed");
  if (cudaEventCreateWithFlags(&c->dec_ready, cudaEventDisableTiming) != cudaSuccess)
    return bail(HB_ECUDA, "event creation failed");
  c->router_set.assign(L, 0);
  if (resident) {
    c->dev_blob.assign((size_t)L * E * 4, nullptr);
    if (!dm((void**)&c->dev_blob_table, sizeof(void*) * (size_t)L * E * 4))
      return bail(HB_ENOMEM, "blob table allocation failed");
    cudaMemset(c->dev_blob_table, 0, sizeof(void*) * (size_t)L * E * 4);
  } else {
    c->host_blob.assign((size_t)L * E * 4, nullptr);
    const int cap[2] = {k.cap_high, k.cap_low};
    const int enc[2] = {k.hi_enc, k.lo_enc};
    for (int p = 0; p < 2; ++p) {
      c->slot_bytes[p] = align_up(c->bbytes[enc[p]], 4096);
      if (cap[p] > 0 && !dm((void**)&c->pool_mem[p], c->slot_bytes[p] * cap[p]))
        return bail(HB_ENOMEM, "expert pool allocation failed");
      c->slot_ready[p].resize(cap[p]);
      c->slot_free[p].resize(cap[p]);
      for (int s = 0; s < cap[p]; ++s) {
        cudaEventCreateWithFlags(&c->slot_ready[p][s], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&c->slot_free[p][s], cudaEventDisableTiming);
      }
    }
    if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(HB_ECUDA, "copy stream creation failed");
    const int w[4] = {k.w_lru, k.w_lfu, k.w_lhu, k.w_fld};
    c->cache = new (std::nothrow) ExpertCache(L, E, K, k.cap_high, k.cap_low, w, k.hi_enc,
                                              k.lo_enc, k.allow_upgrade != 0, k.rank, k.world,
                                              k.prefetch_both != 0);
    if (!c->cache) return bail(HB_ENOMEM, "cache allocation failed");
    if (k.device_cache) {
      if (int rc = dc_create(c)) return bail(rc, c->err);
    }
  }
  if (k.token_sharded) {
    c->ts = true;
    c->ts_C = k.max_batch;
    const size_t nr = (size_t)k.world * c->ts_C;
    bool tok = dm((void**)&c->ts_dec, sizeof(hb_decision) * k.max_batch * K) &&
               dm((void**)&c->ts_pos, sizeof(int) * k.max_batch * K) &&
               dm((void**)&c->ts_rowbad, sizeof(int) * k.max_batch);
    for (int i = 0; i < 2; ++i)
      tok = tok && dm((void**)&c->ts_meta[i], sizeof(hb_ts_meta) * nr) &&
            dm((void**)&c->ts_rows[i], nr * H * 2) && dm((void**)&c->ts_ret[i], nr * H * 4);
    if (!tok) return bail(HB_ENOMEM, "token-sharded buffers allocation failed");
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(HB_ECUDA, "device sync failed");
  *out = c;
  return HB_OK;
}

int hb_destroy(hb_ctx* c) {
  if (!c) return fail(nullptr, HB_EINVAL, "null ctx");
  free_ctx(c);
  return HB_OK;
}

int hb_set_router(hb_ctx* c, int layer, const void* w, int on_device) {
  if (!c || !w) return fail(c, HB_EINVAL, "null argument");
  if (layer < 0 || layer >= c->cfg.n_layers) return fail(c, HB_EINVAL, "bad layer");
  const size_t n = (size_t)c->cfg.n_experts * c->cfg.hidden * 2;
  CUDA_TRY(c, cudaSetDevice(c->device));
  // host copy: finiteness check and the row norms of the fused router's error bound
  std::vector<uint16_t> hw(n / 2);
  CUDA_TRY(c, cudaMemcpy(hw.data(), w, n, on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
  const int E = c->cfg.n_experts, H = c->cfg.hidden;
  std::vector<float> wn(E);
  for (int e = 0; e < E; ++e) {
    double ss = 0.0;
    for (int i = 0; i < H; ++i) {
      const uint16_t b = hw[(size_t)e * H + i];
      if ((b & 0x7C00) == 0x7C00) return fail(c, HB_EINVAL, "router weights must be finite");
      const int ex = (b >> 10) & 0x1F, man = b & 0x3FF;
      const double v = ex ? std::ldexp((double)(man | 0x400), ex - 25) : std::ldexp((double)man, -24);
      ss += v * v;
    }
    wn[e] = (float)(std::sqrt(ss) * (1.0 + 1e-9)) * (1.0f + 1e-6f);   // rounded up
  }
  CUDA_TRY(c, cudaMemcpy((uint8_t*)c->wg + (size_t)layer * n, w, n,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy(c->wnorm + (size_t)layer * E, wn.data(), 4 * E, cudaMemcpyHostToDevice));
  c->router_set[layer] = 1;
  return HB_OK;
}

// a blob in device memory (library-owned), converted from the canonical
// layout when asked: src is host or device memory of nbytes
static int copy_to_device(hb_ctx* c, const void* src, bool src_host, bool canonical,
                          size_t nbytes, int enc, uint8_t** out) {
  uint8_t* dst = nullptr;
  if (cudaMalloc((void**)&dst, nbytes) != cudaSuccess) return fail(c, HB_ENOMEM, "device blob allocation failed");
  uint8_t* tmp = nullptr;
  cudaError_t e = cudaSuccess;
  if (!canonical) {
    e = cudaMemcpy(dst, src, nbytes, src_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice);
  } else {
    const uint8_t* csrc = (const uint8_t*)src;
    if (src_host) {
      e = cudaMalloc((void**)&tmp, nbytes);
      if (e == cudaSuccess) e = cudaMemcpy(tmp, src, nbytes, cudaMemcpyHostToDevice);
      csrc = tmp;
    }
    if (e == cudaSuccess &&
        launch_repack_canonical(enc, c->cfg.hidden, c->cfg.ffn, csrc, dst, nullptr) != HB_OK)
      e = cudaErrorLaunchFailure;
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (tmp) cudaFree(tmp);
  if (e != cudaSuccess) {
    cudaFree(dst);
    return fail(c, HB_ECUDA, std::string("blob copy / repack: ") + cudaGetErrorString(e));
  }
  *out = dst;
  return HB_OK;
}

int hb_register_expert(hb_ctx* c, int layer, int expert, int enc, const void* blob,
                       size_t nbytes, int flags) {
  if (!c || !blob) return fail(c, HB_EINVAL, "null argument");
  const hb_config& k = c->cfg;
  const int enc_ext = enc;                      // the caller's encoding (repack format)
  if (enc == HB_Q2K) {
    if (!c->kq) return fail(c, HB_EINVAL, "HB_Q2K blob for a context without HB_Q2K");
    enc = HB_Q2;
  } else if (enc == HB_Q2 && c->kq) {
    return fail(c, HB_EINVAL, "this context's low-bit encoding is HB_Q2K");
  }
  if (layer < 0 || layer >= k.n_layers || expert < 0 || expert >= k.n_experts)
    return fail(c, HB_EINVAL, "bad layer / expert");
  if (enc != k.hi_enc && enc != k.lo_enc) return fail(c, HB_EINVAL, "encoding is neither hi_enc nor lo_enc");
  if (nbytes != c->bbytes[enc]) return fail(c, HB_EINVAL, "blob size != hb_blob_bytes(enc, H, F)");
  if (expert % k.world != k.rank) return fail(c, HB_EINVAL, "expert not owned by this rank");
  const bool canonical = (flags & HB_REG_CANONICAL) != 0;
  const int mode = flags & ~HB_REG_CANONICAL;
  const size_t idx = ((size_t)layer * k.n_experts + expert) * 4 + enc;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->resident) {
    const uint8_t* dblob = (const uint8_t*)blob;
    if (mode == HB_REG_DEVICE_BORROW) {
      if (canonical) return fail(c, HB_EINVAL, "a borrowed blob must be in the device layout");
    } else if (mode == HB_REG_DEVICE_COPY || mode == HB_REG_HOST_COPY) {
      uint8_t* owned = nullptr;
      if (int rc = copy_to_device(c, blob, mode == HB_REG_HOST_COPY, canonical, nbytes, enc_ext, &owned))
        return rc;
      c->dev_owned.push_back(owned);
      dblob = owned;
    } else {
      return fail(c, HB_EINVAL, "resident mode takes HB_REG_DEVICE_BORROW / DEVICE_COPY / HOST_COPY");
    }
    c->dev_blob[idx] = dblob;
    if (c->k3_tmap) {                           // K3: TMA tensor maps of W1, W3, W2
      CUtensorMap m[6];
      std::memset(m, 0, sizeof(m));
      const int rows[3] = {k.ffn, k.ffn, k.hidden}, cols[3] = {k.hidden, k.hidden, k.ffn};
      for (int i = 0; i < 3; ++i) {
        const MatLayout& ML = c->lay[enc].mat[i];
        const int rc = enc == HB_F16 ? k3_encode_f16_map(&m[i], dblob + ML.q, rows[i], cols[i])
                                     : k3_encode_q_maps(&m[i], &m[3 + i], enc_ext, dblob + ML.q,
                                                        dblob + ML.s, rows[i], cols[i]);
        if (rc) return fail(c, HB_ECUDA, "cuTensorMapEncodeTiled failed");
      }
      CUDA_TRY(c, cudaMemcpy(c->k3_tmap + (((size_t)layer * k.n_experts + expert) * 4 + enc) * 6, m,
                             sizeof(m), cudaMemcpyHostToDevice));
    }
    CUDA_TRY(c, cudaMemcpy(c->dev_blob_table + idx, &c->dev_blob[idx], sizeof(void*),
                           cudaMemcpyHostToDevice));
    return HB_OK;
  }
  if (mode == HB_REG_HOST_PINNED) {
    if (canonical) return fail(c, HB_EINVAL, "a borrowed blob must be in the device layout");
    c->host_blob[idx] = (const uint8_t*)blob;
  } else if (mode == HB_REG_HOST_COPY) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, nbytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
      return fail(c, HB_ENOMEM, "pinned arena allocation failed");
    if (canonical) {                            // convert on the device, back into the arena
      uint8_t* dev = nullptr;
      if (int rc = copy_to_device(c, blob, true, true, nbytes, enc_ext, &dev)) {
        cudaFreeHost(p);
        return rc;
      }
      const cudaError_t e = cudaMemcpy(p, dev, nbytes, cudaMemcpyDeviceToHost);
      cudaFree(dev);
      if (e != cudaSuccess) {
        cudaFreeHost(p);
        return fail(c, HB_ECUDA, "arena copy-back failed");
      }
    } else {
      std::memcpy(p, blob, nbytes);
    }
    c->arena.push_back(p);
    c->host_blob[idx] = (const uint8_t*)p;
  } else {
    return fail(c, HB_EINVAL, "offload mode takes HB_REG_HOST_PINNED / HB_REG_HOST_COPY");
  }
  if (c->dc) {                                  // SM copies read the blob through its mapping
    void* dptr = nullptr;
    if (cudaHostGetDevicePointer(&dptr, (void*)c->host_blob[idx], 0) != cudaSuccess || !dptr) {
      cudaGetLastError();
      return fail(c, HB_EUNSUPPORTED, "device_cache needs mapped pinned host blobs");
    }
    CUDA_TRY(c, cudaMemcpy(c->host_blob_dev + idx, &dptr, sizeof(void*), cudaMemcpyHostToDevice));
  }
  return HB_OK;
}

static int pf_top_up(hb_ctx* c);

int hb_token_begin(hb_ctx* c) {
  if (!c) return fail(nullptr, HB_EINVAL, "null ctx");
  if (c->cache) {
    if (int rc = pf_top_up(c)) return rc;
  }
  if (c->cache) c->cache->token_begin();
  c->dc_tadd += 1;                              // device cache: applied by the next cache op
  c->dc_clear = 1;
  c->token_started = true;
  return HB_OK;
}

int hb_reset_sequence(hb_ctx* c) {
  if (!c) return fail(nullptr, HB_EINVAL, "null ctx");
  if (c->cache) c->cache->reset_sequence();
  c->dc_reset = 1;
  c->dc_tadd = 0;
  // T = 0 after a reset: Eq. 3 divides by T, so the next forward needs
  // hb_token_begin first (T >= 1)
  c->token_started = false;
  return HB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- internals
static RouterParams router_params(hb_ctx* c, const void* x, int batch) {
  const hb_config& k = c->cfg;
  RouterParams p{};
  p.x = (const __half*)x;
  p.B = batch;
  p.E = k.n_experts;
  p.H = k.hidden;
  p.F = k.ffn;
  p.k = k.top_k;
  p.theta1 = hb_theta(k.t1, &p.th1_kind);
  p.theta2 = hb_theta(k.t2, &p.th2_kind);
  p.t1 = k.t1;
  p.t2 = k.t2;
  p.rank = k.rank;
  p.world = k.world;
  p.strict = k.strict || !k.allow_upgrade || !c->resident;
  p.hi_enc = k.hi_enc;
  p.lo_enc = k.lo_enc;
  p.jt = c->jt;
  p.done = c->done;
  p.lbuf = c->lbuf;
  p.rowbad = c->rowbad;
  p.stamps = c->stamps_on ? c->stamps : nullptr;
  p.stamp_cap = c->stamp_cap;
  p.fwd_idx = c->fwd_idx;
  return p;
}

static float* au_buf(hb_ctx* c, int i) {
  return c->au + (size_t)i * c->max_slots * 2 * c->cfg.ffn;
}

static GemvParams gemv_params(hb_ctx* c, int batch, void* y, float* au) {
  const hb_config& k = c->cfg;
  GemvParams g{};
  g.jt = c->jt;
  for (int e = 0; e < 4; ++e) g.lay[e] = c->lay[e];
  g.H = k.hidden;
  g.F = k.ffn;
  g.B = batch;
  g.k = k.top_k;
  g.x_perm = c->x_perm;
  g.xsum = c->xsum;
  g.au = au;
  g.h_hi = c->h_hi;
  g.h_lo = c->h_lo;
  g.hsum = c->hsum;
  // K2b builds h in each CTA's shared memory when every possible slot fits
  // K2b stages one column slice of h per CTA group (one group per vjob and
  // slice; 2 slices when a slice has an even number of groups) when the slots
  // of any vjob fit the stage and every sub-space can get a CTA
  const int max_ns = std::min(kVSlots, batch);
  const int nv_bound = std::min(2 * k.n_experts, batch * k.top_k) +
                       (batch * k.top_k + kVSlots - 1) / kVSlots;
  bool fits = true;
  for (int enc : {k.hi_enc, k.lo_enc}) {
    const int G = k.ffn / epg_of_enc(enc), nh = G % 4 == 0 ? 2 : 1;
    const size_t slice = (size_t)(k.ffn / nh) * 4 + (size_t)(k.ffn / nh / 32) * 4;
    fits = fits && (size_t)max_ns * slice <= (size_t)w2_stage_capacity();
  }
  g.h_global = c->force_h_global || !fits || 2 * nv_bound > kGemvCTAs;
  g.y = (float*)y;
  g.rowbad = c->rowbad;
  g.hfin_tail = c->hfin_tail;
  g.kq = c->kq;
  g.ctas = kGemvCTAs;
  g.clean = !c->hfin_tail;                   // hfin leaves the K2a sums clean, zeroes y
  g.gbar = c->gbar;
  g.ctr = c->gctr;
  g.max_vjobs = c->max_vjobs;
  g.static_frac = c->static_frac;
  g.static_frac2 = c->static_frac2;
  if (k.deterministic) {                     // whole tiles per warp, no column slices of h
    g.det = 1;
    g.h_global = 1;
    g.static_frac = g.static_frac2 = 1.f;
  }
  g.chunk = c->chunk;
  for (int e = 0; e < 4; ++e) g.k2b_w[e] = c->k2b_w[e];
  g.stamps = c->stamps_on ? c->stamps : nullptr;
  g.stamp_cap = c->stamp_cap;
  g.fwd_idx = c->fwd_idx;
  return g;
}

// The legacy GEMV chain's K2a-sum buffer: the router grid zeroes the one it
// uses (the current buffer; the legacy chain keeps using it).  The fused
// kernel switches to the other one, which it expects clean.
static int legacy_au(hb_ctx* c, RouterParams& rp, int batch) {
  const int cn = c->au_cur;
  rp.zero_buf[0] = au_buf(c, cn);
  rp.zero_n[0] = (long long)batch * c->cfg.top_k * 2 * c->cfg.ffn;
  rp.zero_buf[2] = nullptr;
  rp.zero_n[2] = 0;
  c->au_dirty[cn] = rp.zero_n[0];
  return cn;
}

// Fused decode kernel (batch 1): router + K2a + K2b in one launch.  Uses the
// sum buffer the previous GEMV forward did not use (clean) and zeroes the
// other one for the next forward.
static int launch_fused_forward(hb_ctx* c, int layer, const void* x, void* y, cudaStream_t s) {
  const hb_config& k = c->cfg;
  const int cn = c->au_cur ^ 1;
  if (c->au_dirty[cn])                       // not expected: every GEMV forward leaves it clean
    CUDA_TRY(c, cudaMemsetAsync(au_buf(c, cn), 0, (size_t)c->au_dirty[cn] * 4, s));
  FusedParams fp{};
  fp.g = gemv_params(c, 1, y, au_buf(c, cn));
  fp.g.x_raw = (const __half*)x;
  fp.wg = c->wg + (size_t)layer * k.n_experts * k.hidden;
  fp.blob_table = c->dev_blob_table + (size_t)layer * k.n_experts * 4;
  fp.E = k.n_experts;
  fp.wnorm = c->wnorm + (size_t)layer * k.n_experts;
  fp.theta1 = hb_theta(k.t1, &fp.th1_kind);
  fp.theta2 = hb_theta(k.t2, &fp.th2_kind);
  fp.rank = k.rank;
  fp.world = k.world;
  fp.hi_enc = k.hi_enc;
  fp.lo_enc = k.lo_enc;
  fp.dec = c->dec;
  fp.x_save = c->x_save;
  fp.zero_other = au_buf(c, cn ^ 1);
  fp.zero_n = c->au_dirty[cn ^ 1];
  fp.gbar = c->gbar;
  fp.stamps = fp.g.stamps;
  fp.stamp_cap = fp.g.stamp_cap;
  fp.fwd_idx = fp.g.fwd_idx;
  const GemvParams gp2 = fp.g;               // split mode: hfin + K2b (legacy) stamp through it
  fp.g.stamps = nullptr;                     // the fused kernel stamps through fp
  cudaEvent_t* ev = nullptr;
  if (c->prof_n < c->prof_max) ev = &c->prof_ev[3 * c->prof_n++];
  if (ev) cudaEventRecord(ev[0], s);
  fp.router_only = c->fused_router;
  launch_fused(fp, c->fused_split, s);
  if (c->fused_router) {
    launch_w13(gp2, s);
    c->launches += 1;
  }
  if (c->fused_split || c->fused_router) {
    launch_hfin(gp2, 2, s);
    if (ev) cudaEventRecord(ev[1], s);
    launch_w2(gp2, s);
    c->launches += 2;
    if (ev) cudaEventRecord(ev[2], s);
  } else if (ev) {
    cudaEventRecord(ev[1], s);
    cudaEventRecord(ev[2], s);
  }
  c->au_dirty[cn ^ 1] = 0;
  c->au_dirty[cn] = (long long)2 * 2 * k.ffn;      // top-2: at most two slots
  c->au_cur = cn;
  c->launches += 1;
  return HB_OK;
}

// K2a + K2b, bracketed by timing events when hb_profile is on
static void launch_gemv(hb_ctx* c, const GemvParams& gp, cudaStream_t s) {
  cudaEvent_t* ev = nullptr;
  if (c->prof_n < c->prof_max) ev = &c->prof_ev[3 * c->prof_n++];
  if (ev) cudaEventRecord(ev[0], s);
  launch_w13(gp, s);
  if (!gp.hfin_tail) {
    launch_hfin(gp, c->last_batch * c->cfg.top_k, s);
    c->launches += 1;
  }
  if (ev) cudaEventRecord(ev[1], s);
  launch_w2(gp, s);
  if (ev) cudaEventRecord(ev[2], s);
  c->launches += 2;
}

// A10: sum this rank's partial y over the EP ranks (in place, on the stream)
static int ep_reduce(hb_ctx* c, void* y, int batch, cudaStream_t s) {
  if (!c->nccl_comm) return HB_OK;
  const int r = nccl_api().all_reduce(y, y, (size_t)batch * c->cfg.hidden, kNcclFloat32, kNcclSum,
                                      c->nccl_comm, s);
  if (r != 0)
    return fail(c, HB_ENCCL, std::string("ncclAllReduce: ") +
                                 (nccl_api().error_string ? nccl_api().error_string(r) : "error"));
  return HB_OK;
}

// K3 chain (batched decode / prefill): vjob3 table + X gather, K3a, K3b
static void launch_batched(hb_ctx* c, int layer, const void* x, void* y, cudaStream_t s) {
  K3Params kp{};
  kp.jt = c->jt;
  for (int e = 0; e < 4; ++e) kp.lay[e] = c->lay[e];
  kp.H = c->cfg.hidden;
  kp.F = c->cfg.ffn;
  kp.ks = c->k3_ks;
  kp.xg = c->k3_xg;
  kp.hB = c->k3_hB;
  kp.y = (float*)y;
  kp.rowbad = c->rowbad;
  kp.B = c->last_batch;
  kp.tab = c->k3_tab;
  kp.tmap = c->k3_tmap + (size_t)layer * c->cfg.n_experts * 24;
  kp.has_f16 = c->cfg.hi_enc == HB_F16 || c->cfg.lo_enc == HB_F16;
  kp.has_q = c->cfg.hi_enc != HB_F16 || c->cfg.lo_enc != HB_F16;
  kp.ts = c->k3_ts;
  kp.kq = c->kq;
  cudaEvent_t* ev = nullptr;
  if (c->prof_n < c->prof_max) ev = &c->prof_ev[3 * c->prof_n++];
  launch_k3_prep(kp, (const __half*)x, s);
  if (ev) cudaEventRecord(ev[0], s);
  launch_k3a(kp, s);
  if (ev) cudaEventRecord(ev[1], s);
  launch_k3b(kp, s);
  if (ev) cudaEventRecord(ev[2], s);
  c->launches += 1 + 2 * (kp.has_f16 + kp.has_q);
}

static const __half* router_of(hb_ctx* c, int layer) {
  return c->wg + (size_t)layer * c->cfg.n_experts * c->cfg.hidden;
}

// ---- copies of expert loads (the Dynamic Expert Loader)
static int pf_issue_chunk(hb_ctx* c, hb_ctx::PfLoad& L) {
  const size_t n = std::min(c->pf_chunk, L.total - L.issued);
  if (L.issued == 0)   // WAR: every earlier reader of the slot is done before it is overwritten
    CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->slot_free[L.pool][L.slot], 0));
  CUDA_TRY(c, cudaMemcpyAsync(L.dst + L.issued, L.src + L.issued, n, cudaMemcpyHostToDevice,
                              c->copy_stream));
  L.issued += n;
  c->copied[1] += n;
  cudaEvent_t ev;
  if (c->pf_event_pool.empty()) {
    CUDA_TRY(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  } else {
    ev = c->pf_event_pool.back();
    c->pf_event_pool.pop_back();
  }
  CUDA_TRY(c, cudaEventRecord(ev, c->copy_stream));
  c->pf_inflight.emplace_back(ev, n);
  if (L.issued == L.total) CUDA_TRY(c, cudaEventRecord(c->slot_ready[L.pool][L.slot], c->copy_stream));
  return HB_OK;
}

// keep up to pf_window bytes of prefetch chunks in flight on the copy stream
static int pf_top_up(hb_ctx* c) {
  size_t busy = 0;
  std::vector<std::pair<cudaEvent_t, size_t>> keep;
  for (auto& pe : c->pf_inflight) {
    if (cudaEventQuery(pe.first) == cudaSuccess) {
      c->pf_event_pool.push_back(pe.first);
    } else {
      busy += pe.second;
      keep.push_back(pe);
    }
  }
  c->pf_inflight.swap(keep);
  while (!c->pf_queue.empty() && (busy < c->pf_window || c->pf_window == 0)) {
    hb_ctx::PfLoad& L = c->pf_queue.front();
    const size_t before = L.issued;
    if (int rc = pf_issue_chunk(c, L)) return rc;
    busy += L.issued - before;
    if (L.issued == L.total) c->pf_queue.erase(c->pf_queue.begin());
  }
  return HB_OK;
}

// a queued prefetch into (pool, slot): issue the rest now (a hit needs the
// data) or drop it (the slot is being reused for another key)
static int pf_settle(hb_ctx* c, int pool, int slot, bool issue) {
  for (size_t i = 0; i < c->pf_queue.size(); ++i) {
    hb_ctx::PfLoad& L = c->pf_queue[i];
    if (L.pool != pool || L.slot != slot) continue;
    if (issue)
      while (L.issued < L.total)
        if (int rc = pf_issue_chunk(c, L)) return rc;
    c->pf_queue.erase(c->pf_queue.begin() + i);
    return HB_OK;
  }
  return HB_OK;
}

// queue the host->device copies of the load events [from, end) of the cache
// log: on-demand / explicit loads at once, prefetch loads into the chunk queue
static int issue_loads(hb_ctx* c, size_t from) {
  std::vector<hb_event>& ev = c->cache->events;
  for (size_t i = from; i < ev.size(); ++i) {
    const hb_event& e = ev[i];
    if (e.type != 1) continue;
    const int pool = c->cache->pool_of_enc(e.enc);
    const size_t idx = ((size_t)e.layer * c->cfg.n_experts + e.expert) * 4 + e.enc;
    const uint8_t* src = c->host_blob[idx];
    if (!src) return fail(c, HB_ESTATE, "expert blob not registered for a load");
    uint8_t* dst = c->pool_mem[pool] + (size_t)e.slot * c->slot_bytes[pool];
    if (int rc = pf_settle(c, pool, e.slot, false)) return rc;   // reused: drop its queued prefetch
    if (e.kind == 1 && c->pf_window > 0) {
      c->pf_queue.push_back(hb_ctx::PfLoad{pool, e.slot, src, dst, c->bbytes[e.enc], 0});
      continue;
    }
    // WAR: every earlier reader of this slot must be done before it is overwritten
    CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->slot_free[pool][e.slot], 0));
    CUDA_TRY(c, cudaMemcpyAsync(dst, src, c->bbytes[e.enc], cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_TRY(c, cudaEventRecord(c->slot_ready[pool][e.slot], c->copy_stream));
    c->copied[e.kind == 0 ? 0 : 1] += c->bbytes[e.enc];
  }
  return HB_OK;
}

// ------------------------------------------- token-sharded EP (f3)
static int ts_dispatch(hb_ctx* c, int layer, const void* x, int batch, hb_ts_meta* meta,
                       __half* rows, cudaStream_t s) {
  const hb_config& k = c->cfg;
  RouterParams rp = router_params(c, x, batch);
  rp.wg[0] = router_of(c, layer);
  rp.n_route = 1;
  rp.dec = c->ts_dec;
  rp.rowbad = c->ts_rowbad;
  rp.logits = nullptr;
  rp.x_perm = nullptr;
  rp.xsum = nullptr;
  rp.blob_table = nullptr;
  launch_router(rp, s);
  CUDA_TRY(c, cudaMemsetAsync(meta, 0xff, sizeof(hb_ts_meta) * (size_t)k.world * c->ts_C, s));
  TsParams tp{};
  tp.dec = c->ts_dec;
  tp.x = (const __half*)x;
  tp.B = batch;
  tp.k = k.top_k;
  tp.H = k.hidden;
  tp.R = k.world;
  tp.C = c->ts_C;
  tp.pos = c->ts_pos;
  tp.meta_send = meta;
  tp.rows_send = rows;
  launch_ts_pack(tp, s);
  c->launches += 2;
  c->ts_batch = batch;
  CUDA_TRY(c, cudaGetLastError());
  return HB_OK;
}

static int ts_compute(hb_ctx* c, int layer, const hb_ts_meta* meta, const __half* rows, float* ret,
                      cudaStream_t s) {
  const hb_config& k = c->cfg;
  const int n = k.world * c->ts_C;
  RouterParams rp = router_params(c, rows, n);
  rp.strict = 1;
  rp.dec = c->dec;
  rp.x_perm = c->x_perm;
  rp.xsum = c->xsum;
  rp.blob_table = c->dev_blob_table + (size_t)layer * k.n_experts * 4;
  launch_ts_jobs(rp, meta, rows, ret, s);
  c->launches += 1;
  c->last_batch = n;
  c->last_layer = layer;
  c->last_fused = false;
  c->last_filtered = true;                   // no exact logits for hb_get_logits here
  c->last_host_decisions = false;
  if (c->k3_ok && c->k3_min_batch > 0 && n >= c->k3_min_batch) {
    launch_batched(c, layer, rows, ret, s);
  } else {
    const int cn = c->au_cur;
    if (c->au_dirty[cn]) CUDA_TRY(c, cudaMemsetAsync(au_buf(c, cn), 0, (size_t)c->au_dirty[cn] * 4, s));
    c->au_dirty[cn] = 0;
    GemvParams gp = gemv_params(c, n, ret, au_buf(c, cn));
    launch_gemv(c, gp, s);
  }
  CUDA_TRY(c, cudaGetLastError());
  return HB_OK;
}

static int ts_combine(hb_ctx* c, const float* ret, int batch, void* y, cudaStream_t s) {
  TsParams tp{};
  tp.B = batch;
  tp.k = c->cfg.top_k;
  tp.H = c->cfg.hidden;
  tp.R = c->cfg.world;
  tp.C = c->ts_C;
  tp.pos = c->ts_pos;
  tp.ret = ret;
  tp.y = (float*)y;
  tp.rowbad = c->ts_rowbad;
  launch_ts_combine(tp, s);
  c->launches += 1;
  CUDA_TRY(c, cudaGetLastError());
  return HB_OK;
}

// block r of send -> rank r, block r of recv <- rank r (bytes per block)
static int ts_exchange(hb_ctx* c, const void* send, void* recv, size_t block, cudaStream_t s) {
  NcclApi& api = nccl_api();
  if (!api.send || !api.recv || !api.group_start || !api.group_end)
    return fail(c, HB_EUNSUPPORTED, "ncclSend / ncclRecv not found");
  int r = api.group_start();
  for (int q = 0; q < c->cfg.world && r == 0; ++q) {
    r = api.send((const char*)send + q * block, block, kNcclInt8, q, c->nccl_comm, s);
    if (r == 0) r = api.recv((char*)recv + q * block, block, kNcclInt8, q, c->nccl_comm, s);
  }
  const int r2 = api.group_end();
  if (r == 0) r = r2;
  if (r != 0)
    return fail(c, HB_ENCCL, std::string("token-sharded exchange: ") +
                                 (api.error_string ? api.error_string(r) : "error"));
  return HB_OK;
}

static int ts_forward(hb_ctx* c, int layer, const void* x, int batch, void* y, cudaStream_t s) {
  const hb_config& k = c->cfg;
  if (!c->nccl_comm && k.world > 1)
    return fail(c, HB_ESTATE, "token-sharded forward with world > 1 needs hb_nccl_init");
  const size_t nr = (size_t)k.world * c->ts_C;
  if (int rc = ts_dispatch(c, layer, x, batch, c->ts_meta[0], c->ts_rows[0], s)) return rc;
  const int in = c->nccl_comm ? 1 : 0;       // world 1 without NCCL: the send buffers are the input
  if (c->nccl_comm) {
    if (int rc = ts_exchange(c, c->ts_meta[0], c->ts_meta[1], sizeof(hb_ts_meta) * c->ts_C, s)) return rc;
    if (int rc = ts_exchange(c, c->ts_rows[0], c->ts_rows[1], (size_t)c->ts_C * k.hidden * 2, s)) return rc;
  }
  if (int rc = ts_compute(c, layer, c->ts_meta[in], c->ts_rows[in], c->ts_ret[0], s)) return rc;
  if (c->nccl_comm)
    if (int rc = ts_exchange(c, c->ts_ret[0], c->ts_ret[1], (size_t)c->ts_C * k.hidden * 4, s)) return rc;
  (void)nr;
  return ts_combine(c, c->ts_ret[in], batch, y, s);
}

// ------------------------------------------- device-resident cache (f1)
static int dc_create(hb_ctx* c) {
  const hb_config& k = c->cfg;
  const int L = k.n_layers, E = k.n_experts, nk = L * E;
  DcState& h = c->dc_h;
  h.L = L;
  h.E = E;
  h.K = k.top_k;
  h.cap[0] = k.cap_high;
  h.cap[1] = k.cap_low;
  h.w[0] = k.w_lru;
  h.w[1] = k.w_lfu;
  h.w[2] = k.w_lhu;
  h.w[3] = k.w_fld;
  h.random = k.w_lru + k.w_lfu + k.w_lhu + k.w_fld == 0;
  h.hi_enc = k.hi_enc;
  h.lo_enc = k.lo_enc;
  h.upgrade = k.allow_upgrade != 0;
  h.both = k.prefetch_both != 0;
  h.rank = k.rank;
  h.world = k.world;
  h.log_cap = 1 << 16;
  for (int p = 0; p < 2; ++p) {
    h.pool_mem[p] = c->pool_mem[p];
    h.slot_bytes[p] = c->slot_bytes[p];
  }
  for (int e = 0; e < 4; ++e) h.bbytes[e] = c->bbytes[e];
  const char* v = std::getenv("HB_DC_CHUNK_KB");
  if (v) c->dc_chunk = (size_t)std::max(16, std::atoi(v)) << 10;
  v = std::getenv("HB_DC_FG_CTAS");
  if (v) c->dc_fg_ctas = std::min(kGemvCTAs, std::max(1, std::atoi(v)));
  v = std::getenv("HB_DC_BG_CTAS");
  if (v) c->dc_bg_ctas = std::min(kGemvCTAs / 2, std::max(1, std::atoi(v)));
  h.chunk = c->dc_chunk;
  auto dm = [&](void** p, size_t n, int fill) {
    if (cudaMalloc(p, std::max<size_t>(n, 16)) != cudaSuccess) return false;
    return cudaMemset(*p, fill, std::max<size_t>(n, 16)) == cudaSuccess;
  };
  bool ok = true;
  for (int p = 0; p < 2; ++p)
    ok = ok && dm((void**)&h.pool[p], 4 * (size_t)h.cap[p], 0xff) &&
         dm((void**)&h.where[p], 4 * (size_t)nk, 0xff) &&
         dm((void**)&h.task[p], sizeof(DcTask) * h.cap[p], 0);
  ok = ok && dm((void**)&h.R, 8 * (size_t)nk, 0) && dm((void**)&h.F, 8 * (size_t)nk, 0) &&
       dm((void**)&h.H, 8 * (size_t)nk, 0) && dm((void**)&h.mask_exp, 4 * (size_t)nk, 0xff) &&
       dm((void**)&h.masked_keys, 4 * (size_t)nk, 0) && dm((void**)&h.cur, (size_t)nk, 0) &&
       dm((void**)&h.cur_list, 4 * (size_t)kMaxTopK, 0) &&
       dm((void**)&h.log, sizeof(hb_event) * h.log_cap, 0) &&
       dm((void**)&c->host_blob_dev, sizeof(void*) * (size_t)nk * 4, 0) &&
       dm((void**)&c->dc, sizeof(DcState), 0);
  if (!ok) return fail(c, HB_ENOMEM, "device cache allocation failed");
  if (cudaMemcpy(c->dc, &h, sizeof(DcState), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(c, HB_ECUDA, "device cache init failed");
  if (cudaHostAlloc((void**)&c->err_host, 16, cudaHostAllocMapped) != cudaSuccess)
    return fail(c, HB_ENOMEM, "mapped error word allocation failed");
  *c->err_host = 0;
  void* eh = nullptr;
  if (cudaHostGetDevicePointer(&eh, c->err_host, 0) != cudaSuccess)
    return fail(c, HB_ECUDA, "mapped error word has no device address");
  c->err_dev = (int*)eh;
  if (cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming) != cudaSuccess)
    return fail(c, HB_ECUDA, "event creation failed");
  return HB_OK;
}

static int dc_sticky(hb_ctx* c) {
  const int e = *(volatile int*)c->err_host;
  if (!e) return HB_OK;
  return fail(c, e, e == HB_ECAPACITY ? "device cache: a pool was full and every member masked or in use"
                                      : "device cache: forward before hb_token_begin (T = 0)");
}

// one op of the device state machine on stream s (pending token_begin /
// reset_sequence calls ride along)
static int dc_op(hb_ctx* c, int op, int layer, hb_decision* dec, int n_pred, int expert, int enc,
                 cudaStream_t s) {
  DcParams p{};
  p.op = op;
  p.layer = layer;
  p.n_pred = n_pred;
  p.expert = expert;
  p.enc = enc;
  p.do_reset = c->dc_reset;
  p.t_add = c->dc_tadd;
  p.clear_masks = c->dc_clear;
  c->dc_reset = c->dc_tadd = c->dc_clear = 0;
  p.dec = dec;
  p.host_blob = c->host_blob_dev;
  p.jt = c->jt;
  p.H = c->cfg.hidden;
  p.F = c->cfg.ffn;
  p.err_host = c->err_dev;
  CUDA_TRY(c, launch_dc_op(c->dc, p, s));
  c->launches += 1;
  return HB_OK;
}

// background copier on the side stream, forked from s (joined by the next forward)
static int dc_fork_bg(hb_ctx* c, cudaStream_t s) {
  CUDA_TRY(c, cudaEventRecord(c->ev_fork, s));
  CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->ev_fork, 0));
  CUDA_TRY(c, launch_dc_copy_bg(c->dc, c->dc_bg_ctas, c->copy_stream));
  CUDA_TRY(c, cudaEventRecord(c->ev_side, c->copy_stream));
  c->side_pending = true;
  c->launches += 1;
  return HB_OK;
}

static int dc_forward(hb_ctx* c, int layer, RouterParams& rp, void* y, cudaStream_t s) {
  const hb_config& k = c->cfg;
  const int cn = legacy_au(c, rp, 1);
  launch_router(rp, s);
  c->launches += 1;
  if (int rc = dc_op(c, DC_FORWARD, layer, c->dec, 0, 0, 0, s)) return rc;   // raises yield
  if (c->side_pending) {                     // join the (yielding) background copier
    CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_side, 0));
    c->side_pending = false;
  }
  CUDA_TRY(c, launch_dc_copy_fg(c->dc, c->dc_fg_ctas, s));
  c->launches += 1;
  if (layer + 1 < k.n_layers)                // background chunks during K2
    if (int rc = dc_fork_bg(c, s)) return rc;
  GemvParams gp = gemv_params(c, 1, y, au_buf(c, cn));
  gp.ctas = kGemvCTAs - c->dc_bg_ctas;       // the background copier keeps its SMs
  launch_gemv(c, gp, s);
  if (gp.clean) c->au_dirty[cn] = 0;
  c->last_host_decisions = false;
  CUDA_TRY(c, cudaGetLastError());
  return ep_reduce(c, y, 1, s);
}

static int dc_events(hb_ctx* c, hb_event* out, int cap) {
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  DcState h;
  CUDA_TRY(c, cudaMemcpy(&h, c->dc, sizeof(DcState), cudaMemcpyDeviceToHost));
  if (h.log_overflow) return fail(c, HB_ECAPACITY, "device cache event log overflowed (drain it more often)");
  if (int rc = dc_sticky(c)) return rc;
  const int n = std::min(cap, h.log_n);
  if (n > 0) CUDA_TRY(c, cudaMemcpy(out, h.log, sizeof(hb_event) * n, cudaMemcpyDeviceToHost));
  // keep the undrained tail at the front of the log
  if (n < h.log_n) {
    std::vector<hb_event> rest(h.log_n - n);
    CUDA_TRY(c, cudaMemcpy(rest.data(), h.log + n, sizeof(hb_event) * rest.size(), cudaMemcpyDeviceToHost));
    CUDA_TRY(c, cudaMemcpy(h.log, rest.data(), sizeof(hb_event) * rest.size(), cudaMemcpyHostToDevice));
  }
  const int left = h.log_n - n;
  CUDA_TRY(c, cudaMemcpy((char*)c->dc + offsetof(DcState, log_n), &left, sizeof(int), cudaMemcpyHostToDevice));
  return n;
}

static void drain_events(hb_ctx* c) {
  std::vector<hb_event>& ev = c->cache->events;
  c->log.insert(c->log.end(), ev.begin(), ev.end());
  ev.clear();
}

extern "C" {

int moe_layer_forward(hb_ctx* c, int layer, const void* x, int batch, void* y, void* stream) {
  if (!c || !x || !y) return fail(c, HB_EINVAL, "null argument");
  const hb_config& k = c->cfg;
  if (layer < 0 || layer >= k.n_layers) return fail(c, HB_EINVAL, "bad layer");
  if (batch <= 0 || batch > k.max_batch) return fail(c, HB_EINVAL, "batch must be in [1, max_batch]");
  if (((uintptr_t)x & 15) || ((uintptr_t)y & 15))
    return fail(c, HB_EINVAL, "x and y must be 16-byte aligned");
  if (!c->router_set[layer]) return fail(c, HB_ESTATE, "router of this layer not set");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(c, cudaSetDevice(c->device));
  RouterParams rp = router_params(c, x, batch);
  rp.wg[0] = router_of(c, layer);
  rp.n_route = 1;
  rp.dec = c->dec;
  rp.logits = c->logits;
  rp.x_perm = c->x_perm;
  rp.xsum = c->xsum;
  rp.zero_buf[1] = (float*)y;
  rp.zero_n[1] = (long long)batch * k.hidden;

  c->last_batch = batch;
  c->last_layer = layer;

  if (c->ts) return ts_forward(c, layer, x, batch, y, s);
  if (c->resident) {
    rp.blob_table = c->dev_blob_table + (size_t)layer * k.n_experts * 4;
    const bool k3 = c->k3_ok && c->k3_min_batch > 0 && batch >= c->k3_min_batch;
    c->last_host_decisions = false;
    // the filtered routers (exact decisions, logits on demand): batch-1 decode
    // (HB_ROUTER=filtered, diagnostic) and batches of >= 16 tokens (default;
    // HB_ROUTER=exact turns it off)
    if (batch == 1 && k.top_k == 2 && k.n_experts <= 32 && c->router_filtered) rp.filtered = 1;
    if (batch >= 16 && k.top_k == 2 && k.n_experts <= 64 && c->router_batch) rp.filtered_batch = 1;
    if (rp.filtered || rp.filtered_batch) {
      rp.wnorm = c->wnorm + (size_t)layer * k.n_experts;
      rp.x_save = c->x_save;
      rp.logits = nullptr;
    }
    c->last_filtered = rp.filtered || rp.filtered_batch;
    if (!k3 && batch == 1 && c->fused_ok) {
      c->last_fused = true;
      c->last_filtered = false;
      if (int rc = launch_fused_forward(c, layer, x, y, s)) return rc;
      CUDA_TRY(c, cudaGetLastError());
      return ep_reduce(c, y, batch, s);
    }
    c->last_fused = false;
    if (!k3 && batch == 1 && c->router_solo && !c->hfin_tail &&
        router_solo_fits(k.n_experts, k.hidden, k.top_k)) {
      // batch-1 decode: the router on one reserved SM, K2a / K2b on the
      // others; nothing to zero (hfin cleaned the sums of the previous forward)
      const int cn = c->au_cur;
      if (c->au_dirty[cn])
        CUDA_TRY(c, cudaMemsetAsync(au_buf(c, cn), 0, (size_t)c->au_dirty[cn] * 4, s));
      c->au_dirty[cn] = 0;
      rp.wnorm = c->wnorm + (size_t)layer * k.n_experts;
      rp.x_save = c->x_save;
      rp.logits = nullptr;
      c->last_filtered = true;
      launch_router_solo(rp, s);
      c->launches += 1;
      GemvParams gp = gemv_params(c, batch, y, au_buf(c, cn));
      gp.ctas = kGemvCTAs - 1;
      launch_gemv(c, gp, s);
      CUDA_TRY(c, cudaGetLastError());
      return ep_reduce(c, y, batch, s);
    }
    if (k3) rp.zero_n[0] = 0;                          // K3 does not use the K2a sums
    rp.no_vjobs = k3;                                  // ... nor the GEMV vjob table
    const int cn = k3 ? 0 : legacy_au(c, rp, batch);
    launch_router(rp, s);
    c->launches += 1;
    if (k3) {
      launch_batched(c, layer, x, y, s);
    } else {
      GemvParams gp = gemv_params(c, batch, y, au_buf(c, cn));
      launch_gemv(c, gp, s);
      if (gp.clean) c->au_dirty[cn] = 0;
    }
    CUDA_TRY(c, cudaGetLastError());
    return ep_reduce(c, y, batch, s);
  }

  // ---- offload mode: decisions to the host, cache state machine, loads ----
  if (batch != 1) return fail(c, HB_EUNSUPPORTED, "constrained cache supports batch 1 decode (v1)");
  if (!c->token_started) return fail(c, HB_ESTATE, "forward before hb_token_begin");
  rp.blob_table = nullptr;
  c->last_fused = false;
  c->last_filtered = false;
  if (c->dc) {
    if (int rc = dc_sticky(c)) return rc;
    return dc_forward(c, layer, rp, y, s);
  }
  const int cn = legacy_au(c, rp, batch);
  launch_router(rp, s);
  c->launches += 1;
  const int K = k.top_k;
  CUDA_TRY(c, cudaMemcpyAsync(c->dec_host, c->dec, sizeof(hb_decision) * K, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaEventRecord(c->dec_ready, s));
  CUDA_TRY(c, cudaEventSynchronize(c->dec_ready));
  int32_t ex[kMaxTopK];
  uint8_t pr[kMaxTopK], served[kMaxTopK], hit[kMaxTopK];
  int pool[kMaxTopK], slot[kMaxTopK];
  for (int i = 0; i < K; ++i) {
    ex[i] = c->dec_host[i].expert;
    pr[i] = c->dec_host[i].prec;
  }
  const size_t ev0 = c->cache->events.size();
  int rc = c->cache->forward(layer, ex, pr, served, pool, slot, hit);
  if (rc) {
    // inserts made before the failing selection are real: their copies must
    // still be issued, or the cache would map keys to slots holding the
    // victims' weights
    const std::string why = c->cache->err;
    const int lrc = issue_loads(c, ev0);
    drain_events(c);
    return lrc ? lrc : fail(c, rc, why);
  }
  rc = issue_loads(c, ev0);
  drain_events(c);
  if (rc) return rc;
  for (int i = 0; i < K; ++i)               // served slots with a queued prefetch: issue it now
    if (served[i] != HB_ENC_NONE)
      if (int r2 = pf_settle(c, pool[i], slot[i], true)) return r2;
  if (int r2 = pf_top_up(c)) return r2;
  for (int i = 0; i < K; ++i) {
    c->dec_host[i].served_enc = served[i];
    c->dec_host[i].hit = hit[i];
  }
  // Hits compute while the misses load (improving on P:349's
  // "waits for all"): when the layer has both, the hits' K2 chain runs
  // first, waiting only on the hit slots; the misses' chain follows on their
  // ready events and adds into the same y (its hfin leaves y alone).
  bool any_hit = false, any_miss = false;
  for (int i = 0; i < K; ++i)
    if (served[i] != HB_ENC_NONE) (hit[i] ? any_hit : any_miss) = true;
  const bool split = c->hit_first && any_hit && any_miss;
  c->split_fwds += split;
  for (int part = 0; part < (split ? 2 : 1); ++part) {
    auto in_part = [&](int i) {
      return served[i] != HB_ENC_NONE && (!split || (part == 0) == (hit[i] != 0));
    };
    // job table on the host: one job per non-skipped selection of this part
    void* tdev = part ? c->jt2_dev : c->jt_dev;
    uint8_t* jh = (uint8_t*)(part ? c->jt2_host : c->jt_host);
    auto at = [&](const void* p) { return jh + ((const uint8_t*)p - (const uint8_t*)c->jt_dev); };
    int32_t* hdr = (int32_t*)jh;
    Job* jobs = (Job*)at(c->jt.jobs);
    int32_t* stok = (int32_t*)at(c->jt.slot_token);
    float* sgate = (float*)at(c->jt.slot_gate);
    int32_t* tslots = (int32_t*)at(c->jt.tok_slots);
    int nj = 0;
    for (int i = 0; i < K; ++i) {
      tslots[i] = in_part(i) ? nj : -1;
      if (!in_part(i)) continue;
      Job j;
      j.blob = c->pool_mem[pool[i]] + (size_t)slot[i] * c->slot_bytes[pool[i]];
      j.enc = served[i];
      j.expert = ex[i];
      j.n_tok = 1;
      j.slot_off = nj;
      jobs[nj] = j;
      stok[nj] = 0;
      sgate[nj] = c->dec_host[i].gate;
      ++nj;
    }
    hdr[0] = nj;
    hdr[1] = nj;
    hdr[2] = build_vjobs(jobs, nj, k.hidden, k.ffn, (VJobD*)at(c->jt.vjobs),
                         (long long*)at(c->jt.vcum13), (long long*)at(c->jt.vcum2));
    CUDA_TRY(c, cudaMemcpyAsync(tdev, jh, c->jt_bytes, cudaMemcpyHostToDevice, s));
    for (int i = 0; i < K; ++i)
      if (in_part(i)) CUDA_TRY(c, cudaStreamWaitEvent(s, c->slot_ready[pool[i]][slot[i]], 0));
    GemvParams gp = gemv_params(c, batch, y, au_buf(c, cn));
    if (part) {
      gp.jt = c->jt2;
      gp.keep_y = 1;
    }
    launch_gemv(c, gp, s);
    if (gp.clean) c->au_dirty[cn] = 0;
    for (int i = 0; i < K; ++i)
      if (in_part(i)) CUDA_TRY(c, cudaEventRecord(c->slot_free[pool[i]][slot[i]], s));
  }
  c->last_host_decisions = true;
  CUDA_TRY(c, cudaGetLastError());
  return ep_reduce(c, y, batch, s);
}

int expert_cache_load(hb_ctx* c, int layer, int expert, int enc, void* stream) {
  if (!c) return fail(nullptr, HB_EINVAL, "null ctx");
  if (enc == HB_Q2K && c->kq) enc = HB_Q2;
  else if ((enc == HB_Q2 && c->kq) || enc == HB_Q2K)
    return fail(c, HB_EINVAL, "encoding is neither hi_enc nor lo_enc");
  if (c->resident) return fail(c, HB_ESTATE, "expert_cache_load needs a constrained cache");
  const hb_config& k = c->cfg;
  if (layer < 0 || layer >= k.n_layers || expert < 0 || expert >= k.n_experts)
    return fail(c, HB_EINVAL, "bad layer / expert");
  if (expert % k.world != k.rank) return fail(c, HB_EINVAL, "expert not owned by this rank");
  if (c->dc) {
    if (enc != k.hi_enc && enc != k.lo_enc) return fail(c, HB_EINVAL, "encoding is neither hi_enc nor lo_enc");
    if (int rc = dc_sticky(c)) return rc;
    CUDA_TRY(c, cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = dc_op(c, DC_LOAD, layer, nullptr, 0, expert, enc, s)) return rc;
    return dc_fork_bg(c, s);
  }
  const size_t ev0 = c->cache->events.size();
  bool queued = false;
  int rc = c->cache->load(layer, expert, enc, &queued);
  if (rc) return fail(c, rc, c->cache->err);
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (queued) {                    // the copy starts after the caller's work queued on `stream`
    CUDA_TRY(c, cudaEventRecord(c->dec_ready, (cudaStream_t)stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->dec_ready, 0));
  }
  rc = issue_loads(c, ev0);
  drain_events(c);
  if (!rc) rc = pf_top_up(c);
  return rc;
}

int prefetch_next_layer(hb_ctx* c, int layer, const void* x, int batch, void* stream) {
  if (!c || !x) return fail(c, HB_EINVAL, "null argument");
  const hb_config& k = c->cfg;
  if (layer < 0 || layer >= k.n_layers) return fail(c, HB_EINVAL, "bad layer");
  if (c->resident) return 0;
  if (batch != 1) return fail(c, HB_EUNSUPPORTED, "prefetch supports batch 1 decode (v1)");
  const int n = std::min(k.lookahead_p, k.n_layers - 1 - layer);
  if (c->dc && n <= 0) {                             // still expires masks
    CUDA_TRY(c, cudaSetDevice(c->device));
    return dc_op(c, DC_PREFETCH, layer, c->dec_pred, 0, 0, 0, (cudaStream_t)stream);
  }
  if (n <= 0) {
    int pl;
    c->cache->prefetch(layer, 0, nullptr, nullptr, &pl);   // still expires masks
    return 0;
  }
  for (int j = 0; j < n; ++j)
    if (!c->router_set[layer + 1 + j]) return fail(c, HB_ESTATE, "router of a lookahead layer not set");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(c, cudaSetDevice(c->device));
  RouterParams rp = router_params(c, x, batch);
  rp.n_route = n;
  for (int j = 0; j < n; ++j) rp.wg[j] = router_of(c, layer + 1 + j);   // Stacking Computer
  rp.dec = c->dec_pred;
  rp.blob_table = nullptr;
  c->last_fused = false;
  c->last_filtered = false;
  const int cn = legacy_au(c, rp, batch);
  launch_router(rp, s);
  c->launches += 1;
  if (c->dc) {                                       // device walk + background loads
    (void)cn;
    if (int rc = dc_op(c, DC_PREFETCH, layer, c->dec_pred, n, 0, 0, s)) return rc;
    if (int rc = dc_fork_bg(c, s)) return rc;
    return 0;
  }
  const int K = k.top_k;
  hb_decision* hd = c->dec_host + K;                 // after the forward's record
  CUDA_TRY(c, cudaMemcpyAsync(hd, c->dec_pred, sizeof(hb_decision) * n * K, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaEventRecord(c->dec_ready, s));
  CUDA_TRY(c, cudaEventSynchronize(c->dec_ready));
  std::vector<int32_t> ex(n * K);
  std::vector<uint8_t> pr(n * K);
  for (int i = 0; i < n * K; ++i) {
    ex[i] = hd[i].expert;
    pr[i] = hd[i].prec;
  }
  const size_t ev0 = c->cache->events.size();
  int pl = -1;
  int rc = c->cache->prefetch(layer, n, ex.data(), pr.data(), &pl);
  if (rc) {                                          // issue the inserts made so far
    const std::string why = c->cache->err;
    const int lrc = issue_loads(c, ev0);
    drain_events(c);
    return lrc ? lrc : fail(c, rc, why);
  }
  int queued = 0;
  for (size_t i = ev0; i < c->cache->events.size(); ++i) queued += c->cache->events[i].type == 1;
  rc = issue_loads(c, ev0);
  drain_events(c);
  if (!rc) rc = pf_top_up(c);
  return rc ? rc : queued;
}

int hb_get_decisions(hb_ctx* c, hb_decision* out, int cap) {
  if (!c || (cap > 0 && !out)) return fail(c, HB_EINVAL, "null argument");
  const int n = std::min(cap, c->last_batch * c->cfg.top_k);
  if (n <= 0) return 0;
  if (c->last_host_decisions) {
    std::memcpy(out, c->dec_host, sizeof(hb_decision) * n);
  } else {
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaDeviceSynchronize());
    CUDA_TRY(c, cudaMemcpy(out, c->dec, sizeof(hb_decision) * n, cudaMemcpyDeviceToHost));
  }
  if (c->kq)                                    // the Q2 slot holds HB_Q2K
    for (int i = 0; i < n; ++i)
      if (out[i].served_enc == HB_Q2) out[i].served_enc = HB_Q2K;
  return n;
}

int hb_get_logits(hb_ctx* c, int64_t* out, int cap_pairs) {
  if (!c || (cap_pairs > 0 && !out)) return fail(c, HB_EINVAL, "null argument");
  const int n = std::min(cap_pairs, c->last_batch * c->cfg.n_experts);
  if (n <= 0) return 0;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  if (c->last_fused || c->last_filtered) {
    // the fused kernel decides without materialising the exact logits: run
    // the exact router on its saved copy of x (inspection only)
    RouterParams rp = router_params(c, c->x_save, c->last_batch);
    rp.wg[0] = router_of(c, c->last_layer);
    rp.n_route = 1;
    rp.dec = c->dec_pred;
    rp.logits = c->logits;
    launch_router(rp, nullptr);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaDeviceSynchronize());
  }
  CUDA_TRY(c, cudaMemcpy(out, c->logits, sizeof(long long) * 2 * n, cudaMemcpyDeviceToHost));
  return n;
}

int hb_get_events(hb_ctx* c, hb_event* out, int cap) {
  if (!c || (cap > 0 && !out)) return fail(c, HB_EINVAL, "null argument");
  int n;
  if (c->dc) {
    n = dc_events(c, out, cap);
    if (n < 0) return n;
  } else {
    n = std::min<int>(cap, (int)c->log.size());
    for (int i = 0; i < n; ++i) out[i] = c->log[i];
    c->log.erase(c->log.begin(), c->log.begin() + n);
  }
  if (c->kq)
    for (int i = 0; i < n; ++i)
      if (out[i].enc == HB_Q2) out[i].enc = HB_Q2K;
  return n;
}

int hb_copy_stats(hb_ctx* c, uint64_t* out) {
  if (!c || !out) return fail(c, HB_EINVAL, "null argument");
  if (c->dc) {
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaDeviceSynchronize());
    DcState h;
    CUDA_TRY(c, cudaMemcpy(&h, c->dc, sizeof(DcState), cudaMemcpyDeviceToHost));
    out[0] = h.bytes_fg;
    out[1] = h.bytes_bg;
  } else {
    out[0] = c->copied[0];
    out[1] = c->copied[1];
  }
  return HB_OK;
}

int hb_ts_buffer_bytes(hb_ctx* c, size_t* meta_bytes, size_t* rows_bytes, size_t* ret_bytes) {
  if (!c) return fail(nullptr, HB_EINVAL, "null ctx");
  if (!c->ts) return fail(c, HB_ESTATE, "context is not token-sharded");
  const size_t nr = (size_t)c->cfg.world * c->ts_C;
  if (meta_bytes) *meta_bytes = sizeof(hb_ts_meta) * nr;
  if (rows_bytes) *rows_bytes = nr * c->cfg.hidden * 2;
  if (ret_bytes) *ret_bytes = nr * c->cfg.hidden * 4;
  return HB_OK;
}

static int ts_check(hb_ctx* c, int layer) {
  if (!c) return fail(nullptr, HB_EINVAL, "null ctx");
  if (!c->ts) return fail(c, HB_ESTATE, "context is not token-sharded");
  if (layer < 0 || layer >= c->cfg.n_layers) return fail(c, HB_EINVAL, "bad layer");
  if (!c->router_set[layer]) return fail(c, HB_ESTATE, "router of this layer not set");
  return HB_OK;
}

int hb_ts_dispatch(hb_ctx* c, int layer, const void* x, int batch, void* meta_send, void* rows_send,
                   void* stream) {
  if (int rc = ts_check(c, layer)) return rc;
  if (!x || !meta_send || !rows_send) return fail(c, HB_EINVAL, "null argument");
  if (batch <= 0 || batch > c->cfg.max_batch) return fail(c, HB_EINVAL, "batch must be in [1, max_batch]");
  if (((uintptr_t)x & 15) || ((uintptr_t)rows_send & 15)) return fail(c, HB_EINVAL, "x / rows must be 16-byte aligned");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return ts_dispatch(c, layer, x, batch, (hb_ts_meta*)meta_send, (__half*)rows_send, (cudaStream_t)stream);
}

int hb_ts_compute(hb_ctx* c, int layer, const void* meta_recv, const void* rows_recv, void* ret_send,
                  void* stream) {
  if (int rc = ts_check(c, layer)) return rc;
  if (!meta_recv || !rows_recv || !ret_send) return fail(c, HB_EINVAL, "null argument");
  if (((uintptr_t)rows_recv & 15) || ((uintptr_t)ret_send & 15)) return fail(c, HB_EINVAL, "buffers must be 16-byte aligned");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return ts_compute(c, layer, (const hb_ts_meta*)meta_recv, (const __half*)rows_recv, (float*)ret_send,
                    (cudaStream_t)stream);
}

int hb_ts_combine(hb_ctx* c, const void* ret_recv, int batch, void* y, void* stream) {
  if (!c) return fail(nullptr, HB_EINVAL, "null ctx");
  if (!c->ts) return fail(c, HB_ESTATE, "context is not token-sharded");
  if (!ret_recv || !y) return fail(c, HB_EINVAL, "null argument");
  if (batch != c->ts_batch) return fail(c, HB_ESTATE, "combine needs the dispatch of the same batch");
  if (((uintptr_t)ret_recv & 15) || ((uintptr_t)y & 15)) return fail(c, HB_EINVAL, "buffers must be 16-byte aligned");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return ts_combine(c, (const float*)ret_recv, batch, y, (cudaStream_t)stream);
}

int hb_last_expert_bytes(hb_ctx* c, uint64_t* out) {
  if (!c || !out) return fail(c, HB_EINVAL, "null argument");
  std::vector<hb_decision> d(c->last_batch * c->cfg.top_k);
  int n = hb_get_decisions(c, d.data(), (int)d.size());
  if (n < 0) return n;
  // one stream of each served (expert, enc) per forward
  std::vector<char> seen((size_t)c->cfg.n_experts * 4, 0);
  uint64_t tot = 0;
  for (int i = 0; i < n; ++i) {
    if (d[i].served_enc == HB_ENC_NONE) continue;
    const int se = d[i].served_enc == HB_Q2K ? HB_Q2 : d[i].served_enc;
    const size_t key = (size_t)d[i].expert * 4 + se;
    if (seen[key]) continue;
    seen[key] = 1;
    tot += c->bbytes[se];
  }
  *out = tot;
  return HB_OK;
}

int hb_nccl_unique_id(void* out) {
  if (!out) return fail(nullptr, HB_EINVAL, "null argument");
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(nullptr, HB_EUNSUPPORTED, "libnccl.so.2 not found (HB_NCCL_LIB)");
  NcclId id;
  const int r = api.get_unique_id(&id);
  if (r != 0) return fail(nullptr, HB_ENCCL, "ncclGetUniqueId failed");
  std::memcpy(out, &id, sizeof(id));
  return HB_OK;
}

static int nccl_init_ranks(hb_ctx* c, const void* unique_id, int nranks, int rank);

int hb_nccl_init(hb_ctx* c, const void* unique_id) {
  if (!c || !unique_id) return fail(c, HB_EINVAL, "null argument");
  return nccl_init_ranks(c, unique_id, c->cfg.world, c->cfg.rank);
}

int hb_nccl_init_ranks(hb_ctx* c, const void* unique_id, int nranks, int rank) {
  if (!c || !unique_id) return fail(c, HB_EINVAL, "null argument");
  if (nranks <= 0 || rank < 0 || rank >= nranks) return fail(c, HB_EINVAL, "bad nranks / rank");
  return nccl_init_ranks(c, unique_id, nranks, rank);
}

static int nccl_init_ranks(hb_ctx* c, const void* unique_id, int nranks, int rank) {
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(c, HB_EUNSUPPORTED, "libnccl.so.2 not found (HB_NCCL_LIB)");
  if (c->nccl_comm) return fail(c, HB_ESTATE, "NCCL communicator already initialised");
  NcclId id;
  std::memcpy(&id, unique_id, sizeof(id));
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int r = api.comm_init_rank(&c->nccl_comm, nranks, id, rank);
  if (r != 0) {
    c->nccl_comm = nullptr;
    return fail(c, HB_ENCCL, std::string("ncclCommInitRank: ") +
                                 (api.error_string ? api.error_string(r) : "error"));
  }
  return HB_OK;
}

int hb_ep_broadcast_x(hb_ctx* c, void* x, int batch, int root, void* stream) {
  if (!c || !x) return fail(c, HB_EINVAL, "null argument");
  if (batch <= 0 || batch > c->cfg.max_batch) return fail(c, HB_EINVAL, "batch must be in [1, max_batch]");
  if (root < 0 || root >= c->cfg.world) return fail(c, HB_EINVAL, "bad root rank");
  if (!c->nccl_comm) return fail(c, HB_ESTATE, "hb_nccl_init first");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int r = nccl_api().broadcast(x, x, (size_t)batch * c->cfg.hidden, kNcclFloat16, root,
                                     c->nccl_comm, (cudaStream_t)stream);
  if (r != 0)
    return fail(c, HB_ENCCL, std::string("ncclBroadcast: ") +
                                 (nccl_api().error_string ? nccl_api().error_string(r) : "error"));
  return HB_OK;
}

int hb_set_batched_min(hb_ctx* c, int min_batch) {
  if (!c || min_batch < 0) return fail(c, HB_EINVAL, "bad argument");
  if (min_batch > 0 && !c->k3_ok)
    return fail(c, HB_EUNSUPPORTED, "batched GEMM path needs max_batch > 1 (and <= 64 vjob3 per forward)");
  c->k3_min_batch = min_batch;
  return HB_OK;
}

int hb_launch_count(hb_ctx* c, uint64_t* out) {
  if (!c || !out) return fail(c, HB_EINVAL, "null argument");
  *out = c->launches;
  return HB_OK;
}

int hb_profile(hb_ctx* c, int max_calls) {
  if (!c || max_calls < 0) return fail(c, HB_EINVAL, "bad argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  while ((int)c->prof_ev.size() < 3 * max_calls) {
    cudaEvent_t e;
    CUDA_TRY(c, cudaEventCreate(&e));
    c->prof_ev.push_back(e);
  }
  c->prof_max = max_calls;
  c->prof_n = 0;
  return HB_OK;
}

int hb_profile_read(hb_ctx* c, float* ms, int cap) {
  if (!c || (cap > 0 && !ms)) return fail(c, HB_EINVAL, "bad argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int n = std::min(cap, c->prof_n);
  for (int i = 0; i < n; ++i) {
    CUDA_TRY(c, cudaEventSynchronize(c->prof_ev[3 * i + 2]));
    CUDA_TRY(c, cudaEventElapsedTime(&ms[2 * i], c->prof_ev[3 * i], c->prof_ev[3 * i + 1]));
    CUDA_TRY(c, cudaEventElapsedTime(&ms[2 * i + 1], c->prof_ev[3 * i + 1], c->prof_ev[3 * i + 2]));
  }
  return n;
}

int hb_stamps(hb_ctx* c, int max_forwards) {
  if (!c || max_forwards < 0) return fail(c, HB_EINVAL, "bad argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  if (max_forwards > c->stamp_cap) {
    if (c->stamps) cudaFree(c->stamps);
    c->stamps = nullptr;
    c->stamp_cap = 0;
    CUDA_TRY(c, cudaMalloc((void**)&c->stamps, sizeof(unsigned long long) * kStampStride * (size_t)max_forwards));
    c->stamp_cap = max_forwards;
  }
  if (c->stamps)
    CUDA_TRY(c, cudaMemset(c->stamps, 0, sizeof(unsigned long long) * kStampStride * (size_t)c->stamp_cap));
  CUDA_TRY(c, cudaMemset(c->fwd_idx, 0, 16));
  c->stamps_on = max_forwards > 0;
  return HB_OK;
}

int hb_stamps_read(hb_ctx* c, uint64_t* out, int cap) {
  if (!c || (cap > 0 && !out)) return fail(c, HB_EINVAL, "bad argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  unsigned idx[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpy(idx, c->fwd_idx, 8, cudaMemcpyDeviceToHost));
  const int n = std::min<int>(std::min<int>((int)idx[0], c->stamp_cap), cap);
  if (n <= 0) return 0;
  std::vector<unsigned long long> raw((size_t)n * kStampStride);
  CUDA_TRY(c, cudaMemcpy(raw.data(), c->stamps, raw.size() * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) {
    const unsigned long long* r = &raw[(size_t)i * kStampStride];
    uint64_t* o = out + (size_t)i * 15;
    o[0] = ~r[0];                 // first CTA past griddepcontrol.wait
    o[1] = r[1];                  // last CTA with its decisions / job table
    o[2] = r[2];                  // last CTA done with K2a (grid barrier arrival)
    o[3] = ~r[3];                 // first CTA released by the grid barrier
    o[4] = r[4];                  // last CTA done
    o[5] = r[5];                  // last CTA with the router rows in shared memory
    o[6] = r[6];                  // last CTA with its (filtered) logits
    o[7] = r[7];                  // last CTA past decisions + job table
    o[8] = r[8];                  // last CTA with h staged (fused kernel)
    o[9] = r[9] ? ~r[9] : 0;      // first CTA with h staged (fused kernel)
    for (int j = 10; j < 15; ++j) o[j] = r[j];   // router sub-steps (diagnostic), [14] fallbacks
  }
  return n;
}

int hb_quantize_expert(int enc, int hidden, int ffn, const void* w1, const void* w3, const void* w2,
                       void* blob, void* stream) {
  if (!w1 || !w3 || !w2 || !blob) return fail(nullptr, HB_EINVAL, "null argument");
  int rc = launch_quantize_expert(enc, hidden, ffn, (const __half*)w1, (const __half*)w3,
                                  (const __half*)w2, (uint8_t*)blob, (cudaStream_t)stream);
  if (rc) return fail(nullptr, rc, "quantize failed (bad dims/enc or CUDA error)");
  return HB_OK;
}

int hb_synth_fill_f16(void* dst, size_t n, uint64_t key, float scale, uint64_t start, void* stream) {
  if (!dst) return fail(nullptr, HB_EINVAL, "null argument");
  launch_synth((__half*)dst, n, key, scale, start, (cudaStream_t)stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(nullptr, HB_ECUDA, cudaGetErrorString(e));
  return HB_OK;
}

}  // extern "C"
