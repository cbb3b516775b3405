// Device-resident expert cache manager with GPU-initiated, chunk-preemptible
// expert loads (hb_config.device_cache = 1).
//
// Paper: the two-pool cache and Eq. 3 (Sec. 3.4), the stacked
// next-layer prediction and prefetch walk (Sec. 3.3), and the
// motivation for preemptible loads: "a started cudaMemcpy cannot be
// interrupted", so a wrong prefetch delays the correct load (P:521,
// fig:prefetch).  Readings: DESIGN.md R5, R6, R13-R20, R29.
//
// The same state machine as the host ExpertCache (cache.cpp) -- identical
// event sequence, bit-exact with the oracle's O9/O10 -- but kept in HBM and
// run by a one-thread kernel right after the router, so the offload forward
// never synchronises with the host and can be captured in a CUDA graph.
//
// Loads are done by SMs, not copy engines: every (pool, slot) has one task
// (source = the expert's blob in mapped pinned host memory, destination = the
// slot), cut into chunks that copier CTAs claim one at a time.
//  * foreground (dc_copy_fg, on the forward's stream, before K2): the slots the
//    current forward computes from -- on-demand inserts and hits on a slot
//    whose (prefetch) task is still incomplete -- copied until complete;
//  * background (dc_copy_bg, on the library's side stream): any incomplete
//    task, oldest first, while the link would otherwise idle (during K2, the
//    prefetch routers); it stops claiming chunks as soon as the next forward's
//    cache kernel raises `yield`, so an on-demand load waits for at most one
//    chunk per background CTA instead of a whole mispredicted expert.
//  * a slot whose task is replaced (its key evicted) drops the unclaimed
//    chunks of the old task: the replacement takes the slot exclusively
//    (waits for the copiers holding it -- running CTAs, each finishing one
//    chunk) before the new task is published.
#include <cuda_runtime.h>

#include "dcache.h"

namespace hb {

namespace {

constexpr unsigned kExcl = 0x80000000u;
constexpr int kCopyThreads = 512;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_vol(const int* p) { return *(const volatile int*)p; }

// ------------------------------------------------------------ cache logic
// One thread.  Mirrors ExpertCache (cache.cpp) step for step.
struct Logic {
  DcState& s;
  const DcParams& p;

  __device__ int key(int layer, int e) const { return layer * s.E + e; }
  __device__ bool owned(int e) const { return e % s.world == s.rank; }
  __device__ bool masked(int k) const { return s.mask_exp[k] >= 0; }

  // Eq. 3 scaled by T * l_n * (a+b+c+d): an exact integer (R13)
  __device__ long long priority(int k, int cur_layer) const {
    const long long ln = s.L;
    const int lt = k / s.E;
    const long long dist = ((lt - cur_layer) % s.L + s.L) % s.L;
    return ln * (s.w[0] * s.R[k] + s.w[1] * s.F[k] + s.w[2] * s.H[k]) +
           (long long)s.w[3] * s.T * (ln - dist);
  }
  __device__ static unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __device__ void log(int type, int kind, int layer, int e, int enc, int slot, int victim) {
    if (s.log_n >= s.log_cap) {
      s.log_overflow = 1;
      return;
    }
    hb_event& v = s.log[s.log_n++];
    v.type = type;
    v.kind = kind;
    v.layer = layer;
    v.expert = e;
    v.enc = enc;
    v.slot = slot;
    v.victim = victim;
  }
  __device__ void drop_masks(int upto_layer) {
    int n = 0;
    for (int i = 0; i < s.n_masked; ++i) {
      const int k = s.masked_keys[i];
      if (s.mask_exp[k] <= upto_layer) s.mask_exp[k] = -1;
      else s.masked_keys[n++] = k;
    }
    s.n_masked = n;
  }
  __device__ void use(int k, bool high) {  // R = T, F += 1, H += [High]
    s.R[k] = s.T;
    s.F[k] += 1;
    if (high) s.H[k] += 1;
  }
  // returns the slot or -1; *victim = evicted key or -1
  __device__ int insert(int pool, int k, int cur_layer, bool exclude_current, int* victim) {
    int* slots = s.pool[pool];
    const int cap = s.cap[pool];
    int vs = -1;
    *victim = -1;
    for (int i = 0; i < cap; ++i)
      if (slots[i] < 0) { vs = i; break; }
    if (vs < 0) {
      long long bp = 0;
      unsigned long long br = 0;
      int bk = -1;
      for (int i = 0; i < cap; ++i) {
        const int m = slots[i];
        if (masked(m) || (exclude_current && s.cur[m])) continue;
        if (s.random) {                  // Random policy (all-zero weights, R29)
          const unsigned long long r =
              mix64(mix64(((unsigned long long)s.T << 32) + s.n_evict) + (unsigned long long)m);
          if (bk < 0 || r < br || (r == br && m < bk)) { br = r; bk = m; vs = i; }
          continue;
        }
        const long long pr = priority(m, cur_layer);
        if (bk < 0 || pr < bp || (pr == bp && m < bk)) { bp = pr; bk = m; vs = i; }
      }
      if (bk < 0) return -1;
      *victim = bk;
      ++s.n_evict;
      s.where[pool][bk] = -1;
    }
    slots[vs] = k;
    s.where[pool][k] = vs;
    return vs;
  }
  __device__ bool present(int layer, int e, int prec) const {
    const int k = key(layer, e);
    if (prec == HB_HIGH) return s.where[0][k] >= 0;
    return s.where[1][k] >= 0 || (s.upgrade && s.where[0][k] >= 0);
  }
  // new task for (pool, slot): the blob of (layer, e, enc); waits for the
  // copiers still holding the slot's old task
  __device__ void new_task(int pool, int slot, int layer, int e, int enc, int fg) {
    DcTask& t = s.task[pool][slot];
    atomicOr(&t.rw, kExcl);
    while ((ld_acq(&t.rw) & ~kExcl) != 0) __nanosleep(256);
    const unsigned gen = t.gen + 1;
    t.gen = gen;
    t.src = p.host_blob[((size_t)layer * s.E + e) * 4 + enc];
    t.dst = s.pool_mem[pool] + (size_t)slot * s.slot_bytes[pool];
    t.bytes = s.bbytes[enc];
    t.nchunks = (unsigned)((t.bytes + s.chunk - 1) / s.chunk);
    t.ctl = (unsigned long long)gen << 32;
    t.done = (unsigned long long)gen << 32;
    t.fg = fg;
    t.seq = ++s.seq;
    t.live = 1;
    t.layer = layer;
    t.bg = fg ? 0 : 1;
    __threadfence();
    atomicAnd(&t.rw, ~kExcl);
  }
  __device__ void need(int pool, int slot) {
    for (int i = 0; i < s.n_need; ++i)
      if (s.need[i] == pool * 65536 + slot) return;
    s.need[s.n_need++] = pool * 65536 + slot;
    s.task[pool][slot].fg = 1;
    s.task[pool][slot].bg = 0;
  }
  __device__ void fault(int code) {
    if (!s.err) s.err = code;
    if (p.err_host) *(volatile int*)p.err_host = s.err;
  }

  __device__ void apply_pending() {
    if (p.do_reset) {            // records and T only
      for (int k = 0; k < s.L * s.E; ++k) s.R[k] = s.F[k] = s.H[k] = 0;
      s.T = 0;
    }
    s.T += p.t_add;
    if (p.clear_masks) {         // token_begin: every mask has expired
      for (int i = 0; i < s.n_masked; ++i) s.mask_exp[s.masked_keys[i]] = -1;
      s.n_masked = 0;
    }
  }

  // O9 for one token (batch 1) at p.layer; writes served/hit into dec, the
  // job table, the need list
  __device__ void forward() {
    const int K = s.K, layer = p.layer;
    hb_decision* dec = p.dec;
    int served[kMaxTopK], pool_of[kMaxTopK], slot_of[kMaxTopK];
    s.n_need = 0;
    if (s.T == 0) {              // Eq. 3 divides by T: a forward needs token_begin first
      fault(HB_ESTATE);
      for (int i = 0; i < K; ++i) served[i] = HB_ENC_NONE;
    } else {
      drop_masks(layer - 1);
      for (int i = 0; i < s.n_cur; ++i) s.cur[s.cur_list[i]] = 0;
      s.n_cur = 0;
      for (int i = 0; i < K; ++i) {
        served[i] = HB_ENC_NONE;
        pool_of[i] = slot_of[i] = -1;
        dec[i].hit = 0;
        if (dec[i].prec != HB_SKIP && owned(dec[i].expert)) {
          const int k = key(layer, dec[i].expert);
          if (!s.cur[k]) { s.cur[k] = 1; s.cur_list[s.n_cur++] = k; }
        }
      }
      for (int i = 0; i < K; ++i) {
        const int e = dec[i].expert;
        if (dec[i].prec == HB_SKIP || !owned(e)) continue;
        const int k = key(layer, e);
        int pool, slot, enc, victim;
        if (dec[i].prec == HB_HIGH) {
          pool = 0;
          enc = s.hi_enc;
          slot = s.where[0][k];
          if (slot >= 0) {
            use(k, true);
            log(0, 0, layer, e, enc, slot, -1);
            dec[i].hit = 1;
          } else {
            slot = insert(0, k, layer, true, &victim);
            if (slot < 0) { fault(HB_ECAPACITY); continue; }
            use(k, true);
            log(1, 0, layer, e, enc, slot, victim);
            new_task(0, slot, layer, e, enc, 1);
          }
        } else {
          const int sl = s.where[1][k], sh = s.where[0][k];
          if (sl >= 0) {
            use(k, false);
            pool = 1; enc = s.lo_enc; slot = sl;
            log(0, 0, layer, e, enc, slot, -1);
            dec[i].hit = 1;
          } else if (s.upgrade && sh >= 0) {   // Low served by the High copy
            use(k, true);
            pool = 0; enc = s.hi_enc; slot = sh;
            log(0, 0, layer, e, enc, slot, -1);
            dec[i].hit = 1;
          } else {
            pool = 1;
            enc = s.lo_enc;
            slot = insert(1, k, layer, true, &victim);
            if (slot < 0) { fault(HB_ECAPACITY); continue; }
            use(k, false);
            log(1, 0, layer, e, enc, slot, victim);
            new_task(1, slot, layer, e, enc, 1);
          }
        }
        served[i] = enc;
        pool_of[i] = pool;
        slot_of[i] = slot;
        need(pool, slot);
      }
    }
    // job table: one job per served selection (the host path's table)
    const JobTable& jt = p.jt;
    int nj = 0;
    for (int i = 0; i < K; ++i) {
      dec[i].served_enc = (uint8_t)served[i];
      jt.tok_slots[i] = served[i] == HB_ENC_NONE ? -1 : nj;
      if (served[i] == HB_ENC_NONE) continue;
      Job j;
      j.blob = s.pool_mem[pool_of[i]] + (size_t)slot_of[i] * s.slot_bytes[pool_of[i]];
      j.enc = served[i];
      j.expert = dec[i].expert;
      j.n_tok = 1;
      j.slot_off = nj;
      jt.jobs[nj] = j;
      jt.slot_token[nj] = 0;
      jt.slot_gate[nj] = dec[i].gate;
      ++nj;
    }
    jt.hdr[0] = nj;
    jt.hdr[1] = nj;
    jt.hdr[2] = build_vjobs(jt.jobs, nj, p.H, p.F, jt.vjobs, jt.vcum13, jt.vcum2);
  }

  // O10: the stacked routers' predictions for layers layer+1 .. layer+n
  __device__ void prefetch() {
    const int K = s.K, layer = p.layer;
    drop_masks(layer);
    for (int j = 0; j < p.n_pred; ++j) {
      const int lp = layer + 1 + j;
      if (lp >= s.L) break;
      const hb_decision* d = p.dec + (size_t)j * K;
      bool any_missing = false;
      for (int i = 0; i < K; ++i) {
        if (d[i].prec == HB_SKIP || !owned(d[i].expert)) continue;
        const int k = key(lp, d[i].expert);
        if (s.mask_exp[k] < 0) s.masked_keys[s.n_masked++] = k;
        s.mask_exp[k] = s.mask_exp[k] > lp ? s.mask_exp[k] : lp;
      }
      for (int i = 0; i < K; ++i)
        if (d[i].prec != HB_SKIP && owned(d[i].expert) && !present(lp, d[i].expert, d[i].prec))
          any_missing = true;
      if (!any_missing) continue;
      for (int i = 0; i < K; ++i) {
        if (d[i].prec == HB_SKIP || !owned(d[i].expert) || present(lp, d[i].expert, d[i].prec))
          continue;
        // R30 (both): the Low version, then the High one, each if its pool
        // lacks the key; else the predicted precision only
        int pools[2], np = 0;
        const int kk = key(lp, d[i].expert);
        if (s.both) {
          if (s.where[1][kk] < 0) pools[np++] = 1;
          if (s.where[0][kk] < 0) pools[np++] = 0;
        } else {
          pools[np++] = d[i].prec == HB_HIGH ? 0 : 1;
        }
        for (int q = 0; q < np; ++q) {
          const int pool = pools[q];
          const int enc = pool == 0 ? s.hi_enc : s.lo_enc;
          int victim;
          const int slot = insert(pool, kk, layer, true, &victim);
          if (slot < 0) {
            log(2, 1, lp, d[i].expert, enc, -1, -1);
            continue;
          }
          log(1, 1, lp, d[i].expert, enc, slot, victim);
          new_task(pool, slot, lp, d[i].expert, enc, 0);
        }
      }
      return;
    }
  }

  // expert_cache_load: logical insert without record update (idempotent)
  __device__ void load() {
    const int pool = p.enc == s.hi_enc ? 0 : 1;
    const int k = key(p.layer, p.expert);
    if (s.where[pool][k] >= 0) return;
    int victim;
    const int slot = insert(pool, k, p.layer, false, &victim);
    if (slot < 0) { fault(HB_ECAPACITY); return; }
    log(1, 2, p.layer, p.expert, p.enc, slot, victim);
    new_task(pool, slot, p.layer, p.expert, p.enc, 0);
    s.task[pool][slot].bg = 2;                   // explicit: never stale
  }
};

__global__ void dc_op_kernel(DcState* st, DcParams p) {
  if (threadIdx.x != 0) return;
  DcState& s = *st;
  Logic lg{s, p};
  lg.apply_pending();
  if (p.op == DC_FORWARD) {
    // stop the background copiers: this forward's loads go first
    *(volatile int*)&s.yield = 1;
    __threadfence();
    s.cur_layer = p.layer;
    lg.forward();
  } else if (p.op == DC_PREFETCH) {
    lg.prefetch();
  } else if (p.op == DC_LOAD) {
    lg.load();
  }
  __threadfence();
}

// ------------------------------------------------------------ copiers
// Try to take one chunk of task t: returns the chunk index or -1.  On success
// the caller holds a reader share of t (t.rw) until chunk_done().
__device__ int claim(DcTask& t) {
  const unsigned long long c0 = ld_acq64(&t.ctl);
  if ((unsigned)c0 >= *(const volatile unsigned*)&t.nchunks) return -1;   // racy pre-check
  const unsigned v = atomicAdd(&t.rw, 1u);
  if (v & kExcl) {                                     // being replaced
    atomicSub(&t.rw, 1u);
    return -1;
  }
  __threadfence();
  const unsigned n = *(volatile unsigned*)&t.nchunks;
  const unsigned long long c = atomicAdd(&t.ctl, 1ull);
  if ((unsigned)c >= n) {
    atomicSub(&t.rw, 1u);
    return -1;
  }
  return (int)(unsigned)c;
}

__device__ bool complete(const DcTask& t) {
  const unsigned long long d = ld_acq64(&t.done);
  return (unsigned)d >= *(const volatile unsigned*)&t.nchunks;
}

// the whole CTA copies chunk `ci` of t (t.src is host memory mapped into the
// device's address space: the loads cross PCIe)
__device__ void copy_chunk(const DcTask& t, int ci, size_t chunk) {
  const size_t off = (size_t)ci * chunk;
  const size_t n = min(chunk, (size_t)t.bytes - off);
  const uint4* src = (const uint4*)(t.src + off);
  uint4* dst = (uint4*)(t.dst + off);
  const size_t n16 = n / 16;          // blob sizes are multiples of 256 bytes
  constexpr int U = 4;
  size_t i = threadIdx.x;
  for (; i + (U - 1) * kCopyThreads < n16; i += U * kCopyThreads) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcv(src + i + u * kCopyThreads);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(dst + i + u * kCopyThreads, v[u]);
  }
  for (; i < n16; i += kCopyThreads) __stcg(dst + i, __ldcv(src + i));
}

__device__ void chunk_done(DcTask& t, size_t chunk, int ci, unsigned long long* bytes) {
  __threadfence();
  atomicAdd(bytes, (unsigned long long)min(chunk, (size_t)t.bytes - (size_t)ci * chunk));
  atomicAdd(&t.done, 1ull);
  atomicSub(&t.rw, 1u);
}

// foreground: the current forward's need list, until every entry is complete
__global__ void __launch_bounds__(kCopyThreads) dc_copy_fg(DcState* st) {
  DcState& s = *st;
  __shared__ int sh_task, sh_chunk;
  const int nn = s.n_need;
  for (;;) {
    if (threadIdx.x == 0) {
      sh_task = -1;
      bool all = true;
      for (int r = 0; r < nn && sh_task < 0; ++r) {
        const int i = (r + blockIdx.x) % nn;
        const int pool = s.need[i] >> 16, slot = s.need[i] & 0xffff;
        DcTask& t = s.task[pool][slot];
        const int ci = claim(t);
        if (ci >= 0) { sh_task = s.need[i]; sh_chunk = ci; }
        else if (!complete(t)) all = false;
      }
      if (sh_task < 0 && !all) { __nanosleep(500); sh_task = -2; }
    }
    __syncthreads();
    const int ti = sh_task, ci = sh_chunk;
    __syncthreads();
    if (ti == -1) break;
    if (ti == -2) continue;
    DcTask& t = s.task[ti >> 16][ti & 0xffff];
    copy_chunk(t, ci, s.chunk);
    __syncthreads();
    if (threadIdx.x == 0) chunk_done(t, s.chunk, ci, &s.bytes_fg);
  }
  // the last CTA out lowers `yield`: the background copiers may resume
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&s.fg_exit, 1u);
    if (prev == gridDim.x - 1) {
      s.fg_exit = 0;
      for (int i = 0; i < nn; ++i) s.task[s.need[i] >> 16][s.need[i] & 0xffff].fg = 0;
      *(volatile int*)&s.yield = 0;
      __threadfence();
    }
  }
}

// background: oldest incomplete task first, until none is left or `yield`
__global__ void __launch_bounds__(kCopyThreads) dc_copy_bg(DcState* st) {
  DcState& s = *st;
  __shared__ int sh_task, sh_chunk;
  for (;;) {
    if (threadIdx.x == 0) {
      sh_task = -1;
      const int cur = ld_vol(&s.cur_layer);
      if (!ld_vol(&s.yield)) {
        for (int tries = 0; tries < 4 && sh_task < 0; ++tries) {
          unsigned long long best = ~0ull;
          int bi = -1;
          for (int pool = 0; pool < 2; ++pool)
            for (int slot = 0; slot < s.cap[pool]; ++slot) {
              const DcTask& t = s.task[pool][slot];
              if (!*(const volatile int*)&t.live) continue;
              // a prefetch for a layer this token has passed was mispredicted: its
              // chunks move only if a forward needs the key (foreground)
              if (*(const volatile int*)&t.bg == 1 && *(const volatile int*)&t.layer <= cur) continue;
              if ((unsigned)ld_acq64(&t.ctl) >= *(const volatile unsigned*)&t.nchunks) continue;
              const unsigned long long q = *(const volatile unsigned long long*)&t.seq;
              if (q < best) { best = q; bi = pool * 65536 + slot; }
            }
          if (bi < 0) break;
          const int ci = claim(s.task[bi >> 16][bi & 0xffff]);
          if (ci >= 0) { sh_task = bi; sh_chunk = ci; }
        }
      }
    }
    __syncthreads();
    const int ti = sh_task, ci = sh_chunk;
    __syncthreads();
    if (ti < 0) break;
    DcTask& t = s.task[ti >> 16][ti & 0xffff];
    copy_chunk(t, ci, s.chunk);
    __syncthreads();
    if (threadIdx.x == 0) chunk_done(t, s.chunk, ci, &s.bytes_bg);
  }
}

}  // namespace

cudaError_t launch_dc_op(DcState* st, const DcParams& p, cudaStream_t s) {
  dc_op_kernel<<<1, 32, 0, s>>>(st, p);
  return cudaGetLastError();
}
cudaError_t launch_dc_copy_fg(DcState* st, int ctas, cudaStream_t s) {
  dc_copy_fg<<<ctas, kCopyThreads, 0, s>>>(st);
  return cudaGetLastError();
}
cudaError_t launch_dc_copy_bg(DcState* st, int ctas, cudaStream_t s) {
  dc_copy_bg<<<ctas, kCopyThreads, 0, s>>>(st);
  return cudaGetLastError();
}

}  // namespace hb
