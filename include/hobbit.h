/*
 * hobbit.h — C ABI of the B200-native mixed-precision MoE expert layer
 * (HOBBIT, arXiv 2411.01433).  libhobbit.so, built for sm_100a.
 *
 * Citations: P:n = PAPER.md line n (the paper), S:n = SPEC.md line n.
 *
 * The paper states the per-token, per-layer problem (Sec. 3.1
 * steps 1-9; Sec. 3.2): given the gating input, select the top-k
 * experts; score the selected experts (Eq. 2); for a cache miss pick the
 * precision by the thresholds T1/T2 (High / Low / Skip); load; and compute
 * Eq. 1, y = sum_i G(x)_{e_i} E_{e_i}(x).  Sec. 3.3 adds the
 * stacked next-layer prediction + prefetch, Sec. 3.4 (Eq. 3) the
 * two-pool cache policy.  The three calls the paper's problem needs are
 * moe_layer_forward, expert_cache_load and prefetch_next_layer; the rest is
 * setup, inspection and the offline quantiser.
 *
 * Conventions
 *  - Every call returns HB_OK (0) or a negative HB_E* code; hb_last_error()
 *    returns the message of the last failure on that context (thread-local
 *    message for calls without a context).
 *  - "stream" is a cudaStream_t passed as void* (e.g. torch's current stream).
 *    Device work is stream-ordered; no call allocates device memory after
 *    hb_create, so the resident path can be captured in a CUDA graph.
 *  - x is fp16 [batch, hidden] row-major on the device (the MoE block input,
 *    post-norm, "gating input"); y is fp32 [batch, hidden] row-major on
 *    the device and is OVERWRITTEN with this rank's part of Eq. 1.
 *  - A context is not thread-safe: one context per GPU per host thread.
 *  - Expert-parallel (EP): rank r owns experts e with e % world == r.  Each
 *    rank computes the exact router itself (no decision exchange).  Without
 *    hb_nccl_init y is this rank's part of Eq. 1; after it the library sums y
 *    over the ranks itself (in-place NCCL all-reduce at the end of
 *    moe_layer_forward), and hb_ep_broadcast_x replicates x from a root rank.
 */
#ifndef HOBBIT_H
#define HOBBIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define HB_OK            0
#define HB_EINVAL       -1  /* bad argument: dims, t1>t2, K%256, bad ids */
#define HB_ECAPACITY    -2  /* pool full and every member masked or in use */
#define HB_ESTATE       -3  /* expert/router not registered; forward before hb_token_begin */
#define HB_ECUDA        -4  /* CUDA runtime error */
#define HB_ENOMEM       -5  /* host or device allocation failed */
#define HB_EUNSUPPORTED -6  /* e.g. constrained cache with batch > 1 */
#define HB_ENCCL        -7  /* NCCL call failed (EP exchange) */

/* ------------------------------------------------------ encodings, levels */
/* Expert encodings (fp16+int4 and int8+int2 pairs).  Block = 32
 * consecutive K elements of one row; d, m fp16 per block:
 *   HB_F16  w = fp16                      16   bits/weight
 *   HB_Q8   w = d*q,      q int8 [-127,127] 8.5 bits/weight
 *   HB_Q4   w = d*(q-8),  q in [0,15]       4.5 bits/weight
 *   HB_Q2   w = d*q + m,  q in [0,3]        3.0 bits/weight
 * Blob = W1 [F,H], W3 [F,H], W2 [H,F], two layouts of the same size:
 *  - CANONICAL (the interchange format): per matrix the code
 *    section q, [N,K] row-major, element k of a row at bit (k*b) mod 8 of
 *    byte floor(k*b/8) (LSB first; Q4 low nibble = even element; Q8 int8),
 *    F16 values row-major; then d [N][K/32] fp16; then (Q2) m [N][K/32] fp16;
 *    each section 256-byte aligned (hb_canonical_section()).
 *  - DEVICE (what the kernels stream): per matrix a code
 *    section stored tile-major -- 16 rows x one 64-byte group of K = one
 *    contiguous 1 KB "unit" -- and one scale section of per-(unit,row) d/m
 *    records (hb_blob_section()).  hb_repack_canonical converts; the
 *    quantiser writes it directly. */
enum { HB_F16 = 0, HB_Q8 = 1, HB_Q4 = 2, HB_Q2 = 3, HB_Q2K = 4 };
/* HB_Q2K: llama.cpp's Q2_K arithmetic (R32/R33): super-block of 256
 * elements of a row = 16 sub-blocks of 16; per sub-block j a byte sc_j (low
 * nibble scale, high nibble min), per super-block fp16 d and dmin:
 *   w = d * (sc_j & 15) * q - dmin * (sc_j >> 4),  q in [0, 3]   (2.625 bits/weight)
 * CANONICAL: per matrix q (as Q2), sc [N][K/16] bytes, d [N][K/256] fp16,
 * dmin [N][K/256] fp16 (hb_canonical_section sec 0..3).  DEVICE: the Q2 code
 * layout; the 20-byte record of (unit, row) holds d, dmin, sc[16]; the blob is
 * padded to the canonical size.  The kernels (GEMV and tcgen05) form each
 * weight in fp16 (two roundings) before the MMA.  A pair may use HB_Q2K or
 * HB_Q2, not both. */
/* Precision decision of one selected expert. */
enum { HB_HIGH = 0, HB_LOW = 1, HB_SKIP = 2 };
#define HB_ENC_NONE 255

typedef struct {
  int n_layers, n_experts, top_k;   /* l_n (Eq. 3), E, K (Eq. 1) */
  int hidden, ffn;                  /* H, F: multiples of 256 */
  int hi_enc, lo_enc;               /* precision pair, default HB_F16 / HB_Q4 */
  double t1, t2;                    /* thresholds, default 0.6 / 0.9; 0<=t1<=t2 */
  int lookahead_p;                  /* prefetch depth p in [0, 4]; 0 = off */
  int w_lru, w_lfu, w_lhu, w_fld;   /* Eq. 3 weights as integer numerators >= 0; all 0 =
                                       the Random policy (P:1040 normaliser, R29) */
  int cap_high, cap_low;            /* slots per pool on this rank; -1 = fully resident */
  int allow_upgrade;                /* Low request served by a cached High copy (1) */
  int rank, world;                  /* EP: owner(e) = e % world */
  int max_batch;                    /* tokens per forward call */
  int strict;                       /* 1 (default): every Low selection is computed from
                                       lo_enc.  0: in resident mode a Low selection of an
                                       expert that some token of the same forward selected
                                       High is served by the hi_enc copy -- one weight stream
                                       per touched expert (R27; needs allow_upgrade) */
  int device_cache;                 /* offload mode only.  0 (default): the cache state machine
                                       runs on the host, loads are copy-engine memcpys on a copy
                                       stream (one host sync per layer).  1: the state machine
                                       (Eq. 3, the prefetch walk, the event log) lives in HBM and
                                       runs in a kernel after the router; loads are done by SMs
                                       reading the mapped pinned host blobs in chunks --
                                       on-demand chunks first, prefetch chunks in the background
                                       and pre-empted by the next forward -- so the
                                       offload forward never syncs with the host and can be
                                       captured in a CUDA graph.  In this
                                       mode prefetch_next_layer returns 0 (the queued loads are
                                       in hb_get_events), errors of the state machine (pool full)
                                       are sticky and reported by the next call, and a captured
                                       sequence must end with a moe_layer_forward (it joins the
                                       background copier) */
  int token_sharded;                /* resident mode, strict.  1: token-sharded expert
                                       parallelism: each rank passes ITS OWN
                                       max_batch tokens; the router runs on them, every
                                       token's non-skipped selections go to the ranks owning their
                                       experts (e % world): one row (x + hb_ts_meta) per (token,
                                       owner) in a fixed-capacity block (C = max_batch rows per
                                       peer); the owner computes its received rows as one batch and
                                       sends each row's gate-weighted expert sum back; y[b] = the
                                       sum of the token's returned rows.
                                       moe_layer_forward does the two exchanges with NCCL
                                       (hb_nccl_init) -- for world 1 without NCCL, locally; the
                                       staged calls hb_ts_dispatch / hb_ts_compute / hb_ts_combine
                                       leave the exchanges to the caller */
  int prefetch_both;                /* offload mode: 0 (default) prefetch the predicted
                                       precision; 1 prefetch both versions of each missing
                                       predicted expert, Low first ("versions of the experts
                                       with different precision levels", read as SPEC S:195;
                                       DESIGN.md R30) */
  int deterministic;                /* 1: bit-reproducible y for top_k <= 2 (debugging): the
                                       GEMV kernels deal whole row tiles statically (no dynamic
                                       chunks), so every a/u element and every (expert, y row)
                                       term is one fp32 reduction; h is read from global memory;
                                       the batched GEMM does not split K.  Slower (R24) */
} hb_config;

/* One routed (token, rank) pair of the last forward (inspection / parity). */
typedef struct {
  int32_t token;
  int32_t expert;                   /* e_i */
  uint8_t sel_rank;                 /* i, position in the top-k order */
  uint8_t prec;                     /* HB_HIGH / HB_LOW / HB_SKIP */
  uint8_t served_enc;               /* encoding computed, HB_ENC_NONE if skipped / not owned */
  uint8_t hit;                      /* 1 if the expert was cache-resident (offload mode) */
  float gate;                       /* G(x)_{e_i}, softmax over the selected logits */
} hb_decision;

/* Cache event (offload mode), identical to the oracle's event tuples. */
typedef struct {
  int32_t type;                     /* 0 hit, 1 load, 2 prefetch dropped (no eligible victim) */
  int32_t kind;                     /* 0 on-demand, 1 prefetch, 2 explicit expert_cache_load */
  int32_t layer, expert, enc;
  int32_t slot;                     /* slot index in the pool of enc */
  int32_t victim;                   /* evicted key layer*E+expert, or -1 */
} hb_event;

/* Token-sharded EP (hb_config.token_sharded): one dispatched ROW = one source
 * token's selections owned by one rank (the token's x row travels once per
 * owner in a parallel rows buffer). */
typedef struct {
  int32_t token;                    /* source token index, -1 = empty row */
  int32_t n;                        /* selections of the token this rank owns (1..top_k) */
  int32_t expert[8];                /* their experts e_i, in rank order */
  uint8_t prec[8];                  /* HB_HIGH / HB_LOW */
  float gate[8];                    /* G(x)_{e_i} computed by the source's router */
} hb_ts_meta;

typedef struct hb_ctx hb_ctx;

/* ------------------------------------------------------------ host helpers */
void        hb_config_default(hb_config* cfg);
size_t      hb_blob_bytes(int enc, int hidden, int ffn);
/* Offset/size of section sec (0 codes / fp16 values, 1 scales) of matrix mat
 * (0 W1, 1 W3, 2 W2) inside a DEVICE-layout blob.  HB_EINVAL if the section
 * does not exist (F16 has no scale section). */
int         hb_blob_section(int enc, int hidden, int ffn, int mat, int sec,
                            size_t* offset, size_t* nbytes);
/* Same for a CANONICAL blob: sec 0 codes / fp16 values, 1 d, 2 m (Q2 only);
 * HB_Q2K: 1 sc, 2 d, 3 dmin. */
int         hb_canonical_section(int enc, int hidden, int ffn, int mat, int sec,
                                 size_t* offset, size_t* nbytes);
/* Convert a canonical blob into the device layout: src and dst are device
 * pointers of hb_blob_bytes(enc, H, F) bytes each, not overlapping, owned by
 * the caller; stream-ordered (SURVEY.md 8(b) "canonical expert blob"). */
int         hb_repack_canonical(int enc, int hidden, int ffn, const void* src, void* dst,
                                void* stream);
/* k = 2 gap threshold floor(ln(T/(1-T)) * 2^48) (exact-integer form of the
 * T1/T2 test, R9).  *kind = 0 finite, +1 T>=1 (always), -1 T<=0. */
int64_t     hb_theta(double t, int* kind);
const char* hb_last_error(const hb_ctx* ctx);   /* ctx may be NULL */
const char* hb_version(void);

/* ---------------------------------------------------------------- context */
/* Allocate pools (cap_* slots of blob_bytes(hi/lo)) or the resident slot
 * table, the router table, scratch for max_batch tokens, a copy stream and
 * events on `device`.  The caller owns *out and must hb_destroy it. */
int hb_create(const hb_config* cfg, int device, hb_ctx** out);
int hb_destroy(hb_ctx* ctx);

/* Router weights W_g of `layer`, fp16 [E, H] ("linear layer").
 * w is a host pointer (copied) or, with on_device=1, a device pointer (D2D
 * copy on the null stream).  Stacked prediction reads these per layer. */
int hb_set_router(hb_ctx* ctx, int layer, const void* w, int on_device);

/* Register the blob of expert (layer, expert) in encoding enc.  flags = a
 * mode, optionally | HB_REG_CANONICAL:
 *   HB_REG_DEVICE_BORROW  blob is device memory owned by the caller that
 *                         outlives ctx (fully resident mode: cap_* = -1);
 *                         device layout only;
 *   HB_REG_DEVICE_COPY    blob is device memory; copied into HBM owned by
 *                         the library (resident mode); the caller may free it
 *                         on return;
 *   HB_REG_HOST_PINNED    blob is caller-owned pinned host memory that
 *                         outlives ctx (offload mode: next-level storage);
 *                         device layout only;
 *   HB_REG_HOST_COPY      blob is any host memory; copied into the library's
 *                         pinned arena (offload mode) or its HBM (resident).
 *   HB_REG_CANONICAL      the blob is in the canonical layout; the library
 *                         converts it (hb_repack_canonical) while copying.
 * nbytes must equal hb_blob_bytes(enc, H, F).  Only owned experts.  The COPY
 * modes synchronise the device. */
#define HB_REG_DEVICE_BORROW 1
#define HB_REG_HOST_PINNED   2
#define HB_REG_HOST_COPY     3
#define HB_REG_DEVICE_COPY   4
#define HB_REG_CANONICAL     0x100
int hb_register_expert(hb_ctx* ctx, int layer, int expert, int enc,
                       const void* blob, size_t nbytes, int flags);

/* Eq. 3 bookkeeping: T += 1 per forward step (a prefill is one step); masks
 * of the previous step expire.  reset zeroes R, F, H and T;
 * pools and masks are kept. */
int hb_token_begin(hb_ctx* ctx);
int hb_reset_sequence(hb_ctx* ctx);

/* ------------------------------------------------------------- the path */
/* Expert load into the expert cache (P:349 steps 6-8): a logical
 * insert of (layer, expert) into the high pool if enc == hi_enc, the low
 * pool if enc == lo_enc (evicting by Eq. 3 if full, no record update), and
 * an async host->device copy on the library's copy stream, ordered after
 * the work already queued on `stream` and after every earlier reader of the
 * reused slot (device_cache: the load is a background task forked from
 * `stream`).  No-op if already resident.  Offload mode only (HB_ESTATE in
 * resident mode). */
int expert_cache_load(hb_ctx* ctx, int layer, int expert, int enc, void* stream);

/* Stacked next-layer prediction + prefetch (Sec. 3.3): runs the
 * routers of layers layer+1 .. layer+p on x (one launch, the "Stacking
 * Computer"), masks the predicted experts, and queues loads of the first
 * lookahead layer with a miss in the PREDICTED precision (R14)
 * behind the on-demand loads.  Returns the number of loads queued (>= 0).
 * Blocks the host until the prediction is visible.  Resident mode: 0. */
int prefetch_next_layer(hb_ctx* ctx, int layer, const void* x, int batch, void* stream);

/* One MoE layer (P:347-349 + Eq. 1): exact router + top-k + softmax gates +
 * Eq. 2 scores + T1/T2 decision; cache lookup / victim / loads (offload
 * mode; blocks the host until the 1-layer decision record is visible); then
 * the grouped dequant-GEMV W1/W3 + SwiGLU and W2 + gate-weighted sum.
 * y[b,:] = sum over this rank's non-skipped selections of g * E_served(x_b).
 * Resident mode never blocks the host.  batch <= max_batch; batch > 1 with
 * a constrained cache returns HB_EUNSUPPORTED. */
int moe_layer_forward(hb_ctx* ctx, int layer, const void* x, int batch,
                      void* y, void* stream);

/* Batched decode / prefill (P:820 batch 1 only, P:1018
 * "prefill ... nearly all experts"): resident-mode forwards with
 * batch >= min_batch run the expert FFN as a grouped GEMM on the tcgen05
 * tensor cores (weights dequantised to fp16 in shared memory, fp32 TMEM
 * accumulation, h rounded to fp16: DESIGN.md R26) instead of the dequant-GEMV.
 * Decisions are unchanged.  0 = never.  Default 4 (env HB_K3_MIN_BATCH).
 * HB_EUNSUPPORTED if the context was created with max_batch == 1. */
int hb_set_batched_min(hb_ctx* ctx, int min_batch);

/* Expert-parallel exchange: after hb_nccl_init the
 * library sums y over the cfg.world EP ranks itself -- moe_layer_forward
 * ends with an in-place ncclAllReduce(sum, fp32) of y [batch, hidden] on the
 * forward's stream, so y is the full Eq. 1 output on every rank (without it
 * y is this rank's part and the caller reduces).  unique_id: 128 bytes from
 * hb_nccl_unique_id on one rank, shared by the caller (e.g. torch.distributed
 * broadcast); collective over the ranks (cfg.rank / cfg.world).  NCCL is
 * resolved at run time (the process's libnccl.so.2, or HB_NCCL_LIB);
 * HB_EUNSUPPORTED if it cannot be found. */
int hb_nccl_unique_id(void* unique_id_out /* 128 bytes */);
int hb_nccl_init(hb_ctx* ctx, const void* unique_id);
/* The same over an explicit group of nranks ranks (this one = rank), for
 * TP-within-expert: every rank owns every expert (cfg.world
 * = 1) but holds the slice [r F/R, (r+1) F/R) of each expert's W1/W3 rows
 * and W2 columns (a context created with ffn = F/R and blobs quantised from
 * those slices); the library sums the partial y over the group. */
int hb_nccl_init_ranks(hb_ctx* ctx, const void* unique_id, int nranks, int rank);
/* X1: replicate the gating input x [batch, hidden] fp16 (device,
 * caller-owned) from EP rank `root` to every rank, in place, on `stream`
 * (ncclBroadcast; collective, after hb_nccl_init; HB_ESTATE without it). */
int hb_ep_broadcast_x(hb_ctx* ctx, void* x, int batch, int root, void* stream);

/* ------------------------------------------------------------ inspection */
/* Decisions of the last forward: batch*top_k records (synchronises). */
int hb_get_decisions(hb_ctx* ctx, hb_decision* out, int cap);
/* Exact router logits of the last forward, L = logit * 2^48 as int128 split
 * into (lo uint64, hi int64) pairs, [batch][E][2] (synchronises). */
int hb_get_logits(hb_ctx* ctx, int64_t* out, int cap_pairs);
/* Cache events since the last call (offload mode). Returns the count. */
int hb_get_events(hb_ctx* ctx, hb_event* out, int cap);
/* Token-sharded EP, staged (hb_config.token_sharded = 1).
 * Buffers are device memory owned by the caller, laid out per peer rank r:
 * meta [world][C] hb_ts_meta, rows [world][C][hidden] fp16, ret [world][C][hidden]
 * fp32, C = max_batch; hb_ts_buffer_bytes gives the sizes.
 *  hb_ts_dispatch: routes x [batch, hidden] (this rank's tokens, exact decisions)
 *    and writes block r of meta_send / rows_send: one row per token with
 *    selections owned by rank r, tokens in order (empty rows: token = -1).  The caller then sends block r to rank r
 *    (all-to-all) and receives block r from rank r into meta_recv / rows_recv.
 *  hb_ts_compute: the received rows as one batch (each row's selections: the
 *    Eq. 1 terms sum_i g_i E_{e_i}(x) this rank owns) -> ret_send block r = the
 *    rows that came from rank r.  The caller returns block r to rank r (all-to-all).
 *  hb_ts_combine: y [batch, hidden] fp32 <- per token the sum of its returned
 *    rows (owners in the order of the token's selections), NaN rows for
 *    non-finite x (R28).  Needs the dispatch of
 *    the same batch on this context just before.
 * Errors: HB_ESTATE if the context is not token-sharded; HB_EINVAL on bad
 * sizes / pointers. */
int hb_ts_buffer_bytes(hb_ctx* ctx, size_t* meta_bytes, size_t* rows_bytes, size_t* ret_bytes);
int hb_ts_dispatch(hb_ctx* ctx, int layer, const void* x, int batch, void* meta_send,
                   void* rows_send, void* stream);
int hb_ts_compute(hb_ctx* ctx, int layer, const void* meta_recv, const void* rows_recv,
                  void* ret_send, void* stream);
int hb_ts_combine(hb_ctx* ctx, const void* ret_recv, int batch, void* y, void* stream);

/* Bytes moved host -> HBM for expert loads since hb_create (offload mode;
 * synchronises the device): out[0] foreground (on the forward's critical
 * path: on-demand loads, and in device_cache mode the rest of a prefetch the
 * forward needed), out[1] background (prefetch / expert_cache_load chunks).
 * In device_cache mode a prefetch whose slot is reused before its chunks were
 * copied never moves them: out[] counts what crossed the link, the events
 * count logical loads. */
int hb_copy_stats(hb_ctx* ctx, uint64_t out[2]);
/* Realised bytes of expert weights read by the GEMV kernels in the last
 * forward (sum of served blob bytes), for the roofline. */
int hb_last_expert_bytes(hb_ctx* ctx, uint64_t* out);
/* Number of kernel launches issued by the library since creation. */
int hb_launch_count(hb_ctx* ctx, uint64_t* out);
/* Kernel timing for the roofline: with max_calls > 0 every following
 * moe_layer_forward records CUDA events around its W1/W3 (K2a) and W2 (K2b)
 * kernels on the forward's stream (up to max_calls forwards); 0 disables.
 * hb_profile_read synchronises and returns, per recorded forward, the K2a
 * and K2b durations in ms as [n][2] floats; returns n. */
int hb_profile(hb_ctx* ctx, int max_calls);
int hb_profile_read(hb_ctx* ctx, float* ms, int cap);

/* In-kernel timing of the fused batch-1 decode kernel (router + K2a + K2b in
 * one launch), for the roofline: with max_forwards > 0
 * the next max_forwards fused forwards -- including replays of CUDA graphs
 * captured while it is on -- record %globaltimer stamps from inside the
 * kernel (device atomics, no events, no serialisation).  Synchronises and
 * clears the records; 0 disables for forwards issued afterwards.
 * hb_stamps_read synchronises and returns n records of 15 uint64 each (ns):
 * [kernel start (first CTA past its wait on the previous kernel), decisions
 * done (last CTA), K2a done (last CTA), grid barrier passed / K2b h staged
 * (first CTA), kernel end (last CTA), router rows landed (last CTA), logits
 * done (last CTA), decisions + job table done (last CTA), h staged (last
 * CTA), h staged (first CTA), router sub-steps (diagnostic) x4, number of
 * exact-fallback decisions]; 0 where a path has no such point; returns n. */
int hb_stamps(hb_ctx* ctx, int max_forwards);
int hb_stamps_read(hb_ctx* ctx, uint64_t* out, int cap);

/* ------------------------------------------- offline quantiser, generator */
/* Quantise an fp16 expert (W1 [F,H], W3 [F,H], W2 [H,F], device pointers)
 * into a device blob of hb_blob_bytes(enc, H, F) bytes (R8). */
int hb_quantize_expert(int enc, int hidden, int ffn, const void* w1, const void* w3,
                       const void* w2, void* blob, void* stream);
/* Seeded synthetic fp16 fill (the counter-based generator of synthgen/):
 * dst[i] = fp16_rne(fp32(s(key, start+i)) * scale). */
int hb_synth_fill_f16(void* dst, size_t n, uint64_t key, float scale, uint64_t start,
                      void* stream);

/* ------------------------------------------- host-only cache (no GPU) */
/* The Eq. 3 two-pool cache state machine used by the offload path, exposed
 * for CPU-only parity tests.  Same semantics and events as the device ctx. */
typedef struct hb_cache hb_cache;
int hbc_create(const hb_config* cfg, hb_cache** out);
int hbc_destroy(hb_cache* c);
int hbc_token_begin(hb_cache* c);
int hbc_reset_sequence(hb_cache* c);
/* experts/prec: top_k entries in rank order; served: out, top_k encodings. */
int hbc_forward(hb_cache* c, int layer, const int32_t* experts, const uint8_t* prec,
                uint8_t* served);
/* n_pred lookahead layers layer+1..layer+n_pred, [n_pred][top_k] each.
 * *prefetched = the layer whose loads were queued, or -1. */
int hbc_prefetch(hb_cache* c, int layer, int n_pred, const int32_t* experts,
                 const uint8_t* prec, int* prefetched);
int hbc_load(hb_cache* c, int layer, int expert, int enc);
int hbc_get_events(hb_cache* c, hb_event* out, int cap);
const char* hbc_last_error(const hb_cache* c);

#ifdef __cplusplus
}
#endif
#endif /* HOBBIT_H */
