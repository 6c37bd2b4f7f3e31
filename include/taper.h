/*
 * taper.h -- C ABI of the B200-native TAPER hot path (arXiv 2605.06914).
 *
 * Two calls follow the paper's problem statement:
 *   taper_admit            admit(batch state, slack, latency model) -> admitted-branch set
 *                          Sec. 3.3 "Slack-budgeted admission" and
 *                          Algorithm 1 "TAPER Per-Step Planner" (L147-181).
 *   taper_decode_attention decode_attention(admitted set, paged prefix/branch KV, queries)
 *                          -> per-sequence outputs.  Sec. 3.1 visibility rule (L100-103):
 *                          a branch token attends to P (+) H (+) h_i (+) y_{i,<t}; the
 *                          prefix P (+) H is served "from a single set of prefix blocks"
 *                          (L108).
 * plus the work-list rebuild used after the admission broadcast on G > 1 GPUs
 * (taper_build_work) and host helpers.
 *
 * Conventions (all calls):
 *   * Pointers inside the structs are DEVICE pointers unless marked [host].  The caller
 *     owns every buffer; no call allocates device memory or synchronises the stream.
 *     Every kernel is enqueued on `stream` (a cudaStream_t passed as void*; NULL = the
 *     legacy default stream).
 *   * Return value = host-side validation / launch result (TAPER_OK or a negative
 *     TAPER_ERR_*).  Data errors that only the device can see are OR-ed into the device
 *     status word `taper_admission.status` (TAPER_STATUS_* bits); outputs are undefined
 *     when it is non-zero, and the caller reads it whenever it chooses.
 *   * Stateless and thread-safe: no state survives a call except thread-local host
 *     strings (last error, launch count) and the opt-in thread-local debug hooks
 *     taper_set_profile_events / taper_set_trace_buffer (timing events and a pipeline
 *     trace; they change what is recorded, never what is computed).
 *   * bf16 tensors are passed as void* to raw bf16 storage (no torch or CUDA types here).
 */
#ifndef TAPER_H_
#define TAPER_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TAPER_API __attribute__((visibility("default")))
#else
#define TAPER_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------------- return codes */
#define TAPER_OK 0
#define TAPER_ERR_ARG (-1)          /* null pointer, negative count, bad struct field     */
#define TAPER_ERR_RHO (-2)          /* rho outside (0, 1]                 */
#define TAPER_ERR_NONMONOTONE (-3)  /* b <= 0 or c <= 0 or a < 0 (App. C.1)          */
#define TAPER_ERR_CAPACITY (-4)     /* R or S > TAPER_MAX_SLOTS, page size unsupported,
                                       workspace too small                                 */
#define TAPER_ERR_CUDA (-5)         /* a CUDA launch / driver call failed                 */
#define TAPER_ERR_UNSUPPORTED (-6)  /* reserved (no call returns it at present)           */

/* ----------------------------------------------------------------- device status bits */
#define TAPER_STATUS_EMPTY_REQUEST 1   /* a request had no ready slot; it is skipped     */
#define TAPER_STATUS_BAD_LENGTH 2      /* negative length / CSR offsets not monotone     */
#define TAPER_STATUS_PRECISION 4       /* c < budget * 2^-46: fp64 may tie candidates of
                                          different cost, so the sort+scan is no longer
                                          guaranteed bit-identical to Alg. 1             */
#define TAPER_STATUS_WORK_OVERFLOW 8   /* attention partials exceed the workspace        */
#define TAPER_STATUS_WORK_MISMATCH 16  /* taper_decode_attention was given a workspace /
                                          h_local other than the taper_admit or
                                          taper_build_work call that wrote the work list:
                                          nothing is computed, out is not written       */
#define TAPER_STATUS_EMPTY_CONTEXT 32  /* an admitted slot has no context (Lsh_r + Lloc_s
                                          = 0, [C-att-4]): softmax over an empty set; its
                                          output rows are written as zeros, lse as -inf  */

#define TAPER_MAX_SLOTS 4096   /* capacity of the single-CTA admission kernel (R and S)  */
#define TAPER_HEAD_DIM 128     /* Qwen3-32B head_dim                     */
#define TAPER_GQA_GROUP 8      /* 64 Q heads / 8 KV heads (L359)                         */
#ifndef TAPER_CHUNK_TOKENS
#define TAPER_CHUNK_TOKENS 4096 /* largest shared-prefix split (one work item's span)    */
#endif
/* Shared-prefix split of request r on a rank holding h_local KV heads, in a batch of n_req
 * requests: chunks of
 *     clamp(roundup_64(Lsh_r * h_local * n_req / TAPER_CHUNK_TARGET), 1024, TAPER_CHUNK_TOKENS)
 * tokens, i.e. about TAPER_CHUNK_TARGET shared work items per rank whatever the batch (a few
 * per SM of the 148: enough to balance the dynamic schedule, few enough to amortise each
 * item's Q load and partial) -- 4096 for the C2 step at h_local = 8, 1024 at h_local = 1; a
 * 32-request long-context batch splits its 16-32k prefixes finer than a 256-request one.
 * Chunk boundaries depend only on Lsh_r, h_local and n_req, never on which branches are
 * admitted (schedule invariance, Lemma 1); the split is finest at h_local = 1.    */
#if defined(__CUDACC__)
#define TAPER_HD __host__ __device__
#else
#define TAPER_HD
#endif
#ifndef TAPER_CHUNK_TARGET
#define TAPER_CHUNK_TARGET 512
#endif
#ifndef TAPER_CHUNK_MIN
#define TAPER_CHUNK_MIN 1024
#endif
static inline TAPER_HD int32_t taper_chunk_tokens(int32_t lsh, int32_t h_local, int32_t n_req) {
  int64_t c = (int64_t)lsh * h_local * n_req / TAPER_CHUNK_TARGET;
  c = (c + 63) / 64 * 64;
  if (c < TAPER_CHUNK_MIN) c = TAPER_CHUNK_MIN;
  if (c > TAPER_CHUNK_TOKENS) c = TAPER_CHUNK_TOKENS;
  return (int32_t)c;
}

/* App. C.1 display eq. (L316): T(S) = a + b*n_tokens + c*L_context, in ms. [host]      */
typedef struct {
  double a; /* ms, >= 0          */
  double b; /* ms per sequence, > 0  */
  double c; /* ms per context token, > 0 */
} taper_latency_model;

/* Step-width policies: App. D "Baselines" (L393-400) and Alg. 1.                      */
typedef enum {
  TAPER_POLICY_OFF = 0,   /* IRP-Off:   w_{r,t} = 1                                   */
  TAPER_POLICY_CAP = 1,   /* IRP-Ck:    w_{r,t} = min(n_r, cap)                        */
  TAPER_POLICY_EAGER = 2, /* IRP-Eager: w_{r,t} = n_r                                  */
  TAPER_POLICY_GREEDY = 3 /* TAPER: Alg. 1 greedy under the slack budget               */
} taper_policy_kind;

/* What the latency model's L_context counts (App. C.1).                        */
typedef enum {
  TAPER_CTX_PER_SEQUENCE = 0, /* the paper's reading: every admitted sequence counts its
                                 whole context Lsh_r + Lloc_s ([C-adm-6], L318)         */
  TAPER_CTX_PER_REQUEST = 1   /* cascade-aware: request r's prefix
                                 counts once, each admitted slot adds its Lloc_s -- the
                                 bytes taper_decode_attention actually reads           */
} taper_ctx_counting;

typedef struct {            /* [host] */
  int32_t kind;             /* taper_policy_kind                                       */
  int32_t cap;              /* TAPER_POLICY_CAP: k >= 1                                */
  double rho;               /* slack fraction, (0, 1] (Sec. 3.3; default 0.8 L391) */
  const double *utility;    /* DEVICE [R][utility_stride], or NULL.  Sec. 3.4 (L142) "a
                               monotone utility curve u_r(k)", k = opportunistic branches
                               granted to r; Alg. 1 line 15 (L167) scores
                               du = u_r(g+1) - u_r(g).  utility[r*stride + k] = u_r(k) for
                               k < stride; past the table u_r is flat (u_r(stride-1)).
                               NULL = the paper's linear utility u_r(k) = k (L391), run as
                               sort + scan; a table runs Alg. 1's loop literally (one
                               block-wide argmax per commit).  Read by TAPER_POLICY_GREEDY
                               only.  Concave = fairness, weighted = priority (L142).   */
  int32_t ctx_counting;     /* taper_ctx_counting (0 = the paper's per-sequence count) */
  int32_t utility_stride;   /* columns of `utility` (>= 2 when utility != NULL)         */
} taper_policy;

/* Batch state, structure-of-arrays (device).  Request r's ready slots are the slot
 * indices [req_slot_off[r], req_slot_off[r+1]); a serial-stage request has one slot,
 * a parallel-stage request one slot per exposed-but-incomplete branch (L128).          */
typedef struct {
  int32_t n_req;                  /* R  (host value), 0 <= R <= TAPER_MAX_SLOTS       */
  int32_t n_slot;                 /* S  (host value), 0 <= S <= TAPER_MAX_SLOTS       */
  const int32_t *req_shared_len;  /* [R]   Lsh_r: tokens of P (+) H (serial: whole ctx) */
  const int32_t *req_slot_off;    /* [R+1] CSR offsets, req_slot_off[0]=0, [R]=S        */
  const double *req_slack_ms;     /* [R]   d_r(t) - t in ms (L130)                      */
  const int32_t *slot_local_len;  /* [S]   Lloc_s: branch-local tokens h_i (+) y_{i,<=t},
                                     the current token already appended (0 for serial) */
  /* Optional multi-segment local context (NULL = one segment of Lloc_s tokens per slot).
   * Sec. 3.1 (L104-107): at a reduce step the context is P (+) H (+) every branch's
   * h_i (+) y_i in canonical order (+) z -- a concatenation of segments that already sit
   * in the cache in their own pages.  Slot s's local context is then its segments
   * [slot_seg_off[s], slot_seg_off[s+1]) in order, each starting on a page boundary
   * (taper_kv.seg_page_off), so a reduce step reads the branches' KV where it lies
   * instead of copying it.  sum of slot s's seg_len == slot_local_len[s], else
   * TAPER_STATUS_BAD_LENGTH.                                                          */
  const int32_t *slot_seg_off;    /* [S+1] CSR over slots, or NULL                      */
  const int32_t *seg_len;         /* [n_seg] tokens of each local segment (>= 0)        */
} taper_batch;

/* Admission outputs (device, caller-allocated).                                         */
typedef struct {
  int32_t *req_width;     /* [R] w_{r,t} = 1 + k_r (0 for an empty request)            */
  uint8_t *slot_admitted; /* [S] 1 iff the slot advances this step                     */
  int32_t *adm_list;      /* [S] admitted slots in ascending slot index; first n_adm   */
  int32_t *n_adm;         /* [1]                                                        */
  double *diag;           /* [5] T0, budget = T0 + rho*B_t, T(S), E = T(S)-T0 (Sec. 2.3
                             L83-85), min_r slack                                       */
  int32_t *status;        /* [1] TAPER_STATUS_* bits (0 = OK)                           */
} taper_admission;

/* One layer's paged KV cache on this rank (device).                                     */
typedef struct {
  const void *k_pages;  /* bf16 [num_pages, h_local, page_size, 128], 16-B aligned       */
  const void *v_pages;  /* bf16 [num_pages, h_local, page_size, 128]                     */
  int32_t num_pages;
  int32_t page_size;    /* 16, 32, 64 or 128                                            */
  int32_t h_local;      /* KV heads held by this rank (8 / G), 1..8                      */
  const int32_t *req_page_off; /* [R+1] CSR: pages of request r's shared segment        */
  const int32_t *req_pages;    /* token t of the segment is row t % page_size of page
                                  req_pages[req_page_off[r] + t / page_size]            */
  const int32_t *slot_page_off; /* [S+1] CSR: pages of slot s's local segment          */
  const int32_t *slot_pages;
  const int32_t *seg_page_off;  /* [n_seg] with taper_batch.slot_seg_off: token t of local
                                   segment q is row t % page_size of page
                                   slot_pages[seg_page_off[q] + t / page_size]
                                   (slot_page_off is then unused); else NULL            */
} taper_kv;

/* Workspace bytes for a batch of at most n_req requests / n_slot slots on a rank with
 * h_local KV heads.  max_chunk_slots bounds the partial rows' count
 *     sum_r w_r * ceil(Lsh_r / taper_chunk_tokens(Lsh_r, h_local, n_req))  +  sum_{s admitted} ceil(Lloc_s / 1024)
 * (prefix chunks per admitted branch, plus one per local item of <= 16 64-token tiles;
 * with local segments the second sum runs over segments: sum ceil(seg_len / 1024));
 * the Eager value of that sum over all ready slots is always enough.  An undersized
 * workspace is reported as TAPER_STATUS_WORK_OVERFLOW, never overrun.  [host]           */
TAPER_API int taper_workspace_size(int32_t n_req, int32_t n_slot, int32_t h_local,
                         int64_t max_chunk_slots, size_t *bytes);

/* The Eager bound of max_chunk_slots above, computed from HOST copies of the batch
 * arrays (req_shared_len [R], req_slot_off [R+1], slot_local_len [S]; slot_seg_off /
 * seg_len or NULL): every ready slot admitted, prefix chunks of
 * taper_chunk_tokens(Lsh_r, h_local, n_req) tokens.  A bound for h_local = 1 holds for every
 * h_local (the finest split).  Errors: TAPER_ERR_ARG (null array, non-monotone CSR,
 * negative length).  [host]                                                            */
TAPER_API int taper_max_chunk_slots(int32_t n_req, int32_t n_slot,
                                    const int32_t *req_shared_len, const int32_t *req_slot_off,
                                    const int32_t *slot_local_len, const int32_t *slot_seg_off,
                                    const int32_t *seg_len, int32_t h_local,
                                    int64_t *max_chunk_slots);

/* ------------------------------------------------------------------ latency model refit
 * App. C.1 "Fitting": T(S) = a + b n + c L is fitted by ordinary least
 * squares and "refreshed every 10 minutes using a rolling window of the most recent 200
 * observed step latencies".  The window keeps the last TAPER_LATENCY_WINDOW observations
 * (n = sequences in the step, L = its context count -- per sequence or per request, as the
 * admission counts it -- and the measured step time in ms); taper_latency_refit solves the
 * 3x3 normal equations in fp64.  The fitted model replaces *model only if it keeps T
 * monotone (a >= 0, b > 0, c > 0; L341) and the window holds >= 3 observations with a
 * non-singular design; otherwise *model is left as it was and TAPER_ERR_NONMONOTONE /
 * TAPER_ERR_ARG is returned.  fit_out (optional, [3]): R^2, MAPE (fraction), RMSE (ms)
 * of the new fit over the window.  All [host], no GPU.                                   */
#define TAPER_LATENCY_WINDOW 200
typedef struct {
  int32_t count;  /* observations held (<= TAPER_LATENCY_WINDOW)  */
  int32_t head;   /* next slot to overwrite                        */
  double n[TAPER_LATENCY_WINDOW], L[TAPER_LATENCY_WINDOW], t_ms[TAPER_LATENCY_WINDOW];
} taper_latency_window;
TAPER_API int taper_latency_observe(taper_latency_window *w, double n, double L, double t_ms);
TAPER_API int taper_latency_refit(const taper_latency_window *w, taper_latency_model *model,
                                  double *fit_out);

/* One admission step (Sec. 3.3 + Alg. 1; fixed policies of App. D), then the attention
 * work list for this rank (h_local KV heads) is written into `workspace`.
 * Greedy with linear utility is evaluated as a sort of candidates by (dL, r, slot)
 * followed by a prefix scan and the budget predicate on T(n0+m, L0+S_m); see DESIGN.md
 * for why this equals Alg. 1 bit for bit.  fp64, IEEE round-to-nearest, no FMA.
 * Errors: TAPER_ERR_ARG, _RHO, _NONMONOTONE, _CAPACITY, _CUDA.                         */
TAPER_API int taper_admit(const taper_batch *batch, const taper_latency_model *model,
                const taper_policy *policy, const taper_admission *out, int32_t h_local,
                void *workspace, size_t workspace_bytes, void *stream);

/* Rebuild adm_list / n_adm / req_width and the work list from slot_admitted alone (used
 * on every rank after rank 0's slot_admitted is broadcast, so ranks cannot diverge).
 * adm->status is overwritten with this call's data-error bits (the caller owns it for
 * the step: a rank that only calls taper_build_work never keeps a stale bit).  diag is
 * not written.                                                                          */
TAPER_API int taper_build_work(const taper_batch *batch, const taper_admission *adm, int32_t h_local,
                     void *workspace, size_t workspace_bytes, void *stream);

/* Cascade decode attention for one layer on this rank.
 *   q   : bf16 [S, 8*h_local, 128], slot-indexed (RoPE/QK-norm already applied)
 *   out : bf16 [S, 8*h_local, 128]; written for admitted slots only
 *   lse : fp32 [S, 8*h_local] natural-log LSE of each row, or NULL
 *   scale: softmax scale (1/sqrt(128))
 * Q head j of the rank's local KV head g is q[s, 8*g + j, :] (HF repeat_kv mapping).
 * The current token's K/V must already be in the cache (local segment, or the shared
 * segment of a serial request).  Rows of a page past a segment's end may hold any bits
 * (NaN included): their scores are masked and their V rows zeroed before the PV product.
 * An admitted slot with an empty context writes zero rows (TAPER_STATUS_EMPTY_CONTEXT).
 * Ordering contract (programmatic dependent launch): the kernels may start while the
 * previous kernel on `stream` is still running.  A work item may be resolved from the
 * work list before the grid dependency; its results are kept only if every work-list word
 * it was resolved from reads the same after the dependency (otherwise they are discarded
 * and the item is resolved again); q / the K/V pools are read only after the grid
 * dependency.  The page tables
 * (req_page_off ... seg_page_off) and the lengths in `batch` may be read early: they
 * must be written before the taper_admit / taper_build_work call that produced the work
 * list is enqueued (between that call and the attention calls only q and the K/V pool
 * contents may change, e.g. by taper_append_kv or the QKV projection).  `workspace`
 * and h_local must be the ones that call used (checked on the device:
 * TAPER_STATUS_WORK_MISMATCH in adm->status).
 * Errors: TAPER_ERR_ARG, _CAPACITY, _CUDA.                                             */
TAPER_API int taper_decode_attention(const taper_batch *batch, const taper_admission *adm,
                           const taper_kv *kv, const void *q, void *out, float *lse,
                           float scale, void *workspace, size_t workspace_bytes,
                           void *stream);

/* ------------------------------------------------------------------ fused output gather
 * SURVEY 8(f) NEXT-4; App. D L357 (tensor parallelism over NVLink): with the KV heads
 * split over G ranks (rank g holds heads [g h, (g+1) h), h = 8 / G), every rank needs all
 * 64 query heads' outputs of each layer.  Instead of a separate all-gather after the layer,
 * the merge epilogue of taper_decode_attention_gather stores each output row straight into
 * EVERY rank's gathered buffer (NVLink peer stores), then -- once all of this rank's rows
 * are stored -- sets flag[rank] = 1 in every rank's flag array (release, system scope).
 * taper_gather_wait on rank j waits until its flags of all G ranks are set and clears them
 * (acquire), so work enqueued after it reads the complete gathered output.               */
#define TAPER_MAX_RANKS 8
typedef struct {            /* [host] */
  int32_t world;            /* G in {1, 2, 4, 8}; h_local of the call must be 8 / G        */
  int32_t rank;             /* this rank, 0 <= rank < G                                     */
  void *out[TAPER_MAX_RANKS];        /* DEVICE pointers valid in this process: rank j's
                                        gathered output, bf16 [S][64][128] (Q head 8 h g + i
                                        of rank g at column block 8 h g + i); out[rank] is this
                                        rank's own (peer pointers: taper_ipc_open)          */
  int32_t *flags[TAPER_MAX_RANKS];   /* DEVICE pointers: rank j's flag array for THIS call,
                                        int32 [TAPER_MAX_RANKS], zero before the call; a flag
                                        array may be reused once its taper_gather_wait has run
                                        (e.g. one array per layer, reused every step)       */
} taper_gather;

/* taper_decode_attention whose outputs land in every rank's gathered buffer (see above)
 * instead of a per-rank `out`; rows of non-admitted slots are not written.  Same ordering
 * contract and errors as taper_decode_attention, plus TAPER_ERR_ARG for a gather struct
 * that does not match kv->h_local.                                                       */
TAPER_API int taper_decode_attention_gather(const taper_batch *batch, const taper_admission *adm,
                                            const taper_kv *kv, const void *q,
                                            const taper_gather *gather, float *lse, float scale,
                                            void *workspace, size_t workspace_bytes, void *stream);
/* Enqueue the wait for all G ranks' rows of the matching taper_decode_attention_gather call
 * (spins on gather->flags[gather->rank], then zeroes it; a lost flag traps after ~17 s
 * instead of hanging).  Errors: TAPER_ERR_ARG, _CUDA.                                    */
TAPER_API int taper_gather_wait(const taper_gather *gather, void *stream);

/* CUDA IPC for the gathered buffers of other processes on the node.  taper_ipc_handle
 * writes the 64-byte cudaIpcMemHandle_t of the allocation holding dev_ptr and dev_ptr's
 * offset in it; taper_ipc_open maps a peer's handle and returns the peer pointer
 * (base + offset); taper_ipc_close unmaps it.  [host]                                   */
TAPER_API int taper_ipc_handle(const void *dev_ptr, void *handle_64_bytes, size_t *offset);
TAPER_API int taper_ipc_open(const void *handle_64_bytes, size_t offset, void **dev_ptr);
TAPER_API int taper_ipc_close(void *dev_ptr, size_t offset);

/* Append the step's new token K/V of every admitted slot to the cache (Sec. 3.1,
 * [C-att-3]: the current token is the last token of the slot's context).  Call after the
 * lengths in `batch` include the new token and before taper_decode_attention:
 *   * branch (Lloc_s >= 1): local position Lloc_s - 1 -- with local segments, the last
 *     token of the last non-empty segment;
 *   * serial request (Lloc_s = 0): shared position Lsh_r - 1.
 *   k_new, v_new: bf16 [S, h_local, 128], slot-indexed (RoPE already applied to k_new).
 * WRITES kv->k_pages / kv->v_pages (declared const for the attention call).  Slots with
 * no position (Lsh_r + Lloc_s = 0) set TAPER_STATUS_BAD_LENGTH in adm->status.
 * Errors: TAPER_ERR_ARG, _CAPACITY, _CUDA.                                              */
TAPER_API int taper_append_kv(const taper_batch *batch, const taper_admission *adm,
                              const taper_kv *kv, const void *k_new, const void *v_new,
                              void *stream);

/* Profiling hook (bench.py): when `events` is non-NULL, every later
 * taper_decode_attention call on this thread records events[0] before the shared-prefix
 * kernel, events[1] between it and the local/merge kernel and events[2] after, on the
 * call's stream (cudaEvent_t handles passed as void*).  NULL disables.  [host]          */
TAPER_API int taper_set_profile_events(void *const *events, int n_events);

/* Debug hook (libraries built with -DTAPER_TRACE=1; the product build records nothing
 * and ignores the buffer): when non-NULL, attend_kernel records clock64() timestamps of its pipeline
 * events (TMA issue, MMA issue/commit, softmax start/end, epilogue) for CTA 0 into
 * device_buffer[tile * 16 + event] (int64, capacity_tiles * 16 entries).  [host]        */
TAPER_API int taper_set_trace_buffer(void *device_buffer, int capacity_tiles);

/* Human-readable text for a TAPER_ERR_* code or TAPER_STATUS_* bit set.  [host]        */
TAPER_API const char *taper_status_string(int code);
/* Last error message of this thread (detail of the most recent failing call).  [host]  */
TAPER_API const char *taper_last_error(void);
/* Number of kernel launches the most recent taper_admit / taper_decode_attention /
 * taper_build_work call on this thread enqueued.  [host]                               */
TAPER_API int taper_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TAPER_H_ */
