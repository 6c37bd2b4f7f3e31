// taper_internal.cuh -- shared definitions of the CUDA path (sm_100a only).
// Workspace layout, work-list encoding and the inline-PTX wrappers for mbarrier,
// TMA (cp.async.bulk.tensor), tcgen05 (MMA / TMEM) used by the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/taper.h"

namespace taper {

constexpr int kHeadDim = TAPER_HEAD_DIM;
constexpr int kGroup = TAPER_GQA_GROUP;
constexpr int kChunk = TAPER_CHUNK_TOKENS;  // largest prefix chunk (taper_chunk_tokens)
constexpr int kMaxSlots = TAPER_MAX_SLOTS;
constexpr int kTileTokens = 64;       // tokens per pipeline tile (one TMA stage)
constexpr int kLocalItemTiles = 16;   // branch-local tiles per local work item
constexpr int kMaxItemBranches = 16;  // admitted branches stacked in one shared item (<= 128 rows)

// ------------------------------------------------------------------ workspace layout
// hdr[0] = n_rc    : number of (request, prefix chunk) pairs (shared items per KV head)
// hdr[1] = n_cs    : sum_r w_r * (nchunk_r + nloc_r)  (partial "chunk-slots")
// hdr[2] = n_adm   : admitted slots
// hdr[3] = cap_cs  : chunk-slot capacity of the partial buffers (for this h_local)
// hdr[4] = h_local
// hdr[5] = n_rl    : number of (request, local item) pairs (local items per KV head)
// hdr[8] = work counter of attend_kernel's dynamic scheduler (reset by admit and by the
//          last attend CTA to exit, counted in hdr[9])
struct WsLayout {
  size_t hdr, slot_req, slot_rank, slot_lbase, req_chunk_off, req_loc_off, req_part_off,
      req_adm_off, adm_by_req, merge_desc, done, part_lse, part_o, fixed;
};

__host__ __device__ inline size_t ws_align(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline WsLayout ws_layout(int R, int S) {
  WsLayout w;
  size_t o = 0;
  w.hdr = o;           o = ws_align(o + 16 * sizeof(int32_t));
  w.slot_req = o;      o = ws_align(o + size_t(S) * sizeof(int32_t));
  w.slot_rank = o;     o = ws_align(o + size_t(S) * sizeof(int32_t));
  w.slot_lbase = o;    o = ws_align(o + size_t(S) * sizeof(int32_t));  // first local item of r
  w.req_chunk_off = o; o = ws_align(o + size_t(R + 1) * sizeof(int32_t));
  w.req_loc_off = o;   o = ws_align(o + size_t(R + 1) * sizeof(int32_t));
  w.req_part_off = o;  o = ws_align(o + size_t(R + 1) * sizeof(int32_t));
  w.req_adm_off = o;   o = ws_align(o + size_t(R + 1) * sizeof(int32_t));
  w.adm_by_req = o;    o = ws_align(o + size_t(S) * sizeof(int32_t));
  w.merge_desc = o;    o = ws_align(o + size_t(S) * 8 * sizeof(int32_t));
  // per (request, KV head): [0, R*8) items whose partials are written (attend -> merge),
  // [R*8, 2*R*8) merge warps done reading them (the last one re-arms both)
  w.done = o;          o = ws_align(o + size_t(R) * 2 * kGroup * sizeof(int32_t));
  w.fixed = o;
  w.part_lse = o;  // sized at run time from the workspace bytes
  w.part_o = o;
  return w;
}

// Per chunk-slot (one (work item, admitted slot) pair: prefix chunks and local items) the
// workspace holds, per KV head, 8 partial rows (128 fp32 o + 1 fp32 lse), plus one item
// descriptor and 16 local-tile descriptors (items and local items never outnumber
// chunk-slots because every item covers >= 1 admitted slot).
constexpr size_t kPartBytesPerCsHead = size_t(kGroup) * (kHeadDim + 1) * sizeof(float);
constexpr size_t kItemDescBytes = 32;                 // ItemDesc
constexpr size_t kLocalTileBytes = 16;                // int4 {slot, tok0, valid, jrow}
constexpr size_t kWorkBytesPerCs = kItemDescBytes + kLocalItemTiles * kLocalTileBytes + kItemDescBytes;

// Work item descriptor emitted by the admission kernel (A5).  Items are numbered per KV
// head, request-major: request r's prefix chunks, then its local items.
struct ItemDesc {
  int32_t r;        // request
  int32_t w;        // admitted branches (stacked rows = 8 w)
  int32_t adm_off;  // first admitted slot of r in adm_by_req
  int32_t cs0;      // chunk-slot of this item's first stacked branch
  int32_t tb;       // prefix chunk: first token; local item: first local-tile entry
  int32_t te;       // prefix chunk: end token;   local item: unused
  int32_t nt;       // 64-token tiles
  int32_t flags;    // bit 0: local item; bit 1: row mode; bit 2: row mode with M = 128
};
constexpr int32_t kItemLocal = 1, kItemRow = 2, kItemM128 = 4;

// Shared items of a request with >= kRowMin ready slots run in ROW mode (stacked rows on the
// MMA's M; M = 128 when the request has > 8 ready slots, else 64), the others (and every
// local item) in SWAP mode (tokens on M).  The mode and M depend on the request's ready
// slots n_r, never on how many of them are admitted, so a slot's arithmetic -- and its
// output bits -- do not depend on its co-admitted siblings (Lemma 1).
#ifndef TAPER_ROW_MIN
#define TAPER_ROW_MIN 9
#endif
constexpr int kRowMin = TAPER_ROW_MIN;
#ifndef TAPER_ROW_ENABLE
#define TAPER_ROW_ENABLE 1
#endif
constexpr bool kRowEnabled = TAPER_ROW_ENABLE;  // 0: every item in swap mode (A/B builds)
static_assert(kRowMin >= 2 && kRowMin <= 9, "swap mode covers at most 8 branches");

__host__ __device__ inline int64_t ws_cap_cs(size_t bytes, int R, int S, int h_local) {
  WsLayout w = ws_layout(R, S);
  if (bytes < w.fixed + 1024) return 0;
  return int64_t((bytes - w.fixed - 1024) / (kPartBytesPerCsHead * size_t(h_local) + kWorkBytesPerCs));
}

// part_lse, part_o (partial row prow = ((cs * h_local + g) * 8 + qh)), item descriptors,
// local-tile descriptors
struct WsTables {
  size_t lse, o, items, ltiles, sorted;  // sorted: the item descriptors in claim order
  int64_t cap_cs;
};
__host__ __device__ inline WsTables ws_tables(size_t bytes, int R, int S, int h_local) {
  WsLayout w = ws_layout(R, S);
  WsTables t;
  t.cap_cs = ws_cap_cs(bytes, R, S, h_local);
  t.lse = w.fixed;
  t.o = ws_align(t.lse + size_t(t.cap_cs) * h_local * kGroup * sizeof(float));
  t.items = ws_align(t.o + size_t(t.cap_cs) * h_local * kGroup * kHeadDim * sizeof(float));
  t.ltiles = ws_align(t.items + size_t(t.cap_cs) * kItemDescBytes);
  t.sorted = ws_align(t.ltiles + size_t(t.cap_cs) * kLocalItemTiles * kLocalTileBytes);
  return t;
}

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a lost arrival traps (error 700-class) instead of hanging the GPU.  The
// clock read between polls doubles as a short backoff: a tight try_wait loop (measured)
// slows the kernel ~5 %, the polls competing with the SMEM traffic of the busy warps.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
#if defined(TAPER_POLL_NS) && TAPER_POLL_NS > 0
    __nanosleep(TAPER_POLL_NS);  // experiment: back off between polls (power-capped runs)
#endif
    if (clock64() - t0 > (1ll << 35)) __trap();  // ~17 s at 2 GHz
  }
}

// Programmatic dependent launch (PDL): let the next kernel in the stream launch / wait
// for the previous one's completion and memory.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA: 4-D tiled load global -> shared, completion on an mbarrier (transaction bytes).
__device__ __forceinline__ void tma_load_4d(void *smem_dst, const void *tmap, uint64_t *bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}
// TMA: 5-D tiled load (one box lands both 64-column halves of a K or V tile).
__device__ __forceinline__ void tma_load_5d(void *smem_dst, const void *tmap, uint64_t *bar,
                                            int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}
// The same load with an L2 cache-policy hint (e.g. evict-first for KV tiles read once).
__device__ __forceinline__ void tma_load_5d_hint(void *smem_dst, const void *tmap, uint64_t *bar,
                                                 int c0, int c1, int c2, int c3, int c4,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
#ifndef TAPER_KV_EVICT_FRACTION
#define TAPER_KV_EVICT_FRACTION 1.0
#endif
#define TAPER_STR2(x) #x
#define TAPER_STR(x) TAPER_STR2(x)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, " TAPER_STR(TAPER_KV_EVICT_FRACTION) ";"
               : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_prefetch_desc(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// ---- tcgen05 (5th-gen tensor cores, TMEM accumulators)
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t *smem_slot) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T (kind::f16, bf16 inputs, fp32 accumulate)
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T ("TS": A operand read from tensor memory, K-major,
// two bf16 per 32-bit column); lanes whose bit is set in `mask` keep their old D.
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate,
                                              const uint32_t (&mask)[4]) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(mask[0]), "r"(mask[1]),
      "r"(mask[2]), "r"(mask[3])
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem] with every output lane enabled (A K-major in TMEM).
__device__ __forceinline__ void tc_mma_f16_tsa(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05 ops of this thread complete.
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

#define TAPER_R4(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3])
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TAPER_R4(0), TAPER_R4(4), TAPER_R4(8), TAPER_R4(12), TAPER_R4(16), TAPER_R4(20),
        TAPER_R4(24), TAPER_R4(28)
      : "r"(taddr));
}
#undef TAPER_R4
#define TAPER_W4(i) "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3])
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
          taddr),
      TAPER_W4(0), TAPER_W4(4), TAPER_W4(8), TAPER_W4(12), TAPER_W4(16), TAPER_W4(20),
      TAPER_W4(24), TAPER_W4(28)
      : "memory");
}
#undef TAPER_W4
// N = 8 / 16 consecutive 32-bit columns per lane (32 lanes of the warp's quadrant)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                   taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
               "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}
// generic N-column helpers built from the fixed-width instructions
template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, uint32_t *v) {
  if constexpr (N == 16) {
    tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(v));
  } else {
#pragma unroll
    for (int i = 0; i < N / 32; ++i)
      tmem_ld32(taddr + 32 * i, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * i));
  }
}
template <int N>
__device__ __forceinline__ void tmem_st_n(uint32_t taddr, const uint32_t *v) {
  if constexpr (N == 8) {
    tmem_st8(taddr, *reinterpret_cast<const uint32_t(*)[8]>(v));
  } else if constexpr (N == 16) {
    tmem_st16(taddr, *reinterpret_cast<const uint32_t(*)[16]>(v));
  } else {
#pragma unroll
    for (int i = 0; i < N / 32; ++i)
      tmem_st32(taddr + 32 * i, *reinterpret_cast<const uint32_t(*)[32]>(v + 32 * i));
  }
}
// 16 lanes, two threads per lane ("16x32bx2"): thread t < 16 reads / writes lane t columns
// [taddr + j], thread t >= 16 lane t - 16 columns [taddr + IMM + j], j < N.  Used for M = 64
// accumulators, whose rows live in lanes 0-15 of each quadrant.
#define TAPER_X2_LD(N, ADDR, IMMOP, REGS, ...)                                                 \
  template <int IMM>                                                                           \
  __device__ __forceinline__ void tmem_ld_x2_##N(uint32_t taddr, uint32_t *v) {                \
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x" #N ".b32 {" REGS "}, [" ADDR "], " IMMOP \
                 ";"                                                                           \
                 : __VA_ARGS__                                                                 \
                 : "r"(taddr), "n"(IMM));                                                      \
  }
#define TAPER_O4(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3])
TAPER_X2_LD(8, "%8", "%9", "%0,%1,%2,%3,%4,%5,%6,%7", TAPER_O4(0), TAPER_O4(4))
TAPER_X2_LD(16, "%16", "%17", "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15", TAPER_O4(0),
            TAPER_O4(4), TAPER_O4(8), TAPER_O4(12))
TAPER_X2_LD(32, "%32", "%33",
            "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,"
            "%23,%24,%25,%26,%27,%28,%29,%30,%31",
            TAPER_O4(0), TAPER_O4(4), TAPER_O4(8), TAPER_O4(12), TAPER_O4(16), TAPER_O4(20),
            TAPER_O4(24), TAPER_O4(28))
#undef TAPER_O4
#undef TAPER_X2_LD
template <int IMM>
__device__ __forceinline__ void tmem_st_x2_4(uint32_t taddr, const uint32_t *v) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x4.b32 [%0], %1, {%2,%3,%4,%5};" ::"r"(taddr),
               "n"(IMM), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
template <int IMM>
__device__ __forceinline__ void tmem_st_x2_8(uint32_t taddr, const uint32_t *v) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x8.b32 [%0], %1, {%2,%3,%4,%5,%6,%7,%8,%9};" ::"r"(
                   taddr),
               "n"(IMM), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
               "r"(v[6]), "r"(v[7])
               : "memory");
}
template <int IMM>
__device__ __forceinline__ void tmem_st_x2_32(uint32_t taddr, const uint32_t *v) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x32.b32 [%0], %1, {%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33};" ::"r"(
          taddr),
      "n"(IMM), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
      "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
      "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]),
      "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int n_threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n_threads) : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// UMMA shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bit.
//   K-major : rows of 128 B (64 bf16 of K), 8-row atoms of 1024 B, SBO = atom stride.
//   MN-major: K-rows of 128 B (64 bf16 of MN), LBO = stride between 64-wide MN blocks,
//             SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (sm_100)
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: bf16 x bf16 -> fp32, dense.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, bool a_mn_major,
                                                       bool b_mn_major) {
  return (1u << 4)                           // D format fp32
         | (1u << 7)                         // A bf16
         | (1u << 10)                        // B bf16
         | (uint32_t(a_mn_major) << 15)      // A major
         | (uint32_t(b_mn_major) << 16)      // B major
         | (uint32_t(N >> 3) << 17)          // N / 8
         | (uint32_t(M >> 4) << 24);         // M / 16
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace taper
