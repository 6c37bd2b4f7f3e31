// attention.cu -- cascade decode attention for one continuous-batching step.
//
// Sec. 3.1: branch i of a parallel phase attends to
//     P (+) H (+) h_i (+) y_{i,<t}
// and "a backend with paged or radix-tree KV caches can serve all branches from a single
// set of prefix blocks".  Two kernels:
//
//  A6+A7  attend_kernel (tcgen05 + TMA, one persistent CTA per SM, dynamic scheduling)
//     Work items of one request r and local KV head g; the stacked query operand is
//     [8 GQA heads] x [w admitted branches] (8 w <= 128 rows):
//       * shared item : one chunk of P (+) H (taper_chunk_tokens(Lsh, h, R) <= 4096 tokens,
//                       include/taper.h) for a group of <= 16 admitted branches -- every
//                       page read ONCE from HBM and contracted against all stacked rows
//                       (the cascade);
//       * local item  : <= 16 64-token tiles of ONE admitted branch's h_i (+) y_i (w = 1),
//                       or of one local segment of a reduce step's context (L104-107).
//     Per 64-token tile, SWAP mode (requests with < 9 ready slots, local items; tokens on
//     the MMA's M, stacked rows on N):
//       S^T = K Q^T    tcgen05.mma SS, M = 64 tokens, N = 8 w, K = 128 (A = the K tile by
//                      TMA, B = Q^T by TMA, both SMEM; fp32 S^T in TMEM)
//       online softmax (two groups of 4 warps; lazy running max) -> P = hi + lo bf16,
//                      stored transposed into SMEM with stmatrix.trans
//       O^T += V^T P^T tcgen05.mma SS, M = 128 (d), N = 16 w (hi and lo rows), K = 64
//                      (A = the V tile as an MN-major operand, B = P^T)
//     so the tensor and softmax work of a tile scale with the live rows; ROW mode (requests
//     with >= 9 ready slots; 128 stacked rows on M):
//       S = Q K^T      SS, M = 128 rows, N = 64 tokens; softmax thread = row; P = hi + lo
//                      to TMEM; O += P V as two TS MMAs (A = P from TMEM, B = the V tile).
//     Output: a normalised partial (o, lse) per stacked row and item, published per
//     (request, KV head) on a completion counter.
//  A8     merge_kernel: per admitted slot and KV head, log-sum-exp merge of its partials
//     (prefix chunks in order, then its local items) into bf16 out[s, 8g:8g+8, :];
//     launched with PDL, each warp starts once its request's items are published.
//
// Item boundaries depend only on segment lengths, and a stacked row's arithmetic does not
// depend on which other rows share the operand, so a slot's output does not depend on
// which siblings are co-admitted (Lemma 1; tests/test_gpu_attention.py).
#include <cuda.h>
#include <cuda_bf16.h>

#include <atomic>
#include <mutex>

#include "host_common.h"
#include "taper_internal.cuh"

namespace taper {

constexpr int kTile = kTileTokens;   // 64 tokens per pipeline stage
constexpr int kItemTiles = (kChunk / kTileTokens > kLocalItemTiles) ? kChunk / kTileTokens
                                                                    : kLocalItemTiles;
static_assert(kItemTiles <= 64, "scheduler lanes resolve at most two tiles each");
// K and V tiles ride separate TMA rings: a K stage is released as soon as QK(t) completes,
// a V stage only after PV(t); each stage is 64 tokens x 128 d bf16 = 16 KB.  Four + four
// stages keep ~128 KB in flight per SM, as fast as 5 + 5 (same-box A/B, r2 ab_rings:
// C2 191.3 vs 192.2 us, C3 846 vs 842 us) and they leave room for 16-branch Q operands.
#ifndef TAPER_KSTAGES
#define TAPER_KSTAGES 4
#endif
#ifndef TAPER_VSTAGES
#define TAPER_VSTAGES 4
#endif
#ifndef TAPER_DBG_FORCE_RERESOLVE
#define TAPER_DBG_FORCE_RERESOLVE 0  // test builds: always take the re-resolve path
#endif
#ifndef TAPER_MERGE_PDL
#define TAPER_MERGE_PDL 1  // 0: merge_kernel launches without PDL (A/B experiments)
#endif
#ifndef TAPER_MERGE_GRID
#define TAPER_MERGE_GRID 0  // > 0: at most this many merge CTAs (A/B experiments)
#endif
#ifndef TAPER_CLAIM_LEAD
#define TAPER_CLAIM_LEAD 8  // tiles before an item's end at which the next item is claimed
#endif
constexpr int kClaimLead = TAPER_CLAIM_LEAD;
#ifndef TAPER_PDL
#define TAPER_PDL 1  // 0: attend_kernel launches without PDL (A/B experiments)
#endif
// Row mode (kItemRow, taper_internal.cuh): stacked rows on the MMA's M, S = Q K^T, thread =
// row, P kept in TMEM for a TS MMA O += P V.  Swap mode: tokens on M ("swap-AB"), tensor and
// softmax work proportional to the live rows -- requests with < kRowMin ready slots and
// every local item (w = 1).  See DESIGN.md "row mode".
constexpr int kSwapMaxW = kRowMin - 1;       // widest swap-mode item
constexpr int kSwapMaxWB = (kSwapMaxW + 1) / 2;  // 8-row blocks per softmax group (swap mode)
constexpr int kKStages = TAPER_KSTAGES;
constexpr int kVStages = TAPER_VSTAGES;
constexpr int kStageBytes = 2 * 8192;
constexpr int kOffV = kKStages * kStageBytes;
constexpr int kOffQ = kOffV + kVStages * kStageBytes;   // Q operand, 2 buffers x 128 rows
constexpr int kQBytes = kMaxItemBranches * kGroup * 256;  // 32 KB: [branch][d-half][8][128 B]
constexpr int kOffPT = kOffQ + 2 * kQBytes;              // swap-mode P^T operand
// Swap items with <= kNarrowPT branches (P^T <= 8 KB) alternate between two P^T halves by
// tile parity, so softmax(n) only waits for PV(n-2); wider ones use the whole buffer.
#ifndef TAPER_NARROW_PT
#define TAPER_NARROW_PT 4
#endif
constexpr int kNarrowPT = TAPER_NARROW_PT < kSwapMaxW ? TAPER_NARROW_PT : kSwapMaxW;
constexpr int kPTHalf = 2 * kNarrowPT * kGroup * 128;  // hi + lo rows of kNarrowPT branches
constexpr int kPTBytes = (2 * kPTHalf > 2 * kSwapMaxW * kGroup * 128)
                             ? 2 * kPTHalf : 2 * kSwapMaxW * kGroup * 128;
constexpr int kOffML = kOffPT + kPTBytes;  // (m, l) of the <= 128 stacked rows, 2 buffers
// swap mode, cross-warp tile maxima per softmax group: [2 parities][4 warps][kRedCols] (a
// group owns <= kSwapMaxWB 8-row blocks)
constexpr int kRedCols = 8 * kSwapMaxWB;
constexpr int kRedFloats = 2 * 4 * kRedCols;
constexpr int kOffRed = kOffML + 2 * 128 * 8;
// row mode: per-row tile maxima of the two token halves [2 parities][2 groups][128]; then
// the softmax warps' partial row sums [2 O buffers][4 slots][128 rows] (swap: slot = TMEM
// quadrant warp, row: slot = group), summed by the epilogue
constexpr int kOffRowRed = kOffRed + 2 * kRedFloats * 4;
constexpr int kOffLPart = kOffRowRed + 2 * 2 * 128 * 4;
constexpr int kOffAlpha = kOffLPart + 2 * 4 * 128 * 4;  // swap: rescale factors [8][kRedCols]
constexpr int kRecBytes = kItemTiles <= 32 ? 1024 : 2048;  // ItemRec slot
// claimed-item ring: the scheduler resolves one item ahead of the K producer, the softmax
// warps hold theirs to the item's end, the MMA and epilogue warps copy the record at once --
// three 2 KB records suffice
constexpr int kItemRing = kRecBytes == 2048 ? 3 : 8;
constexpr int kOffRec = kOffAlpha + 8 * kRedCols * 4;
constexpr int kOffBar = kOffRec + kItemRing * kRecBytes;
constexpr int kSmemUsed = kOffBar + 512;
constexpr int kSmemBytes = kSmemUsed + 1024;  // + alignment slack
static_assert(kSmemBytes <= 232448, "exceeds 227 KB of dynamic SMEM per CTA");
// warp 0: K producer; warp 1: MMA issuer; warps 2-5: softmax group 0; warps 6-9:
// epilogue; warp 10: V producer; warp 11: item scheduler (claims, resolves tiles, loads Q);
// warps 12-15: softmax group 1.  A group owns 8-row blocks of the stacked rows.
constexpr int kAttnThreads = 512;
// Every lane of the 15 consumer warps releases each record (and every scheduler lane
// publishes it): each thread's own arrive orders its own SMEM accesses, which is also
// the pattern compute-sanitizer's racecheck models (a lane-0 arrive after __syncwarp is
// equally correct but reported as a hazard).
constexpr int kRingConsumers = 15 * 32;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0;     // swap: S^T 0 [0, 64), S^T 1 [64, 128) (64 tokens x N rows);
                                  // row: S 0 / S 1 (rows x 64 tokens)
constexpr uint32_t kColO = 128;   // swap: O^T 0 [128, 256), O^T 1 [256, 384) (128 d x 2N rows);
                                  // row: O 0 / O 1 (rows x 128 d)
constexpr uint32_t kColP = 384;   // row: P 0 [384, 448), P 1 [448, 512): hi then lo halves of P,
                                  // rows x 64 tokens bf16 each
// Row mode splits P = hi + lo (bf16 each) like swap mode: with P rounded to one bf16 the
// peaked parity case misses allclose(2e-3, 1e-2) (max abs 8.2e-3, r2 run e).
#ifndef TAPER_ROW_PLO
#define TAPER_ROW_PLO 1
#endif
constexpr bool kRowPlo = TAPER_ROW_PLO;
// A/B isolation (timing only, on batches without row items): drop row support from one role
#ifndef TAPER_DBG_ROW_ROLES
#define TAPER_DBG_ROW_ROLES 7  // bit 0: MMA warp, bit 1: softmax warps, bit 2: epilogue
#endif
constexpr bool kRowMma = kRowEnabled && (TAPER_DBG_ROW_ROLES & 1);
constexpr bool kRowSm = kRowEnabled && (TAPER_DBG_ROW_ROLES & 2);
constexpr bool kRowEpi = kRowEnabled && (TAPER_DBG_ROW_ROLES & 4);

struct AttnParams {
  // slot_page_off: per slot (local tiles with segment -1) or, when the batch has local
  // segments, taper_kv.seg_page_off per segment.  (One pointer for both: an extra kernel
  // parameter measurably slowed the kernel, 200 -> 212 us per C2 layer.)
  const int32_t *slot_page_off, *slot_pages, *req_page_off, *req_pages;
  int32_t *hdr;        // hdr[8]: work counter, hdr[9]: CTAs exited
  const int32_t *adm_by_req;
  int32_t *done;       // [r * 8 + g]: items of (request, KV head) whose partials are written
  const ItemDesc *sorted;  // the item descriptors in claim order (admit: longest first)
  const int4 *ltiles;
  float *part_lse, *part_o;
  int h_local, page_size;
  int tma5d;  // 1: page_size >= 64, one 5-D box per full tile; 0: 4-D boxes of one page
  int cap_cs;  // partial capacity this call's workspace gives (checked against hdr[3])
  float scale_log2;
  long long *trace;  // debug: pipeline event timestamps of CTA 0 (taper_set_trace_buffer)
  int trace_cap;
};

// Debug trace (builds with -DTAPER_TRACE=1 only; the product build compiles every probe
// out -- their checks alone cost ~5 % of the softmax warps' issue slots, ncu r2a):
// event e of tile/item index n -> trace[(n * 16 + e)] = clock64 (CTA 0 only).
#ifndef TAPER_TRACE
#define TAPER_TRACE 0
#endif
constexpr bool kTrace = TAPER_TRACE;
__device__ __forceinline__ bool tracing(const AttnParams &p) { return kTrace && p.trace != nullptr; }
__device__ __forceinline__ void trace_cta(const AttnParams &p, int e) {  // globaltimer, CTA row
  if (tracing(p)) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3000 + blockIdx.x) * 16 + e] = (long long)g;
  }
}
// as trace_cta, but the timestamp is taken once `dep` is available (waits for its load)
__device__ __forceinline__ void trace_cta_dep(const AttnParams &p, int e, int dep) {
  if (tracing(p)) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g) : "r"(dep) : "memory");
    p.trace[(size_t)(3000 + blockIdx.x) * 16 + e] = (long long)g + (dep == 0x7fffffff);
  }
}
__device__ __forceinline__ void trace_ev(const AttnParams &p, int e, uint32_t n) {
  if (tracing(p) && blockIdx.x == 0 && int(n) < p.trace_cap)
    p.trace[(size_t)n * 16 + e] = clock64();
}

template <bool B> struct BoolC { static constexpr bool value = B; };

struct Item {
  int r, g, local, w, adm_off, cs0, nt, tb, te, row, m128;
};

// A claimed work item as the scheduler warp resolves it into SMEM: the descriptor plus, per
// 64-token tile, its first token, valid tokens and the page of each 16-token box.  Every
// other role reads only this record (no global loads per item).
struct ItemRec {
  int32_t it, g, desc[8];  // desc = ItemDesc {r, w, adm_off, cs0, tb, te, nt, flags}
  int32_t pad[6];
  int32_t tok0[kItemTiles], valid[kItemTiles];
  int32_t pg[kItemTiles][4];
};
static_assert(sizeof(ItemRec) <= kRecBytes, "ItemRec size");

__device__ __forceinline__ void decode_item(const ItemRec *rec, Item &x) {
  x.g = rec->g;
  x.r = rec->desc[0]; x.w = rec->desc[1]; x.adm_off = rec->desc[2]; x.cs0 = rec->desc[3];
  x.tb = rec->desc[4]; x.te = rec->desc[5]; x.nt = rec->desc[6];
  x.local = rec->desc[7] & kItemLocal;
  x.row = (rec->desc[7] & kItemRow) != 0;
  x.m128 = (rec->desc[7] & kItemM128) != 0;
}

struct TileInfo {
  const int32_t *pages;
  int tok0, valid;
  int4 lt;  // local item: the work-list entry the tile was resolved from
};

__device__ __forceinline__ TileInfo tile_info(const AttnParams &p, const Item &x, int t) {
  TileInfo ti;
  if (!x.local) {
    ti.pages = p.req_pages + __ldcg(p.req_page_off + x.r);
    ti.tok0 = x.tb + t * kTile;
    ti.lt = make_int4(0, 0, 0, 0);
    ti.valid = min(kTile, x.te - ti.tok0);
  } else {
    const int4 lt = __ldcg(p.ltiles + x.tb + t);  // {slot, tok0, valid, segment or -1}
    ti.lt = lt;
    ti.pages = p.slot_pages + __ldcg(p.slot_page_off + (lt.w >= 0 ? lt.w : lt.x));
    ti.tok0 = lt.y;
    ti.valid = lt.z;
  }
  return ti;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// S^T[tS] = K Q^T ("swap-AB": tokens on M = 64, stacked rows on N = 8 wpad).  A = the K tile
// (SW128 K-major: [d-half][64 tokens][64 d], halves 8 KB apart), B = Q^T (SW128 K-major:
// [branch][d-half][8 rows][64 d], 8-row groups 2 KB apart, halves 1 KB apart); 8 k-steps of
// 16 over d = 128.
__device__ __forceinline__ void issue_qk(uint32_t tS, uint32_t kb, uint32_t qb, uint32_t idesc) {
  const uint64_t a0 = umma_desc_sw128(kb, 16, 1024);
  const uint64_t b0 = umma_desc_sw128(qb, 16, 2048);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint64_t a = a0 + uint64_t((((kk >> 2) * 8192) + (kk & 3) * 32) >> 4);
    const uint64_t b = b0 + uint64_t((((kk >> 2) * 1024) + (kk & 3) * 32) >> 4);
    tc_mma_f16(tS, a, b, idesc, kk > 0 ? 1u : 0u);
  }
}

// O^T[tO] (+)= V^T P^T: M = 128 (d), N = 16 wpad (per branch: 8 hi rows then 8 lo rows of
// P = hi + lo), K = 64 tokens in 4 k-steps.  A = the V tile as an MN-major SW128 operand
// (d halves 8 KB apart, 8-token groups 1 KB apart), B = P^T (SW128 K-major, 8-row groups
// 1 KB apart).
__device__ __forceinline__ void issue_pv(uint32_t tO, uint32_t vb, uint32_t pb, bool first,
                                         uint32_t idesc) {
  const uint64_t a0 = umma_desc_sw128(vb, 8192, 1024);
  const uint64_t b0 = umma_desc_sw128(pb, 16, 1024);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t a = a0 + uint64_t((kk * 2048) >> 4);
    const uint64_t b = b0 + uint64_t((kk * 32) >> 4);
    tc_mma_f16(tO, a, b, idesc, (first && kk == 0) ? 0u : 1u);
  }
}

// Row mode.  S[tS] = Q K^T: M = stacked rows (64 or 128; rows past 8 w are padding), N = 64
// tokens, K = 128 d.  A = Q (the same SMEM buffer as swap mode's Q^T: SW128 K-major, 8-row
// groups 2 KB apart, d-halves 1 KB apart), B = the K tile (SW128 K-major, 8-token groups
// 1 KB apart, d-halves 8 KB apart).  Verified against fp64 by scripts/rowmode_check.cu.
__device__ __forceinline__ void issue_qk_row(uint32_t tS, uint32_t qb, uint32_t kb, uint32_t idesc) {
  const uint64_t a0 = umma_desc_sw128(qb, 16, 2048);
  const uint64_t b0 = umma_desc_sw128(kb, 16, 1024);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint64_t a = a0 + uint64_t((((kk >> 2) * 1024) + (kk & 3) * 32) >> 4);
    const uint64_t b = b0 + uint64_t((((kk >> 2) * 8192) + (kk & 3) * 32) >> 4);
    tc_mma_f16(tS, a, b, idesc, kk > 0 ? 1u : 0u);
  }
}
// Row mode.  O[tO] (+)= P V: M = stacked rows, N = 128 d, K = 64 tokens in 4 k-steps.  A = P
// from TMEM (bf16 pairs, 8 columns per 16 tokens), B = the V tile as an MN-major SW128
// operand (d-halves 8 KB apart, 8-token groups 1 KB apart).
__device__ __forceinline__ void issue_pv_row(uint32_t tO, uint32_t tP, uint32_t vb, bool first,
                                             uint32_t idesc) {
  const uint64_t b0 = umma_desc_sw128(vb, 8192, 1024);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t b = b0 + uint64_t((kk * 2048) >> 4);
    tc_mma_f16_tsa(tO, tP + 8 * kk, b, idesc, (first && kk == 0) ? 0u : 1u);
    if (kRowPlo) tc_mma_f16_tsa(tO, tP + 32 + 8 * kk, b, idesc, 1u);  // + P_lo V
  }
}

// 16 TMEM lanes x 8 wpad columns in the 16x256b pattern: for column block b, registers
// 4b..4b+3 hold (token lane/4, col 8b + 2(lane%4)), (same, +1), (token lane/4 + 8, col),
// (same, +1) -- the mma.m16n8 accumulator fragment.
template <int WPAD>
__device__ __forceinline__ void tmem_ld_16x256(uint32_t taddr, uint32_t (&v)[4 * WPAD]) {
  if constexpr (WPAD == 1) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(taddr));
  } else if constexpr (WPAD == 2) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
  } else if constexpr (WPAD == 3) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]) : "r"(taddr + 16));
  } else if constexpr (WPAD == 4) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
  }
}

__device__ __forceinline__ void stmatrix_x4_trans(uint32_t addr, uint32_t r0, uint32_t r1,
                                                  uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr),
               "r"(r0), "r"(r1), "r"(r2), "r"(r3)
               : "memory");
}

// bar.red.or over a named barrier: true iff any of the n participating threads passes true
__device__ __forceinline__ bool bar_red_or(int id, int n_threads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(uint32_t(pred)), "r"(id), "r"(n_threads)
      : "memory");
  return r != 0;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&h2);
}
// P = hi + lo, both bf16 pairs.  kTrunc: hi is the upper half of
// each fp32 word (one byte permute instead of a conversion), lo = P - hi rounded to bf16
// (|error| <= 2^-16 P instead of 2^-17).  Swap mode truncates (same-box: C2 188.0 -> 186.1
// us per layer, -0.7 % at the power cap); row mode rounds (truncating there measured 3 %
// slower on C3).
#ifndef TAPER_PHI_TRUNC_SWAP
#define TAPER_PHI_TRUNC_SWAP 1
#endif
template <bool kTrunc>
__device__ __forceinline__ void split_hi_lo(float a, float b, uint32_t &hi, uint32_t &lo) {
  if constexpr (kTrunc) {
    const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
    hi = __byte_perm(ua, ub, 0x7632);
    lo = pack_bf16(a - __uint_as_float(ua & 0xffff0000u), b - __uint_as_float(ub & 0xffff0000u));
  } else {
    hi = pack_bf16(a, b);
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&hi));
    lo = pack_bf16(a - f.x, b - f.y);
  }
}

// Butterfly plan for NC columns over lane bits 4, 3, 2: an even count is halved by a
// transposing exchange (each lane keeps one half), an odd one is reduced in place.
__host__ __device__ constexpr int bfly_cnt(int nc, int st) {
  int c = nc;
  for (int i = 0; i < st; ++i) c = (c % 2 == 0) ? c / 2 : c;
  return c;
}

struct SoftmaxCtx {  // per-thread constants of a softmax warp
  const AttnParams *p;
  uint8_t *smem;
  uint64_t *s_full, *pv_done, *vfull, *p_full_g, *o_free, *ml_full;
  float2 *xml;
  float *red_g, *alpha_s;
  float *row_red;  // row mode: [2][2][128] tile maxima
  float *lpart;    // [2][4][128] partial row sums (item end, read by the epilogue)
  uint32_t tmem, lane_off, pt_base;
  int grp, wq, lane, warp, tid, bar_id;
  float c;
};

// One item of a softmax group in the transposed layout.  This thread holds tokens
// tA = lane/4 and tA + 8 of its warp's 16-token slice and, per 8-row block b < WB of the
// group's blocks [blk0, blk0 + WB), stacked rows 8 (blk0 + b) + 2 (lane%4) + {0, 1}
// (column index i = 2b + e).  Running max (lazy: moves only when a tile's max exceeds it
// by > 8 in log2 units) and this thread's partial row sums live in registers.  Column max
// per tile: a transposing butterfly over the 8 lanes sharing columns, one SMEM exchange
// across the group's 4 warps for the columns a lane ends up owning, the lazy update there,
// and the mirrored butterfly broadcasting the maxima back.  P = hi + lo (bf16 each) goes to
// SMEM as P^T (the PV MMA's B operand) via stmatrix.trans once PV(n-1) has released it.
// WB = 0: the group has no rows in this item and only keeps the barrier phases in step.
template <int WB>
__device__ __forceinline__ void softmax_item(const SoftmaxCtx &C, const ItemRec *rec, const Item &x,
                                             int blk0, uint32_t item_idx, uint32_t &n,
                                             bool &prev_wide) {
  constexpr int NC = WB > 0 ? 2 * WB : 2;    // columns per thread
  constexpr int NF = bfly_cnt(NC, 3);        // columns a lane owns after the butterfly
  const int lane = C.lane, wq = C.wq;
  const int c0 = 2 * (lane & 3);
  const int tA = 16 * wq + (lane >> 2);      // token within the 64-token tile
  const uint32_t ob = item_idx & 1;
  const uint32_t tO = C.tmem + C.lane_off + kColO + ob * 128;
  const int n_live = 8 * x.w;
  // lane-invariant butterfly ownership and stmatrix addresses
  int off = 0;
#pragma unroll
  for (int st = 0; st < 3; ++st) {
    const int cnt = bfly_cnt(NC, st);
    if (cnt % 2 == 0 && (lane & (16 >> st))) off += cnt / 2;
  }
  int col[NF];
#pragma unroll
  for (int j = 0; j < NF; ++j) col[j] = 8 * ((off + j) >> 1) + c0 + ((off + j) & 1);
  uint32_t st_addr[WB > 0 ? WB : 1];
  {
    const int mi = lane >> 3, k = lane & 7;
    const int ch = 2 * wq + (mi & 1);
#pragma unroll
    for (int b = 0; b < WB; ++b) {
      const int R = 16 * (blk0 + b) + ((mi >> 1) << 3) + k;
      st_addr[b] = C.pt_base + (R >> 3) * 1024 + (R & 7) * 128 + (((ch ^ (R & 7)) & 7) << 4);
    }
  }
  const bool rows_live = 8 * (blk0 + WB) <= n_live;
  const bool wide = x.w > kNarrowPT;
  float m_run[NC], l_run[NC], m_red[NF];
#pragma unroll
  for (int i = 0; i < NC; ++i) { m_run[i] = -INFINITY; l_run[i] = 0.f; }
#pragma unroll
  for (int j = 0; j < NF; ++j) m_red[j] = -INFINITY;

  for (int t = 0; t < x.nt; ++t) {
    const uint32_t sb = n & 1;
    const int nvalid = x.local ? rec->valid[t] : min(kTile, x.te - (x.tb + t * kTile));
    mbar_wait(C.s_full + sb, (n >> 1) & 1);
    if (C.warp == 2 && lane == 0) trace_ev(*C.p, 7, n);
    tc_fence_after();
    if constexpr (WB > 0) {
      const uint32_t tS = C.tmem + C.lane_off + kColS + sb * 64;
      float *red_max = C.red_g + (n & 1) * 4 * kRedCols;
      uint32_t s[4 * WB];
      tmem_ld_16x256<WB>(tS + 8 * blk0, s);
      tmem_ld_wait();
      if (C.warp == 2 && lane == 0) trace_ev(*C.p, 4, n);
      float x2[4 * WB];
#pragma unroll
      for (int i = 0; i < 4 * WB; ++i) x2[i] = __uint_as_float(s[i]);
      if (nvalid < kTile || !rows_live) {
        const bool vA = tA < nvalid, vB = tA + 8 < nvalid;
#pragma unroll
        for (int b = 0; b < WB; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool live = 8 * (blk0 + b) + c0 + e < n_live;
            if (!(live && vA)) x2[4 * b + e] = -INFINITY;
            if (!(live && vB)) x2[4 * b + 2 + e] = -INFINITY;
          }
      }
      // Lazy max: the running maxima only move when some score exceeds them by > 8 (log2
      // units).  One barrier-reduction tells the group whether any thread sees such a
      // score; only then is the exact column max reduced (butterfly + SMEM exchange).
      float v[NC];
      bool exceed = false;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        v[i] = fmaxf(x2[4 * (i >> 1) + (i & 1)], x2[4 * (i >> 1) + 2 + (i & 1)]);
        exceed |= v[i] * C.c > m_run[i] + 8.f;
      }
      if (bar_red_or(C.bar_id, 128, exceed)) {
#pragma unroll
        for (int st = 0; st < 3; ++st) {
          const int M = 16 >> st;
          const int cnt = bfly_cnt(NC, st);
          if (cnt % 2 == 0) {
            const bool up = (lane & M) != 0;
#pragma unroll
            for (int j = 0; j < cnt / 2; ++j) {
              const float send = up ? v[j] : v[cnt / 2 + j];
              const float keep = up ? v[cnt / 2 + j] : v[j];
              v[j] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, M));
            }
          } else {
#pragma unroll
            for (int j = 0; j < cnt; ++j) v[j] = fmaxf(v[j], __shfl_xor_sync(0xffffffffu, v[j], M));
          }
        }
#pragma unroll
        for (int j = 0; j < NF; ++j) red_max[wq * kRedCols + col[j]] = v[j];
        named_bar_sync(C.bar_id, 128);
        if (C.warp == 2 && lane == 0) trace_ev(*C.p, 13, n);
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          float mx = fmaxf(fmaxf(red_max[col[j]], red_max[kRedCols + col[j]]),
                           fmaxf(red_max[2 * kRedCols + col[j]], red_max[3 * kRedCols + col[j]]));
          mx *= C.c;  // log2 units (c = softmax scale * log2 e > 0)
          if (mx > m_red[j] + 8.f) m_red[j] = mx;
          v[j] = m_red[j];
        }
#pragma unroll
        for (int st = 2; st >= 0; --st) {
          const int M = 16 >> st;
          const int cnt = bfly_cnt(NC, st);
          if (cnt % 2 == 0) {
            const bool up = (lane & M) != 0;
            float lo[NC], hi[NC];
#pragma unroll
            for (int j = 0; j < cnt / 2; ++j) {
              const float recv = __shfl_xor_sync(0xffffffffu, v[j], M);
              lo[j] = up ? recv : v[j];
              hi[j] = up ? v[j] : recv;
            }
#pragma unroll
            for (int j = 0; j < cnt / 2; ++j) { v[j] = lo[j]; v[cnt / 2 + j] = hi[j]; }
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < NC; ++i) v[i] = m_run[i];
      }
      if (C.warp == 2 && lane == 0) trace_ev(*C.p, 9, n);
      bool need_any = false;
      float alpha[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        alpha[i] = 1.f;
        if (v[i] != m_run[i]) {
          alpha[i] = ex2(m_run[i] - v[i]);  // 0 when m_run = -inf
          l_run[i] *= alpha[i];
          m_run[i] = v[i];
          need_any = true;
        }
      }
      // P = 2^(x c - m) = hi + lo (bf16 each), packed for stmatrix before waiting on the MMA
      uint32_t pk[4 * WB];
#pragma unroll
      for (int b = 0; b < WB; ++b) {
        float pA[2], pB[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 2 * b + e;
          const float neg_m = m_run[i] == -INFINITY ? 0.f : -m_run[i];
          pA[e] = ex2(fmaf(x2[4 * b + e], C.c, neg_m));
          pB[e] = ex2(fmaf(x2[4 * b + 2 + e], C.c, neg_m));
          l_run[i] += pA[e] + pB[e];
        }
        split_hi_lo<TAPER_PHI_TRUNC_SWAP>(pA[0], pA[1], pk[4 * b], pk[4 * b + 2]);
        split_hi_lo<TAPER_PHI_TRUNC_SWAP>(pB[0], pB[1], pk[4 * b + 1], pk[4 * b + 3]);
      }
      if (C.warp == 2 && lane == 0) trace_ev(*C.p, 10, n);
      // the P^T (half) buffer this tile writes was last read by PV(n-2) when this and the
      // previous tile are narrow, else by PV(n-1); an O rescale needs PV(n-1) complete
      const bool rescale = t > 0 && __any_sync(0xffffffffu, need_any);
      if ((rescale || wide || prev_wide) && n >= 1)
        mbar_wait(C.pv_done + ((n - 1) & 1), ((n - 1) >> 1) & 1);
      else if (n >= 2)
        mbar_wait(C.pv_done + (n & 1), ((n - 2) >> 1) & 1);
      if (rescale) {
        // O^T *= alpha for the group's rows: every warp holds every factor (lanes 0-3 cover
        // all of the group's columns), published in the warp's own SMEM slice
        if (lane < 4) {
#pragma unroll
          for (int b = 0; b < WB; ++b) {
            C.alpha_s[8 * b + c0] = alpha[2 * b];
            C.alpha_s[8 * b + c0 + 1] = alpha[2 * b + 1];
          }
        }
        __syncwarp();
        tc_fence_after();
#pragma unroll 1
        for (int b = 0; b < WB; ++b) {
          uint32_t o[16];
          tmem_ld16(tO + 16 * (blk0 + b), o);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            o[j] = __float_as_uint(__uint_as_float(o[j]) * C.alpha_s[8 * b + (j & 7)]);
          tmem_st16(tO + 16 * (blk0 + b), o);
        }
        tmem_st_wait();
      }
      if (C.warp == 2 && lane == 0) trace_ev(*C.p, 14, n);
      const uint32_t pbuf = wide ? 0u : (n & 1) * kPTHalf;
#pragma unroll
      for (int b = 0; b < WB; ++b)
        stmatrix_x4_trans(st_addr[b] + pbuf, pk[4 * b], pk[4 * b + 1], pk[4 * b + 2], pk[4 * b + 3]);
      if (C.warp == 2 && lane == 0) trace_ev(*C.p, 15, n);
    } else if (n >= 2) {  // no rows: keep in step with the writers (p_full parity phases)
      mbar_wait(C.pv_done + (n & 1), ((n - 2) >> 1) & 1);
    }
    prev_wide = wide;
    if (C.grp == 1 && nvalid < kTile) {  // group 1 has fewer (w = 1: no) rows
      // partial tile: V rows past the last valid token were not loaded (or hold tokens
      // past the sequence end); zero them so 0 * garbage cannot reach O
      const uint32_t vs = n % kVStages;
      mbar_wait(C.vfull + vs, (n / kVStages) & 1);
      uint8_t *vt = C.smem + kOffV + vs * kStageBytes;
      const int nz = (kTile - nvalid) * 8;  // 16 B chunks per d-half (128 B per row)
      for (int i = C.tid - 384; i < 2 * nz; i += 128) {
        const int hf = i / nz, j = i - hf * nz;
        *reinterpret_cast<uint4 *>(vt + hf * 8192 + nvalid * 128 + j * 16) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    fence_proxy_async_smem();  // P^T / V zeros (generic stores) -> visible to the MMA
    tc_fence_before();
    if (lane == 0 && C.warp == 2) trace_ev(*C.p, 8, n);
    mbar_arrive(C.p_full_g + (n & 1));
    ++n;
  }
  // row sums: this thread's partial over its 2 tokens per tile -> 16 tokens of its warp; the
  // 4 warps' partials go to SMEM without a group barrier and the epilogue adds them (the
  // slowest warp's item end then overlaps the next item's first tile)
  if constexpr (WB > 0) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      l_run[i] += __shfl_xor_sync(0xffffffffu, l_run[i], 4);
      l_run[i] += __shfl_xor_sync(0xffffffffu, l_run[i], 8);
      l_run[i] += __shfl_xor_sync(0xffffffffu, l_run[i], 16);
    }
  }
  if (C.warp == 2 && lane == 0) trace_ev(*C.p, 1, 2048 + item_idx);
  // publish (m, l) for the epilogue; xml[ob] / lpart[ob] were consumed by epilogue item_idx-2
  mbar_wait(C.o_free + ob, ((item_idx >> 1) & 1) ^ 1);
  if (C.warp == 2 && lane == 0) trace_ev(*C.p, 2, 2048 + item_idx);
  if constexpr (WB > 0) {
    if (lane < 4) {
      float *lp = C.lpart + (ob * 4 + wq) * 128 + 8 * blk0;
#pragma unroll
      for (int b = 0; b < WB; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          lp[8 * b + c0 + e] = l_run[2 * b + e];
          if (wq == 0) C.xml[ob * 128 + 8 * (blk0 + b) + c0 + e] = make_float2(m_run[2 * b + e], 0.f);
        }
    }
  }
  mbar_arrive(C.ml_full + ob);
  if (C.warp == 2 && lane == 0) trace_ev(*C.p, 3, 2048 + item_idx);
}

// Row mode: one shared item of w >= kRowMin branches (8 w <= 128 stacked rows; M = 128 when
// 8 w > 64, else 64).  Thread = stacked row: with M = 128 row 32 wq + lane holds 32 tokens of
// the tile; with M = 64 (rows in lanes 0-15 of each quadrant, 16x32bx2 accesses) row
// 16 wq + lane % 16 holds 16 tokens, lanes l and l ^ 16 the two halves.  Group g takes tokens
// [32 g, 32 g + 32) of every tile; the two groups' tile maxima of a row meet in SMEM behind a
// 64-thread barrier of the warp pair sharing the TMEM quadrant, so both apply the same lazy
// running max (moves only when a tile max exceeds it by > 8 in log2 units) and each rescales
// its half of O's 128 columns.  P = 2^(x c - m) = hi + lo goes to TMEM as two sets of bf16
// pairs, the A operands of two PV TS-MMAs accumulating into the same O.
#ifndef TAPER_ROW_NOINLINE
#define TAPER_ROW_NOINLINE 0
#endif
#if TAPER_ROW_NOINLINE
#define TAPER_ROW_INLINE __noinline__
#else
#define TAPER_ROW_INLINE __forceinline__
#endif
// (TAPER_ROW_NOINLINE=1 moves it out of line: measured worse -- a 320 B stack frame and
// spills in the kernel -- so it is inlined; the 1.7 % a row path once cost swap-only
// layers came from the MMA warp's loop, fixed there.)
template <bool M128>
__device__ TAPER_ROW_INLINE void softmax_item_row(const SoftmaxCtx C, const Item x,
                                                  uint32_t item_idx, uint32_t &n) {
  constexpr int NT = M128 ? 32 : 16;  // tokens per thread per tile
  const int lane = C.lane, wq = C.wq, grp = C.grp;
  const int half = M128 ? 0 : (lane >> 4);
  const int row = M128 ? 32 * wq + lane : 16 * wq + (lane & 15);
  const int n_live = 8 * x.w;
  const bool warp_live = (M128 ? 32 * wq : 16 * wq) < n_live;  // same for the warp pair
  const bool writer = M128 || half == 0;                      // one thread per row and group
  const int tk0 = 32 * grp + 16 * half;                       // first token of this thread
  const uint32_t ob = item_idx & 1;
  const uint32_t tO = C.tmem + C.lane_off + kColO + ob * 128;
  const int pair_bar = 4 + wq;
  float m_run = -INFINITY, l_run = 0.f;
  for (int t = 0; t < x.nt; ++t) {
    const uint32_t sb = n & 1;
    const int nvalid = min(kTile, x.te - (x.tb + t * kTile));
    mbar_wait(C.s_full + sb, (n >> 1) & 1);
    tc_fence_after();
    if (warp_live) {
      uint32_t s[NT];
      const uint32_t tS = C.tmem + C.lane_off + kColS + sb * 64 + 32 * grp;
      if constexpr (M128) tmem_ld32(tS, s); else tmem_ld_x2_16<16>(tS, s);
      tmem_ld_wait();
      float xv[NT];
      float mh = -INFINITY;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        xv[j] = tk0 + j < nvalid ? __uint_as_float(s[j]) : -INFINITY;
        mh = fmaxf(mh, xv[j]);
      }
      if constexpr (!M128) mh = fmaxf(mh, __shfl_xor_sync(0xffffffffu, mh, 16));
      float *rb = C.row_red + sb * 256;  // [grp][row], by tile parity
      if (writer) rb[grp * 128 + row] = mh;
      named_bar_sync(pair_bar, 64);
      const float mt = fmaxf(mh, rb[(grp ^ 1) * 128 + row]) * C.c;  // log2 units
      float alpha = 1.f;
      if (mt > m_run + 8.f) {
        alpha = ex2(m_run - mt);  // 0 when m_run = -inf
        l_run *= alpha;
        m_run = mt;
      }
      const float neg_m = m_run == -INFINITY ? 0.f : -m_run;
      uint32_t pk[NT / 2], pl[kRowPlo ? NT / 2 : 1];
      float ls = 0.f;
#pragma unroll
      for (int i = 0; i < NT / 2; ++i) {
        const float pA = ex2(fmaf(xv[2 * i], C.c, neg_m)), pB = ex2(fmaf(xv[2 * i + 1], C.c, neg_m));
        if constexpr (kRowPlo) {
          split_hi_lo<false>(pA, pB, pk[i], pl[i]);
          ls += pA + pB;
        } else {
          pk[i] = pack_bf16(pA, pB);
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&pk[i]));
          ls += f.x + f.y;  // the row sum of what the MMA multiplies
        }
      }
      l_run += ls;
      // O rows *= alpha needs PV(n-1) complete (and PV(n) waits for this tile's p_full); the
      // P buffer this tile writes was last read by PV(n-2)
      const bool rescale = t > 0 && __any_sync(0xffffffffu, alpha != 1.f);
      if (rescale) {
        mbar_wait(C.pv_done + ((n - 1) & 1), ((n - 1) >> 1) & 1);
        tc_fence_after();
        uint32_t o[32];
        if constexpr (M128) {
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            tmem_ld32(tO + 64 * grp + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
            tmem_st32(tO + 64 * grp + 32 * c, o);
          }
        } else {
          tmem_ld_x2_32<32>(tO + 64 * grp, o);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
          tmem_st_x2_32<32>(tO + 64 * grp, o);
        }
      } else if (n >= 2) {
        mbar_wait(C.pv_done + (n & 1), ((n - 2) >> 1) & 1);
      }
      const uint32_t tP = C.tmem + C.lane_off + kColP + sb * 64 + 16 * grp;
      if constexpr (M128) {
        tmem_st16(tP, *reinterpret_cast<const uint32_t(*)[16]>(pk));
        if constexpr (kRowPlo) tmem_st16(tP + 32, *reinterpret_cast<const uint32_t(*)[16]>(pl));
      } else {
        tmem_st_x2_8<8>(tP, pk);
        if constexpr (kRowPlo) tmem_st_x2_8<8>(tP + 32, pl);
      }
      tmem_st_wait();
    }
    if (C.grp == 1 && nvalid < kTile) {  // zero V rows past the last valid token (as swap mode)
      const uint32_t vs = n % kVStages;
      mbar_wait(C.vfull + vs, (n / kVStages) & 1);
      uint8_t *vt = C.smem + kOffV + vs * kStageBytes;
      const int nz = (kTile - nvalid) * 8;
      for (int i = C.tid - 384; i < 2 * nz; i += 128) {
        const int hf = i / nz, j = i - hf * nz;
        *reinterpret_cast<uint4 *>(vt + hf * 8192 + nvalid * 128 + j * 16) = make_uint4(0u, 0u, 0u, 0u);
      }
      fence_proxy_async_smem();
    }
    tc_fence_before();
    mbar_arrive(C.p_full_g + (n & 1));
    ++n;
  }
  if constexpr (!M128) l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
  // publish (m, l) for the epilogue (which adds the two groups' partial sums); xml[ob] and
  // lpart[ob] were consumed by epilogue item_idx-2
  mbar_wait(C.o_free + ob, ((item_idx >> 1) & 1) ^ 1);
  if (warp_live && writer && row < n_live) {
    C.lpart[(ob * 4 + grp) * 128 + row] = l_run;
    if (grp == 0) C.xml[ob * 128 + row] = make_float2(m_run, 0.f);
  }
  mbar_arrive(C.ml_full + ob);
}

// Consumer side of the claimed-item ring: the k-th item this CTA processes (-1 = done).
__device__ __forceinline__ int ring_item(uint64_t *it_full, const ItemRec *recs, uint32_t k) {
  const uint32_t slot = k % kItemRing;
  mbar_wait(it_full + slot, (k / kItemRing) & 1);
  return *reinterpret_cast<const volatile int32_t *>(&recs[slot].it);
}
__device__ __forceinline__ void ring_release(uint64_t *it_empty, uint32_t k, int lane) {
  (void)lane;
  mbar_arrive(it_empty + (k % kItemRing));
}

__global__ void __launch_bounds__(kAttnThreads, 1)
    attend_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const __grid_constant__ CUtensorMap tmK16,
                  const __grid_constant__ CUtensorMap tmV16,
                  const __grid_constant__ CUtensorMap tmQ, AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment (SW128) by pointer arithmetic on the shared array, so the compiler
  // keeps the shared address space (LDS/STS instead of generic loads)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kOffBar);
  uint64_t *kfull = bars;                      // [kKStages] TMA -> MMA (K tile landed)
  uint64_t *kempty = kfull + kKStages;         // [kKStages] QK done -> TMA
  uint64_t *vfull = kempty + kKStages;         // [kVStages] TMA -> MMA (V tile landed)
  uint64_t *vempty = vfull + kVStages;         // [kVStages] PV done -> TMA
  uint64_t *s_full = vempty + kVStages;        // [2] QK done -> softmax
  uint64_t *p_full = s_full + 2;               // [group][tile parity] P^T written -> PV
  uint64_t *pv_done = p_full + 4;              // [2] PV done -> softmax (P^T free, O stable)
  uint64_t *q_full = pv_done + 2;              // [2] Q^T landed (TMA) -> MMA
  uint64_t *q_free = q_full + 2;               // [2] last QK of the item done -> scheduler
  uint64_t *o_full = q_free + 2;               // [2] last PV of an item -> epilogue
  uint64_t *o_free = o_full + 2;               // [2] epilogue done -> MMA / softmax
  uint64_t *ml_full = o_free + 2;              // [2] softmax (m, l) published -> epilogue
  uint64_t *it_full = ml_full + 2;             // [kItemRing] scheduler published an item
  uint64_t *it_empty = it_full + kItemRing;    // [kItemRing] all consumer warps are done
  uint64_t *sched_go = it_empty + kItemRing;   // K producer started an item -> scheduler
  uint64_t *val_bar = sched_go + 1;            // scheduler validated record 0 -> epilogue
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sched_go + 2);
  volatile int32_t *first_ok = reinterpret_cast<volatile int32_t *>(tmem_slot + 1);  // record 0 valid
  ItemRec *recs = reinterpret_cast<ItemRec *>(smem + kOffRec);
  float2 *xml = reinterpret_cast<float2 *>(smem + kOffML);
  const float *lpart = reinterpret_cast<const float *>(smem + kOffLPart);
  float *red = reinterpret_cast<float *>(smem + kOffRed);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = p.h_local;
  if (tracing(p) && tid == 0) {  // per-CTA wall-clock span (debug trace)
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3000 + blockIdx.x) * 16 + 0] = (long long)g;
  }

  // No zero-fill of the K/V rings: token rows of a partial tile that TMA does not load hold
  // stale data, which never reaches O -- their scores are masked to -inf before the max,
  // and softmax group 1 zeroes the V rows past the last valid token of every partial tile
  // before the PV MMA reads them (0 * NaN would otherwise poison O).  Measured without PDL
  // overlap (a foreign kernel between calls): 47.3 -> 46.0 us per call at h = 1.
  // (-DTAPER_ZERO_FILL restores the fill.)
#ifdef TAPER_ZERO_FILL
  for (int i = tid; i < kOffQ / 16; i += kAttnThreads)
    reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
#endif
  if (tid == 0) {
    for (int i = 0; i < kKStages; ++i) { mbar_init(kfull + i, 1); mbar_init(kempty + i, 1); }
    for (int i = 0; i < kVStages; ++i) { mbar_init(vfull + i, 1); mbar_init(vempty + i, 1); }
    for (int i = 0; i < 4; ++i) mbar_init(p_full + i, 128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(pv_done + i, 1);
      mbar_init(q_full + i, 1);
      mbar_init(q_free + i, 1);
      mbar_init(o_full + i, 1);
      mbar_init(o_free + i, 128);
      mbar_init(ml_full + i, 256);
    }
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(it_full + i, 32);
      mbar_init(it_empty + i, kRingConsumers);
    }
    mbar_init(sched_go, 1);
    mbar_init(val_bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK); tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmK16); tma_prefetch_desc(&tmV16); tma_prefetch_desc(&tmQ);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) trace_cta(p, 5);  // prologue done
  // PDL: the prologue above overlapped the previous kernel; wait for its memory, then let
  // the merge kernel launch (it reads the work list, which is complete and visible once
  // this grid's dependency has resolved; its warps then wait for per-request completion
  // counters).  The scheduler warp resolves its first item before waiting (see below).
  if (warp != 11) {
    pdl_wait();
    pdl_launch_dependents();
  }

  if (warp == 11) {
    // ======================= item scheduler ==================================================
    // Claims work items (global atomic counter -> dynamic scheduling) one item ahead of the
    // K producer, resolves each into an SMEM ItemRec (descriptor, tile geometry, page
    // indices: lane l resolves tile l), publishes it, then loads the item's stacked queries
    // Q^T (one 2 KB TMA box per branch: its 8 GQA rows, SW128) into Q buffer k & 1.  The
    // dependent global loads of an item thus overlap the previous item.
    const int box_tok = p.page_size < kTile ? p.page_size : kTile;
    // The first item is resolved speculatively, before the grid dependency, from plain
    // loads of the work list issued all at once (no acquire chain); after the dependency
    // resolves, every work-list word the record was built from is read again and compared
    // (include/taper.h ordering contract): equal values give the same record, otherwise it
    // is resolved again from the values now visible.
    // Control snapshot: one work-list word per lane from a fixed address -- lanes 0-7 the
    // descriptor of claim index blockIdx.x, 8-11 header words -- so the first item costs one
    // load latency before its pages, and validating it after the grid dependency another.
    const int32_t *snap_addr =
        lane < 8 ? reinterpret_cast<const int32_t *>(
                       p.sorted + min(int(blockIdx.x) / h, p.cap_cs > 0 ? p.cap_cs - 1 : 0)) + lane
                 : p.hdr + (lane == 8 ? 0 : lane == 9 ? 5 : lane == 10 ? 3 : lane == 11 ? 4 : 0);
    int32_t snap = __ldcg(snap_addr);
    // claims per launch (items x KV heads), or none if the work list was written for another
    // workspace / h_local (warp-uniform)
    int n_items = 0;
    auto derive = [&]() {
      const bool ok = __shfl_sync(0xffffffffu, snap, 11) == h && __shfl_sync(0xffffffffu, snap, 10) == p.cap_cs;
      n_items = ok ? (__shfl_sync(0xffffffffu, snap, 8) + __shfl_sync(0xffffffffu, snap, 9)) * h : 0;
    };
    derive();
    if (lane == 0) trace_cta_dep(p, 12, n_items);  // header loaded
    int *work_counter = p.hdr + 8;
    // the descriptor of claim index `it` (longest first, then KV head), loaded before the
    // claim is known to be valid (the index is clamped into the table) so that its latency
    // overlaps the header loads: one dependent global load less on the way to the first TMA
    auto load_desc = [&](int it) -> int32_t {
      int qi = (it > 0 ? it : 0) / h;
      qi = qi < p.cap_cs - 1 ? qi : (p.cap_cs > 0 ? p.cap_cs - 1 : 0);
      return lane < 8 ? __ldcg(reinterpret_cast<const int32_t *>(p.sorted + qi) + lane) : 0;
    };
    // claim index `it` (-1: none) -> the SMEM record (descriptor, per-tile geometry and
    // pages); slot_j = the admitted slot of the item's branch `lane` (its Q rows), loaded
    // alongside the pages
    int4 lt_seen = make_int4(0, 0, 0, 0);  // local item: the entry of tile `lane`
    auto resolve = [&](ItemRec *rec, int it, int32_t d, int &w, int &adm_off, int &g, int &slot_j) {
      w = 0; adm_off = 0; g = 0; slot_j = 0;
      if (it >= 0) {
        const int qi = it / h;
        g = it - qi * h;
        const int nt = __shfl_sync(0xffffffffu, d, 6);
        Item x;
        x.r = __shfl_sync(0xffffffffu, d, 0);
        w = __shfl_sync(0xffffffffu, d, 1);
        adm_off = __shfl_sync(0xffffffffu, d, 2);
        x.tb = __shfl_sync(0xffffffffu, d, 4);
        x.te = __shfl_sync(0xffffffffu, d, 5);
        x.local = __shfl_sync(0xffffffffu, d, 7) & kItemLocal;
        if (lane < 8) rec->desc[lane] = d;
        if (lane < w) slot_j = __ldcg(p.adm_by_req + adm_off + lane);
        for (int t = lane; t < nt; t += 32) {
          const TileInfo ti = tile_info(p, x, t);
          if (t == lane) lt_seen = ti.lt;
          rec->tok0[t] = ti.tok0;
          rec->valid[t] = ti.valid;
#pragma unroll
          for (int b = 0; b < kTile / 16; ++b)
            rec->pg[t][b] =
                b * box_tok < ti.valid ? __ldcg(ti.pages + (ti.tok0 + b * box_tok) / p.page_size) : 0;
        }
      }
      if (lane == 0) { rec->it = it; rec->g = g; }
    };
    // claim index of the k-th item of this CTA: blockIdx.x first, then from the counter
    auto claim = [&](uint32_t k) -> int {
      int c = int(blockIdx.x);
      if (k > 0 && lane == 0) c = int(gridDim.x) + atomicAdd(work_counter, 1);
      return __shfl_sync(0xffffffffu, c, 0);
    };
    auto first_desc = [&]() -> int32_t { return lane < 8 ? snap : 0; };
    // publish record k (every lane arrives) and load its Q^T: box {64 d, 8 rows, 2 d-halves}
    // of q viewed as (d-lo, GQA row, d-half, slot * h + g) -> [d-half][8 rows][128 B] per branch
    auto publish = [&](uint32_t k, uint32_t slot, int it, int w, int g, int slot_j) {
      __syncwarp();
      mbar_arrive(it_full + slot);  // release (every lane): the record is visible
      if (it < 0) return;
      const uint32_t qb = k & 1;
      mbar_wait(q_free + qb, ((k >> 1) & 1) ^ 1);
      if (elect_one()) mbar_arrive_expect_tx(q_full + qb, w * 2048);
      __syncwarp();
      if (lane < w)
        tma_load_4d(smem + kOffQ + qb * kQBytes + lane * 2048, &tmQ, q_full + qb, 0, 0, 0,
                    slot_j * h + g);
      if (k == 0 && lane == 0) trace_cta(p, 9);  // first Q load issued
      __syncwarp();
    };
    bool redo = false;  // record 0 failed validation: record 1 is the first claim again
    for (uint32_t k = 0;; ++k) {
      if (k >= 1) mbar_wait(sched_go, (k - 1) & 1);  // K producer started item k-1
      const bool first = k == 0 || (k == 1 && redo);
      int it = claim(first ? 0 : k);
      int32_t d = first ? first_desc() : load_desc(it);
      if (k == 0 && lane == 0) trace_cta_dep(p, 13, d);  // descriptor loaded
      const uint32_t slot = k % kItemRing;
      ItemRec *rec = recs + slot;
      mbar_wait(it_empty + slot, ((k / kItemRing) & 1) ^ 1);
      int w, adm_off, g, slot_j;
      resolve(rec, it < n_items ? it : -1, d, w, adm_off, g, slot_j);
      if (k == 0 && lane == 0) trace_cta(p, 6);  // first record resolved
      if (k == 0) {
        // The first record was resolved while the previous kernel drained.  Wait for it (q,
        // the K/V pools and a just-written work list become visible) and let the merge
        // kernel launch.  A record that names an item is published at once; then the
        // header, the descriptor, the branches' slots and (local item) the tile entries
        // are loaded again -- independent loads, one latency -- and compared with the
        // values it was resolved from.  On a difference the item runs anyway (its loads
        // stay in bounds: TMA drops out-of-range boxes) but the epilogue discards its
        // partials (first_ok = 0), and record 1 is the first claim resolved again.
        pdl_wait();
        pdl_launch_dependents();
        if (lane == 0) trace_cta(p, 8);  // grid dependency resolved
        const bool early_item = it >= 0 && it < n_items;
        if (early_item) publish(0, slot, it, w, g, slot_j);
        const int32_t snap2 = __ldcg(snap_addr);
        const int nt_e = __shfl_sync(0xffffffffu, d, 6), tb_e = __shfl_sync(0xffffffffu, d, 4);
        const bool local_e = __shfl_sync(0xffffffffu, d, 7) & kItemLocal;
        const int sj2 = (early_item && lane < w) ? __ldcg(p.adm_by_req + adm_off + lane) : slot_j;
        const int4 lt2 = (early_item && local_e && lane < nt_e) ? __ldcg(p.ltiles + tb_e + lane) : lt_seen;
        const bool same = !TAPER_DBG_FORCE_RERESOLVE & (snap2 == snap) & (sj2 == slot_j) & (lt2.x == lt_seen.x) &
                          (lt2.y == lt_seen.y) & (lt2.z == lt_seen.z) & (lt2.w == lt_seen.w);
        const bool ok = __all_sync(0xffffffffu, same);
        if (!ok) {
          snap = snap2;
          derive();
        }
        if (lane == 0) {
          *first_ok = (!early_item || ok) ? 1 : 0;
          mbar_arrive(val_bar);
        }
        if (early_item) {
          redo = !ok;
          continue;
        }
        if (!ok) {  // nothing published yet: resolve the first claim from the visible words
          it = claim(0);
          d = first_desc();
          resolve(rec, it < n_items ? it : -1, d, w, adm_off, g, slot_j);
        }
      }
      if (it >= n_items) it = -1;
      publish(k, slot, it, w, g, slot_j);
      if (it < 0) break;
    }
  } else if (warp == 0 || warp == 10) {
    // ======================= TMA producers: warp 0 = K, warp 10 = V =======================
    // Tile geometry and pages come from the item record in SMEM; the whole warp runs the
    // loop with warp-uniform operands and one elected lane issues (no waterfall loops).
    const bool is_k = warp == 0;
    const CUtensorMap *tmap = is_k ? &tmK : &tmV;
    const CUtensorMap *tmap16 = is_k ? &tmK16 : &tmV16;
    uint64_t *ring_full = is_k ? kfull : vfull;
    uint64_t *ring_empty = is_k ? kempty : vempty;
    const int n_stages = is_k ? kKStages : kVStages;
    uint8_t *ring = smem + (is_k ? 0 : kOffV);
    const int box_tok = p.page_size < kTile ? p.page_size : kTile;
    const uint32_t half_box_bytes = box_tok * 128;
    uint32_t n_prod = 0;  // global tile counter
    for (uint32_t k = 0;; ++k) {
      const int it = ring_item(it_full, recs, k);
      if (it < 0) {
        ring_release(it_empty, k, lane);
        break;
      }
      const ItemRec *rec = recs + (k % kItemRing);
      const int g_u = rec->g;
      const int nt_u = rec->desc[6];
      // the scheduler may claim the next item once this one's producer is kClaimLead tiles
      // from its end (enough for the next record's dependent loads; an earlier claim keeps
      // work reserved on a busy CTA while others run dry at the end of the queue)
      const int t_go = nt_u > kClaimLead ? nt_u - kClaimLead : 0;
      // (Tiles issued in pairs by lanes 0 and 1 -- a higher TMA issue ceiling in isolation,
      // scripts/tma_issue_probe.cu -- measured 2.3 % slower on C2, r2 run l; one lane issues.)
      for (int t = 0; t < nt_u; ++t, ++n_prod) {
        if (is_k && t == t_go) {
          __syncwarp();
          if (lane == 0) mbar_arrive(sched_go);
        }
        const int tok0 = rec->tok0[t];
        const int valid = rec->valid[t];
        const uint32_t st = n_prod % n_stages;
        uint8_t *dst = ring + st * kStageBytes;
        mbar_wait(ring_empty + st, ((n_prod / n_stages) & 1) ^ 1);
        if (is_k && lane == 0) trace_ev(p, 0, n_prod);
        if (is_k && lane == 0 && tracing(p) && t == 0 && n_prod == 0) {
          unsigned long long g;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
          p.trace[(size_t)(3000 + blockIdx.x) * 16 + 2] = (long long)g;  // first TMA issued
        }
        if (elect_one()) {
          if (p.tma5d && valid == kTile) {
            // one box: {64 d, 64 tokens, 2 d-halves} -> [d-half][token][64] (two SW128 atoms)
            mbar_arrive_expect_tx(ring_full + st, 2 * kTile * 128);
#ifndef TAPER_KV_EVICT_FIRST
#define TAPER_KV_EVICT_FIRST 1
#endif
#if TAPER_KV_EVICT_FIRST
            // K / V tiles are read once per layer: evict-first keeps L2 for the page tables,
            // q and the partials (same-box A/B: C2 192.2 -> 189.3 us, C5 1723 -> 1739 us)
            tma_load_5d_hint(dst, tmap, ring_full + st, 0, tok0 % p.page_size, 0, g_u, rec->pg[t][0],
                             l2_policy_evict_first());
#else
            tma_load_5d(dst, tmap, ring_full + st, 0, tok0 % p.page_size, 0, g_u, rec->pg[t][0]);
#endif
          } else if (p.tma5d) {
            // partial tile: {64 d, 16 tokens} boxes per d-half up to the last valid token
            // (rows past it are zeroed by the softmax warps before PV)
            const int n16 = (valid + 15) >> 4;
            const int pg0 = rec->pg[t][0];
            mbar_arrive_expect_tx(ring_full + st, n16 * 2 * 2048);
            for (int b = 0; b < n16; ++b)
              for (int hf = 0; hf < 2; ++hf)
                tma_load_5d(dst + hf * 8192 + b * 2048, tmap16, ring_full + st, 0,
                            tok0 % p.page_size + 16 * b, hf, g_u, pg0);
          } else {
            int pg[kTile / 16];
#pragma unroll
            for (int b = 0; b < kTile / 16; ++b) pg[b] = rec->pg[t][b];
            const int n_box = (valid + box_tok - 1) / box_tok;
            mbar_arrive_expect_tx(ring_full + st, n_box * half_box_bytes * 2);
#pragma unroll
            for (int b = 0; b < kTile / 16; ++b) {
              if (b < n_box) {
                const int row = (tok0 + b * box_tok) % p.page_size;
                const int o = b * half_box_bytes;
                tma_load_4d(dst + o, tmap, ring_full + st, 0, row, g_u, pg[b]);
                tma_load_4d(dst + 8192 + o, tmap, ring_full + st, 64, row, g_u, pg[b]);
              }
            }
          }
        }
        __syncwarp();
        if (is_k && lane == 0) trace_ev(p, 12, n_prod);
      }
      ring_release(it_empty, k, lane);
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (whole warp, one elected lane issues) =========
    // Every lane runs the loop so all operands stay warp-uniform (uniform registers); the
    // tcgen05.mma / commit instructions are issued by elect.sync's lane (CUTLASS pattern).
    const uint32_t sK = smem_u32(smem), sV = smem_u32(smem + kOffV);
    const uint32_t sQ = smem_u32(smem + kOffQ), sPT = smem_u32(smem + kOffPT);
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    uint32_t n = 0;  // global tile counter (S double buffer index = n & 1)
    for (uint32_t item_idx = 0;; ++item_idx) {
      const int it = ring_item(it_full, recs, item_idx);
      Item x;
      decode_item(recs + item_idx % kItemRing, x);
      ring_release(it_empty, item_idx, lane);
#ifdef TAPER_TRACE_ITEMS
      if (it < 0 && lane == 0 && tracing(p)) {  // per-CTA items and tiles (debug)
        p.trace[(size_t)(3000 + blockIdx.x) * 16 + 3] = item_idx;
        p.trace[(size_t)(3000 + blockIdx.x) * 16 + 4] = n;
      }
#endif
      if (it < 0) break;
      const int wi = __shfl_sync(0xffffffffu, x.w, 0);
      const int nt = __shfl_sync(0xffffffffu, x.nt, 0);
      const bool row = kRowMma && __shfl_sync(0xffffffffu, x.row, 0);
      const uint32_t qb = item_idx & 1;
      const uint32_t ob = item_idx & 1;  // O double buffer
      const uint32_t tO = tmem_u + kColO + ob * 128;
      mbar_wait(q_full + qb, (item_idx >> 1) & 1);
      if (lane == 0) trace_ev(p, 6, n);
      if (item_idx == 0 && lane == 0) trace_cta(p, 10);  // first Q landed
      tc_fence_after();
      // One tile loop per mode (selected once per item): a per-tile mode branch in this
      // latency-critical loop slowed swap-only layers by ~1.7 % (r2 run m).
      auto tile_loop = [&](auto row_c) {
        constexpr bool kRow = decltype(row_c)::value;
        uint32_t idesc_qk, idesc_pv;
        if constexpr (kRow) {
          const int mrow = __shfl_sync(0xffffffffu, x.m128, 0) ? 128 : 64;  // rows on M (padded)
          idesc_qk = umma_idesc_bf16(mrow, 64, false, false);
          idesc_pv = umma_idesc_bf16(mrow, 128, false, true);
        } else {
          idesc_qk = umma_idesc_bf16(64, 8 * wi, false, false);
          idesc_pv = umma_idesc_bf16(128, 16 * wi, true, false);
        }
        for (int t = 0; t <= nt; ++t) {
          if (t < nt) {
            const uint32_t ks = n % kKStages;
            mbar_wait(kfull + ks, (n / kKStages) & 1);
            if (lane == 0) trace_ev(p, 1, n);
            tc_fence_after();
            if (elect_one()) {
              if constexpr (kRow)
                issue_qk_row(tmem_u + kColS + (n & 1) * 64, sQ + qb * kQBytes, sK + ks * kStageBytes,
                             idesc_qk);
              else
                issue_qk(tmem_u + kColS + (n & 1) * 64, sK + ks * kStageBytes, sQ + qb * kQBytes,
                         idesc_qk);
              tc_commit(kempty + ks);
              tc_commit(s_full + (n & 1));
              if (t == nt - 1) tc_commit(q_free + qb);
            }
            __syncwarp();
            if (lane == 0) trace_ev(p, 2, n);
          }
          if (t > 0) {
            // PV of the previous tile (its P is ready once the softmax arrives on p_full)
            const uint32_t m = n - 1;
            mbar_wait(p_full + (m & 1), (m >> 1) & 1);
            mbar_wait(p_full + 2 + (m & 1), (m >> 1) & 1);
            if (lane == 0) trace_ev(p, 3, m);
            const bool first = t == 1;
            if (first) mbar_wait(o_free + ob, ((item_idx >> 1) & 1) ^ 1);  // epilogue item-2 done
            const uint32_t vs = m % kVStages;
            mbar_wait(vfull + vs, (m / kVStages) & 1);
            tc_fence_after();
            if (elect_one()) {
              if constexpr (kRow)
                issue_pv_row(tO, tmem_u + kColP + (m & 1) * 64, sV + vs * kStageBytes, first, idesc_pv);
              else
                issue_pv(tO, sV + vs * kStageBytes,
                         sPT + (wi > kNarrowPT ? 0u : (m & 1) * kPTHalf), first, idesc_pv);
              tc_commit(vempty + vs);
              tc_commit(pv_done + (m & 1));
              if (t == nt) tc_commit(o_full + ob);
            }
            __syncwarp();
            if (lane == 0) trace_ev(p, 5, m);
          }
          if (t < nt) ++n;
        }
      };
      if (__builtin_expect(!row, 1)) {
        tile_loop(BoolC<false>{});
      } else {
        if constexpr (kRowMma) tile_loop(BoolC<true>{});
      }
    }
  } else if (warp < 6 || warp >= 12) {
    // ======================= softmax / O correction (2 groups x 128 threads) ==========
    // Group 0 (warps 2-5) owns the first ceil(w/2) 8-row blocks of the item's stacked rows,
    // group 1 (warps 12-15) the rest; each group covers all four TMEM lane quadrants.
    SoftmaxCtx C;
    C.p = &p;
    C.smem = smem;
    C.grp = warp >= 12 ? 1 : 0;
    C.wq = warp & 3;  // TMEM lane quadrant: tokens 16 wq .. 16 wq + 15
    C.lane = lane;
    C.warp = warp;
    C.tid = tid;
    C.bar_id = C.grp ? 3 : 1;
    C.tmem = tmem;
    C.lane_off = uint32_t(C.wq * 32) << 16;
    C.pt_base = smem_u32(smem + kOffPT);
    C.c = p.scale_log2;
    C.s_full = s_full;
    C.pv_done = pv_done;
    C.vfull = vfull;
    C.p_full_g = p_full + 2 * C.grp;
    C.o_free = o_free;
    C.ml_full = ml_full;
    C.xml = xml;
    C.red_g = red + C.grp * kRedFloats;
    C.alpha_s = reinterpret_cast<float *>(smem + kOffAlpha) + (C.grp * 4 + C.wq) * kRedCols;
    C.row_red = reinterpret_cast<float *>(smem + kOffRowRed);
    C.lpart = reinterpret_cast<float *>(smem + kOffLPart);
    uint32_t n = 0;
    bool prev_wide = true;
    for (uint32_t item_idx = 0;; ++item_idx) {
      const int it = ring_item(it_full, recs, item_idx);
      if (it < 0) {
        ring_release(it_empty, item_idx, lane);
        break;
      }
      const ItemRec *rec = recs + item_idx % kItemRing;
      Item x;
      decode_item(rec, x);
      if (warp == 2 && lane == 0) trace_ev(p, 0, 2048 + item_idx);
      if (kRowSm && x.row) {
        // (M = 64 row items exist only when kRowMin <= 8; n_r >= 9 means M = 128)
        if (kRowMin > 8 || x.m128) softmax_item_row<true>(C, x, item_idx, n);
        else if constexpr (kRowMin <= 8) softmax_item_row<false>(C, x, item_idx, n);
        prev_wide = false;  // the swap P^T halves were last read before this item's tiles
      } else {
        const int wb0 = (x.w + 1) >> 1;
        const int wb = C.grp ? x.w - wb0 : wb0;   // 8-row blocks of this group
        const int blk0 = C.grp ? wb0 : 0;
        switch (wb) {
          case 0: softmax_item<0>(C, rec, x, blk0, item_idx, n, prev_wide); break;
          case 1: softmax_item<1>(C, rec, x, blk0, item_idx, n, prev_wide); break;
          case 2: if constexpr (kSwapMaxWB >= 2) softmax_item<2>(C, rec, x, blk0, item_idx, n, prev_wide); break;
          case 3: if constexpr (kSwapMaxWB >= 3) softmax_item<3>(C, rec, x, blk0, item_idx, n, prev_wide); break;
          default: if constexpr (kSwapMaxWB >= 4) softmax_item<4>(C, rec, x, blk0, item_idx, n, prev_wide); break;
        }
      }
      ring_release(it_empty, item_idx, lane);
    }
  } else {
    // ======================= epilogue (128 threads, warps 6-9) =======================
    // O^T[d][16 b + e (hi) / 16 b + 8 + e (lo)] -> partial row (branch b, GQA row e):
    // thread = d, so every row is written by 128 consecutive threads (coalesced), while the
    // next item's tiles run (O^T is double-buffered in TMEM).
    const int wq = warp & 3;
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const int d = wq * 32 + lane;
    const int etid = tid - 192;  // 0..127
    for (uint32_t item_idx = 0;; ++item_idx) {
      const int it = ring_item(it_full, recs, item_idx);
      Item x;
      decode_item(recs + item_idx % kItemRing, x);
      ring_release(it_empty, item_idx, lane);
      if (it < 0) break;
      const uint32_t ob = item_idx & 1;
      const uint32_t tO = tmem + lane_off + kColO + ob * 128;
      mbar_wait(ml_full + ob, (item_idx >> 1) & 1);
      mbar_wait(o_full + ob, (item_idx >> 1) & 1);
      // record 0 was published before its validation: a record that failed it writes and
      // publishes nothing (its item is resolved again as record 1)
      bool keep = true;
      if (item_idx == 0) {
        mbar_wait(val_bar, 0);
        keep = *first_ok != 0;
        if (!keep) x.w = 0;
      }
      if (warp == 6 && lane == 0) trace_ev(p, 10, 2048 + item_idx);
      if (tracing(p) && blockIdx.x == 0 && warp == 6 && lane == 0 &&
          2048 + int(item_idx) < p.trace_cap) {
        long long *tr = p.trace + (size_t)(2048 + item_idx) * 16;
        tr[13] = x.w; tr[14] = x.nt; tr[15] = x.local;
      }
      tc_fence_after();
      if (kRowEpi && x.row) {
        // row mode: O[row][d], thread = row (M = 128) or half a row (M = 64, 16x32bx2);
        // each thread writes its row's contiguous 512 B (256 B) of the partial
        const bool m128 = kRowMin > 8 || x.m128;
        const int row = m128 ? 32 * wq + lane : 16 * wq + (lane & 15);
        const int hf = m128 ? 0 : (lane >> 4);
        if ((m128 ? 32 * wq : 16 * wq) < 8 * x.w) {
          const bool live = row < 8 * x.w;
          const size_t prow = ((size_t)(x.cs0 + (row >> 3)) * h + x.g) * kGroup + (row & 7);
          const float *lp = lpart + ob * 512 + row;
          const float2 ml = live ? make_float2(xml[ob * 128 + row].x, lp[0] + lp[128]) : make_float2(0.f, 0.f);
          const float inv = ml.y > 0.f ? 1.f / ml.y : 0.f;
          float4 *dst = reinterpret_cast<float4 *>(p.part_o + prow * kHeadDim + 64 * hf);
#pragma unroll 1
          for (int c = 0; c < (m128 ? 4 : 2); ++c) {
            uint32_t o[32];
            if (m128) tmem_ld32(tO + 32 * c, o); else tmem_ld_x2_32<64>(tO + 32 * c, o);
            tmem_ld_wait();
            if (live) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                dst[8 * c + j] = make_float4(__uint_as_float(o[4 * j]) * inv, __uint_as_float(o[4 * j + 1]) * inv,
                                             __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
            }
          }
          if (live && hf == 0)
            p.part_lse[prow] = ml.y > 0.f ? (ml.x + __log2f(ml.y)) * 0.69314718055994531f : -INFINITY;
        }
      }
#pragma unroll 1
      for (int b = 0; b < ((kRowEpi && x.row) ? 0 : x.w); ++b) {
        uint32_t o[16];
        tmem_ld16(tO + 16 * b, o);
        tmem_ld_wait();
        const size_t prow0 = ((size_t)(x.cs0 + b) * h + x.g) * kGroup;
        const float *lp = lpart + ob * 512 + 8 * b;  // the 4 quadrant warps' partial sums
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float L = (lp[e] + lp[128 + e]) + (lp[256 + e] + lp[384 + e]);
          const float inv = L > 0.f ? 1.f / L : 0.f;
          p.part_o[(prow0 + e) * kHeadDim + d] = (__uint_as_float(o[e]) + __uint_as_float(o[8 + e])) * inv;
        }
        if (etid < 8) {
          const float L = (lp[etid] + lp[128 + etid]) + (lp[256 + etid] + lp[384 + etid]);
          p.part_lse[prow0 + etid] =
              L > 0.f ? (xml[ob * 128 + 8 * b + etid].x + __log2f(L)) * 0.69314718055994531f : -INFINITY;
        }
      }
      // hand O^T / (m, l) back, then publish the item: the barrier orders every epilogue
      // thread's partial stores before one thread's gpu-scope fence + counter increment
      // (release pattern), so only that thread waits for the stores to drain
      named_bar_sync(2, 128);
      if (warp == 6 && lane == 0) trace_ev(p, 11, 2048 + item_idx);
      tc_fence_before();
      mbar_arrive(o_free + ob);
      if (etid == 0 && keep) {
        __threadfence();
        atomicAdd(p.done + x.r * kGroup + x.g, 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  if (tid == 0) {
    // the last CTA to exit re-arms the work counter for the next launch (all claims are done)
    __threadfence();
    if (atomicAdd(p.hdr + 9, 1) == int(gridDim.x) - 1) {
      __threadfence();
      p.hdr[8] = 0;
      p.hdr[9] = 0;
    }
  }
  if (tracing(p) && tid == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3000 + blockIdx.x) * 16 + 1] = (long long)g;
  }
}

// ------------------------------------------------------------------ A8: LSE merge
constexpr int kMergeThreads = 256;  // one CTA per admitted slot, warps over (KV head, row)

struct MergeParams {
  long long *trace;  // debug: per-CTA globaltimer span at rows 3200 + CTA (taper_set_trace_buffer)
  int trace_cap;
  const int32_t *hdr;
  const int4 *merge_desc;
  int32_t *done;  // [R * 8] completion counters (attend), [R * 8, 2 R * 8) readers done
  int R;
  const float *part_lse, *part_o;
  __nv_bfloat16 *out;
  float *lse_out;
  int h_local;
  int cap_cs;       // partial capacity of this call's workspace (checked against hdr[3])
  int32_t *status;  // taper_admission.status (TAPER_STATUS_WORK_MISMATCH)
  // fused gather (taper_decode_attention_gather): world > 0 stores every row into all
  // world ranks' gathered buffers [S][64][128] at Q-head column head0 + 8 g + a
  int world, rank, head0;
  __nv_bfloat16 *gout[TAPER_MAX_RANKS];
  int32_t *gflags[TAPER_MAX_RANKS];
  int32_t *gcount;  // merge CTAs done (workspace hdr[11]); the last one raises the flags
};

__device__ __forceinline__ int ld_acquire_sys(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int32_t *p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Per (admitted slot, KV head, GQA row): a warp merges the row's partials (lane: dims
// 4 lane .. 4 lane + 3, 512 B per partial row) with an online LSE, partials in work order
// (prefix chunks, then local items), up to kMergeBatch partials' loads in flight at a time.
// Launched with PDL while attend_kernel is still running: a warp starts as soon as the
// attend epilogues have published all items of its (request, KV head) (acquire on the
// completion counter), so the merge overlaps the attend kernel's tail.
// Units of RPW rows of one KV head; NB partials in flight per round (NB * RPW <= 32 lanes
// carry the lse values).  Partials merge in work order (prefix chunks, then local items), so
// each row's arithmetic does not depend on RPW / NB.
template <int RPW, int NB>
__device__ __forceinline__ void merge_slot(const MergeParams &p, int s, int r, int w, const int4 md,
                                           const int4 ml, int target, int warp, int wps, int lane,
                                           int qheads) {
  static_assert(NB * RPW <= 32 && kGroup % RPW == 0, "lse lanes");
  constexpr int kUnitsPerHead = kGroup / RPW;
  const int h = p.h_local, nc = md.z, nq = nc + ml.y;
  for (int u = warp; u < h * kUnitsPerHead; u += wps) {
    const int g = u / kUnitsPerHead, a0 = (u - g * kUnitsPerHead) * RPW;
    int32_t *cnt = p.done + r * kGroup + g;
    if (ld_acquire(cnt) < target) {  // bounded spin: a lost publication traps, never hangs
      const long long t0 = clock64();
      while (ld_acquire(cnt) < target) {
        __nanosleep(128);
        if (clock64() - t0 > (1ll << 35)) __trap();
      }
    }
    float M[RPW], Z[RPW];
    float4 acc[RPW];
#pragma unroll
    for (int a = 0; a < RPW; ++a) {
      M[a] = -INFINITY; Z[a] = 0.f; acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int q0 = 0; q0 < nq; q0 += NB) {
      float4 v[NB][RPW];
      float l2 = -INFINITY;  // lane u * RPW + a: lse of row a0 + a of partial q0 + u (log2 units)
#pragma unroll
      for (int u2 = 0; u2 < NB; ++u2) {
        const int q = q0 + u2;  // prefix chunk q (stride w), then the slot's own local items
        const bool ok = q < nq;
        const size_t cs = q < nc ? (size_t)md.y + (size_t)q * w : (size_t)ml.x + (q - nc);
        const size_t prow = (cs * h + g) * kGroup + a0;
        if (ok && lane / RPW == u2) l2 = __ldcg(p.part_lse + prow + lane % RPW) * 1.4426950408889634f;
#pragma unroll
        for (int a = 0; a < RPW; ++a)
          v[u2][a] = ok ? __ldcg(reinterpret_cast<const float4 *>(p.part_o + (prow + a) * kHeadDim) + lane)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u2 = 0; u2 < NB; ++u2) {
#pragma unroll
        for (int a = 0; a < RPW; ++a) {
          const float lq = __shfl_sync(0xffffffffu, l2, u2 * RPW + a);
          if (lq == -INFINITY) continue;
          const float Mn = fmaxf(M[a], lq);
          const float sc = ex2(M[a] - Mn), wgt = ex2(lq - Mn);  // ex2(-inf) = 0
          acc[a].x = acc[a].x * sc + wgt * v[u2][a].x; acc[a].y = acc[a].y * sc + wgt * v[u2][a].y;
          acc[a].z = acc[a].z * sc + wgt * v[u2][a].z; acc[a].w = acc[a].w * sc + wgt * v[u2][a].w;
          Z[a] = Z[a] * sc + wgt;
          M[a] = Mn;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < RPW; ++a) {
      const float inv = Z[a] > 0.f ? 1.f / Z[a] : 0.f;  // empty context: zeros, lse -inf
      __align__(8) __nv_bfloat162 o2[2];
      o2[0] = __floats2bfloat162_rn(acc[a].x * inv, acc[a].y * inv);
      o2[1] = __floats2bfloat162_rn(acc[a].z * inv, acc[a].w * inv);
      const int qh = g * kGroup + a0 + a;
      if (p.world == 0) {
        *reinterpret_cast<uint2 *>(p.out + ((size_t)s * qheads + qh) * kHeadDim + 4 * lane) =
            *reinterpret_cast<uint2 *>(o2);
      } else {  // fused gather: the row goes to every rank's buffer (NVLink peer stores)
        const size_t off = ((size_t)s * (kGroup * kGroup) + p.head0 + qh) * kHeadDim + 4 * lane;
        for (int j = 0; j < p.world; ++j)
          *reinterpret_cast<uint2 *>(p.gout[j] + off) = *reinterpret_cast<uint2 *>(o2);
      }
      if (p.lse_out && lane == a)
        p.lse_out[(size_t)s * qheads + qh] = (M[a] + __log2f(Z[a])) * 0.69314718055994531f;
    }
    // the last of the request's w * kUnitsPerHead readers re-arms the counters for the next call
    __syncwarp();
    if (lane == 0 && atomicAdd(cnt + p.R * kGroup, 1) == w * kUnitsPerHead - 1) {
      *cnt = 0;
      cnt[p.R * kGroup] = 0;
    }
  }
}

// One instantiation per rows-per-unit (RPW = the largest power of two <= h_local), chosen by
// the host: each gets its own register allocation (one kernel holding all four spilled).
#ifndef TAPER_MERGE_MIN_RPW
#define TAPER_MERGE_MIN_RPW 1  // 2: two slots per merge CTA at h = 1 (A/B: C2, C3 slower, C5 faster)
#endif
constexpr int kMergeMinRpw = TAPER_MERGE_MIN_RPW;
#ifndef TAPER_MERGE_ONE_WAITER
#define TAPER_MERGE_ONE_WAITER 0  // 1 (A/B): C5 h = 1 216.7 -> 212.3 us, C2 h = 1 37.0 -> 37.9: off
#endif
constexpr bool kMergeOneWaiter = TAPER_MERGE_ONE_WAITER;
template <int RPW, int NB>
__global__ void __launch_bounds__(kMergeThreads, 2) merge_kernel(MergeParams p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool tr = kTrace && p.trace != nullptr && threadIdx.x == 0 && 3200 + int(blockIdx.x) < p.trace_cap;
  if (tr) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3200 + blockIdx.x) * 16 + 0] = (long long)g;
  }
  pdl_launch_dependents();
  const int h = p.h_local;
  // the work list is visible: attend_kernel triggers this launch only after its own grid
  // dependency (the admission) resolved.  A work list written for another workspace or
  // h_local computes nothing (attend_kernel claims no items either).
  const bool match = __ldcg(p.hdr + 4) == h && __ldcg(p.hdr + 3) == p.cap_cs;
  if (!match && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.status, TAPER_STATUS_WORK_MISMATCH);
  const int n_adm = match ? __ldcg(p.hdr + 2) : 0;
  const int qheads = kGroup * h;
  // spc slots per CTA (RPW > h: a slot has fewer units than the CTA has warps), wps warps each
  const int spc = RPW > h ? RPW / h : 1, wps = (kMergeThreads / 32) / spc;
  for (int k = blockIdx.x * spc + warp / wps; k < n_adm; k += gridDim.x * spc) {
    // {slot, first shared partial, prefix chunks, width}, {first local partial, local items,
    // request, items of the request per KV head}
    const int4 md = __ldcg(p.merge_desc + 2 * k);
    const int4 ml = __ldcg(p.merge_desc + 2 * k + 1);
    const int s = md.x, nc = md.z, w = md.w, r = ml.z;
    const int target = ml.w;
    (void)nc;
    // one warp per (KV head, RPW GQA rows), RPW = the largest power of two <= h: the 8 warps
    // cover all units of a slot at once whatever h is, so the merge after the request's last
    // item costs about one load latency (a warp per KV head left 7 of 8 warps idle at h = 1:
    // same-box C2 h = 1 41.7 -> 36.9 us per call, C3 h = 1 106 -> 97)
    merge_slot<RPW, NB>(p, s, r, w, md, ml, target, warp % wps, wps, lane, qheads);
  }
  if (p.world > 0) {
    // every row of this CTA is stored (system-scope fence by each thread), then the last CTA
    // to finish raises this rank's flag in every rank's flag array (release, system scope)
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(p.gcount, 1) == int(gridDim.x) - 1) {
      __threadfence_system();
      for (int j = 0; j < p.world; ++j) st_release_sys(p.gflags[j] + p.rank, 1);
      *p.gcount = 0;  // re-armed before this kernel completes (the next merge waits for it)
    }
  }
  // The merge grid must complete only after attend_kernel (its counter re-arm) has.  One
  // CTA waiting would be enough and would let the others leave early, freeing SMs for the
  // next call's attend CTAs -- which then also take SMs the merge CTAs not yet running
  // need (TAPER_MERGE_ONE_WAITER, mixed: off)
  if (!kMergeOneWaiter || blockIdx.x == gridDim.x - 1) pdl_wait();
  if (tr) {
    __syncwarp();
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3200 + blockIdx.x) * 16 + 1] = (long long)g;
  }
}

// taper_gather_wait: one thread per rank polls this rank's flag of that rank (acquire,
// system scope), then the flags are cleared for the array's next use.
__global__ void __launch_bounds__(32, 1) gather_wait_kernel(int32_t *flags, int world) {
  const int j = threadIdx.x;
  if (j < world && ld_acquire_sys(flags + j) == 0) {
    const long long t0 = clock64();
    while (ld_acquire_sys(flags + j) == 0) {
      __nanosleep(128);
      if (clock64() - t0 > (1ll << 35)) __trap();  // a lost flag traps, never hangs
    }
  }
  __syncwarp();
  if (j < world) flags[j] = 0;
}

}  // namespace taper

// ---------------------------------------------------------------------- host side
using namespace taper;

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

static int make_kv_map(CUtensorMap *map, const void *pool, const taper_kv *kv, bool box16 = false) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(TAPER_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t row = 128 * 2;
  const cuuint64_t ps = (cuuint64_t)kv->page_size, hl = (cuuint64_t)kv->h_local;
  CUresult r;
  if (kv->page_size >= kTile) {
    // (d-lo 64, token, d-half 2, head, page): one {64, 64, 2} box = a full K or V tile in
    // the [d-half][token][64] layout of two SW128 K-major atoms
    cuuint64_t dims[5] = {64, ps, 2, hl, (cuuint64_t)kv->num_pages};
    cuuint64_t strides[4] = {row, 128, row * ps, row * ps * hl};
    // box16: {64 d, 16 tokens, one d-half} for the partial last tile of a segment
    cuuint32_t box[5] = {64, box16 ? 16u : (cuuint32_t)kTile, box16 ? 1u : 2u, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(pool), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[4] = {128, ps, hl, (cuuint64_t)kv->num_pages};
    cuuint64_t strides[3] = {row, row * ps, row * ps * hl};
    cuuint32_t box[4] = {64, (cuuint32_t)kv->page_size, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(pool), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return fail(TAPER_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return TAPER_OK;
}

// q [S][8 h][128] bf16 viewed as (d-lo 64, GQA row 8, d-half 2, slot * h + g): one
// {64, 8, 2, 1} box = the 8 rows of one (slot, KV head) as [d-half][8][128 B] with SW128,
// the K-major B-operand layout of Q^T.
static int make_q_map(CUtensorMap *map, const void *q, int S, int h) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(TAPER_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {64, (cuuint64_t)kGroup, 2, (cuuint64_t)S * (cuuint64_t)h};
  cuuint64_t strides[3] = {256, 128, 256 * kGroup};
  cuuint32_t box[4] = {64, (cuuint32_t)kGroup, 2, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(q), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TAPER_ERR_CUDA, "cuTensorMapEncodeTiled (q) failed");
  return TAPER_OK;
}

static thread_local cudaEvent_t g_prof_ev[3] = {nullptr, nullptr, nullptr};
static thread_local long long *g_trace = nullptr;
static thread_local int g_trace_cap = 0;

extern "C" int taper_set_trace_buffer(void *device_buffer, int capacity_tiles) {
  g_trace = static_cast<long long *>(device_buffer);
  g_trace_cap = device_buffer ? capacity_tiles : 0;
  return TAPER_OK;
}

extern "C" int taper_set_profile_events(void *const *events, int n_events) {
  if (events && n_events != 3) return fail(TAPER_ERR_ARG, "need 3 events");
  for (int i = 0; i < 3; ++i) g_prof_ev[i] = events ? static_cast<cudaEvent_t>(events[i]) : nullptr;
  return TAPER_OK;
}

static int device_sms() {
  static thread_local int dev = -1, sms = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    dev = d;
  }
  return sms;
}

static int decode_attention(const taper_batch *batch, const taper_admission *adm,
                            const taper_kv *kv, const void *q, void *out, const taper_gather *gather,
                            float *lse, float scale, void *workspace, size_t workspace_bytes,
                            void *stream) {
  if (gather) {
    const int G = gather->world;
    if (!(G == 1 || G == 2 || G == 4 || G == 8) || gather->rank < 0 || gather->rank >= G)
      return fail(TAPER_ERR_ARG, "gather: world must be 1, 2, 4 or 8 and 0 <= rank < world");
    if (!kv || kv->h_local * G != 8) return fail(TAPER_ERR_ARG, "gather: kv->h_local must be 8 / world");
    for (int j = 0; j < G; ++j) {
      if (!gather->out[j] || !gather->flags[j]) return fail(TAPER_ERR_ARG, "gather: null out / flags");
      if (reinterpret_cast<uintptr_t>(gather->out[j]) & 15)
        return fail(TAPER_ERR_ARG, "gather: out buffers must be 16-byte aligned");
    }
    out = gather->out[gather->rank];
  }
  if (!batch || !adm || !kv || !q || !out || !workspace)
    return fail(TAPER_ERR_ARG, "null argument");
  const int R = batch->n_req, S = batch->n_slot;
  if (R < 0 || S < 0) return fail(TAPER_ERR_ARG, "negative n_req/n_slot");
  if (R > kMaxSlots || S > kMaxSlots) return fail(TAPER_ERR_CAPACITY, "R or S exceeds TAPER_MAX_SLOTS");
  if (kv->h_local < 1 || kv->h_local > 8) return fail(TAPER_ERR_ARG, "h_local must be in [1, 8]");
  if (!(kv->page_size == 16 || kv->page_size == 32 || kv->page_size == 64 || kv->page_size == 128))
    return fail(TAPER_ERR_CAPACITY, "page_size must be 16, 32, 64 or 128");
  if (!kv->k_pages || !kv->v_pages || !kv->req_page_off || !kv->req_pages ||
      !kv->slot_page_off || !kv->slot_pages || kv->num_pages < 1)
    return fail(TAPER_ERR_ARG, "null kv array or empty pool");
  if ((reinterpret_cast<uintptr_t>(kv->k_pages) | reinterpret_cast<uintptr_t>(kv->v_pages) |
       reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(TAPER_ERR_ARG, "K/V pools, q and out must be 16-byte aligned");
  if (!adm->adm_list || !adm->slot_admitted) return fail(TAPER_ERR_ARG, "null admission arrays");
  if ((batch->slot_seg_off != nullptr) != (kv->seg_page_off != nullptr))
    return fail(TAPER_ERR_ARG, "batch.slot_seg_off and kv.seg_page_off must be given together");
  WsLayout L = ws_layout(R, S);
  if (workspace_bytes < L.fixed + 512) return fail(TAPER_ERR_CAPACITY, "workspace too small");
  if (S == 0) { set_launches(0); return TAPER_OK; }
  const int h = kv->h_local;
  char *w = static_cast<char *>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  CUtensorMap tmK, tmV, tmK16, tmV16, tmQ;
  int rc = make_kv_map(&tmK, kv->k_pages, kv);
  if (rc == TAPER_OK) rc = make_kv_map(&tmV, kv->v_pages, kv);
  if (rc == TAPER_OK) rc = make_kv_map(&tmK16, kv->k_pages, kv, kv->page_size >= kTile);
  if (rc == TAPER_OK) rc = make_kv_map(&tmV16, kv->v_pages, kv, kv->page_size >= kTile);
  if (rc == TAPER_OK) rc = make_q_map(&tmQ, q, S, kv->h_local);
  if (rc != TAPER_OK) return rc;

  {  // the SMEM opt-in is a per-device function attribute
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kSmemBytes);
      if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(attend_kernel)");
      attr_set.fetch_or(bit);
    }
  }
  WsTables tabs = ws_tables(workspace_bytes, R, S, h);
  if (!adm->status) return fail(TAPER_ERR_ARG, "null admission status");
  AttnParams ap;
  ap.slot_page_off = batch->slot_seg_off ? kv->seg_page_off : kv->slot_page_off;
  ap.slot_pages = kv->slot_pages;
  ap.req_page_off = kv->req_page_off;
  ap.req_pages = kv->req_pages;
  ap.hdr = reinterpret_cast<int32_t *>(w + L.hdr);
  ap.done = reinterpret_cast<int32_t *>(w + L.done);
  ap.adm_by_req = reinterpret_cast<const int32_t *>(w + L.adm_by_req);
  ap.ltiles = reinterpret_cast<const int4 *>(w + tabs.ltiles);
  ap.sorted = reinterpret_cast<const ItemDesc *>(w + tabs.sorted);
  ap.part_lse = reinterpret_cast<float *>(w + tabs.lse);
  ap.part_o = reinterpret_cast<float *>(w + tabs.o);
  ap.h_local = h;
  ap.page_size = kv->page_size;
  ap.tma5d = kv->page_size >= kTile ? 1 : 0;
  ap.cap_cs = int(tabs.cap_cs > 0x7fffffff ? 0x7fffffff : tabs.cap_cs);  // as admit stores it
  ap.scale_log2 = scale * 1.4426950408889634f;
  ap.trace = g_trace;
  ap.trace_cap = g_trace_cap;
  const int sms = device_sms();
  if (g_prof_ev[0]) cudaEventRecord(g_prof_ev[0], st);
  // both kernels launch with programmatic stream serialization (PDL): each may start while
  // its predecessor drains and synchronises in-kernel (griddepcontrol / completion counters)
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cfg.attrs = pdl;
  cfg.numAttrs = TAPER_PDL ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, attend_kernel, tmK, tmV, tmK16, tmV16, tmQ, ap);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "attend_kernel launch");
  if (g_prof_ev[1]) cudaEventRecord(g_prof_ev[1], st);

  MergeParams mp;
  mp.trace = g_trace;
  mp.trace_cap = g_trace_cap;
  mp.hdr = ap.hdr;
  mp.done = ap.done;
  mp.R = R;
  mp.merge_desc = reinterpret_cast<const int4 *>(w + L.merge_desc);
  mp.part_lse = ap.part_lse;
  mp.part_o = ap.part_o;
  mp.out = static_cast<__nv_bfloat16 *>(out);
  mp.lse_out = lse;
  mp.h_local = h;
  mp.cap_cs = ap.cap_cs;
  mp.status = adm->status;
  mp.world = gather ? gather->world : 0;
  mp.rank = gather ? gather->rank : 0;
  mp.head0 = gather ? kGroup * h * gather->rank : 0;
  for (int j = 0; j < TAPER_MAX_RANKS; ++j) {
    mp.gout[j] = gather && j < gather->world ? static_cast<__nv_bfloat16 *>(gather->out[j]) : nullptr;
    mp.gflags[j] = gather && j < gather->world ? gather->flags[j] : nullptr;
  }
  mp.gcount = ap.hdr + 11;
  int grid = S > 0 ? S : 1;  // CTAs beyond the admitted count exit at once
  if (TAPER_MERGE_GRID > 0 && grid > TAPER_MERGE_GRID) grid = TAPER_MERGE_GRID;  // (A/B knob)
  cfg.gridDim = dim3(grid);
  cfg.numAttrs = TAPER_MERGE_PDL ? 1 : 0;
  cfg.blockDim = dim3(kMergeThreads);
  cfg.dynamicSmemBytes = 0;
  // rows per merge unit: the largest power of two <= h, at least kMergeMinRpw (2 at h = 1:
  // one CTA takes two slots -- half the merge CTAs holding SMs the next call's attend CTAs
  // need; same-box C5 h = 1 216.3 -> 213.3 us but C2 36.9 -> 38.3, C3 97.4 -> 101.0: off)
  const int rpw = h >= 8 ? 8 : h >= 4 ? 4 : (h >= 2 || kMergeMinRpw >= 2) ? 2 : 1;
  if (rpw > h) cfg.gridDim = dim3((grid + rpw / h - 1) / (rpw / h));
  e = rpw == 8   ? cudaLaunchKernelEx(&cfg, merge_kernel<8, 2>, mp)
      : rpw == 4 ? cudaLaunchKernelEx(&cfg, merge_kernel<4, 4>, mp)
      : rpw == 2 ? cudaLaunchKernelEx(&cfg, merge_kernel<2, 8>, mp)
                 : cudaLaunchKernelEx(&cfg, merge_kernel<1, 8>, mp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "merge_kernel launch");
  if (g_prof_ev[2]) cudaEventRecord(g_prof_ev[2], st);
  set_launches(2);
  return TAPER_OK;
}

extern "C" int taper_decode_attention(const taper_batch *batch, const taper_admission *adm,
                                      const taper_kv *kv, const void *q, void *out, float *lse,
                                      float scale, void *workspace, size_t workspace_bytes,
                                      void *stream) {
  return decode_attention(batch, adm, kv, q, out, nullptr, lse, scale, workspace, workspace_bytes,
                          stream);
}

extern "C" int taper_decode_attention_gather(const taper_batch *batch, const taper_admission *adm,
                                             const taper_kv *kv, const void *q,
                                             const taper_gather *gather, float *lse, float scale,
                                             void *workspace, size_t workspace_bytes, void *stream) {
  if (!gather) return fail(TAPER_ERR_ARG, "null gather");
  return decode_attention(batch, adm, kv, q, nullptr, gather, lse, scale, workspace, workspace_bytes,
                          stream);
}

extern "C" int taper_gather_wait(const taper_gather *gather, void *stream) {
  if (!gather || gather->world < 1 || gather->world > TAPER_MAX_RANKS || gather->rank < 0 ||
      gather->rank >= gather->world || !gather->flags[gather->rank])
    return fail(TAPER_ERR_ARG, "bad gather struct");
  gather_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(gather->flags[gather->rank],
                                                                       gather->world);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "gather_wait_kernel launch");
  set_launches(1);
  return TAPER_OK;
}
