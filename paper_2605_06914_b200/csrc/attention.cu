// attention.cu -- cascade decode attention for one continuous-batching step.
//
// Sec. 3.1: branch i of a parallel phase attends to
//     P (+) H (+) h_i (+) y_{i,<t}
// and "a backend with paged or radix-tree KV caches can serve all branches from a single
// set of prefix blocks".  Two kernels:
//
//  A6+A7  attend_kernel (tcgen05 + TMA, one persistent CTA per SM)
//     Work items of one request r and local KV head g, all sharing the same stacked query
//     operand Q_stack = [8 GQA heads] x [w_r admitted branches] (rows = 8 w_r <= 128):
//       * shared item : one 1024-token chunk of P (+) H -- every page read ONCE from HBM
//                       and contracted against all stacked rows (the cascade);
//       * local item  : up to 16 64-token tiles of the branches' own segments h_i (+) y_i,
//                       each tile masked to the 8 rows of the branch that owns it.
//     Per 64-token tile:  S = Q_stack K^T (tcgen05.mma, A = Q in TMEM, B = K via TMA in
//     SMEM, fp32 S in TMEM) -> online softmax (one TMEM lane per row) -> P = hi + lo bf16
//     written back into the S columns of TMEM -> O += P V (tcgen05.mma, A = P in TMEM,
//     B = V straight from the TMA tile as an MN-major operand).  When <= 32 (<= 64) rows
//     are live, Q_stack is replicated into 4 (2) TMEM lane quadrants and each copy owns a
//     16 (32)-token slice of every tile (split-K inside the CTA, PV lanes masked per copy),
//     so the softmax work is spread over all four SM sub-partitions; the copies are merged
//     in the epilogue.  Output: a normalised partial (o, lse) per stacked row and item.
//  A8     merge_kernel: per admitted slot and KV head, log-sum-exp merge of its partials
//     (prefix chunks in order, then local items) into bf16 out[s, 8g:8g+8, :].
//
// Item boundaries depend only on segment lengths, and a stacked row's arithmetic does not
// depend on which other rows share the operand, so a slot's output does not depend on
// which siblings are co-admitted (Lemma 1; tests/test_gpu_attention.py).
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>

#include "host_common.h"
#include "taper_internal.cuh"

namespace taper {

constexpr int kTile = kTileTokens;   // 64 tokens per pipeline stage
// K and V tiles ride separate TMA rings: a K stage is released as soon as QK(t) completes,
// a V stage only after PV(t); each stage is 64 tokens x 128 d bf16 = two 8 KB boxes.
constexpr int kKStages = 6;
constexpr int kVStages = 6;
constexpr int kStageBytes = 2 * 8192;
constexpr int kOffV = kKStages * kStageBytes;                 // 64 KB
constexpr int kOffQS = kOffV + kVStages * kStageBytes;        // 160 KB: next item's queries
constexpr int kQSRows = 64;                                   // staged rows per pass
constexpr int kQSStride = 256 + 16;  // padded row stride: conflict-free 16 B row reads
constexpr int kQSBytes = kQSRows * kQSStride;                 // 64 rows x 128 bf16
constexpr int kXCols = 16;                                    // epilogue pass width
constexpr int kXStride = kXCols + 4;                          // floats per staged row (+pad)
constexpr int kOffX = kOffQS + kQSBytes;                      // epilogue staging 128 rows
constexpr int kXBytes = 128 * kXStride * 4;
constexpr int kOffML = kOffX + kXBytes;           // (m, l) of the 128 M-rows, 2 buffers
constexpr int kItemRing = 8;                      // claimed-item ring (ItemRec, 512 B each)
constexpr int kOffRec = kOffML + 2 * 128 * 8;
constexpr int kOffBar = kOffRec + kItemRing * 512;
constexpr int kSmemUsed = kOffBar + 512;
constexpr int kSmemBytes = kSmemUsed + 1024;      // + alignment slack
// warp 0: K producer; warp 1: MMA issuer; warps 2-5: softmax; warps 6-9: epilogue;
// warp 10: V producer; warp 11: item scheduler (claims, resolves tiles, stages queries)
constexpr int kAttnThreads = 384;
constexpr int kRingConsumers = 11;  // warps 0-10 release every item record
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0;     // S0 / P0 [0, 64), S1 / P1 [64, 128)
constexpr uint32_t kColO = 128;   // O0 [128, 256), O1 [256, 384)
constexpr uint32_t kColQ = 384;   // Q0 [384, 448), Q1 [448, 512): 128 bf16 per row, 64 packed cols

constexpr uint32_t kIdescQK = umma_idesc_bf16(128, 64, false, false);
constexpr uint32_t kIdescPV = umma_idesc_bf16(128, 128, false, true);
constexpr uint32_t kIdescQK64 = umma_idesc_bf16(64, 64, false, false);
constexpr uint32_t kIdescPV64 = umma_idesc_bf16(64, 128, false, true);

struct AttnParams {
  const int32_t *slot_page_off, *slot_pages, *req_page_off, *req_pages;
  int32_t *hdr;        // hdr[8]: work counter, hdr[9]: CTAs exited
  const int32_t *adm_by_req;
  int32_t *done;       // [r * 8 + g]: items of (request, KV head) whose partials are written
  const ItemDesc *items;
  const int4 *ltiles;
  const __nv_bfloat16 *q;
  float *part_lse, *part_o;
  int h_local, page_size;
  int tma5d;  // 1: page_size >= 64, one 5-D box per tile; 0: two 4-D boxes per page
  float scale_log2;
  long long *trace;  // debug: pipeline event timestamps of CTA 0 (taper_set_trace_buffer)
  int trace_cap;
};

// Debug trace: event e of tile/item index n -> trace[(n * 16 + e)] = clock64 (CTA 0 only).
__device__ __forceinline__ void trace_ev(const AttnParams &p, int e, uint32_t n) {
  if (p.trace != nullptr && blockIdx.x == 0 && int(n) < p.trace_cap)
    p.trace[(size_t)n * 16 + e] = clock64();
}

struct Item {
  int r, g, local, w, adm_off, cs0, nt, tb, te, rep, m64;
};

// TMEM row layout of the MMA accumulator (cta_group::1): M = 128 puts row m in lane m; M = 64
// puts rows 16q..16q+15 in lanes 32q..32q+15 (16 rows per lane quadrant).  Returns the M-row
// held by (quadrant wq, lane) or -1.
__device__ __forceinline__ int mrow_of(int m64, int wq, int lane) {
  if (!m64) return wq * 32 + lane;
  return lane < 16 ? wq * 16 + lane : -1;
}

// A claimed work item as the scheduler warp resolves it into SMEM: the descriptor plus, per
// 64-token tile, its first token, valid tokens, owning branch (-1: all rows) and the page of
// each 16-token box.  Every other role reads only this record (no global loads per item).
struct ItemRec {
  int32_t it, g, desc[8];  // desc = ItemDesc {r, w, adm_off, cs0, tb, te, nt, flags}
  int32_t pad[6];
  int32_t tok0[kLocalItemTiles], valid[kLocalItemTiles], jrow[kLocalItemTiles];
  int32_t pg[kLocalItemTiles][4];
};
static_assert(sizeof(ItemRec) == 512, "ItemRec size");

__device__ __forceinline__ void decode_item(const ItemRec *rec, Item &x) {
  x.g = rec->g;
  x.r = rec->desc[0]; x.w = rec->desc[1]; x.adm_off = rec->desc[2]; x.cs0 = rec->desc[3];
  x.tb = rec->desc[4]; x.te = rec->desc[5]; x.nt = rec->desc[6];
  const int f = rec->desc[7];
  x.local = f & 1;
  x.rep = (f >> 1) & 7;
  x.m64 = (f >> 4) & 1;
}

struct TileInfo {
  const int32_t *pages;
  int tok0, valid, jrow;  // jrow = owning branch (local tiles) or -1 (all rows)
};

__device__ __forceinline__ TileInfo tile_info(const AttnParams &p, const Item &x, int t) {
  TileInfo ti;
  if (!x.local) {
    ti.pages = p.req_pages + __ldg(p.req_page_off + x.r);
    ti.tok0 = x.tb + t * kTile;
    ti.valid = min(kTile, x.te - ti.tok0);
    ti.jrow = -1;
  } else {
    const int4 lt = __ldg(p.ltiles + x.tb + t);  // {slot, tok0, valid, branch}
    ti.pages = p.slot_pages + __ldg(p.slot_page_off + lt.x);
    ti.tok0 = lt.y;
    ti.valid = lt.z;
    ti.jrow = lt.w;
  }
  return ti;
}

// valid tokens and owning branch of tile t (softmax side)
__device__ __forceinline__ int2 tile_rows(const ItemRec *rec, int t) {
  return make_int2(rec->valid[t], rec->jrow[t]);
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Move the item's staged stacked queries (SMEM, [row][128] bf16, filled by the producer's
// bulk copies in passes of 64 rows) into TMEM columns [qcol, qcol + 64), replicated over
// the row copies; each pass's buffer is released after use.  Ends with the tcgen05 stores
// complete and fenced.  `pass` counts staging passes consumed so far (updated).
__device__ __forceinline__ void stage_q_tmem(const Item &x, const uint8_t *qs, uint64_t *qs_full,
                                             uint64_t *qs_free, uint32_t &pass, uint32_t tmem,
                                             uint32_t lane_off, int wq, int lane, uint32_t qcol) {
  const int R8 = 8 * x.w;
  const int m = mrow_of(x.m64, wq, lane);
  const int rpc = (x.m64 ? 64 : 128) / x.rep;
  const int i = m >= 0 ? m % rpc : 1 << 20;
  uint32_t v[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) v[c] = 0u;
  for (int r0 = 0; r0 < R8; r0 += kQSRows, ++pass) {
    mbar_wait(qs_full, pass & 1);
    if (i >= r0 && i < min(R8, r0 + kQSRows)) {
      const uint4 *src = reinterpret_cast<const uint4 *>(qs + (i - r0) * kQSStride);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const uint4 u = src[c];
        v[4 * c] = u.x; v[4 * c + 1] = u.y; v[4 * c + 2] = u.z; v[4 * c + 3] = u.w;
      }
    }
    mbar_arrive(qs_free);
  }
  tmem_st_n<64>(tmem + lane_off + qcol, v);
  tmem_st_wait();
  tc_fence_before();
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// S[tS] = Q[tQ] * K^T: 8 k-steps of 16 over d = 128 (A = Q from TMEM, B = K tile in SMEM,
// SW128 K-major: d 0..63 in the first 8 KB box, 64..127 in the second).
__device__ __forceinline__ void issue_qk(uint32_t tS, uint32_t tQ, uint32_t kb, uint32_t idesc) {
  const uint32_t nomask[4] = {0u, 0u, 0u, 0u};
  const uint64_t b0 = umma_desc_sw128(kb, 16, 1024);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint64_t b = b0 + uint64_t((((kk >> 2) * 8192) + (kk & 3) * 32) >> 4);
    tc_mma_f16_ts(tS, tQ + kk * 8, b, idesc, kk > 0 ? 1u : 0u, nomask);
  }
}

// O[tO] += P[tP] * V: P = hi (columns 0..31) + lo (32..63), 4 k-steps of 16 tokens;
// B = V tile as an MN-major SW128 operand (d 0..63 / 64..127 boxes 8 KB apart).  With REP
// replicated row copies, copy c owns tokens [c*64/REP, (c+1)*64/REP): its k-steps run
// with the other copies' TMEM lanes masked off.
template <int REP>
__device__ __forceinline__ void issue_pv(uint32_t tO, uint32_t tP, uint32_t vb, bool first,
                                         uint32_t idesc) {
  const uint64_t b0 = umma_desc_sw128(vb, 8192, 1024);
  constexpr int KPC = 4 / REP;
#pragma unroll
  for (int c = 0; c < REP; ++c) {
    uint32_t mask[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) mask[q] = (REP == 1 || q / (4 / REP) == c) ? 0u : 0xffffffffu;
    constexpr int kParts = 2;  // P = hi + lo
#pragma unroll
    for (int part = 0; part < kParts; ++part) {
#pragma unroll
      for (int k = 0; k < KPC; ++k) {
        const int kk = c * KPC + k;
        const uint64_t b = b0 + uint64_t((kk * 2048) >> 4);
        tc_mma_f16_ts(tO, tP + part * 32 + kk * 8, b, idesc,
                      (first && part == 0 && k == 0) ? 0u : 1u, mask);
      }
    }
  }
}

// One tile of the online softmax for a thread's row, branch-free.  CW = tokens of the tile
// handled by this thread; nvalid = live tokens among them (0 for a row that is dead in this
// tile).  Updates m_run and this thread's share of l_run, and writes P (hi, lo) into the
// row's S columns.  M = 128 (SPLIT = false): one thread per row (TMEM lane), tokens
// [colbase, colbase + CW).  M = 64 (SPLIT = true): rows live in lanes 0-15 of the quadrant and
// two threads share a row -- lane t < 16 takes tokens [colbase, +CW), lane t + 16 the next CW
// (16x32bx2 accesses); the row max is combined across the pair, the row sum at the end of
// the item.
template <int CW, bool SPLIT>
__device__ __forceinline__ void softmax_tile(uint32_t tS, int colbase, int nvalid, bool o_live,
                                             float c, float &m_run, float &l_run, uint32_t tO,
                                             uint64_t *pv_prev, uint32_t pv_prev_parity) {
  uint32_t s[CW];
  if constexpr (SPLIT) {
    if constexpr (CW == 8) tmem_ld_x2_8<CW>(tS + colbase, s);
    else if constexpr (CW == 16) tmem_ld_x2_16<CW>(tS + colbase, s);
    else tmem_ld_x2_32<CW>(tS + colbase, s);
  } else {
    tmem_ld_n<CW>(tS + colbase, s);
  }
  tmem_ld_wait();
  float x[CW];
#pragma unroll
  for (int j = 0; j < CW; ++j) x[j] = j < nvalid ? __uint_as_float(s[j]) : -INFINITY;
  float mx = x[0];
#pragma unroll
  for (int j = 1; j < CW; ++j) mx = fmaxf(mx, x[j]);
  if constexpr (SPLIT) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  mx *= c;  // scores in log2 units (c = softmax scale * log2 e > 0)
  // lazy rescale: only raise the running max when it grows by more than 8 (log2 units)
  const bool need = mx > m_run + 8.f;
  float alpha = 1.f;
  if (need) {
    alpha = ex2(m_run - mx);  // 0 when m_run = -inf
    l_run *= alpha;
    m_run = mx;
  }
  if (o_live && __any_sync(0xffffffffu, need)) {
    mbar_wait(pv_prev, pv_prev_parity);  // O *= alpha needs PV(n-1) complete
    tc_fence_after();
#pragma unroll 1
    for (int q = 0; q < (SPLIT ? 2 : 4); ++q) {
      uint32_t o[32];
      if constexpr (SPLIT) tmem_ld_x2_32<64>(tO + q * 32, o);
      else tmem_ld32(tO + q * 32, o);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
      if constexpr (SPLIT) tmem_st_x2_32<64>(tO + q * 32, o);
      else tmem_st32(tO + q * 32, o);
    }
    tmem_st_wait();
  }
  // P = 2^(x - m) split into hi + lo bf16 (DESIGN.md Sec. 6 "P precision"), written back
  // into this row's S columns in groups of up to 16 tokens (8 packed columns per part)
  constexpr int G = CW < 16 ? CW : 16;
  const float neg_m = m_run == -INFINITY ? 0.f : -m_run;
  float lsum = 0.f;
#pragma unroll
  for (int g = 0; g < CW / G; ++g) {
    uint32_t hi[G / 2], lo[G / 2];
#pragma unroll
    for (int jj = 0; jj < G / 2; ++jj) {
      const int j = g * (G / 2) + jj;
      const float e0 = ex2(fmaf(x[2 * j], c, neg_m));
      const float e1 = ex2(fmaf(x[2 * j + 1], c, neg_m));
      lsum += e0 + e1;
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
      const float2 f2 = __bfloat1622float2(h2);
      const __nv_bfloat162 l2 = __floats2bfloat162_rn(e0 - f2.x, e1 - f2.y);
      hi[jj] = *reinterpret_cast<const uint32_t *>(&h2);
      lo[jj] = *reinterpret_cast<const uint32_t *>(&l2);
    }
    const uint32_t col = colbase / 2 + g * (G / 2);
    if constexpr (SPLIT) {
      if constexpr (G == 8) {
        tmem_st_x2_4<CW / 2>(tS + col, hi);
        tmem_st_x2_4<CW / 2>(tS + 32 + col, lo);
      } else {
        tmem_st_x2_8<CW / 2>(tS + col, hi);
        tmem_st_x2_8<CW / 2>(tS + 32 + col, lo);
      }
    } else {
      tmem_st8(tS + col, hi);
      tmem_st8(tS + 32 + col, lo);
    }
  }
  l_run += lsum;
  tmem_st_wait();
}

// Consumer side of the claimed-item ring: the k-th item this CTA processes (-1 = done).
__device__ __forceinline__ int ring_item(uint64_t *it_full, const ItemRec *recs, uint32_t k) {
  const uint32_t slot = k % kItemRing;
  mbar_wait(it_full + slot, (k / kItemRing) & 1);
  return *reinterpret_cast<const volatile int32_t *>(&recs[slot].it);
}
__device__ __forceinline__ void ring_release(uint64_t *it_empty, uint32_t k, int lane) {
  __syncwarp();
  if (lane == 0) mbar_arrive(it_empty + (k % kItemRing));
}

__global__ void __launch_bounds__(kAttnThreads, 1)
    attend_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  AttnParams p) {
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
  uint64_t *p_full = s_full + 2;           // [2] softmax -> PV
  uint64_t *pv_done = p_full + 2;          // [2] PV done -> softmax (O rescale)
  uint64_t *q_full = pv_done + 2;          // softmax (Q staged) -> MMA
  uint64_t *o_full = q_full + 1;           // [2] last PV of an item -> epilogue
  uint64_t *o_free = o_full + 2;           // [2] epilogue done -> MMA / softmax
  uint64_t *ml_full = o_free + 2;          // [2] softmax (m, l) published -> epilogue
  uint64_t *qs_full = ml_full + 2;         // producer's Q staging copy landed
  uint64_t *qs_free = qs_full + 1;         // softmax moved the staged Q into TMEM
  uint64_t *it_full = qs_free + 1;         // [kItemRing] scheduler published an item record
  uint64_t *it_empty = it_full + kItemRing;  // [kItemRing] all consumer warps are done with it
  uint64_t *sched_go = it_empty + kItemRing;  // K producer started an item -> scheduler
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sched_go + 1);
  ItemRec *recs = reinterpret_cast<ItemRec *>(smem + kOffRec);
  float *xo = reinterpret_cast<float *>(smem + kOffX);
  float2 *xml = reinterpret_cast<float2 *>(smem + kOffML);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = p.h_local;
  const int n_items = (__ldg(p.hdr) + __ldg(p.hdr + 5)) * h;
  if (p.trace != nullptr && tid == 0) {  // per-CTA wall-clock span (debug trace)
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3000 + blockIdx.x) * 16 + 0] = (long long)g;
  }

  // Zero the K/V rings once: rows of a partial tile that TMA does not load must hold finite
  // values (P = 0 there, but 0 * NaN would still poison O).
  for (int i = tid; i < kOffQS / 16; i += kAttnThreads)
    reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int i = 0; i < kKStages; ++i) { mbar_init(kfull + i, 1); mbar_init(kempty + i, 1); }
    for (int i = 0; i < kVStages; ++i) { mbar_init(vfull + i, 1); mbar_init(vempty + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
      mbar_init(pv_done + i, 1);
      mbar_init(o_full + i, 1);
      mbar_init(o_free + i, 128);
      mbar_init(ml_full + i, 128);
    }
    mbar_init(q_full, 128);
    mbar_init(qs_full, 1);
    mbar_init(qs_free, 128);
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(it_full + i, 1);
      mbar_init(it_empty + i, kRingConsumers);
    }
    mbar_init(sched_go, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmK); tma_prefetch_desc(&tmV); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the prologue above overlapped the previous kernel; the merge kernel may launch now
  // (it waits for per-request completion counters); wait for the previous kernel's memory.
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 11) {
    // ======================= item scheduler ==================================================
    // Claims work items (global atomic counter -> dynamic scheduling) one item ahead of the
    // K producer, resolves each into an SMEM ItemRec (descriptor, tile geometry, page
    // indices: lane l resolves tile l), publishes it, then stages the item's stacked queries
    // (w slots x 8 heads x 256 B, 2 KB per slot) into SMEM by bulk copies in passes of 8
    // slots for the softmax warps.  The dependent global loads of an item thus overlap the
    // previous item instead of stalling the pipeline at every item boundary.
    const int box_tok = p.page_size < kTile ? p.page_size : kTile;
    const int n_items = (__ldg(p.hdr) + __ldg(p.hdr + 5)) * p.h_local;
    int *work_counter = p.hdr + 8;
    uint32_t qs_pass = 0;
    for (uint32_t k = 0;; ++k) {
      if (k >= 1) mbar_wait(sched_go, (k - 1) & 1);  // K producer started item k-1
      int it = 0;
      if (lane == 0) it = atomicAdd(work_counter, 1);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= n_items) it = -1;
      const uint32_t slot = k % kItemRing;
      ItemRec *rec = recs + slot;
      mbar_wait(it_empty + slot, ((k / kItemRing) & 1) ^ 1);
      int w = 0, adm_off = 0, g = 0;
      if (it >= 0) {
        const int q = it / p.h_local;
        g = it - q * p.h_local;
        const int32_t d = lane < 8 ? __ldg(reinterpret_cast<const int32_t *>(p.items + q) + lane) : 0;
        const int nt = __shfl_sync(0xffffffffu, d, 6);
        Item x;
        x.r = __shfl_sync(0xffffffffu, d, 0);
        w = __shfl_sync(0xffffffffu, d, 1);
        adm_off = __shfl_sync(0xffffffffu, d, 2);
        x.tb = __shfl_sync(0xffffffffu, d, 4);
        x.te = __shfl_sync(0xffffffffu, d, 5);
        x.local = __shfl_sync(0xffffffffu, d, 7) & 1;
        if (lane < 8) rec->desc[lane] = d;
        if (lane < nt) {
          const TileInfo ti = tile_info(p, x, lane);
          rec->tok0[lane] = ti.tok0;
          rec->valid[lane] = ti.valid;
          rec->jrow[lane] = ti.jrow;
#pragma unroll
          for (int b = 0; b < kTile / 16; ++b)
            rec->pg[lane][b] =
                b * box_tok < ti.valid ? __ldg(ti.pages + (ti.tok0 + b * box_tok) / p.page_size) : 0;
        }
      }
      if (lane == 0) { rec->it = it; rec->g = g; }
      __syncwarp();
      if (lane == 0) mbar_arrive(it_full + slot);  // release: the record is visible
      if (it < 0) break;
      const int slot_j = lane < w ? __ldg(p.adm_by_req + adm_off + lane) : 0;
      for (int j0 = 0; j0 < w; j0 += kQSRows / 8, ++qs_pass) {
        const int nj = min(kQSRows / 8, w - j0);
        mbar_wait(qs_free, (qs_pass & 1) ^ 1);
        if (elect_one()) mbar_arrive_expect_tx(qs_full, nj * 2048);
        __syncwarp();
        // one 256 B copy per stacked row (slot j, head e) into the padded staging rows
        for (int rr = lane; rr < kQSRows; rr += 32) {
          const int j = rr >> 3;
          const int s_j = __shfl_sync(0xffffffffu, slot_j, min(j0 + j, 31));
          if (j < nj)
            bulk_g2s(smem + kOffQS + rr * kQSStride,
                     p.q + ((size_t)s_j * (kGroup * p.h_local) + g * kGroup + (rr & 7)) * kHeadDim,
                     256, qs_full);
        }
        __syncwarp();
      }
    }
  } else if (warp == 0 || warp == 10) {
    // ======================= TMA producers: warp 0 = K, warp 10 = V =======================
    // Tile geometry and pages come from the item record in SMEM; the whole warp runs the
    // loop with warp-uniform operands and one elected lane issues (no waterfall loops).
    const bool is_k = warp == 0;
    const CUtensorMap *tmap = is_k ? &tmK : &tmV;
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
      if (is_k) {
        __syncwarp();
        if (lane == 0) mbar_arrive(sched_go);  // the scheduler may claim the next item
      }
      const int g_u = rec->g;
      const int nt_u = rec->desc[6];
      for (int t = 0; t < nt_u; ++t, ++n_prod) {
        const int tok0 = rec->tok0[t];
        const int valid = rec->valid[t];
        int pg[kTile / 16];
#pragma unroll
        for (int b = 0; b < kTile / 16; ++b) pg[b] = rec->pg[t][b];
        const uint32_t st = n_prod % n_stages;
        const int n_box = (valid + box_tok - 1) / box_tok;
        uint8_t *dst = ring + st * kStageBytes;
        mbar_wait(ring_empty + st, ((n_prod / n_stages) & 1) ^ 1);
        if (is_k && lane == 0) trace_ev(p, 0, n_prod);
        if (is_k && lane == 0 && p.trace != nullptr && t == 0 && n_prod == 0) {
          unsigned long long g;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
          p.trace[(size_t)(3000 + blockIdx.x) * 16 + 2] = (long long)g;  // first TMA issued
        }
        if (elect_one()) {
          if (p.tma5d) {
            // one box: {64 d, 64 tokens, 2 d-halves} -> [d-half][token][64] (two SW128 atoms)
            mbar_arrive_expect_tx(ring_full + st, 2 * kTile * 128);
            tma_load_5d(dst, tmap, ring_full + st, 0, tok0 % p.page_size, 0, g_u, pg[0]);
          } else {
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
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    uint32_t n = 0;  // global tile counter (S/P double buffer index = n & 1)
    for (uint32_t item_idx = 0;; ++item_idx) {
      const int it = ring_item(it_full, recs, item_idx);
      Item x;
      decode_item(recs + item_idx % kItemRing, x);
      ring_release(it_empty, item_idx, lane);
      if (it < 0) break;
      const int rep = __shfl_sync(0xffffffffu, x.rep, 0);
      const int m64 = __shfl_sync(0xffffffffu, x.m64, 0);
      const uint32_t idesc_qk = m64 ? kIdescQK64 : kIdescQK;
      const uint32_t idesc_pv = m64 ? kIdescPV64 : kIdescPV;
      const uint32_t ob = item_idx & 1;  // O double buffer
      const uint32_t tO = tmem_u + kColO + ob * 128;
      mbar_wait(q_full, item_idx & 1);
      if (lane == 0) trace_ev(p, 6, n);
      tc_fence_after();
      for (int t = 0; t <= x.nt; ++t) {
        if (t < x.nt) {
          const uint32_t ks = n % kKStages;
          mbar_wait(kfull + ks, (n / kKStages) & 1);
          if (lane == 0) trace_ev(p, 1, n);
          tc_fence_after();
          if (elect_one()) {
            issue_qk(tmem_u + kColS + (n & 1) * 64, tmem_u + kColQ + (item_idx & 1) * 64,
                     sK + ks * kStageBytes, idesc_qk);
            tc_commit(kempty + ks);
            tc_commit(s_full + (n & 1));
          }
          __syncwarp();
          if (lane == 0) trace_ev(p, 2, n);
        }
        if (t > 0) {
          // PV of the previous tile (its P is ready once the softmax arrives on p_full)
          const uint32_t m = n - 1;
          mbar_wait(p_full + (m & 1), (m >> 1) & 1);
          if (lane == 0) trace_ev(p, 3, m);
          const bool first = (t == 1);
          const uint32_t vs = m % kVStages;
          // O[ob] is free once the epilogue of item item_idx - 2 has read it
          if (first) mbar_wait(o_free + ob, ((item_idx >> 1) & 1) ^ 1);
          mbar_wait(vfull + vs, (m / kVStages) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t tP = tmem_u + kColS + (m & 1) * 64;
            const uint32_t vb = sV + vs * kStageBytes;
            if (rep == 4) issue_pv<4>(tO, tP, vb, first, idesc_pv);
            else if (rep == 2) issue_pv<2>(tO, tP, vb, first, idesc_pv);
            else issue_pv<1>(tO, tP, vb, first, idesc_pv);
            tc_commit(vempty + vs);
            tc_commit(pv_done + (m & 1));
            if (t == x.nt) tc_commit(o_full + ob);
          }
          __syncwarp();
          if (lane == 0) trace_ev(p, 5, m);
        }
        if (t < x.nt) ++n;
      }
    }
  } else if (warp < 6) {
    // ======================= softmax / O correction (128 threads) =======================
    const int wq = warp & 3;            // TMEM lane quadrant of this warp
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const float c_log2 = p.scale_log2;
    uint32_t qs_pass = 0;
    uint32_t n = 0;
    int it = ring_item(it_full, recs, 0);
    if (it >= 0) {
      Item x0;
      decode_item(recs, x0);
      stage_q_tmem(x0, smem + kOffQS, qs_full, qs_free, qs_pass, tmem, lane_off, wq, lane, kColQ);
      mbar_arrive(q_full);
    }
    for (uint32_t item_idx = 0; it >= 0; ++item_idx) {
      const ItemRec *rec = recs + item_idx % kItemRing;
      Item x;
      decode_item(rec, x);
      const int R8 = 8 * x.w;
      const int rep = x.rep;
      // M-row of this thread; M = 64 rows are shared by lane pairs (t, t + 16), half h
      const int m64 = x.m64;
      const int mrow = m64 ? wq * 16 + (lane & 15) : wq * 32 + lane;
      const int h = m64 ? lane >> 4 : 0;
      const int rpc = (m64 ? 64 : 128) / rep, cw = 64 / rep;
      const int copy = mrow / rpc;
      const int i = mrow - copy * rpc;  // stacked row (dead if >= R8)
      const int colbase = copy * cw;
      const int tw = m64 ? cw / 2 : cw;  // tokens handled by this thread
      const int tok0 = colbase + h * tw;
      const uint32_t ob = item_idx & 1;
      const uint32_t tO = tmem + lane_off + kColO + ob * 128;
      float m_run = -INFINITY, l_run = 0.f;
      bool staged = false;  // next item's Q staged in TMEM (or there is no next item)
      int next = -1;
      for (int t = 0; t < x.nt; ++t) {
        const uint32_t sb = n & 1;
        const int2 tr = tile_rows(rec, t);  // {valid tokens, owning branch or -1}
        const bool live = i < R8 && (tr.y < 0 || (i >> 3) == tr.y);
        const int nvalid = live ? max(0, min(tw, tr.x - tok0)) : 0;
        mbar_wait(s_full + sb, (n >> 1) & 1);
        if (warp == 2 && lane == 0) trace_ev(p, 7, n);
        tc_fence_after();
        // P[sb] aliases S[sb]: PV(n-2) finished reading it before QK(n) was issued.
        const uint32_t tS = tmem + lane_off + kColS + sb * 64;
        uint64_t *pv_prev = pv_done + ((n - 1) & 1);
        const uint32_t pv_par = ((n - 1) >> 1) & 1;
        const bool o_live = t > 0;
        if (m64) {
          if (cw == 16)
            softmax_tile<8, true>(tS, colbase, nvalid, o_live, c_log2, m_run, l_run, tO, pv_prev, pv_par);
          else if (cw == 32)
            softmax_tile<16, true>(tS, colbase, nvalid, o_live, c_log2, m_run, l_run, tO, pv_prev, pv_par);
          else
            softmax_tile<32, true>(tS, colbase, nvalid, o_live, c_log2, m_run, l_run, tO, pv_prev, pv_par);
        } else {
          if (cw == 16)
            softmax_tile<16, false>(tS, colbase, nvalid, o_live, c_log2, m_run, l_run, tO, pv_prev, pv_par);
          else if (cw == 32)
            softmax_tile<32, false>(tS, colbase, nvalid, o_live, c_log2, m_run, l_run, tO, pv_prev, pv_par);
          else
            softmax_tile<64, false>(tS, colbase, nvalid, o_live, c_log2, m_run, l_run, tO, pv_prev, pv_par);
        }
        tc_fence_before();
        if (lane == 0) trace_ev(p, warp == 2 ? 8 : 6 + warp, n);  // warps 3,4,5 -> 9,10,11
        mbar_arrive(p_full + sb);
        ++n;
        // Stage the next item's queries into the other Q buffer as soon as the item is
        // claimed and its rows have landed in SMEM (never blocks here).  Q[(k+1) & 1] was
        // last read by item k-1's QK MMAs, complete since this item's first s_full.
        if (!staged) {
          const uint32_t slot = (item_idx + 1) % kItemRing;
          int ready = lane == 0 ? mbar_try_wait(it_full + slot, ((item_idx + 1) / kItemRing) & 1) : 0;
          ready = __shfl_sync(0xffffffffu, ready, 0);
          if (ready) {
            next = ring_item(it_full, recs, item_idx + 1);
            if (next < 0) {
              staged = true;
            } else {
              int qready = lane == 0 ? mbar_try_wait(qs_full, qs_pass & 1) : 0;
              qready = __shfl_sync(0xffffffffu, qready, 0);
              if (qready) {
                Item xn;
                decode_item(recs + (item_idx + 1) % kItemRing, xn);
                stage_q_tmem(xn, smem + kOffQS, qs_full, qs_free, qs_pass, tmem, lane_off, wq,
                             lane, kColQ + ((item_idx + 1) & 1) * 64);
                mbar_arrive(q_full);
                staged = true;
              }
            }
          }
        }
      }
      if (m64) l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);  // row sum of the lane pair
      if (!staged) {  // not staged during the item: wait for it now
        next = ring_item(it_full, recs, item_idx + 1);
        if (next >= 0) {
          Item xn;
          decode_item(recs + (item_idx + 1) % kItemRing, xn);
          stage_q_tmem(xn, smem + kOffQS, qs_full, qs_free, qs_pass, tmem, lane_off, wq, lane,
                       kColQ + ((item_idx + 1) & 1) * 64);
          mbar_arrive(q_full);
        }
      }
      ring_release(it_empty, item_idx, lane);
      // publish (m, l) for the epilogue warps; xml[ob] was consumed by epilogue item_idx-2
      mbar_wait(o_free + ob, ((item_idx >> 1) & 1) ^ 1);
      if (h == 0) xml[ob * 128 + mrow] = make_float2(m_run, l_run);
      mbar_arrive(ml_full + ob);
      it = next;
    }
  } else {
    // ======================= epilogue (128 threads, warps 6-9) =======================
    // Merges the replicated copies of each stacked row and writes the normalised partial
    // (o, lse), overlapping the next item's tiles (O is double-buffered in TMEM).
    const int wq = warp & 3;
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    for (uint32_t item_idx = 0;; ++item_idx) {
      const int it = ring_item(it_full, recs, item_idx);
      Item x;
      decode_item(recs + item_idx % kItemRing, x);
      ring_release(it_empty, item_idx, lane);
      if (it < 0) break;
      const int R8 = 8 * x.w;
      const int rep = x.rep;
      const int mrow = mrow_of(x.m64, wq, lane);
      const int rpc = (x.m64 ? 64 : 128) / rep;
      const int copy = mrow >= 0 ? mrow / rpc : 0;
      const int i = mrow >= 0 ? mrow - copy * rpc : 1 << 20;
      const uint32_t ob = item_idx & 1;
      const uint32_t tO = tmem + lane_off + kColO + ob * 128;
      mbar_wait(ml_full + ob, (item_idx >> 1) & 1);
      mbar_wait(o_full + ob, (item_idx >> 1) & 1);
      if (warp == 6 && lane == 0) trace_ev(p, 10, 2048 + item_idx);
      tc_fence_after();
      const bool has = mrow >= 0 && i < R8;
      const float2 mine = has ? xml[ob * 128 + mrow] : make_float2(-INFINITY, 0.f);
      float M = -INFINITY, L = 0.f;
      if (has) {
        for (int c = 0; c < rep; ++c) M = fmaxf(M, xml[ob * 128 + c * rpc + i].x);
        for (int c = 0; c < rep; ++c) {
          const float2 ml = xml[ob * 128 + c * rpc + i];
          if (ml.y > 0.f) L += ex2(ml.x - M) * ml.y;
        }
      }
      const float f = (L > 0.f && mine.y > 0.f) ? ex2(mine.x - M) / L : 0.f;
      if (warp == 6 && lane == 0) trace_ev(p, 12, 2048 + item_idx);
      const bool out_row = has;
      const bool warp_out = __any_sync(0xffffffffu, out_row);
      const int etid = tid - 192;  // 0..127
      if (out_row && copy == 0) {
        const size_t prow = ((size_t)(x.cs0 + (i >> 3)) * h + x.g) * kGroup + (i & 7);
        p.part_lse[prow] = L > 0.f ? (M + __log2f(L)) * 0.69314718055994531f : -INFINITY;
      }
      // 16-column passes: every copy stages its scaled O row slice in SMEM, then all 128
      // threads sum the copies and write the rows with coalesced stores
      constexpr int kF4 = kXCols / 4;  // float4 per row slice
#pragma unroll 1
      for (int pass = 0; pass < kHeadDim / kXCols; ++pass) {
        if (warp_out) {
          uint32_t o[16];
          tmem_ld16(tO + pass * kXCols, o);
          tmem_ld_wait();
          if (out_row) {
            float4 *xr = reinterpret_cast<float4 *>(xo + mrow * kXStride);
#pragma unroll
            for (int j = 0; j < kF4; ++j)
              xr[j] = make_float4(__uint_as_float(o[4 * j]) * f, __uint_as_float(o[4 * j + 1]) * f,
                                  __uint_as_float(o[4 * j + 2]) * f,
                                  __uint_as_float(o[4 * j + 3]) * f);
          }
        }
        named_bar_sync(2, 128);
        for (int k = etid; k < R8 * kF4; k += 128) {
          const int row = k / kF4, c4 = k % kF4;
          float4 a = reinterpret_cast<const float4 *>(xo + row * kXStride)[c4];
          for (int cc = 1; cc < rep; ++cc) {
            const float4 b = reinterpret_cast<const float4 *>(xo + (cc * rpc + row) * kXStride)[c4];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
          }
          const size_t prow = ((size_t)(x.cs0 + (row >> 3)) * h + x.g) * kGroup + (row & 7);
          reinterpret_cast<float4 *>(p.part_o + prow * kHeadDim + pass * kXCols)[c4] = a;
        }
        named_bar_sync(2, 128);  // staging reused by the next pass / item
      }
      // publish: this item's partials of (request, KV head) are complete (release)
      __threadfence();
      named_bar_sync(2, 128);
      if (etid == 0) atomicAdd(p.done + x.r * kGroup + x.g, 1);
      if (warp == 6 && lane == 0) trace_ev(p, 14, 2048 + item_idx);
      if (warp == 8 && lane == 0) trace_ev(p, 15, 2048 + item_idx);
      tc_fence_before();
      if (warp == 6 && lane == 0) trace_ev(p, 11, 2048 + item_idx);
      mbar_arrive(o_free + ob);
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
  if (p.trace != nullptr && tid == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3000 + blockIdx.x) * 16 + 1] = (long long)g;
  }
}

// ------------------------------------------------------------------ A8: LSE merge
constexpr int kMergeThreads = 256;  // one CTA per admitted slot, one warp per KV head

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
};

// Per (admitted slot, KV head): the slot's partials are 8 contiguous GQA rows (4 KB) per
// work item, so the warp streams whole 4 KB blocks (lane: dims 4 lane .. 4 lane + 3 of all 8
// rows) and runs the 8 rows' online LSE merges side by side, partials in work order
// (prefix chunks, then local items), two items' loads in flight at a time.
// Launched with PDL while attend_kernel is still running: a warp starts as soon as the
// attend epilogues have published all items of its (request, KV head) (acquire on the
// completion counter), so the merge overlaps the attend kernel's tail.
__global__ void __launch_bounds__(kMergeThreads, 2) merge_kernel(MergeParams p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool tr = p.trace != nullptr && threadIdx.x == 0 && 3200 + int(blockIdx.x) < p.trace_cap;
  if (tr) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3200 + blockIdx.x) * 16 + 0] = (long long)g;
  }
  pdl_launch_dependents();
  const int h = p.h_local;
  const int n_adm = __ldg(p.hdr + 2);
  const int qheads = kGroup * h;
  for (int k = blockIdx.x; k < n_adm; k += gridDim.x) {
    const int4 md = __ldg(p.merge_desc + k);  // {slot, first chunk-slot, partials, width | r << 16}
    const int s = md.x, nq = md.z, w = md.w & 0xffff, r = md.w >> 16;
    for (int g = warp; g < h; g += kMergeThreads / 32) {
      const size_t row0 = ((size_t)md.y * h + g) * kGroup;
      const size_t qstride = (size_t)w * h * kGroup;  // partial rows between items
      int32_t *cnt = p.done + r * kGroup + g;
      if (ld_acquire(cnt) < nq) {  // bounded spin: a lost publication traps, never hangs
        const long long t0 = clock64();
        while (ld_acquire(cnt) < nq) {
          __nanosleep(256);
          if (clock64() - t0 > (1ll << 35)) __trap();
        }
      }
      float M[kGroup], Z[kGroup];
      float4 acc[kGroup];
#pragma unroll
      for (int a = 0; a < kGroup; ++a) {
        M[a] = -INFINITY; Z[a] = 0.f; acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int q0 = 0; q0 < nq; q0 += 2) {
        float4 v[2][kGroup];
        float l2 = -INFINITY;  // lane u * 8 + a: lse of row a of item q0 + u (log2 units)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const bool ok = q0 + u < nq;
          const size_t prow = row0 + (size_t)(q0 + u) * qstride;
          if (ok && (lane >> 3) == u) l2 = __ldcg(p.part_lse + prow + (lane & 7)) * 1.4426950408889634f;
#pragma unroll
          for (int a = 0; a < kGroup; ++a)
            v[u][a] = ok ? __ldcg(reinterpret_cast<const float4 *>(p.part_o + (prow + a) * kHeadDim) + lane)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
          for (int a = 0; a < kGroup; ++a) {
            const float lq = __shfl_sync(0xffffffffu, l2, u * 8 + a);
            if (lq == -INFINITY) continue;
            const float Mn = fmaxf(M[a], lq);
            const float sc = ex2(M[a] - Mn), wgt = ex2(lq - Mn);  // ex2(-inf) = 0
            acc[a].x = acc[a].x * sc + wgt * v[u][a].x; acc[a].y = acc[a].y * sc + wgt * v[u][a].y;
            acc[a].z = acc[a].z * sc + wgt * v[u][a].z; acc[a].w = acc[a].w * sc + wgt * v[u][a].w;
            Z[a] = Z[a] * sc + wgt;
            M[a] = Mn;
          }
        }
      }
#pragma unroll
      for (int a = 0; a < kGroup; ++a) {
        const float inv = 1.f / Z[a];
        __align__(8) __nv_bfloat162 o2[2];
        o2[0] = __floats2bfloat162_rn(acc[a].x * inv, acc[a].y * inv);
        o2[1] = __floats2bfloat162_rn(acc[a].z * inv, acc[a].w * inv);
        *reinterpret_cast<uint2 *>(p.out + ((size_t)s * qheads + g * kGroup + a) * kHeadDim + 4 * lane) =
            *reinterpret_cast<uint2 *>(o2);
        if (p.lse_out && lane == a)
          p.lse_out[(size_t)s * qheads + g * kGroup + a] = (M[a] + __log2f(Z[a])) * 0.69314718055994531f;
      }
      // the last of the request's w readers re-arms the counters for the next call
      __syncwarp();
      if (lane == 0 && atomicAdd(cnt + p.R * kGroup, 1) == w - 1) {
        *cnt = 0;
        cnt[p.R * kGroup] = 0;
      }
    }
  }
  pdl_wait();  // complete only after attend_kernel (its counter re-arm) has completed
  if (tr) {
    __syncwarp();
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[(size_t)(3200 + blockIdx.x) * 16 + 1] = (long long)g;
  }
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

static int make_kv_map(CUtensorMap *map, const void *pool, const taper_kv *kv) {
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
    cuuint32_t box[5] = {64, (cuuint32_t)kTile, 2, 1, 1};
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

extern "C" int taper_decode_attention(const taper_batch *batch, const taper_admission *adm,
                                      const taper_kv *kv, const void *q, void *out, float *lse,
                                      float scale, void *workspace, size_t workspace_bytes,
                                      void *stream) {
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
  WsLayout L = ws_layout(R, S);
  if (workspace_bytes < L.fixed + 512) return fail(TAPER_ERR_CAPACITY, "workspace too small");
  if (S == 0) { set_launches(0); return TAPER_OK; }
  const int h = kv->h_local;
  char *w = static_cast<char *>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  CUtensorMap tmK, tmV;
  int rc = make_kv_map(&tmK, kv->k_pages, kv);
  if (rc != TAPER_OK) return rc;
  rc = make_kv_map(&tmV, kv->v_pages, kv);
  if (rc != TAPER_OK) return rc;

  static thread_local bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes);
    if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(attend_kernel)");
    attr_set = true;
  }
  WsTables tabs = ws_tables(workspace_bytes, R, S, h);
  AttnParams ap;
  ap.slot_page_off = kv->slot_page_off;
  ap.slot_pages = kv->slot_pages;
  ap.req_page_off = kv->req_page_off;
  ap.req_pages = kv->req_pages;
  ap.hdr = reinterpret_cast<int32_t *>(w + L.hdr);
  ap.done = reinterpret_cast<int32_t *>(w + L.done);
  ap.adm_by_req = reinterpret_cast<const int32_t *>(w + L.adm_by_req);
  ap.items = reinterpret_cast<const ItemDesc *>(w + tabs.items);
  ap.ltiles = reinterpret_cast<const int4 *>(w + tabs.ltiles);
  ap.q = static_cast<const __nv_bfloat16 *>(q);
  ap.part_lse = reinterpret_cast<float *>(w + tabs.lse);
  ap.part_o = reinterpret_cast<float *>(w + tabs.o);
  ap.h_local = h;
  ap.page_size = kv->page_size;
  ap.tma5d = kv->page_size >= kTile ? 1 : 0;
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
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, attend_kernel, tmK, tmV, ap);
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
  const int grid = S > 0 ? S : 1;  // CTAs beyond the admitted count exit at once
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kMergeThreads);
  cfg.dynamicSmemBytes = 0;
  e = cudaLaunchKernelEx(&cfg, merge_kernel, mp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "merge_kernel launch");
  if (g_prof_ev[2]) cudaEventRecord(g_prof_ev[2], st);
  set_launches(2);
  return TAPER_OK;
}
