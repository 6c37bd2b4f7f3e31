// attention.cu -- cascade decode attention for one continuous-batching step.
//
// Sec. 3.1: branch i of a parallel phase attends to
//     P (+) H (+) h_i (+) y_{i,<t}
// and "a backend with paged or radix-tree KV caches can serve all branches from a single
// set of prefix blocks".  The kernels below exploit exactly that:
//
//  A6  shared_prefix_kernel (tcgen05 + TMA, one persistent CTA per SM)
//      work item = (request r, local KV head g, 1024-token chunk c of P (+) H).
//      The w_r admitted branches x 8 GQA query heads are stacked into one M = 128 MMA
//      operand (rows = 8 * w_r <= 128), and every K/V page of the chunk is brought into
//      shared memory by TMA ONCE and contracted against all stacked rows:
//          S = Q_stack K^T  (tcgen05.mma, M=128, N=64 tokens, K=128, fp32 in TMEM)
//          online softmax in registers (one TMEM lane = one query row per thread)
//          O += P V         (tcgen05.mma, M=128, N=128, K=64 tokens, P bf16 from SMEM)
//      -> normalised partial (o, lse) per stacked row and chunk.
//  A7+A8 local_merge_kernel (CUDA cores)
//      per admitted slot s and local KV head g: 8 query rows over the branch-local
//      segment h_i (+) y_i -- lane-per-token QK with 16-byte loads, warp-shuffle
//      softmax, coalesced PV -- then the log-sum-exp merge of the shared-chunk partials
//      and the local partial into bf16 out[s, 8g:8g+8, :].
//
// Chunk boundaries depend only on the prefix length, and each row's arithmetic does not
// depend on its position in the stacked operand, so a slot's output does not depend on
// which siblings are co-admitted (Lemma 1; tests/test_gpu_attention.py).
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>

#include "host_common.h"
#include "taper_internal.cuh"

namespace taper {

constexpr int kTile = 64;      // tokens per pipeline stage
constexpr int kStages = 4;     // TMA ring depth (4 x 32 KB in flight per SM)
constexpr int kRowsMax = 128;  // MMA M; 8 * w_r <= 128
constexpr int kKVStageBytes = 4 * 8192;             // K[d0:64], K[d64:128], V[..], V[..]
constexpr int kOffQ = kStages * kKVStageBytes;      // 131072
constexpr int kQBytes = 2 * kRowsMax * 128;         // two 64-column SW128 atoms
constexpr int kOffP = kOffQ + kQBytes;              // 163840
constexpr int kPBytes = kRowsMax * 128;             // 128 rows x 64 tokens bf16
// P precision (DESIGN.md Sec. 9 "P precision"): by default P = hi + lo with both parts
// bf16 and two PV MMAs, so P carries ~16 mantissa bits (a single bf16 P breaks the
// 2e-3 / 1e-2 tolerance on peaked softmaxes).  fp16 P against bf16 V is not a legal
// kind::f16 combination (illegal instruction on sm_100a).  -DTAPER_P_BF16 builds the
// single-bf16 experiment.
#if !defined(TAPER_P_BF16)
#define TAPER_P_SPLIT 1
constexpr int kPParts = 2;
#else
constexpr int kPParts = 1;
#endif
constexpr int kOffBar = kOffP + 2 * kPParts * kPBytes;
constexpr int kSmemUsed = kOffBar + 256;
constexpr int kSmemBytes = kSmemUsed + 1024;        // + alignment slack
constexpr int kSharedThreads = 192;                 // warp0 TMA, warp1 MMA, warps2-5 softmax
constexpr uint32_t kTmemCols = 256;                 // S0 [0,64) S1 [64,128) O [128,256)

constexpr uint32_t kIdescQK = umma_idesc_bf16(128, 64, false, false);
constexpr uint32_t kIdescPV = umma_idesc_bf16(128, 128, false, true);

struct SharedParams {
  const int32_t *Lsh, *req_page_off, *req_pages;
  const int32_t *hdr, *req_chunk_off, *req_part_off, *req_adm_off, *adm_by_req;
  const __nv_bfloat16 *q;
  float *part_lse, *part_o;
  int R, h_local, page_size;
  float scale_log2;
};

struct Item {
  int r, g, tb, te, nt, w, adm_off, part_base;
};

__device__ __forceinline__ void decode_item(const SharedParams &p, int it, Item &x) {
  const int rc = it / p.h_local;
  x.g = it - rc * p.h_local;
  int lo = 0, hi = p.R;  // req_chunk_off[lo] <= rc < req_chunk_off[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(p.req_chunk_off + mid) <= rc) lo = mid; else hi = mid;
  }
  x.r = lo;
  const int c = rc - __ldg(p.req_chunk_off + lo);
  x.tb = c * kChunk;
  x.te = min(x.tb + kChunk, __ldg(p.Lsh + lo));
  x.nt = (x.te - x.tb + kTile - 1) / kTile;
  x.adm_off = __ldg(p.req_adm_off + lo);
  x.w = __ldg(p.req_adm_off + lo + 1) - x.adm_off;
  x.part_base = __ldg(p.req_part_off + lo) + c * x.w;
}

// Stage the stacked queries of an item into the SW128 K-major A-operand layout.
__device__ __forceinline__ void load_q_rows(const SharedParams &p, const Item &x, uint8_t *sQ,
                                            int row) {
  if (row >= 8 * x.w) return;
  const int slot = __ldg(p.adm_by_req + x.adm_off + (row >> 3));
  const uint4 *src = reinterpret_cast<const uint4 *>(
      p.q + ((size_t)slot * (kGroup * p.h_local) + x.g * kGroup + (row & 7)) * kHeadDim);
  uint4 v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) v[c] = __ldg(src + c);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int atom = c >> 3, cc = c & 7;
    uint8_t *dst = sQ + atom * (kRowsMax * 128) + (row >> 3) * 1024 + (row & 7) * 128 +
                   ((cc ^ (row & 7)) << 4);
    *reinterpret_cast<uint4 *>(dst) = v[c];
  }
}

__global__ void __launch_bounds__(kSharedThreads, 1)
    shared_prefix_kernel(const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, SharedParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kOffBar);
  uint64_t *full = bars;               // [kStages]
  uint64_t *empty = bars + kStages;    // [kStages]
  uint64_t *s_full = bars + 2 * kStages;  // [2]
  uint64_t *p_full = s_full + 2;          // [2]
  uint64_t *pv_done = p_full + 2;         // [2]
  uint64_t *q_full = pv_done + 2;
  uint64_t *o_full = q_full + 1;
  uint64_t *o_free = o_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_free + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = __ldg(p.hdr) * p.h_local;

  // zero the operand buffers once: stale rows must be finite (row independence of MMA)
  for (int i = tid; i < kOffBar / 16; i += kSharedThreads)
    reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
      mbar_init(pv_done + i, 1);
    }
    mbar_init(q_full, 128);
    mbar_init(o_full, 1);
    mbar_init(o_free, 128);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmK); tma_prefetch_desc(&tmV); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      const int box_tok = p.page_size < kTile ? p.page_size : kTile;
      const uint32_t half_box_bytes = box_tok * 128;
      int stage = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        Item x;
        decode_item(p, it, x);
        const int32_t *pages = p.req_pages + __ldg(p.req_page_off + x.r);
        for (int t = 0; t < x.nt; ++t) {
          mbar_wait(empty + stage, phase ^ 1);
          const int tok0 = x.tb + t * kTile;
          const int valid = min(kTile, x.te - tok0);
          const int n_box = (valid + box_tok - 1) / box_tok;
          mbar_arrive_expect_tx(full + stage, n_box * half_box_bytes * 4);
          uint8_t *st = smem + stage * kKVStageBytes;
          for (int b = 0; b < n_box; ++b) {
            const int tok = tok0 + b * box_tok;
            const int page = __ldg(pages + tok / p.page_size);
            const int row = tok % p.page_size;
            const int o = b * half_box_bytes;
            tma_load_4d(st + o, &tmK, full + stage, 0, row, x.g, page);
            tma_load_4d(st + 8192 + o, &tmK, full + stage, 64, row, x.g, page);
            tma_load_4d(st + 16384 + o, &tmV, full + stage, 0, row, x.g, page);
            tma_load_4d(st + 24576 + o, &tmV, full + stage, 64, row, x.g, page);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (single thread) =======================
    if (lane == 0) {
      const uint32_t sQ = smem_u32(smem + kOffQ);
      const uint32_t sP0 = smem_u32(smem + kOffP);
      const uint32_t sKV = smem_u32(smem);
      const uint32_t tO = tmem + 128;
      int stage = 0, prev_stage = 0;
      uint32_t phase = 0;
      uint32_t n = 0;  // global tile counter
      uint32_t item_idx = 0;
      auto issue_pv = [&](uint32_t m, int st, bool first) {
        mbar_wait(p_full + (m & 1), (m >> 1) & 1);
        if (first) mbar_wait(o_free, (item_idx & 1) ^ 1);
        tc_fence_after();
        const uint32_t vb = sKV + st * kKVStageBytes + 16384;
#pragma unroll
        for (int part = 0; part < kPParts; ++part) {
          const uint32_t pa = sP0 + (part * 2 + (m & 1)) * kPBytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t a = umma_desc_sw128(pa + kk * 32, 16, 1024);
            const uint64_t b = umma_desc_sw128(vb + kk * 2048, 8192, 1024);
            tc_mma_f16(tO, a, b, kIdescPV, (first && part == 0 && kk == 0) ? 0u : 1u);
          }
        }
        tc_commit(empty + st);
        tc_commit(pv_done + (m & 1));
      };
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        Item x;
        decode_item(p, it, x);
        mbar_wait(q_full, item_idx & 1);
        tc_fence_after();
        for (int t = 0; t < x.nt; ++t) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t kb = sKV + stage * kKVStageBytes;
          const uint32_t tS = tmem + (n & 1) * 64;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t a = umma_desc_sw128(sQ + (kk >> 2) * (kRowsMax * 128) + (kk & 3) * 32, 16, 1024);
            const uint64_t b = umma_desc_sw128(kb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
            tc_mma_f16(tS, a, b, kIdescQK, kk > 0 ? 1u : 0u);
          }
          tc_commit(s_full + (n & 1));
          if (t > 0) issue_pv(n - 1, prev_stage, t == 1);
          prev_stage = stage;
          if (++stage == kStages) { stage = 0; phase ^= 1; }
          ++n;
        }
        issue_pv(n - 1, prev_stage, x.nt == 1);
        tc_commit(o_full);
        ++item_idx;
      }
    }
  } else {
    // ======================= softmax / correction / epilogue (128 threads) ===========
    const int wq = warp & 3;            // TMEM lane quadrant of this warp
    const int row = wq * 32 + lane;     // query row owned by this thread
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    uint8_t *sQ = smem + kOffQ;
    uint32_t n = 0, item_idx = 0;
    if (blockIdx.x < n_items) {
      Item x0;
      decode_item(p, blockIdx.x, x0);
      load_q_rows(p, x0, sQ, row);
      fence_proxy_async_smem();
      mbar_arrive(q_full);
    }
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      Item x;
      decode_item(p, it, x);
      const int R8 = 8 * x.w;
      const bool warp_active = wq * 32 < R8;
      float m_run = -INFINITY, l_run = 0.f;
      for (int t = 0; t < x.nt; ++t) {
        const uint32_t sb = n & 1;
        mbar_wait(s_full + sb, (n >> 1) & 1);
        tc_fence_after();
        if (warp_active) {
          uint32_t s0[32], s1[32];
          const uint32_t tS = tmem + lane_off + sb * 64;
          tmem_ld32(tS, s0);
          tmem_ld32(tS + 32, s1);
          tmem_ld_wait();
          const int valid = min(kTile, x.te - (x.tb + t * kTile));
          float xs[64];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            xs[j] = j < valid ? __uint_as_float(s0[j]) * p.scale_log2 : -INFINITY;
            xs[32 + j] = (32 + j) < valid ? __uint_as_float(s1[j]) * p.scale_log2 : -INFINITY;
          }
          float mx = xs[0];
#pragma unroll
          for (int j = 1; j < 64; ++j) mx = fmaxf(mx, xs[j]);
          // lazy rescale: keep a stale max unless the row max grew by > 8 (2^8 headroom)
          const bool need = mx > m_run + 8.f;
          float alpha = 1.f;
          if (need) {
            alpha = ex2(m_run - mx);  // 0 when m_run = -inf
            l_run *= alpha;
            m_run = mx;
          }
          if (t > 0 && __any_sync(0xffffffffu, need)) {
            // O *= alpha needs PV(n-1) complete
            mbar_wait(pv_done + ((n - 1) & 1), ((n - 1) >> 1) & 1);
            tc_fence_after();
            const uint32_t tO = tmem + lane_off + 128;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t o[32];
              tmem_ld32(tO + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
              tmem_st32(tO + c * 32, o);
            }
            tmem_st_wait();
          }
          // P = 2^(x - m) in bf16; l accumulates the rounded values actually multiplied
          uint32_t pk[kPParts][32];
          float lsum = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float e0 = ex2(xs[2 * j] - m_run), e1 = ex2(xs[2 * j + 1] - m_run);
            __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
            float2 f2 = __bfloat1622float2(h2);
            pk[0][j] = *reinterpret_cast<uint32_t *>(&h2);
#if defined(TAPER_P_SPLIT)
            __nv_bfloat162 l2 = __floats2bfloat162_rn(e0 - f2.x, e1 - f2.y);
            float2 g2 = __bfloat1622float2(l2);
            pk[1][j] = *reinterpret_cast<uint32_t *>(&l2);
            lsum += (f2.x + g2.x) + (f2.y + g2.y);
#else
            lsum += f2.x + f2.y;
#endif
          }
          l_run += lsum;
          if (n >= 2) mbar_wait(pv_done + sb, ((n >> 1) - 1) & 1);  // P[sb] free
#pragma unroll
          for (int part = 0; part < kPParts; ++part) {
            uint8_t *prow = smem + kOffP + (part * 2 + sb) * kPBytes + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<uint4 *>(prow + ((c ^ (row & 7)) << 4)) =
                  make_uint4(pk[part][4 * c], pk[part][4 * c + 1], pk[part][4 * c + 2], pk[part][4 * c + 3]);
          }
          fence_proxy_async_smem();
        }
        tc_fence_before();
        mbar_arrive(p_full + sb);
        ++n;
      }
      // all QK MMAs of this item are complete -> stage the next item's queries
      const int next = it + gridDim.x;
      if (next < n_items) {
        Item xn;
        decode_item(p, next, xn);
        load_q_rows(p, xn, sQ, row);
        fence_proxy_async_smem();
        mbar_arrive(q_full);
      }
      // epilogue: normalised partial (o, lse) for each live row
      mbar_wait(o_full, item_idx & 1);
      tc_fence_after();
      if (warp_active) {
        const bool live = row < R8;
        const size_t prow = ((size_t)(x.part_base + (row >> 3)) * p.h_local + x.g) * kGroup + (row & 7);
        const float inv_l = 1.f / l_run;
        float4 *dst = reinterpret_cast<float4 *>(p.part_o + prow * kHeadDim);
        const uint32_t tO = tmem + lane_off + 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + c * 32, o);
          tmem_ld_wait();
          if (live) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[c * 8 + j] = make_float4(__uint_as_float(o[4 * j]) * inv_l,
                                           __uint_as_float(o[4 * j + 1]) * inv_l,
                                           __uint_as_float(o[4 * j + 2]) * inv_l,
                                           __uint_as_float(o[4 * j + 3]) * inv_l);
          }
        }
        if (live) p.part_lse[prow] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
      }
      tc_fence_before();
      mbar_arrive(o_free);
      ++item_idx;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ------------------------------------------------------------------ local + merge
constexpr int kLocalThreads = 128;

struct LocalParams {
  const int32_t *Lsh, *Lloc, *slot_page_off, *slot_pages;
  const int32_t *hdr, *slot_req, *slot_rank, *req_chunk_off, *req_part_off, *req_adm_off,
      *adm_list;
  const __nv_bfloat16 *q, *k_pages, *v_pages;
  const float *part_lse, *part_o;
  __nv_bfloat16 *out;
  float *lse_out;
  int h_local, page_size;
  float scale_log2;
};

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, d));
  return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
  return x;
}

__global__ void __launch_bounds__(kLocalThreads) local_merge_kernel(LocalParams p) {
  __shared__ __align__(16) float qs[kGroup][kHeadDim];
  __shared__ __align__(16) float wo[4][kGroup][kHeadDim];
  __shared__ float wm[4][kGroup], wl[4][kGroup];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = p.h_local;
  const int n_items = __ldg(p.hdr + 2) * h;
  const int qheads = kGroup * h;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int k = it / h, g = it - k * h;
    const int s = __ldg(p.adm_list + k);
    const int r = __ldg(p.slot_req + s);
    const int j = __ldg(p.slot_rank + s);
    const int adm0 = __ldg(p.req_adm_off + r);
    const int w = __ldg(p.req_adm_off + r + 1) - adm0;
    __syncthreads();  // smem reuse across items
    {
      const int rr = tid >> 4, d0 = (tid & 15) * 8;
      const uint4 raw = __ldg(reinterpret_cast<const uint4 *>(
          p.q + ((size_t)s * qheads + g * kGroup + rr) * kHeadDim + d0));
      const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = __bfloat1622float2(b2[i]);
        qs[rr][d0 + 2 * i] = f.x * p.scale_log2;
        qs[rr][d0 + 2 * i + 1] = f.y * p.scale_log2;
      }
    }
    __syncthreads();
    // ---------------- A7: branch-local segment, split over 4 warps
    const int Ll = __ldg(p.Lloc + s);
    const int32_t *pages = p.slot_pages + __ldg(p.slot_page_off + s);
    float m[kGroup], lsum[kGroup], o[kGroup][4];
#pragma unroll
    for (int a = 0; a < kGroup; ++a) {
      m[a] = -INFINITY; lsum[a] = 0.f;
      o[a][0] = o[a][1] = o[a][2] = o[a][3] = 0.f;
    }
    for (int blk = warp; blk * 32 < Ll; blk += 4) {
      const int t = blk * 32 + lane;
      const bool valid = t < Ll;
      float x[kGroup];
      if (valid) {
        const int page = __ldg(pages + t / p.page_size);
        const uint4 *kr = reinterpret_cast<const uint4 *>(
            p.k_pages + (((size_t)page * h + g) * p.page_size + t % p.page_size) * kHeadDim);
#pragma unroll
        for (int a = 0; a < kGroup; ++a) x[a] = 0.f;
#pragma unroll 4
        for (int c = 0; c < 16; ++c) {
          const uint4 raw = __ldg(kr + c);
          const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&raw);
          float kf[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 f = __bfloat1622float2(b2[i]);
            kf[2 * i] = f.x; kf[2 * i + 1] = f.y;
          }
#pragma unroll
          for (int a = 0; a < kGroup; ++a) {
            const float4 q0 = *reinterpret_cast<const float4 *>(&qs[a][c * 8]);
            const float4 q1 = *reinterpret_cast<const float4 *>(&qs[a][c * 8 + 4]);
            x[a] += q0.x * kf[0] + q0.y * kf[1] + q0.z * kf[2] + q0.w * kf[3] +
                    q1.x * kf[4] + q1.y * kf[5] + q1.z * kf[6] + q1.w * kf[7];
          }
        }
      } else {
#pragma unroll
        for (int a = 0; a < kGroup; ++a) x[a] = -INFINITY;
      }
      float pr[kGroup];
#pragma unroll
      for (int a = 0; a < kGroup; ++a) {
        const float mn = fmaxf(m[a], warp_max(x[a]));
        const float alpha = ex2(m[a] - mn);
        pr[a] = valid ? ex2(x[a] - mn) : 0.f;
        lsum[a] = lsum[a] * alpha + pr[a];
        o[a][0] *= alpha; o[a][1] *= alpha; o[a][2] *= alpha; o[a][3] *= alpha;
        m[a] = mn;
      }
      const int nvalid = min(32, Ll - blk * 32);
      for (int jj = 0; jj < nvalid; ++jj) {
        const int tj = blk * 32 + jj;
        const int page = __ldg(pages + tj / p.page_size);
        const uint2 raw = __ldg(reinterpret_cast<const uint2 *>(
            p.v_pages + (((size_t)page * h + g) * p.page_size + tj % p.page_size) * kHeadDim +
            4 * lane));
        const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&raw);
        const float2 v01 = __bfloat1622float2(b2[0]), v23 = __bfloat1622float2(b2[1]);
#pragma unroll
        for (int a = 0; a < kGroup; ++a) {
          const float pj = __shfl_sync(0xffffffffu, pr[a], jj);
          o[a][0] += pj * v01.x; o[a][1] += pj * v01.y;
          o[a][2] += pj * v23.x; o[a][3] += pj * v23.y;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kGroup; ++a) {
      const float l = warp_sum(lsum[a]);
      if (lane == 0) { wm[warp][a] = m[a]; wl[warp][a] = l; }
      *reinterpret_cast<float4 *>(&wo[warp][a][4 * lane]) = make_float4(o[a][0], o[a][1], o[a][2], o[a][3]);
    }
    __syncthreads();
    // ---------------- A8: log-sum-exp merge (shared chunks in order, then local warps)
    {
      const int rr = tid >> 4, d0 = (tid & 15) * 8;
      const int c0 = __ldg(p.req_chunk_off + r), nch = __ldg(p.req_chunk_off + r + 1) - c0;
      const int cs0 = __ldg(p.req_part_off + r) + j;
      float M = -INFINITY;
      for (int c = 0; c < nch; ++c) {
        const size_t prow = ((size_t)(cs0 + c * w) * h + g) * kGroup + rr;
        M = fmaxf(M, __ldg(p.part_lse + prow) * 1.4426950408889634f);
      }
#pragma unroll
      for (int ww = 0; ww < 4; ++ww) if (wl[ww][rr] > 0.f) M = fmaxf(M, wm[ww][rr]);
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      float Z = 0.f;
      for (int c = 0; c < nch; ++c) {
        const size_t prow = ((size_t)(cs0 + c * w) * h + g) * kGroup + rr;
        const float wgt = ex2(__ldg(p.part_lse + prow) * 1.4426950408889634f - M);
        const float4 *src = reinterpret_cast<const float4 *>(p.part_o + prow * kHeadDim + d0);
        const float4 a0 = __ldg(src), a1 = __ldg(src + 1);
        acc[0] += wgt * a0.x; acc[1] += wgt * a0.y; acc[2] += wgt * a0.z; acc[3] += wgt * a0.w;
        acc[4] += wgt * a1.x; acc[5] += wgt * a1.y; acc[6] += wgt * a1.z; acc[7] += wgt * a1.w;
        Z += wgt;
      }
#pragma unroll
      for (int ww = 0; ww < 4; ++ww) {
        if (wl[ww][rr] > 0.f) {
          const float wgt = ex2(wm[ww][rr] - M);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += wgt * wo[ww][rr][d0 + i];
          Z += wgt * wl[ww][rr];
        }
      }
      const float invZ = 1.f / Z;
      __align__(16) __nv_bfloat162 ob[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ob[i] = __floats2bfloat162_rn(acc[2 * i] * invZ, acc[2 * i + 1] * invZ);
      *reinterpret_cast<uint4 *>(p.out + ((size_t)s * qheads + g * kGroup + rr) * kHeadDim + d0) =
          *reinterpret_cast<uint4 *>(ob);
      if (p.lse_out && (tid & 15) == 0)
        p.lse_out[(size_t)s * qheads + g * kGroup + rr] = (M + __log2f(Z)) * 0.69314718055994531f;
    }
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
  cuuint64_t dims[4] = {128, (cuuint64_t)kv->page_size, (cuuint64_t)kv->h_local,
                        (cuuint64_t)kv->num_pages};
  cuuint64_t strides[3] = {row, row * kv->page_size, row * kv->page_size * kv->h_local};
  const cuuint32_t box_tok = kv->page_size < kTile ? kv->page_size : kTile;
  cuuint32_t box[4] = {64, box_tok, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(pool), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TAPER_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return TAPER_OK;
}

static thread_local cudaEvent_t g_prof_ev[3] = {nullptr, nullptr, nullptr};

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
  size_t lse_off, o_off;
  ws_partials(workspace_bytes, R, S, h, &lse_off, &o_off);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float scale_log2 = scale * 1.4426950408889634f;

  CUtensorMap tmK, tmV;
  int rc = make_kv_map(&tmK, kv->k_pages, kv);
  if (rc != TAPER_OK) return rc;
  rc = make_kv_map(&tmV, kv->v_pages, kv);
  if (rc != TAPER_OK) return rc;

  static thread_local bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(shared_prefix_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(shared_prefix_kernel)");
    attr_set = true;
  }
  SharedParams sp;
  sp.Lsh = batch->req_shared_len;
  sp.req_page_off = kv->req_page_off;
  sp.req_pages = kv->req_pages;
  sp.hdr = reinterpret_cast<const int32_t *>(w + L.hdr);
  sp.req_chunk_off = reinterpret_cast<const int32_t *>(w + L.req_chunk_off);
  sp.req_part_off = reinterpret_cast<const int32_t *>(w + L.req_part_off);
  sp.req_adm_off = reinterpret_cast<const int32_t *>(w + L.req_adm_off);
  sp.adm_by_req = reinterpret_cast<const int32_t *>(w + L.adm_by_req);
  sp.q = static_cast<const __nv_bfloat16 *>(q);
  sp.part_lse = reinterpret_cast<float *>(w + lse_off);
  sp.part_o = reinterpret_cast<float *>(w + o_off);
  sp.R = R;
  sp.h_local = h;
  sp.page_size = kv->page_size;
  sp.scale_log2 = scale_log2;
  const int sms = device_sms();
  if (g_prof_ev[0]) cudaEventRecord(g_prof_ev[0], st);
  shared_prefix_kernel<<<sms, kSharedThreads, kSmemBytes, st>>>(tmK, tmV, sp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "shared_prefix_kernel launch");
  if (g_prof_ev[1]) cudaEventRecord(g_prof_ev[1], st);

  LocalParams lp;
  lp.Lsh = batch->req_shared_len;
  lp.Lloc = batch->slot_local_len;
  lp.slot_page_off = kv->slot_page_off;
  lp.slot_pages = kv->slot_pages;
  lp.hdr = sp.hdr;
  lp.slot_req = reinterpret_cast<const int32_t *>(w + L.slot_req);
  lp.slot_rank = reinterpret_cast<const int32_t *>(w + L.slot_rank);
  lp.req_chunk_off = sp.req_chunk_off;
  lp.req_part_off = sp.req_part_off;
  lp.req_adm_off = sp.req_adm_off;
  lp.adm_list = adm->adm_list;
  lp.q = sp.q;
  lp.k_pages = static_cast<const __nv_bfloat16 *>(kv->k_pages);
  lp.v_pages = static_cast<const __nv_bfloat16 *>(kv->v_pages);
  lp.part_lse = sp.part_lse;
  lp.part_o = sp.part_o;
  lp.out = static_cast<__nv_bfloat16 *>(out);
  lp.lse_out = lse;
  lp.h_local = h;
  lp.page_size = kv->page_size;
  lp.scale_log2 = scale_log2;
  int grid = S * h;
  if (grid > sms * 8) grid = sms * 8;
  local_merge_kernel<<<grid, kLocalThreads, 0, st>>>(lp);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "local_merge_kernel launch");
  if (g_prof_ev[2]) cudaEventRecord(g_prof_ev[2], st);
  set_launches(2);
  return TAPER_OK;
}
