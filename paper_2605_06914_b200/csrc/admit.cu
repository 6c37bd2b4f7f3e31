// admit.cu -- per-step admission (Sec. 3.3, Algorithm 1) as one CTA on the device.
//
// Algorithm 1 widens the protected composition S0 greedily by
// utility per marginal latency cost and prunes a request once its next branch does not
// fit the slack budget.  Under the paper's default linear utility (L391) every score is
// 1 / (EPS + dt) and dt grows with the candidate's added context dL, so the greedy loop
// commits candidates in ascending (dL, r, slot) order and stops at the first one that
// does not fit (monotonicity, L120-123).  This kernel therefore evaluates Alg. 1 as
//     bitonic sort of candidate keys (dL, r, slot)  ->  int64 prefix scan S_m
//     -> predicate T(n0 + m, L0 + S_m) <= budget  ->  longest feasible prefix,
// in fp64 with IEEE round-to-nearest and no contraction, which gives the same set and
// the same T(S) bits as the literal loop.
// The fixed policies IRP-Off / IRP-Ck / IRP-Eager (App. D) reuse the same
// canonical order (ascending Lloc, then slot index).  The kernel then emits the
// attention work list, so the step never round-trips to the host.
#include "taper_internal.cuh"

namespace taper {

constexpr int kAdmitThreads = 1024;
constexpr int kPerThread = kMaxSlots / kAdmitThreads;  // 4
#ifndef TAPER_ITEM_COST0
#define TAPER_ITEM_COST0 0
#endif
constexpr int kItemCost0 = TAPER_ITEM_COST0;  // fixed per-item cost in the claim order
#ifndef TAPER_WIDE_COST
#define TAPER_WIDE_COST 3
#endif
#ifndef TAPER_NARROW_COST
#define TAPER_NARROW_COST 2
#endif
#ifndef TAPER_ROW_COST
#define TAPER_ROW_COST 2
#endif
// per-tile claim costs: swap-mode items with > 4 branches (softmax-bound), narrower swap items
// and row-mode items (both at about the memory rate)
constexpr int kWideCost = TAPER_WIDE_COST, kNarrowCost = TAPER_NARROW_COST, kRowCost = TAPER_ROW_COST;
constexpr double kEps = 1e-9;  // Alg. 1 line 16 "EPS" (no value in the paper) [C-adm-3]

struct AdmitParams {
  int R, S;
  const int32_t *Lsh, *off, *Lloc;
  const int32_t *seg_off, *seg_len;  // local segments (CSR over S), or NULL = one per slot
  const double *slack;
  double a, b, c, rho;
  int kind, cap;
  int ctx_per_request;  // TAPER_CTX_PER_REQUEST: an opportunistic slot adds Lloc only
  const double *util;   // [R][ustride] u_r(k) (flat past the table); NULL = linear
  int ustride;
  int decide;  // 1: admission + work list; 0: work list from slot_admitted only
  int32_t *req_width;
  uint8_t *slot_admitted;
  int32_t *adm_list, *n_adm;
  double *diag;
  int32_t *status;
  int32_t *hdr, *slot_req, *slot_rank, *slot_lbase, *req_chunk_off, *req_loc_off, *req_part_off,
      *req_adm_off, *adm_by_req;
  int4 *merge_desc;  // [2 S] per admitted slot k (adm_list order): {slot, first shared
                     //     partial, prefix chunks, width}, {first local partial, local
                     //     items, request, items of the request per KV head}
  int32_t *done;     // [2 * R * 8] attend -> merge completion counters (zeroed here)
  int64_t cap_cs;
  int h_local;
  ItemDesc *items;   // [cap_cs] work items (A5)
  int4 *ltiles;      // [cap_cs * 16] local tiles {slot, tok0, valid, jrow}
  ItemDesc *sorted;  // [cap_cs] the item descriptors in claim order (longest first)
};

// Local work items of slot s: one per <= kLocalItemTiles 64-token tiles of each of its
// local segments (a tile never spans two segments: each starts on a page boundary).
__device__ __forceinline__ int local_items(const AdmitParams &p, int s) {
  constexpr int per = kTileTokens * kLocalItemTiles;
  if (p.seg_off == nullptr) return (p.Lloc[s] + per - 1) / per;
  int n = 0;
  for (int q = p.seg_off[s]; q < p.seg_off[s + 1]; ++q) n += (max(p.seg_len[q], 0) + per - 1) / per;
  return n;
}

// Prefix chunks of a request (a function of Lsh and h_local only: schedule invariance,
// Lemma 1).  Nominal chunks of ck = taper_chunk_tokens(Lsh, h, R) tokens; with >= 3 chunks and
// TAPER_SKEW_CHUNKS, the first is ck + ck/2 and the others shift by ck/2, so the last one is
// about half a chunk: the longest-first claim order then ends on short items.  Chunk starts
// stay multiples of 64 tokens (a tile never straddles a page).
#ifndef TAPER_SKEW_CHUNKS
#define TAPER_SKEW_CHUNKS 0
#endif
struct ChunkPlan { int ck, half, n; bool skew; };
__device__ __forceinline__ ChunkPlan chunk_plan(int lsh, int h, int R) {
  ChunkPlan c;
  c.ck = taper_chunk_tokens(lsh, h, R);
  c.half = (c.ck / 2) / kTileTokens * kTileTokens;
  const int n = (lsh + c.ck - 1) / c.ck;
  c.skew = TAPER_SKEW_CHUNKS && n >= 3 && c.ck + c.half <= kChunk;
  c.n = (c.skew && (n - 1) * c.ck + c.half >= lsh) ? n - 1 : n;
  return c;
}
__device__ __forceinline__ int chunk_start(const ChunkPlan &c, int lsh, int i) {
  if (i >= c.n) return lsh;
  if (!c.skew || i == 0) return min(i * c.ck, lsh);
  return min(i * c.ck + c.half, lsh);
}

__device__ __forceinline__ double T_eval(double a, double b, double c, long long n,
                                         long long L) {
  // App. C.1: T(S) = a + b*n_tokens + c*L_context, each operation rounded separately.
  return __dadd_rn(__dadd_rn(a, __dmul_rn(b, __ll2double_rn(n))),
                   __dmul_rn(c, __ll2double_rn(L)));
}

// Block-wide exclusive scan of 4 consecutive values per thread (4096 elements).
template <typename T>
__device__ T block_exscan4(T (&v)[kPerThread], T *warp_buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T local[kPerThread];
  T run = 0;
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) { local[k] = run; run += v[k]; }
  T incl = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_buf[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T x = warp_buf[lane];
    T xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += y;
    }
    warp_buf[lane] = xi - x;          // exclusive warp offset
    if (lane == 31) warp_buf[32] = xi;  // total
  }
  __syncthreads();
  T base = warp_buf[warp] + (incl - run);
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) v[k] = base + local[k];
  T total = warp_buf[32];
  __syncthreads();
  return total;
}

// Ascending bitonic sort of n (power of two, <= 4096) keys in shared memory.
__device__ void bitonic_sort(unsigned long long *keys, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          unsigned long long x = keys[i], y = keys[ixj];
          bool up = (i & k) == 0;
          if ((x > y) == up) { keys[i] = y; keys[ixj] = x; }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ long long warp_sum_ll(long long x) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
  return x;
}
__device__ __forceinline__ double warp_min_d(double x) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, d));
  return x;
}

// u_r(k) of the caller's table, flat past its last column (reading R-util)
__device__ __forceinline__ double util_at(const AdmitParams &p, int r, int k) {
  return p.util[(long long)r * p.ustride + min(k, p.ustride - 1)];
}

// (score, r) lexicographic argmax: higher score, ties to the lower request index -- the
// strict '>' of Alg. 1 line 18 scanned in ascending r [C-adm-4].  r < 0 = no candidate.
struct Best { double score; long long dL; int r; };
__device__ __forceinline__ bool better(double s1, int r1, double s2, int r2) {
  if (r2 < 0) return r1 >= 0;
  if (r1 < 0) return false;
  return s1 > s2 || (s1 == s2 && r1 < r2);
}
__device__ __forceinline__ Best warp_argmax(Best b) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    Best o;
    o.score = __shfl_xor_sync(0xffffffffu, b.score, d);
    o.dL = __shfl_xor_sync(0xffffffffu, b.dL, d);
    o.r = __shfl_xor_sync(0xffffffffu, b.r, d);
    if (better(o.score, o.r, b.score, b.r)) b = o;
  }
  return b;
}

// Algorithm 1 executed literally for a caller-supplied utility
// table (Sec. 3.4 "pluggable utility interface").  keys[] holds
// the opportunistic slots sorted request-major (r, Lloc, slot), so request r's next
// branch in canonical order [C-adm-1] is keys[start_r + granted_r].  One iteration of
// the while-loop (L158-178): every live request evaluates its candidate in fp64 exactly
// as the oracle does (T(n+1, L+dL) against the budget -> prune; du / (EPS + max(0, dt))),
// a block-wide argmax picks the commit, and every thread applies it to (n, L).  One named
// barrier per iteration (the per-warp winners are double-buffered by iteration parity).
// Only the first ceil(R / 32) warps (<= 32) take part; thread t owns requests t, t + T, ..
__device__ void greedy_literal(const AdmitParams &p, const unsigned long long *keys,
                               int *scan_i, long long n0, long long L0, double budget,
                               long long *nadd_out, long long *Ladd_out) {
  constexpr int kOwn = kMaxSlots / kAdmitThreads;  // 4 requests per thread at most
  __shared__ double wb_score[2][32];
  __shared__ long long wb_dL[2][32];
  __shared__ int wb_r[2][32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int R = p.R;
  // start_r: exclusive scan of the opportunistic counts, request-major like the keys
  int cnt[kPerThread];
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    int r = tid * kPerThread + k;
    cnt[k] = (r < R) ? max(0, p.off[r + 1] - p.off[r] - 1) : 0;
  }
  block_exscan4<int>(cnt, scan_i);
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    int r = tid * kPerThread + k;
    if (r < R) p.req_part_off[r] = cnt[k];  // scratch: rewritten by the work-list pass
  }
  __syncthreads();
  // one request per thread while R <= 1024 (the fp64 division chain per candidate is the
  // iteration's latency, so candidates are spread over threads, not stacked per thread)
  const int nwarps = min(kAdmitThreads / 32, max(1, (R + 31) / 32));
  const int nthr = nwarps * 32;
  if (tid < nthr) {
    int start[kOwn], count[kOwn], g[kOwn];
    long long lsh[kOwn];
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const int r = tid + k * nthr;
      start[k] = 0; count[k] = 0; g[k] = 0; lsh[k] = 0;
      if (r < R) {
        start[k] = p.req_part_off[r];
        count[k] = max(0, p.off[r + 1] - p.off[r] - 1);
        lsh[k] = p.ctx_per_request ? 0ll : (long long)p.Lsh[r];
      }
    }
    long long n = n0, L = L0;
    for (int it = 0;; ++it) {
      Best b{0.0, 0, -1};
      const double T_step = T_eval(p.a, p.b, p.c, n, L);
#pragma unroll
      for (int k = 0; k < kOwn; ++k) {
        if (g[k] >= count[k]) continue;  // exhausted or pruned (count forced to g)
        const int r = tid + k * nthr;
        const int s = int(keys[start[k] + g[k]] & 0xFFF);
        const long long dL = lsh[k] + (long long)p.Lloc[s];
        const double T_widened = T_eval(p.a, p.b, p.c, n + 1, L + dL);
        if (T_widened > budget) { count[k] = g[k]; continue; }  // L164: prune r
        const double du = __dsub_rn(util_at(p, r, g[k] + 1), util_at(p, r, g[k]));
        const double dt = __dsub_rn(T_widened, T_step);
        const double score = __ddiv_rn(du, __dadd_rn(kEps, dt > 0.0 ? dt : 0.0));
        if (better(score, r, b.score, b.r)) { b.score = score; b.dL = dL; b.r = r; }
      }
      b = warp_argmax(b);
      Best w = b;
      if (nwarps > 1) {
        const int buf = it & 1;
        if (lane == 0) { wb_score[buf][tid >> 5] = b.score; wb_dL[buf][tid >> 5] = b.dL; wb_r[buf][tid >> 5] = b.r; }
        asm volatile("bar.sync 1, %0;" :: "r"(nthr) : "memory");
        w = Best{0.0, 0, -1};
        if (nwarps <= 2) {  // two warps: a broadcast scan beats five shuffle rounds (measured)
          for (int j = 0; j < nwarps; ++j)
            if (better(wb_score[buf][j], wb_r[buf][j], w.score, w.r))
              w = Best{wb_score[buf][j], wb_dL[buf][j], wb_r[buf][j]};
        } else {
          if (lane < nwarps) { w.score = wb_score[buf][lane]; w.dL = wb_dL[buf][lane]; w.r = wb_r[buf][lane]; }
          w = warp_argmax(w);
        }
      }
      if (w.r < 0 || w.score <= 0.0) break;  // L21-22: no feasible increment of value
      n += 1; L += w.dL;                         // L23-26: commit
#pragma unroll
      for (int k = 0; k < kOwn; ++k)
        if (tid + k * nthr == w.r) g[k] += 1;    // owner advances r (drops it when exhausted)
    }
    // admitted opportunistic slots: the first g_r of r's canonical run
#pragma unroll
    for (int k = 0; k < kOwn; ++k)
      for (int j = 0; j < g[k]; ++j) p.slot_admitted[int(keys[start[k] + j] & 0xFFF)] = 1;
    if (tid == 0) { *nadd_out = n - n0; *Ladd_out = L - L0; }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kAdmitThreads, 1) admit_kernel(AdmitParams p) {
  __shared__ unsigned long long keys[kMaxSlots];
  __shared__ long long scan_ll[33];
  __shared__ int scan_i[33];
  __shared__ long long red_ll[32];
  __shared__ double red_d[32];
  __shared__ int sh_status;
  __shared__ long long sh_n0, sh_L0, sh_nadd, sh_Ladd;
  __shared__ double sh_T0, sh_budget, sh_ms;
  __shared__ int sh_ncand, sh_mstar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = p.R, S = p.S;
  if (tid == 0) { sh_status = 0; sh_ncand = 0; sh_mstar = 0; }
  __syncthreads();

  // ---- per-request pass: slot -> request map, validation, protected slot (S0, L128)
  long long my_L0 = 0, my_n0 = 0;
  double my_ms = INFINITY;
  for (int r = tid; r < R; r += blockDim.x) {
    int b = p.off[r], e = p.off[r + 1];
    if (b < 0 || e < b || e > S || p.Lsh[r] < 0) { atomicOr(&sh_status, TAPER_STATUS_BAD_LENGTH); continue; }
    if (e == b) { atomicOr(&sh_status, TAPER_STATUS_EMPTY_REQUEST); continue; }
    int prot = -1, best = 0;
    for (int s = b; s < e; ++s) {
      p.slot_req[s] = r;
      int l = p.Lloc[s];
      if (l < 0) atomicOr(&sh_status, TAPER_STATUS_BAD_LENGTH);
      if (p.seg_off != nullptr) {  // segments must tile the local context exactly
        const int q0 = p.seg_off[s], q1 = p.seg_off[s + 1];
        long long sum = 0;
        bool bad = q1 < q0;
        for (int q = q0; q < q1 && !bad; ++q) { bad = p.seg_len[q] < 0; sum += p.seg_len[q]; }
        if (bad || sum != l) atomicOr(&sh_status, TAPER_STATUS_BAD_LENGTH);
      }
      if (prot < 0 || l < best) { prot = s; best = l; }  // canonical first (Lloc, slot)
    }
    if (p.decide) {
      my_n0 += 1;
      my_L0 += (long long)p.Lsh[r] + (long long)best;
      my_ms = fmin(my_ms, p.slack[r]);
      p.slot_rank[prot] = -1;  // marks the protected slot for the policy pass
    }
  }
  if (p.off[0] != 0 || p.off[R] != S) atomicOr(&sh_status, TAPER_STATUS_BAD_LENGTH);

  if (p.decide) {
    // ---- S0 aggregates and the slack budget (Sec. 3.3; Alg. 1 L2-4)
    my_n0 = warp_sum_ll(my_n0);
    my_L0 = warp_sum_ll(my_L0);
    my_ms = warp_min_d(my_ms);
    if (lane == 0) { red_ll[warp] = my_L0; red_d[warp] = my_ms; scan_ll[warp] = my_n0; }
    __syncthreads();
    if (tid == 0) {
      long long n0 = 0, L0 = 0;
      double ms = INFINITY;
      for (int w = 0; w < 32; ++w) { n0 += scan_ll[w]; L0 += red_ll[w]; ms = fmin(ms, red_d[w]); }
      double T0 = T_eval(p.a, p.b, p.c, n0, L0);
      double budget = T0;
      if (n0 > 0) {
        double residual = __dsub_rn(ms, T0);
        double B = residual > 0.0 ? residual : 0.0;
        budget = __dadd_rn(T0, __dmul_rn(p.rho, B));
      }
      if (p.kind == TAPER_POLICY_GREEDY && !p.util && p.c < __dmul_rn(budget, 0x1p-46))
        atomicOr(&sh_status, TAPER_STATUS_PRECISION);
      sh_n0 = n0; sh_L0 = L0; sh_T0 = T0; sh_budget = budget; sh_ms = ms;
      sh_nadd = 0; sh_Ladd = 0;
    }
    __syncthreads();
    if (sh_status & TAPER_STATUS_BAD_LENGTH) {
      // outputs undefined; keep memory-safe defaults
      for (int s = tid; s < S; s += blockDim.x) p.slot_admitted[s] = 0;
      __syncthreads();
    } else {
      // ---- policy pass: which opportunistic slots join the step
      int n_keys = 1;
      while (n_keys < S) n_keys <<= 1;
      const bool sorted_policy = p.kind == TAPER_POLICY_CAP || p.kind == TAPER_POLICY_GREEDY;
      // request-major keys (r, Lloc, slot): each request's opportunistic slots form one
      // run in canonical order (IRP-Ck, and Alg. 1 with a non-linear utility)
      const bool request_major = p.kind == TAPER_POLICY_CAP || p.util != nullptr;
      long long my_nadd = 0, my_Ladd = 0;
      for (int s = tid; s < n_keys; s += blockDim.x) {
        unsigned long long key = ~0ull;
        if (s < S) {
          int r = p.slot_req[s];
          bool prot = p.slot_rank[s] == -1;
          bool active = r >= 0 && r < R;
          uint8_t adm = prot ? 1 : 0;
          if (active && !prot) {
            // context added by admitting s: its whole sequence (paper, per sequence) or
            // only its local segment (cascade-aware, the prefix already counted once)
            long long dL = (p.ctx_per_request ? 0ll : (long long)p.Lsh[r]) + (long long)p.Lloc[s];
            if (p.kind == TAPER_POLICY_EAGER) {
              adm = 1; my_nadd += 1; my_Ladd += dL;
            } else if (request_major) {
              key = ((unsigned long long)r << 43) | ((unsigned long long)p.Lloc[s] << 12) |
                    (unsigned long long)s;
            } else if (p.kind == TAPER_POLICY_GREEDY) {
              key = ((unsigned long long)dL << 24) | ((unsigned long long)r << 12) |
                    (unsigned long long)s;
              atomicAdd(&sh_ncand, 1);
            }
          }
          p.slot_admitted[s] = adm;
        }
        if (sorted_policy) keys[s] = key;
      }
      __syncthreads();
      if (sorted_policy) {
        bitonic_sort(keys, n_keys);
        if (p.kind == TAPER_POLICY_CAP) {
          // canonical rank among r's non-protected slots -> admit the first cap-1
          for (int i = tid; i < S; i += blockDim.x) {
            unsigned long long k = keys[i];
            if (k == ~0ull) continue;
            int r = int(k >> 43), s = int(k & 0xFFF);
            // non-protected slots of r occupy a contiguous run; rank within it:
            int first = i;
            while (first > 0 && keys[first - 1] != ~0ull && int(keys[first - 1] >> 43) == r) --first;
            if (i - first < p.cap - 1) {
              p.slot_admitted[s] = 1;
              my_nadd += 1;
              my_Ladd += (p.ctx_per_request ? 0ll : (long long)p.Lsh[r]) + (long long)p.Lloc[s];
            }
          }
        } else if (request_major) {
          // GREEDY, non-linear utility: Alg. 1 literally (scores differ per request, so
          // the commit order is no longer a fixed sort of the candidates)
          greedy_literal(p, keys, scan_i, sh_n0, sh_L0, sh_budget, &sh_nadd, &sh_Ladd);
          my_nadd = 0; my_Ladd = 0;
        } else {
          // GREEDY: inclusive prefix sums of dL over the sorted candidates
          const int ncand = sh_ncand;
          long long v[kPerThread];
#pragma unroll
          for (int k = 0; k < kPerThread; ++k) {
            int i = tid * kPerThread + k;
            v[k] = (i < ncand) ? (long long)(keys[i] >> 24) : 0;
          }
          long long ex[kPerThread];
#pragma unroll
          for (int k = 0; k < kPerThread; ++k) ex[k] = v[k];
          block_exscan4<long long>(ex, scan_ll);
          int my_feasible = 0;
#pragma unroll
          for (int k = 0; k < kPerThread; ++k) {
            int i = tid * kPerThread + k;  // candidate position; m = i + 1 admitted
            if (i < ncand) {
              long long Sm = ex[k] + v[k];
              double Tm = T_eval(p.a, p.b, p.c, sh_n0 + i + 1, sh_L0 + Sm);
              if (Tm <= sh_budget) {
                my_feasible += 1;
                int s = int(keys[i] & 0xFFF);
                p.slot_admitted[s] = 1;  // feasible set is a prefix (T monotone in m)
              }
            }
          }
          int tot = my_feasible;
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
          if (lane == 0) atomicAdd(&sh_mstar, tot);
          __syncthreads();
          const int mstar = sh_mstar;
#pragma unroll
          for (int k = 0; k < kPerThread; ++k) {
            int i = tid * kPerThread + k;
            if (mstar > 0 && i == mstar - 1) { sh_nadd = mstar; sh_Ladd = ex[k] + v[k]; }
          }
          my_nadd = 0; my_Ladd = 0;
        }
      }
      if (p.kind != TAPER_POLICY_GREEDY) {
        my_nadd = warp_sum_ll(my_nadd);
        my_Ladd = warp_sum_ll(my_Ladd);
        if (lane == 0) {
          atomicAdd(reinterpret_cast<unsigned long long *>(&sh_nadd), (unsigned long long)my_nadd);
          atomicAdd(reinterpret_cast<unsigned long long *>(&sh_Ladd), (unsigned long long)my_Ladd);
        }
      }
      __syncthreads();
    }
    if (tid == 0) {
      double TS = T_eval(p.a, p.b, p.c, sh_n0 + sh_nadd, sh_L0 + sh_Ladd);
      p.diag[0] = sh_T0;
      p.diag[1] = sh_budget;
      p.diag[2] = TS;
      p.diag[3] = __dsub_rn(TS, sh_T0);  // Sec. 2.3 branch externality E_t(k)
      p.diag[4] = sh_ms;
    }
    __syncthreads();
  } else {
    __syncthreads();
  }

  // ---- work list (A5): per-request widths, item counts and CSR offsets.
  // Shared items: (taper_chunk_tokens(Lsh_r, h_local, R)-token prefix chunk, group of <= 16 admitted branches).  Local items:
  // <= kLocalItemTiles 64-token tiles of ONE admitted branch's local KV.  Partials (8 rows
  // per KV head each): shared (chunk c, branch j) at c * w + j, then one per local item.
  int w_loc[kPerThread], nc_loc[kPerThread], nl_loc[kPerThread], cs_loc[kPerThread];
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    int r = tid * kPerThread + k;
    int w = 0, nc = 0, nl = 0;
    if (r < R) {
      int b = p.off[r], e = p.off[r + 1];
      if (!(sh_status & TAPER_STATUS_BAD_LENGTH)) {
        for (int s = b; s < e; ++s)
          if (p.slot_admitted[s]) {
            w += 1;
            nl += local_items(p, s);
          }
        if (w > 0 && p.Lsh[r] > 0) nc = chunk_plan(p.Lsh[r], p.h_local, R).n;
      }
      p.req_width[r] = w;
    }
    const int groups = (w + kMaxItemBranches - 1) / kMaxItemBranches;
    w_loc[k] = w; nc_loc[k] = nc * groups; nl_loc[k] = nl; cs_loc[k] = w * nc + nl;
  }
  int tot_w = block_exscan4<int>(w_loc, scan_i);
  int tot_nc = block_exscan4<int>(nc_loc, scan_i);
  int tot_nl = block_exscan4<int>(nl_loc, scan_i);
  int tot_cs = block_exscan4<int>(cs_loc, scan_i);
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    int r = tid * kPerThread + k;
    if (r < R) {
      p.req_adm_off[r] = w_loc[k];
      p.req_chunk_off[r] = nc_loc[k];
      p.req_loc_off[r] = nl_loc[k];
      p.req_part_off[r] = cs_loc[k];
    }
  }
  if (tid == 0) {
    p.req_adm_off[R] = tot_w;
    p.req_chunk_off[R] = tot_nc;
    p.req_loc_off[R] = tot_nl;
    p.req_part_off[R] = tot_cs;
  }
  __syncthreads();
  // admitted slots of each request in ascending slot order; rank j of each slot
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    int r = tid * kPerThread + k;
    if (r < R && !(sh_status & TAPER_STATUS_BAD_LENGTH)) {
      int j = 0, base = w_loc[k];
      for (int s = p.off[r]; s < p.off[r + 1]; ++s) {
        if (p.slot_admitted[s]) {
          p.adm_by_req[base + j] = s; p.slot_rank[s] = j; ++j;
          // softmax over an empty context is undefined [C-att-4]: flagged, zero output
          if (p.Lsh[r] == 0 && p.Lloc[s] == 0) atomicOr(&sh_status, TAPER_STATUS_EMPTY_CONTEXT);
        } else {
          p.slot_rank[s] = -2;
        }
      }
    }
  }
  __syncthreads();
  // item and local-tile descriptors (A5): one request per thread
  const bool fits = (long long)tot_cs <= p.cap_cs;
  // (strided over the block: requests are independent here, and a latency-bound chain
  // per thread is shorter when every thread takes at most ceil(R / 1024) requests)
  for (int r = tid; r < R; r += blockDim.x) {
    if (!fits || (sh_status & TAPER_STATUS_BAD_LENGTH)) continue;
    const int w = p.req_adm_off[r + 1] - p.req_adm_off[r];
    if (w == 0) continue;
    const int adm_off = p.req_adm_off[r];
    const int nsh = p.req_chunk_off[r + 1] - p.req_chunk_off[r];  // shared items
    const int groups = (w + kMaxItemBranches - 1) / kMaxItemBranches;
    const int nc = nsh / groups;
    const int cs_r = p.req_part_off[r];
    const int it0 = p.req_chunk_off[r] + p.req_loc_off[r];  // request-major item numbering
    const ChunkPlan cp = chunk_plan(p.Lsh[r], p.h_local, R);
    const int n_ready = p.off[r + 1] - p.off[r];  // the item mode depends on n_r, not on w_r
    for (int c = 0; c < nc; ++c)
      for (int g = 0; g < groups; ++g) {
        ItemDesc d;
        d.r = r;
        d.w = min(kMaxItemBranches, w - g * kMaxItemBranches);
        d.adm_off = adm_off + g * kMaxItemBranches;
        d.cs0 = cs_r + c * w + g * kMaxItemBranches;
        d.tb = chunk_start(cp, p.Lsh[r], c); d.te = chunk_start(cp, p.Lsh[r], c + 1);
        d.nt = (d.te - d.tb + kTileTokens - 1) / kTileTokens;
        d.flags = (kRowEnabled && n_ready >= kRowMin) ? (kItemRow | (n_ready > 8 ? kItemM128 : 0)) : 0;
        p.items[it0 + c * groups + g] = d;
      }
    // local items: per admitted branch, its local tiles in groups of kLocalItemTiles
    const int l0 = p.req_loc_off[r];
    int li = 0;
    for (int j = 0; j < w; ++j) {
      const int s = p.adm_by_req[adm_off + j];
      p.slot_lbase[s] = li;  // local items of the request's branches before j
      const int nseg = p.seg_off ? p.seg_off[s + 1] - p.seg_off[s] : 1;
      for (int qs = 0; qs < nseg; ++qs) {
        const int seg = p.seg_off ? p.seg_off[s] + qs : -1;  // -1: the slot's page list
        const int L = p.seg_off ? p.seg_len[seg] : p.Lloc[s];
        for (int t0 = 0; t0 < L; t0 += kTileTokens * kLocalItemTiles, ++li) {
          const int nt = min(kLocalItemTiles, (L - t0 + kTileTokens - 1) / kTileTokens);
          for (int t = 0; t < nt; ++t) {
            const int tok = t0 + t * kTileTokens;
            p.ltiles[(size_t)(l0 + li) * kLocalItemTiles + t] =
                make_int4(s, tok, min(kTileTokens, L - tok), seg);
          }
          ItemDesc d;
          d.r = r; d.w = 1; d.adm_off = adm_off + j; d.cs0 = cs_r + nc * w + li;
          d.tb = (l0 + li) * kLocalItemTiles; d.te = 0;
          d.nt = nt;
          d.flags = kItemLocal;
          p.items[it0 + nsh + li] = d;
        }
      }
    }
  }
  for (int i = tid; i < 2 * R * kGroup; i += blockDim.x) p.done[i] = 0;
  // adm_list: ascending slot index
  int f[kPerThread];
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    int s = tid * kPerThread + k;
    f[k] = (s < S && !(sh_status & TAPER_STATUS_BAD_LENGTH)) ? p.slot_admitted[s] : 0;
  }
  int fl[kPerThread];
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) fl[k] = f[k];
  int n_adm = block_exscan4<int>(fl, scan_i);
#pragma unroll
  for (int k = 0; k < kPerThread; ++k) {
    int s = tid * kPerThread + k;
    if (s < S && f[k]) {
      p.adm_list[fl[k]] = s;
      // merge descriptor: the slot's shared partials (stride w) and its own local items'
      const int r = p.slot_req[s], j = p.slot_rank[s];
      const int w = p.req_adm_off[r + 1] - p.req_adm_off[r];
      const int groups = (w + kMaxItemBranches - 1) / kMaxItemBranches;
      const int nc = (p.req_chunk_off[r + 1] - p.req_chunk_off[r]) / groups;
      const int n_items = (p.req_chunk_off[r + 1] - p.req_chunk_off[r]) +
                          (p.req_loc_off[r + 1] - p.req_loc_off[r]);
      const int lpre = p.slot_lbase[s];
      const int nl = local_items(p, s);
      const int cs_r = p.req_part_off[r];
      p.merge_desc[2 * fl[k]] = make_int4(s, cs_r + j, nc, w);
      p.merge_desc[2 * fl[k] + 1] = make_int4(cs_r + nc * w + lpre, nl, r, n_items);
    }
  }
  // claim order (longest processing time first): the dynamic scheduler of attend_kernel
  // hands out items in this order, so the last claims are the shortest and the CTAs finish
  // together.  Cost ~ tiles x (2, or 3 for > 4 stacked branches: their softmax is ~1.4x a
  // narrow tile's); ties keep request-major order.  More than 4096 items: as emitted.
  {
    const int D = ((long long)tot_cs <= p.cap_cs && !(sh_status & TAPER_STATUS_BAD_LENGTH)) ? tot_nc + tot_nl : 0;
    if (D <= kMaxSlots) {
      int n_keys = 1;
      while (n_keys < D) n_keys <<= 1;
      for (int i = tid; i < n_keys; i += blockDim.x) {
        unsigned long long key = ~0ull;
        if (i < D) {
          const ItemDesc d = p.items[i];
          // (with > 16 admitted branches the groups of one prefix chunk share the cost of
          // the widest, so they stay adjacent: the later group re-reads the chunk from L2)
          const int wr = (d.flags & kItemLocal) ? d.w : p.req_adm_off[d.r + 1] - p.req_adm_off[d.r];
          const int per_tile = (d.flags & kItemRow) ? kRowCost
                                                    : (min(wr, kMaxItemBranches) > 4 ? kWideCost : kNarrowCost);
          const int cost = d.nt * per_tile + kItemCost0;
          key = ((unsigned long long)(0xffff - cost) << 32) | (unsigned)i;
        }
        keys[i] = key;
      }
      __syncthreads();
      bitonic_sort(keys, n_keys);
      for (int i = tid; i < D; i += blockDim.x) p.sorted[i] = p.items[int(keys[i] & 0xffffffffu)];
    } else {
      for (int i = tid; i < D; i += blockDim.x) p.sorted[i] = p.items[i];
    }
  }
  __syncthreads();  // every table above is written before the header below
  if (tid == 0) {
    int st = sh_status;
    int n_rc = tot_nc, n_rl = tot_nl;
    if ((long long)tot_cs > p.cap_cs) { st |= TAPER_STATUS_WORK_OVERFLOW; n_rc = 0; n_rl = 0; n_adm = 0; }
    if (st & TAPER_STATUS_BAD_LENGTH) { n_rc = 0; n_rl = 0; n_adm = 0; }
    p.hdr[0] = n_rc;
    p.hdr[5] = n_rl;
    p.hdr[1] = tot_cs;
    p.hdr[2] = n_adm;
    p.hdr[3] = int(p.cap_cs > 0x7fffffff ? 0x7fffffff : p.cap_cs);
    p.hdr[4] = p.h_local;
    p.hdr[8] = 0;  // dynamic work counter of the next attend_kernel
    p.hdr[11] = 0;  // merge CTAs done (fused gather), re-armed by every gathered merge
    p.hdr[9] = 0;  // attend CTAs exited
    *p.n_adm = n_adm;
    *p.status = st;  // the caller owns the word for this step (admit and build_work alike)
  }
}

}  // namespace taper

// ---------------------------------------------------------------------- host side
#include "host_common.h"

using namespace taper;

static int launch_admit(const taper_batch *batch, const taper_latency_model *model,
                        const taper_policy *policy, const taper_admission *out, int32_t h_local,
                        void *ws, size_t ws_bytes, void *stream, int decide) {
  if (!batch || !out || !ws) return fail(TAPER_ERR_ARG, "null batch/admission/workspace");
  const int R = batch->n_req, S = batch->n_slot;
  if (R < 0 || S < 0) return fail(TAPER_ERR_ARG, "negative n_req/n_slot");
  if (R > kMaxSlots || S > kMaxSlots) return fail(TAPER_ERR_CAPACITY, "R or S exceeds TAPER_MAX_SLOTS");
  if (h_local < 1 || h_local > 8) return fail(TAPER_ERR_ARG, "h_local must be in [1, 8]");
  if (!batch->req_slot_off || (R > 0 && !batch->req_shared_len) ||
      (S > 0 && !batch->slot_local_len) || (decide && R > 0 && !batch->req_slack_ms))
    return fail(TAPER_ERR_ARG, "null batch array");
  if ((R > 0 && !out->req_width) || (S > 0 && (!out->slot_admitted || !out->adm_list)) ||
      !out->n_adm || !out->status || (decide && !out->diag))
    return fail(TAPER_ERR_ARG, "null admission output");
  AdmitParams p{};
  if (decide) {
    if (!model || !policy) return fail(TAPER_ERR_ARG, "null model/policy");
    if (!(policy->rho > 0.0 && policy->rho <= 1.0)) return fail(TAPER_ERR_RHO, "rho must be in (0, 1]");
    if (!(model->b > 0.0 && model->c > 0.0 && model->a >= 0.0))
      return fail(TAPER_ERR_NONMONOTONE, "latency model needs a >= 0, b > 0, c > 0");
    if (policy->kind < TAPER_POLICY_OFF || policy->kind > TAPER_POLICY_GREEDY)
      return fail(TAPER_ERR_ARG, "unknown policy kind");
    if (policy->kind == TAPER_POLICY_CAP && policy->cap < 1) return fail(TAPER_ERR_ARG, "cap must be >= 1");
    if (policy->utility && policy->utility_stride < 2)
      return fail(TAPER_ERR_ARG, "utility_stride must be >= 2 when a utility table is given");
    // the utility curve matters to Alg. 1 only; the fixed policies ignore it (App. D)
    if (policy->kind == TAPER_POLICY_GREEDY && policy->utility) {
      p.util = policy->utility;
      p.ustride = policy->utility_stride;
    }
    p.a = model->a; p.b = model->b; p.c = model->c; p.rho = policy->rho;
    p.kind = policy->kind; p.cap = policy->cap;
    if (policy->ctx_counting != TAPER_CTX_PER_SEQUENCE && policy->ctx_counting != TAPER_CTX_PER_REQUEST)
      return fail(TAPER_ERR_ARG, "ctx_counting must be TAPER_CTX_PER_SEQUENCE or _PER_REQUEST");
    p.ctx_per_request = policy->ctx_counting == TAPER_CTX_PER_REQUEST;
  }
  WsLayout L = ws_layout(R, S);
  if (ws_bytes < L.fixed) return fail(TAPER_ERR_CAPACITY, "workspace smaller than the fixed part");
  char *w = static_cast<char *>(ws);
  p.R = R; p.S = S;
  p.Lsh = batch->req_shared_len; p.off = batch->req_slot_off; p.Lloc = batch->slot_local_len;
  p.seg_off = batch->slot_seg_off; p.seg_len = batch->seg_len;
  if (p.seg_off && !p.seg_len) return fail(TAPER_ERR_ARG, "slot_seg_off without seg_len");
  p.slack = batch->req_slack_ms;
  p.decide = decide;
  p.req_width = out->req_width; p.slot_admitted = out->slot_admitted;
  p.adm_list = out->adm_list; p.n_adm = out->n_adm; p.diag = out->diag; p.status = out->status;
  p.hdr = reinterpret_cast<int32_t *>(w + L.hdr);
  p.slot_req = reinterpret_cast<int32_t *>(w + L.slot_req);
  p.slot_rank = reinterpret_cast<int32_t *>(w + L.slot_rank);
  p.slot_lbase = reinterpret_cast<int32_t *>(w + L.slot_lbase);
  p.req_chunk_off = reinterpret_cast<int32_t *>(w + L.req_chunk_off);
  p.req_part_off = reinterpret_cast<int32_t *>(w + L.req_part_off);
  p.req_loc_off = reinterpret_cast<int32_t *>(w + L.req_loc_off);
  p.req_adm_off = reinterpret_cast<int32_t *>(w + L.req_adm_off);
  p.adm_by_req = reinterpret_cast<int32_t *>(w + L.adm_by_req);
  p.merge_desc = reinterpret_cast<int4 *>(w + L.merge_desc);
  p.done = reinterpret_cast<int32_t *>(w + L.done);
  WsTables T = ws_tables(ws_bytes, R, S, h_local);
  p.cap_cs = T.cap_cs;
  p.items = reinterpret_cast<ItemDesc *>(w + T.items);
  p.ltiles = reinterpret_cast<int4 *>(w + T.ltiles);
  p.sorted = reinterpret_cast<ItemDesc *>(w + T.sorted);
  p.h_local = h_local;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (S > 0) {
    cudaError_t e = cudaMemsetAsync(p.slot_req, 0xff, sizeof(int32_t) * S, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(p.slot_rank, 0, sizeof(int32_t) * S, st);
    if (e != cudaSuccess) return fail_cuda(e, "memset workspace");
  }
  admit_kernel<<<1, kAdmitThreads, 0, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "admit_kernel launch");
  set_launches(1);
  return TAPER_OK;
}

extern "C" int taper_admit(const taper_batch *batch, const taper_latency_model *model,
                           const taper_policy *policy, const taper_admission *out,
                           int32_t h_local, void *workspace, size_t workspace_bytes,
                           void *stream) {
  return launch_admit(batch, model, policy, out, h_local, workspace, workspace_bytes, stream, 1);
}

extern "C" int taper_build_work(const taper_batch *batch, const taper_admission *adm,
                                int32_t h_local, void *workspace, size_t workspace_bytes,
                                void *stream) {
  return launch_admit(batch, nullptr, nullptr, adm, h_local, workspace, workspace_bytes, stream, 0);
}
