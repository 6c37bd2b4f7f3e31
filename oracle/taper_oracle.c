/*
 * oracle/taper_oracle.c -- fp64 CPU ORACLE for the TAPER hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2605_06914_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * It is plain, slow and written to be checked against PAPER.md by eye:
 *
 *   oracle_T            App. C.1 display eq.:
 *                         T(S) = a + b*n_tokens + c*L_context
 *   oracle_admit        Sec. 3.3 (L126-140) protected composition S0 and slack
 *                       budget, then Algorithm 1 "TAPER Per-Step Planner"
 *                       (L147-181) executed LITERALLY (greedy loop with
 *                       pruning), plus the fixed policies IRP-Off / IRP-Ck /
 *                       IRP-Eager of App. D "Baselines" (L391-400).
 *   oracle_bruteforce   App. B "Width allocation problem" (L290-296): maximise
 *                       sum_r u_r(k_r) s.t. T(S(k)) <= T_max over EVERY subset
 *                       of opportunistic branches (tiny instances only).
 *   oracle_attention    Sec. 3.1 visibility rule (L100-103): a branch token
 *                       attends to P (+) H (+) h_i (+) y_{i,<t}.  Plain
 *                       softmax attention in fp64 over the fully materialised
 *                       per-branch context [shared prefix ; branch-local]
 *                       (prefix duplicated per branch), one (slot, q-head) at
 *                       a time.  oracle_attention_seg: the local context may be
 *                       several segments (reduce step, L104-107).
 *
 * Readings of the paper where it is silent are listed in DESIGN.md
 * ("Readings"); the ones used here are tagged [C-adm-n] / [C-att-n].
 * Compile with -ffp-contract=off: every fp64 operation below is rounded
 * separately, in the order written ([C-adm-5]).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_STATUS_EMPTY_REQUEST 1 /* a request had no ready slot [C-adm-11] */
#define ORACLE_ERR_ARG (-1)
#define ORACLE_ERR_TOO_LARGE (-2)

#define POLICY_OFF 0
#define POLICY_CAP 1
#define POLICY_EAGER 2
#define POLICY_GREEDY 3

/* Algorithm 1 line 16 writes EPS without a value [C-adm-3]. */
static const double ORACLE_EPS = 1e-9;

/* ---------------------------------------------------------------------- */
/* App. C.1: T(S) = a + b*n_tokens + c*L_context (L316).                    */
double oracle_T(double a, double b, double c, int64_t n, int64_t L) {
  double fixed_plus_ffn = a + b * (double)n;
  return fixed_plus_ffn + c * (double)L;
}

/* Sec. 3.3 (L131-137): B_t = max(0, min_r(d_r(t)-t) - T0); the widened step
 * is admitted iff T(S) <= T0 + rho * B_t.  Returns the right-hand side. */
double oracle_budget(double T0, double min_slack, double rho) {
  double residual = min_slack - T0;
  double B = residual > 0.0 ? residual : 0.0;
  return T0 + rho * B;
}

/* Canonical order of a request's ready slots [C-adm-1, C-adm-2]: ascending
 * branch-local length, ties by ascending slot index.  Insertion sort. */
static void canonical_order(const int32_t *Lloc, int32_t begin, int32_t end,
                            int32_t *order /* [end-begin] */) {
  int32_t n = end - begin;
  for (int32_t i = 0; i < n; ++i) order[i] = begin + i;
  for (int32_t i = 1; i < n; ++i) {
    int32_t s = order[i];
    int32_t j = i - 1;
    while (j >= 0 && (Lloc[order[j]] > Lloc[s] ||
                      (Lloc[order[j]] == Lloc[s] && order[j] > s))) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = s;
  }
}

/* Utility u_r(k).  util == NULL means the paper's default linear utility
 * u_r(k) = k (App. D "TAPER configuration", L391).  Otherwise util[r*ustride+k]
 * holds u_r(k) for k in [0, ustride); beyond the table u is flat. */
static double utility(const double *util, int32_t ustride, int32_t r, int32_t k) {
  if (util == NULL) return (double)k;
  if (k >= ustride) k = ustride - 1;
  return util[(int64_t)r * ustride + k];
}

/*
 * oracle_admit: one TAPER step.
 *   batch (host arrays): R requests; ready slots of r are [off[r], off[r+1]);
 *   Lsh[r] = shared-segment length (serial request: whole context);
 *   Lloc[s] = branch-local length of slot s; slack[r] = d_r(t) - t in ms.
 *   Each admitted slot of r contributes Lsh[r] + Lloc[s] context tokens
 *   (per-sequence counting, L318 "their aggregate context length" [C-adm-6]);
 *   oracle_admit_ctx with ctx_per_request = 1 counts r's prefix once: its first
 *   (protected) slot adds Lsh[r] + Lloc[s], every further slot only Lloc[s] (the
 *   bytes a cascade kernel reads, reading R-ctx).
 * Outputs: req_width[r] = w_{r,t} (0 for a request with no ready slot),
 *   slot_admitted[s] in {0,1}, diag = {T0, budget, T(S), E = T(S)-T0, min_slack},
 *   *n_evals = number of T() evaluations performed by the greedy loop.
 * Returns ORACLE_OK, ORACLE_STATUS_EMPTY_REQUEST, or a negative error.
 */
int oracle_admit_ctx(int32_t R, int32_t S, const int32_t *Lsh, const int32_t *off,
                     const double *slack, const int32_t *Lloc, double a, double b,
                     double c, int32_t kind, int32_t cap, double rho,
                     const double *util, int32_t ustride, int32_t ctx_per_request,
                     int32_t *req_width, uint8_t *slot_admitted, double *diag,
                     int64_t *n_evals) {
  if (R < 0 || S < 0 || off[0] != 0 || off[R] != S) return ORACLE_ERR_ARG;
  int status = ORACLE_OK;
  int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
  int32_t *granted = (int32_t *)calloc((size_t)(R > 0 ? R : 1), sizeof(int32_t));
  uint8_t *cand = (uint8_t *)calloc((size_t)(R > 0 ? R : 1), 1);
  uint8_t *infeasible = (uint8_t *)calloc((size_t)(R > 0 ? R : 1), 1);
  for (int32_t s = 0; s < S; ++s) slot_admitted[s] = 0;
  int64_t evals = 0;

  /* BuildBaseline (Alg. 1 line 2; Sec. 3.3): every active request
   * advances exactly one token; the protected slot is the first ready slot
   * in canonical order. */
  int64_t n = 0, L = 0;
  double min_slack = INFINITY;
  for (int32_t r = 0; r < R; ++r) {
    req_width[r] = 0;
    if (off[r + 1] <= off[r]) { status = ORACLE_STATUS_EMPTY_REQUEST; continue; }
    canonical_order(Lloc, off[r], off[r + 1], order + off[r]);
    int32_t prot = order[off[r]];
    slot_admitted[prot] = 1;
    req_width[r] = 1;
    n += 1;
    L += (int64_t)Lsh[r] + (int64_t)Lloc[prot];
    /* Alg. 1 line 3: min over requests of d_r - now. */
    if (slack[r] < min_slack) min_slack = slack[r];
  }
  double T0 = oracle_T(a, b, c, n, L);
  /* Alg. 1 line 4.  With no active request the residual is defined as 0. */
  double budget = (n > 0) ? oracle_budget(T0, min_slack, rho) : T0;

  if (kind == POLICY_CAP || kind == POLICY_EAGER) {
    /* App. D: IRP-Ck w = min(n_r, k); IRP-Eager w = n_r [C-adm-9]. */
    for (int32_t r = 0; r < R; ++r) {
      int32_t nr = off[r + 1] - off[r];
      if (nr <= 0) continue;
      int32_t w = (kind == POLICY_EAGER) ? nr : (nr < cap ? nr : cap);
      for (int32_t p = 1; p < w; ++p) {
        int32_t s = order[off[r] + p];
        slot_admitted[s] = 1;
        n += 1;
        L += (ctx_per_request ? 0 : (int64_t)Lsh[r]) + (int64_t)Lloc[s];
      }
      req_width[r] = w;
    }
  } else if (kind == POLICY_GREEDY) {
    /* Alg. 1 lines 5-6: granted = 0; candidates = requests with ready
     * (opportunistic) branches [C-adm-8]. */
    int32_t n_cand = 0;
    for (int32_t r = 0; r < R; ++r) {
      cand[r] = (off[r + 1] - off[r]) > 1;
      n_cand += cand[r];
    }
    /* Alg. 1 line 8: while candidates. */
    while (n_cand > 0) {
      int32_t best = -1;
      double best_score = 0.0;
      int64_t best_dL = 0;
      /* Alg. 1 line 10: for r in candidates (ascending r [C-adm-4]). */
      for (int32_t r = 0; r < R; ++r) {
        if (!cand[r]) continue;
        /* AddBranch(step, r): r's next ready branch in canonical order. */
        int32_t s = order[off[r] + 1 + granted[r]];
        int64_t dL = (ctx_per_request ? 0 : (int64_t)Lsh[r]) + (int64_t)Lloc[s];
        double T_widened = oracle_T(a, b, c, n + 1, L + dL);
        evals += 1;
        /* Alg. 1 lines 12-14: monotone: prune request r. */
        if (T_widened > budget) { infeasible[r] = 1; continue; }
        /* Alg. 1 lines 15-17. */
        double du = utility(util, ustride, r, granted[r] + 1) -
                    utility(util, ustride, r, granted[r]);
        double T_step = oracle_T(a, b, c, n, L);
        evals += 1;
        double dt = T_widened - T_step;
        double score = du / (ORACLE_EPS + (dt > 0.0 ? dt : 0.0));
        /* Alg. 1 lines 18-19: strict '>' keeps the lowest r on ties. */
        if (best < 0 || score > best_score) {
          best = r;
          best_score = score;
          best_dL = dL;
        }
      }
      /* Alg. 1 line 20: candidates -= infeasible. */
      for (int32_t r = 0; r < R; ++r)
        if (infeasible[r]) { if (cand[r]) { cand[r] = 0; --n_cand; } infeasible[r] = 0; }
      /* Alg. 1 lines 21-22. */
      if (best < 0 || best_score <= 0.0) break;
      /* Alg. 1 lines 23-26: commit the best candidate. */
      int32_t s = order[off[best] + 1 + granted[best]];
      slot_admitted[s] = 1;
      n += 1;
      L += best_dL;
      granted[best] += 1;
      req_width[best] += 1;
      if (granted[best] >= (off[best + 1] - off[best]) - 1 && cand[best]) {
        cand[best] = 0;
        --n_cand;
      }
    }
  } else if (kind != POLICY_OFF) {
    status = ORACLE_ERR_ARG;
  }

  double TS = oracle_T(a, b, c, n, L);
  diag[0] = T0;
  diag[1] = budget;
  diag[2] = TS;
  diag[3] = TS - T0; /* Sec. 2.3 branch externality E_t(k) = T(S(k)) - T(S0). */
  diag[4] = min_slack;
  if (n_evals) *n_evals = evals;
  free(order);
  free(granted);
  free(cand);
  free(infeasible);
  return status;
}

int oracle_admit(int32_t R, int32_t S, const int32_t *Lsh, const int32_t *off,
                 const double *slack, const int32_t *Lloc, double a, double b,
                 double c, int32_t kind, int32_t cap, double rho,
                 const double *util, int32_t ustride, int32_t *req_width,
                 uint8_t *slot_admitted, double *diag, int64_t *n_evals) {
  return oracle_admit_ctx(R, S, Lsh, off, slack, Lloc, a, b, c, kind, cap, rho, util, ustride,
                          0, req_width, slot_admitted, diag, n_evals);
}

/*
 * oracle_bruteforce: App. B width-allocation problem on a tiny batch.
 * Enumerates every subset of the opportunistic slots (all ready slots except
 * each request's protected one), keeps those with T(S) <= budget (the same
 * budget oracle_admit computes), and maximises sum_r u_r(k_r).
 * best_mask receives the lexicographically-first optimal subset as a bitmask
 * over opportunistic slots listed in ascending slot index; *n_opp their count.
 */
int oracle_bruteforce_ctx(int32_t R, int32_t S, const int32_t *Lsh, const int32_t *off,
                          const double *slack, const int32_t *Lloc, double a, double b,
                          double c, double rho, const double *util, int32_t ustride,
                          int32_t ctx_per_request, double *best_utility, int64_t *best_mask,
                          int32_t *n_opp_out, double *budget_out) {
  if (R < 0 || S < 0 || off[0] != 0 || off[R] != S) return ORACLE_ERR_ARG;
  int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
  int32_t opp_slot[24], opp_req[24];
  int32_t n_opp = 0;
  int64_t n0 = 0, L0 = 0;
  double min_slack = INFINITY;
  uint8_t *is_prot = (uint8_t *)calloc((size_t)(S > 0 ? S : 1), 1);
  for (int32_t r = 0; r < R; ++r) {
    if (off[r + 1] <= off[r]) continue;
    canonical_order(Lloc, off[r], off[r + 1], order + off[r]);
    int32_t prot = order[off[r]];
    is_prot[prot] = 1;
    n0 += 1;
    L0 += (int64_t)Lsh[r] + (int64_t)Lloc[prot];
    if (slack[r] < min_slack) min_slack = slack[r];
  }
  for (int32_t r = 0; r < R; ++r)
    for (int32_t s = off[r]; s < off[r + 1]; ++s)
      if (!is_prot[s]) {
        if (n_opp >= 24) { free(order); free(is_prot); return ORACLE_ERR_TOO_LARGE; }
        opp_slot[n_opp] = s;
        opp_req[n_opp] = r;
        ++n_opp;
      }
  double T0 = oracle_T(a, b, c, n0, L0);
  double budget = (n0 > 0) ? oracle_budget(T0, min_slack, rho) : T0;
  int32_t *k = (int32_t *)calloc((size_t)(R > 0 ? R : 1), sizeof(int32_t));
  double best = -INFINITY;
  int64_t best_m = 0;
  for (int64_t mask = 0; mask < ((int64_t)1 << n_opp); ++mask) {
    int64_t n = n0, L = L0;
    for (int32_t r = 0; r < R; ++r) k[r] = 0;
    for (int32_t i = 0; i < n_opp; ++i)
      if (mask & ((int64_t)1 << i)) {
        n += 1;
        L += (ctx_per_request ? 0 : (int64_t)Lsh[opp_req[i]]) + (int64_t)Lloc[opp_slot[i]];
        k[opp_req[i]] += 1;
      }
    if (oracle_T(a, b, c, n, L) > budget) continue;
    double u = 0.0;
    for (int32_t r = 0; r < R; ++r) u += utility(util, ustride, r, k[r]);
    if (u > best) { best = u; best_m = mask; }
  }
  *best_utility = best;
  *best_mask = best_m;
  *n_opp_out = n_opp;
  if (budget_out) *budget_out = budget;
  free(order);
  free(is_prot);
  free(k);
  return ORACLE_OK;
}

int oracle_bruteforce(int32_t R, int32_t S, const int32_t *Lsh, const int32_t *off,
                      const double *slack, const int32_t *Lloc, double a, double b,
                      double c, double rho, const double *util, int32_t ustride,
                      double *best_utility, int64_t *best_mask, int32_t *n_opp_out,
                      double *budget_out) {
  return oracle_bruteforce_ctx(R, S, Lsh, off, slack, Lloc, a, b, c, rho, util, ustride, 0,
                               best_utility, best_mask, n_opp_out, budget_out);
}

/* bf16 bit pattern -> exact fp64 value. */
static double bf16_to_double(uint16_t h) {
  uint32_t bits = (uint32_t)h << 16;
  float f;
  memcpy(&f, &bits, sizeof f);
  return (double)f;
}

/*
 * oracle_attention_seg: plain fp64 softmax attention for selected (slot, q-head)
 * pairs.  KV pages: [num_pages][h_kv][page_size][d] bf16 (bit patterns).
 * Token t of a segment with page list P lives in page P[t / page_size] at
 * row t % page_size.  Slot s of request r sees the concatenation
 *     K = [K_shared(r) tokens 0..Lsh[r]-1 ; K_local(s) tokens 0..Lloc[s]-1]
 * (visibility rule, Sec. 3.1; current token already appended
 * [C-att-3]).  The local context is one segment (page list slot_pages from
 * slot_page_off[s]) or, when slot_seg_off != NULL, the segments
 * slot_seg_off[s] .. slot_seg_off[s+1]-1 in order, segment q holding seg_len[q]
 * tokens in the page list slot_pages from seg_page_off[q] -- the reduce-step
 * context P (+) H (+) h_1 (+) y_1 (+) ... (+) z of Sec. 3.1 (L104-107).
 * Q head hq reads KV head hq / (q_heads / h_kv) [C-att-2].
 *   x_j = scale * q . k_j ;  p = softmax(x) ;  o = sum_j p_j v_j
 *   lse = log(sum_j exp(x_j))   (natural log)
 * q: [S][q_heads][d] bf16 bits.  out: [n_eval][d], lse: [n_eval].
 */
static int attention_pair(int32_t e, int32_t R, const int32_t *off, int32_t h_kv,
                          int32_t q_heads, int32_t d, int32_t page_size, int32_t group,
                          const uint16_t *k_pages, const uint16_t *v_pages, const int32_t *Lsh,
                          const int32_t *req_page_off, const int32_t *req_pages,
                          const int32_t *Lloc, const int32_t *slot_page_off,
                          const int32_t *slot_pages, const int32_t *slot_seg_off,
                          const int32_t *seg_len, const int32_t *seg_page_off,
                          const uint16_t *q, const int32_t *eval_slot,
                          const int32_t *eval_qhead, double scale, double *out, double *lse);
static inline int min_status(int a, int b) { return a < b ? a : b; }

int oracle_attention_seg(int32_t R, const int32_t *off, int32_t h_kv, int32_t q_heads,
                         int32_t d, int32_t page_size, const uint16_t *k_pages,
                         const uint16_t *v_pages, const int32_t *Lsh,
                         const int32_t *req_page_off, const int32_t *req_pages,
                         const int32_t *Lloc, const int32_t *slot_page_off,
                         const int32_t *slot_pages, const int32_t *slot_seg_off,
                         const int32_t *seg_len, const int32_t *seg_page_off,
                         const uint16_t *q, int32_t n_eval, const int32_t *eval_slot,
                         const int32_t *eval_qhead, double scale, double *out, double *lse) {
  if (h_kv <= 0 || q_heads % h_kv != 0 || d <= 0 || page_size <= 0) return ORACLE_ERR_ARG;
  int32_t group = q_heads / h_kv;
  int status = ORACLE_OK;
  /* The (slot, q-head) pairs are independent: with OpenMP (oracle_set_threads) they are
   * spread over the host cores; each pair's arithmetic below is the same either way. */
#pragma omp parallel for schedule(dynamic, 1) reduction(min : status)
  for (int32_t e = 0; e < n_eval; ++e)
    status = min_status(status, attention_pair(e, R, off, h_kv, q_heads, d, page_size, group,
                                               k_pages, v_pages, Lsh, req_page_off, req_pages,
                                               Lloc, slot_page_off, slot_pages, slot_seg_off,
                                               seg_len, seg_page_off, q, eval_slot, eval_qhead,
                                               scale, out, lse));
  return status;
}

/* One (slot, q-head) pair of oracle_attention_seg. */
static int attention_pair(int32_t e, int32_t R, const int32_t *off, int32_t h_kv,
                          int32_t q_heads, int32_t d, int32_t page_size, int32_t group,
                          const uint16_t *k_pages, const uint16_t *v_pages, const int32_t *Lsh,
                          const int32_t *req_page_off, const int32_t *req_pages,
                          const int32_t *Lloc, const int32_t *slot_page_off,
                          const int32_t *slot_pages, const int32_t *slot_seg_off,
                          const int32_t *seg_len, const int32_t *seg_page_off,
                          const uint16_t *q, const int32_t *eval_slot,
                          const int32_t *eval_qhead, double scale, double *out, double *lse) {
  (void)h_kv;
  {
    int32_t s = eval_slot[e];
    int32_t hq = eval_qhead[e];
    int32_t g = hq / group;
    /* request owning slot s: off[r] <= s < off[r+1] */
    int32_t r = -1;
    for (int32_t i = 0; i < R; ++i)
      if (off[i] <= s && s < off[i + 1]) { r = i; break; }
    if (r < 0) return ORACLE_ERR_ARG;
    int64_t n_sh = Lsh[r], n_loc = Lloc[s], n_tok = n_sh + n_loc;
    if (n_tok < 1) return ORACLE_ERR_ARG; /* [C-att-4] */
    if (slot_seg_off) { /* the segments must make up the local context exactly */
      int64_t sum = 0;
      for (int32_t qs = slot_seg_off[s]; qs < slot_seg_off[s + 1]; ++qs) sum += seg_len[qs];
      if (sum != n_loc) return ORACLE_ERR_ARG;
    }
    /* Materialise this branch's K and V (prefix duplicated per branch). */
    double *K = (double *)malloc(sizeof(double) * (size_t)(n_tok * d));
    double *V = (double *)malloc(sizeof(double) * (size_t)(n_tok * d));
    for (int64_t t = 0; t < n_tok; ++t) {
      int64_t page, row;
      if (t < n_sh) {
        page = req_pages[req_page_off[r] + t / page_size];
        row = t % page_size;
      } else if (!slot_seg_off) {
        int64_t u = t - n_sh;
        page = slot_pages[slot_page_off[s] + u / page_size];
        row = u % page_size;
      } else {
        /* find the local segment holding local token u */
        int64_t u = t - n_sh;
        int32_t qs = slot_seg_off[s];
        while (u >= seg_len[qs]) { u -= seg_len[qs]; ++qs; }
        page = slot_pages[seg_page_off[qs] + u / page_size];
        row = u % page_size;
      }
      int64_t base = ((page * h_kv + g) * page_size + row) * d;
      for (int32_t i = 0; i < d; ++i) {
        K[t * d + i] = bf16_to_double(k_pages[base + i]);
        V[t * d + i] = bf16_to_double(v_pages[base + i]);
      }
    }
    double *qv = (double *)malloc(sizeof(double) * (size_t)d);
    for (int32_t i = 0; i < d; ++i)
      qv[i] = bf16_to_double(q[((int64_t)s * q_heads + hq) * d + i]);
    double *x = (double *)malloc(sizeof(double) * (size_t)n_tok);
    double m = -INFINITY;
    for (int64_t t = 0; t < n_tok; ++t) {
      double dot = 0.0;
      for (int32_t i = 0; i < d; ++i) dot += qv[i] * K[t * d + i];
      x[t] = scale * dot;
      if (x[t] > m) m = x[t];
    }
    double Z = 0.0;
    for (int64_t t = 0; t < n_tok; ++t) {
      x[t] = exp(x[t] - m);
      Z += x[t];
    }
    for (int32_t i = 0; i < d; ++i) {
      double acc = 0.0;
      for (int64_t t = 0; t < n_tok; ++t) acc += x[t] * V[t * d + i];
      out[(int64_t)e * d + i] = acc / Z;
    }
    lse[e] = m + log(Z);
    free(K);
    free(V);
    free(qv);
    free(x);
  }
  return ORACLE_OK;
}

/* Host threads for oracle_attention(_seg) (1 = serial; the result does not depend on it). */
int oracle_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
  return n > 0 ? n : 1;
#else
  (void)n;
  return 1;
#endif
}

/* oracle_attention: oracle_attention_seg with one local segment per slot. */
int oracle_attention(int32_t R, const int32_t *off, int32_t h_kv, int32_t q_heads,
                     int32_t d, int32_t page_size, const uint16_t *k_pages,
                     const uint16_t *v_pages, const int32_t *Lsh,
                     const int32_t *req_page_off, const int32_t *req_pages,
                     const int32_t *Lloc, const int32_t *slot_page_off,
                     const int32_t *slot_pages, const uint16_t *q, int32_t n_eval,
                     const int32_t *eval_slot, const int32_t *eval_qhead, double scale,
                     double *out, double *lse) {
  return oracle_attention_seg(R, off, h_kv, q_heads, d, page_size, k_pages, v_pages, Lsh,
                              req_page_off, req_pages, Lloc, slot_page_off, slot_pages, NULL,
                              NULL, NULL, q, n_eval, eval_slot, eval_qhead, scale, out, lse);
}
