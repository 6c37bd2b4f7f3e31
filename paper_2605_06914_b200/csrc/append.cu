// append.cu -- write the step's new token K/V of every admitted slot into its KV pages.
//
// [C-att-3] / Sec. 3.1: the current token's K and V are part of the
// context the step attends to -- the last token of the slot's local segment (a branch, the
// last non-empty local segment when the context has several), or of its request's shared
// segment (a serial request, Lloc = 0).  One CTA per adm_list entry, one warp per local KV
// head, 16 B per lane: K row and V row (2 x 256 B) per (slot, head).
#include "host_common.h"
#include "taper_internal.cuh"

namespace taper {

struct AppendParams {
  const int32_t *Lsh, *off, *Lloc, *seg_off, *seg_len;
  const int32_t *req_page_off, *req_pages, *slot_page_off, *slot_pages, *seg_page_off;
  const int32_t *adm_list, *n_adm;
  const uint4 *k_new, *v_new;  // [S, h, 128] bf16 as 16 x 16 B per row
  uint4 *k_pages, *v_pages;    // [num_pages, h, page, 128]
  int32_t *status;
  int R, h, page_size;
};

__global__ void __launch_bounds__(256) append_kernel(AppendParams p) {
  const int i = blockIdx.x;
  if (i >= *p.n_adm) return;
  const int s = p.adm_list[i];
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (g >= p.h) return;
  int lo = 0, hi = p.R - 1;  // request owning slot s: off[r] <= s < off[r+1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.off[mid] <= s) lo = mid; else hi = mid - 1;
  }
  const int r = lo;
  int page = -1, row = 0;
  const int lloc = p.Lloc[s];
  if (lloc > 0) {
    if (p.seg_off == nullptr) {
      const int t = lloc - 1;
      page = p.slot_pages[p.slot_page_off[s] + t / p.page_size];
      row = t % p.page_size;
    } else {
      for (int q = p.seg_off[s + 1] - 1; q >= p.seg_off[s]; --q)  // last non-empty segment
        if (p.seg_len[q] > 0) {
          const int t = p.seg_len[q] - 1;
          page = p.slot_pages[p.seg_page_off[q] + t / p.page_size];
          row = t % p.page_size;
          break;
        }
    }
  } else if (p.Lsh[r] > 0) {
    const int t = p.Lsh[r] - 1;
    page = p.req_pages[p.req_page_off[r] + t / p.page_size];
    row = t % p.page_size;
  }
  if (page < 0) {  // no token to hold the current step [C-att-4]
    if (g == 0 && lane == 0) atomicOr(p.status, TAPER_STATUS_BAD_LENGTH);
    return;
  }
  if (lane < 16) {
    const size_t dst = ((size_t(page) * p.h + g) * p.page_size + row) * 16 + lane;
    const size_t src = (size_t(s) * p.h + g) * 16 + lane;
    p.k_pages[dst] = p.k_new[src];
    p.v_pages[dst] = p.v_new[src];
  }
}

}  // namespace taper

using namespace taper;

extern "C" int taper_append_kv(const taper_batch *batch, const taper_admission *adm,
                               const taper_kv *kv, const void *k_new, const void *v_new,
                               void *stream) {
  if (!batch || !adm || !kv || !k_new || !v_new) return fail(TAPER_ERR_ARG, "null argument");
  const int R = batch->n_req, S = batch->n_slot;
  if (R < 0 || S < 0) return fail(TAPER_ERR_ARG, "negative n_req/n_slot");
  if (R > kMaxSlots || S > kMaxSlots) return fail(TAPER_ERR_CAPACITY, "R or S exceeds TAPER_MAX_SLOTS");
  if (kv->h_local < 1 || kv->h_local > 8) return fail(TAPER_ERR_ARG, "h_local must be in [1, 8]");
  if (kv->page_size < 1) return fail(TAPER_ERR_ARG, "page_size must be positive");
  if (!kv->k_pages || !kv->v_pages || !kv->req_page_off || !kv->req_pages ||
      !kv->slot_page_off || !kv->slot_pages || !adm->adm_list || !adm->n_adm || !adm->status)
    return fail(TAPER_ERR_ARG, "null kv / admission array");
  if ((batch->slot_seg_off != nullptr) != (kv->seg_page_off != nullptr))
    return fail(TAPER_ERR_ARG, "batch.slot_seg_off and kv.seg_page_off must be given together");
  if ((reinterpret_cast<uintptr_t>(kv->k_pages) | reinterpret_cast<uintptr_t>(kv->v_pages) |
       reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new)) & 15)
    return fail(TAPER_ERR_ARG, "K/V pools and new K/V must be 16-byte aligned");
  if (S == 0 || R == 0) { set_launches(0); return TAPER_OK; }
  AppendParams p;
  p.Lsh = batch->req_shared_len; p.off = batch->req_slot_off; p.Lloc = batch->slot_local_len;
  p.seg_off = batch->slot_seg_off; p.seg_len = batch->seg_len;
  p.req_page_off = kv->req_page_off; p.req_pages = kv->req_pages;
  p.slot_page_off = kv->slot_page_off; p.slot_pages = kv->slot_pages;
  p.seg_page_off = kv->seg_page_off;
  p.adm_list = adm->adm_list; p.n_adm = adm->n_adm;
  p.k_new = static_cast<const uint4 *>(k_new); p.v_new = static_cast<const uint4 *>(v_new);
  p.k_pages = static_cast<uint4 *>(const_cast<void *>(kv->k_pages));
  p.v_pages = static_cast<uint4 *>(const_cast<void *>(kv->v_pages));
  p.status = adm->status;
  p.R = R; p.h = kv->h_local; p.page_size = kv->page_size;
  append_kernel<<<S, 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "append_kernel launch");
  set_launches(1);
  return TAPER_OK;
}
