// api.cu -- host helpers of the C ABI: errors, status strings, workspace sizing.
#include <cuda.h>

#include <cmath>
#include <cstring>
#include <mutex>

#include "host_common.h"
#include "taper_internal.cuh"

namespace taper {
static thread_local char g_last_error[512] = "";
static thread_local int g_launches = 0;

int fail(int code, const char *msg) {
  std::snprintf(g_last_error, sizeof g_last_error, "%s", msg);
  return code;
}
int fail_cuda(cudaError_t e, const char *what) {
  std::snprintf(g_last_error, sizeof g_last_error, "%s: %s", what, cudaGetErrorString(e));
  return TAPER_ERR_CUDA;
}
void set_launches(int n) { g_launches = n; }
void add_launches(int n) { g_launches += n; }
}  // namespace taper

extern "C" const char *taper_last_error(void) { return taper::g_last_error; }
extern "C" int taper_last_launch_count(void) { return taper::g_launches; }

extern "C" const char *taper_status_string(int code) {
  switch (code) {
    case TAPER_OK: return "ok";
    case TAPER_ERR_ARG: return "invalid argument";
    case TAPER_ERR_RHO: return "rho outside (0, 1]";
    case TAPER_ERR_NONMONOTONE: return "latency model not monotone (need a >= 0, b > 0, c > 0)";
    case TAPER_ERR_CAPACITY: return "capacity exceeded (slots, page size or workspace)";
    case TAPER_ERR_CUDA: return "CUDA error";
    case TAPER_ERR_UNSUPPORTED: return "unsupported";
    default: break;
  }
  if (code > 0) {
    static thread_local char buf[256];
    buf[0] = 0;
    if (code & TAPER_STATUS_EMPTY_REQUEST) std::strcat(buf, "empty-request ");
    if (code & TAPER_STATUS_BAD_LENGTH) std::strcat(buf, "bad-length ");
    if (code & TAPER_STATUS_PRECISION) std::strcat(buf, "fp64-precision ");
    if (code & TAPER_STATUS_WORK_OVERFLOW) std::strcat(buf, "work-overflow ");
    if (code & TAPER_STATUS_WORK_MISMATCH) std::strcat(buf, "work-mismatch ");
    if (code & TAPER_STATUS_EMPTY_CONTEXT) std::strcat(buf, "empty-context ");
    return buf;
  }
  return "unknown error";
}

extern "C" int taper_workspace_size(int32_t n_req, int32_t n_slot, int32_t h_local,
                                    int64_t max_chunk_slots, size_t *bytes) {
  if (!bytes || n_req < 0 || n_slot < 0 || max_chunk_slots < 0 || h_local < 1 || h_local > 8)
    return taper::fail(TAPER_ERR_ARG, "bad workspace_size arguments");
  if (n_req > taper::kMaxSlots || n_slot > taper::kMaxSlots)
    return taper::fail(TAPER_ERR_CAPACITY, "R or S exceeds TAPER_MAX_SLOTS");
  taper::WsLayout L = taper::ws_layout(n_req, n_slot);
  // per chunk-slot: partial rows (8 x (128 + 1) fp32 per head) + work descriptors
  size_t part = size_t(max_chunk_slots) *
                (size_t(h_local) * taper::kPartBytesPerCsHead + taper::kWorkBytesPerCs);
  *bytes = L.fixed + 1024 + part + 2048;
  return TAPER_OK;
}

// Eager bound of the partial-row count (include/taper.h): per request, its ready branches x
// prefix chunks, plus one local item per <= kLocalItemTiles tiles of each local segment.
extern "C" int taper_max_chunk_slots(int32_t n_req, int32_t n_slot, const int32_t *lsh,
                                     const int32_t *off, const int32_t *lloc,
                                     const int32_t *seg_off, const int32_t *seg_len,
                                     int32_t h_local, int64_t *out) {
  if (!out || n_req < 0 || n_slot < 0 || h_local < 1 || h_local > 8 || !off ||
      (n_req > 0 && !lsh) || (n_slot > 0 && !lloc) || (seg_off && !seg_len))
    return taper::fail(TAPER_ERR_ARG, "bad taper_max_chunk_slots arguments");
  if (off[0] != 0 || off[n_req] != n_slot)
    return taper::fail(TAPER_ERR_ARG, "req_slot_off must run from 0 to n_slot");
  constexpr int64_t per = int64_t(taper::kTileTokens) * taper::kLocalItemTiles;
  int64_t total = 0;
  for (int r = 0; r < n_req; ++r) {
    if (off[r + 1] < off[r] || lsh[r] < 0)
      return taper::fail(TAPER_ERR_ARG, "non-monotone req_slot_off or negative length");
    const int64_t ck = taper_chunk_tokens(lsh[r], h_local, n_req);
    total += int64_t(off[r + 1] - off[r]) * ((int64_t(lsh[r]) + ck - 1) / ck);
  }
  for (int s = 0; s < n_slot; ++s) {
    if (!seg_off) {
      if (lloc[s] < 0) return taper::fail(TAPER_ERR_ARG, "negative local length");
      total += (int64_t(lloc[s]) + per - 1) / per;
      continue;
    }
    if (seg_off[s + 1] < seg_off[s]) return taper::fail(TAPER_ERR_ARG, "non-monotone slot_seg_off");
    for (int q = seg_off[s]; q < seg_off[s + 1]; ++q) {
      if (seg_len[q] < 0) return taper::fail(TAPER_ERR_ARG, "negative segment length");
      total += (int64_t(seg_len[q]) + per - 1) / per;
    }
  }
  *out = total;
  return TAPER_OK;
}

// ------------------------------------------------------------------ CUDA IPC (fused gather)
typedef CUresult (*GetRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);
static GetRangeFn get_range_fn() {
  static GetRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetRangeFn>(ptr);
  });
  return fn;
}

extern "C" int taper_ipc_handle(const void *dev_ptr, void *handle, size_t *offset) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  if (!dev_ptr || !handle || !offset) return taper::fail(TAPER_ERR_ARG, "null ipc argument");
  GetRangeFn range = get_range_fn();
  if (!range) return taper::fail(TAPER_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return taper::fail(TAPER_ERR_ARG, "pointer is not device memory");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
  if (e != cudaSuccess) return taper::fail_cuda(e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, sizeof h);
  *offset = size_t(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return TAPER_OK;
}

extern "C" int taper_ipc_open(const void *handle, size_t offset, void **dev_ptr) {
  if (!handle || !dev_ptr) return taper::fail(TAPER_ERR_ARG, "null ipc argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void *base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return taper::fail_cuda(e, "cudaIpcOpenMemHandle");
  *dev_ptr = static_cast<char *>(base) + offset;
  return TAPER_OK;
}

extern "C" int taper_ipc_close(void *dev_ptr, size_t offset) {
  if (!dev_ptr) return taper::fail(TAPER_ERR_ARG, "null ipc pointer");
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(dev_ptr) - offset);
  if (e != cudaSuccess) return taper::fail_cuda(e, "cudaIpcCloseMemHandle");
  return TAPER_OK;
}

// ------------------------------------------------------------------ latency model refit
extern "C" int taper_latency_observe(taper_latency_window *w, double n, double L, double t_ms) {
  if (!w || !(n >= 0) || !(L >= 0) || !(t_ms >= 0)) return taper::fail(TAPER_ERR_ARG, "bad observation");
  if (w->count < 0 || w->count > TAPER_LATENCY_WINDOW || w->head < 0 || w->head >= TAPER_LATENCY_WINDOW)
    return taper::fail(TAPER_ERR_ARG, "corrupt latency window");
  w->n[w->head] = n;
  w->L[w->head] = L;
  w->t_ms[w->head] = t_ms;
  w->head = (w->head + 1) % TAPER_LATENCY_WINDOW;
  if (w->count < TAPER_LATENCY_WINDOW) ++w->count;
  return TAPER_OK;
}

// OLS through the normal equations X^T X beta = X^T y, X = [1, n, L], in fp64 with the
// columns centred (the intercept is recovered afterwards) so that L ~ 1e5 does not swamp
// the 3x3 system; Cramer's rule on the centred 2x2 block.
extern "C" int taper_latency_refit(const taper_latency_window *w, taper_latency_model *model,
                                   double *fit_out) {
  if (!w || !model || w->count < 0 || w->count > TAPER_LATENCY_WINDOW)
    return taper::fail(TAPER_ERR_ARG, "bad refit arguments");
  const int m = w->count;
  if (m < 3) return taper::fail(TAPER_ERR_ARG, "fewer than 3 observations");
  double mn = 0, mL = 0, mt = 0;
  for (int i = 0; i < m; ++i) { mn += w->n[i]; mL += w->L[i]; mt += w->t_ms[i]; }
  mn /= m; mL /= m; mt /= m;
  double snn = 0, sLL = 0, snL = 0, snt = 0, sLt = 0, stt = 0;
  for (int i = 0; i < m; ++i) {
    const double dn = w->n[i] - mn, dL = w->L[i] - mL, dt = w->t_ms[i] - mt;
    snn += dn * dn; sLL += dL * dL; snL += dn * dL; snt += dn * dt; sLt += dL * dt; stt += dt * dt;
  }
  const double det = snn * sLL - snL * snL;
  if (!(det > 1e-12 * snn * sLL) || snn <= 0 || sLL <= 0)
    return taper::fail(TAPER_ERR_ARG, "singular design (n and L collinear or constant)");
  const double b = (snt * sLL - sLt * snL) / det;
  const double c = (sLt * snn - snt * snL) / det;
  const double a = mt - b * mn - c * mL;
  if (!(a >= 0) || !(b > 0) || !(c > 0))
    return taper::fail(TAPER_ERR_NONMONOTONE, "refit would make T non-monotone (a < 0, b <= 0 or c <= 0)");
  if (fit_out) {
    double sse = 0, ape = 0;
    for (int i = 0; i < m; ++i) {
      const double r = w->t_ms[i] - (a + b * w->n[i] + c * w->L[i]);
      sse += r * r;
      ape += w->t_ms[i] > 0 ? std::fabs(r) / w->t_ms[i] : 0.0;
    }
    fit_out[0] = stt > 0 ? 1.0 - sse / stt : 1.0;
    fit_out[1] = ape / m;
    fit_out[2] = std::sqrt(sse / m);
  }
  model->a = a;
  model->b = b;
  model->c = c;
  return TAPER_OK;
}
