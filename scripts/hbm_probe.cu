// Dev probe: achievable HBM read bandwidth on this B200 for the attention kernel's access
// pattern -- 16 KB page tiles (64 tokens x 128 d bf16) of a paged pool, fetched with
//   (a) TMA 1-D bulk copies (cp.async.bulk) into an N-stage SMEM ring, one producer lane,
//       consumer releases immediately (no compute);
//   (b) plain 16-byte vectorised loads (ld.global.nc.v4), every thread streaming;
// over a pool larger than L2, pages visited in a random permutation.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o hbm_probe hbm_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#include <cuda.h>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(64, 1) tma_probe(const uint8_t *pool, const int *order, int n_pages,
                                                   int page_bytes, unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int chunks_per_page = page_bytes / CHUNK;
  const long long total = (long long)n_pages * chunks_per_page;
  if (warp == 0) {
    if (lane == 0) {
      int n = 0;
      for (long long c = blockIdx.x; c < total; c += gridDim.x, ++n) {
        const int st = n % STAGES;
        mbar_wait(empty + st, ((n / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(full + st, CHUNK);
        const long long page = order[c / chunks_per_page] % n_pages;
        bulk_g2s(smem + st * CHUNK, pool + page * page_bytes + (c % chunks_per_page) * CHUNK, CHUNK, full + st);
      }
    }
  } else {
    if (lane == 0) {
      unsigned long long acc = 0;
      int n = 0;
      for (long long c = blockIdx.x; c < total; c += gridDim.x, ++n) {
        const int st = n % STAGES;
        mbar_wait(full + st, (n / STAGES) & 1);
        acc += smem[st * CHUNK + (n & 127)];
        mbar_arrive(empty + st);
      }
      if (acc == 0xdeadbeef) *sink = acc;
    }
  }
}

// P producer warps in one CTA, each with its own ring and consumer warp
template <int STAGES, int CHUNK, int P>
__global__ void __launch_bounds__(64 * P, 1) tma_probe_multi(const uint8_t *pool, const int *order,
                                                             int n_pages, int page_bytes,
                                                             unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[P][STAGES], empty[P][STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pid = warp % P, role = warp / P;  // role 0 producer, 1 consumer
  if (threadIdx.x == 0) {
    for (int q = 0; q < P; ++q)
      for (int i = 0; i < STAGES; ++i) { mbar_init(&full[q][i], 1); mbar_init(&empty[q][i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int chunks_per_page = page_bytes / CHUNK;
  const long long total = (long long)n_pages * chunks_per_page;
  uint8_t *ring = smem + pid * STAGES * CHUNK;
  if (lane == 0) {
    unsigned long long acc = 0;
    int n = 0;
    for (long long c = blockIdx.x * P + pid; c < total; c += (long long)gridDim.x * P, ++n) {
      const int st = n % STAGES;
      if (role == 0) {
        mbar_wait(&empty[pid][st], ((n / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[pid][st], CHUNK);
        const long long page = order[c / chunks_per_page] % n_pages;
        bulk_g2s(ring + st * CHUNK, pool + page * page_bytes + (c % chunks_per_page) * CHUNK, CHUNK,
                 &full[pid][st]);
      } else {
        mbar_wait(&full[pid][st], (n / STAGES) & 1);
        acc += ring[st * CHUNK + (n & 127)];
        mbar_arrive(&empty[pid][st]);
      }
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

template <int STAGES, int CHUNK, int P>
void run_multi(const uint8_t *pool, const int *order, int n_pages, int page_bytes,
               unsigned long long *sink, int sms) {
  auto k = tma_probe_multi<STAGES, CHUNK, P>;
  const int smem = P * STAGES * CHUNK;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k<<<sms, 64 * P, smem>>>(pool, order, n_pages, page_bytes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("TMA bulk  %d producer warps/CTA, stages=%d chunk=%d: %7.1f GB/s\n", P, STAGES, CHUNK,
         (double)n_pages * page_bytes / (ms * 1e-3) / 1e9);
}

// Tensor-map TMA: P producer warps, each loading {64 d, 64 tok, 2 halves} 16 KB boxes of a
// [pages, 1 head, 64 tok, 128 d] pool (the attention kernel's 5-D map), SW128.
template <int STAGES, int P, bool FIVE_D>
__global__ void __launch_bounds__(64 * P, 1) tensor_probe(const __grid_constant__ CUtensorMap tm,
                                                          const int *order, int n_pages,
                                                          unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[P][STAGES], empty[P][STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pid = warp % P, role = warp / P;
  if (threadIdx.x == 0) {
    for (int q = 0; q < P; ++q)
      for (int i = 0; i < STAGES; ++i) { mbar_init(&full[q][i], 1); mbar_init(&empty[q][i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  uint8_t *ring = smem + pid * STAGES * 16384;
  if (lane == 0) {
    unsigned long long acc = 0;
    int n = 0;
    for (long long c = blockIdx.x * P + pid; c < n_pages; c += (long long)gridDim.x * P, ++n) {
      const int st = n % STAGES;
      if (role == 0) {
        mbar_wait(&empty[pid][st], ((n / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[pid][st], 16384);
        const int page = order[c] % n_pages;
        if (FIVE_D) {
          tma_load_5d(ring + st * 16384, &tm, &full[pid][st], 0, 0, 0, 0, page);
        } else {
          tma_load_4d(ring + st * 16384, &tm, &full[pid][st], 0, 0, 0, page);
          tma_load_4d(ring + st * 16384 + 8192, &tm, &full[pid][st], 64, 0, 0, page);
        }
      } else {
        mbar_wait(&full[pid][st], (n / STAGES) & 1);
        acc += ring[st * 16384 + (n & 127)];
        mbar_arrive(&empty[pid][st]);
      }
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES, int P, bool FIVE_D>
void run_tensor(void *pool, const int *order, int n_pages, unsigned long long *sink, int sms,
                CUtensorMapL2promotion promo) {
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  CUtensorMap tm;
  CUresult r;
  if (FIVE_D) {
    cuuint64_t dims[5] = {64, 64, 2, 1, (cuuint64_t)n_pages};
    cuuint64_t strides[4] = {256, 128, 256 * 64, 256 * 64};
    cuuint32_t box[5] = {64, 64, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, pool, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[4] = {128, 64, 1, (cuuint64_t)n_pages};
    cuuint64_t strides[3] = {256, 256 * 64, 256 * 64};
    cuuint32_t box[4] = {64, 64, 1, 1}, es[4] = {1, 1, 1, 1};
    r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, pool, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return; }
  auto k = tensor_probe<STAGES, P, FIVE_D>;
  const int smem = P * STAGES * 16384 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k<<<sms, 64 * P, smem>>>(tm, order, n_pages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("tensor TMA %s %d producers stages=%d promo=%d: %7.1f GB/s %s\n", FIVE_D ? "5D 16KB box" : "4D 2x8KB",
         P, STAGES, int(promo), (double)n_pages * 16384 / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

__global__ void ldg_probe(const uint4 *pool, const int *order, int n_pages, int page_bytes,
                          unsigned long long *sink) {
  const int per_page = page_bytes / 16;
  unsigned acc = 0;
  const long long total = (long long)n_pages * per_page;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long page = order[i / per_page] % n_pages;
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(pool + page * per_page + i % per_page));
    acc ^= v.x ^ v.w;
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

template <int STAGES, int CHUNK>
void run_tma(const uint8_t *pool, const int *order, int n_pages, int page_bytes, unsigned long long *sink,
             int sms, int ctas_per_sm) {
  auto k = tma_probe<STAGES, CHUNK>;
  const int smem = STAGES * CHUNK;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k<<<sms * ctas_per_sm, 64, smem>>>(pool, order, n_pages, page_bytes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  printf("TMA bulk  stages=%2d chunk=%6d ctas/sm=%d in-flight/SM=%4d KB: %7.1f GB/s %s\n", STAGES, CHUNK,
         ctas_per_sm, STAGES * CHUNK * ctas_per_sm / 1024,
         (double)n_pages * page_bytes / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char **argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int burn = argc > 1 ? atoi(argv[1]) : 0;  // >0: repeat the 2-producer tensor probe N times (power check)
  const int page_bytes = 16384;  // one (page, head) K block: 64 tokens x 128 d bf16
  const size_t pool_bytes = size_t(4) << 30;  // 4 GiB >> L2
  const int n_pages = int(pool_bytes / page_bytes);
  uint8_t *pool;
  int *order;
  unsigned long long *sink;
  if (cudaMalloc(&pool, pool_bytes) != cudaSuccess) { printf("malloc failed\n"); return 1; }
  cudaMemset(pool, 1, pool_bytes);
  cudaMalloc(&sink, 8);
  std::vector<int> h(n_pages);
  for (int i = 0; i < n_pages; ++i) h[i] = i;
  std::mt19937 rng(1);
  std::shuffle(h.begin(), h.end(), rng);
  cudaMalloc(&order, n_pages * sizeof(int));
  cudaMemcpy(order, h.data(), n_pages * sizeof(int), cudaMemcpyHostToDevice);
  int *seq;
  std::vector<int> hs(n_pages);
  for (int i = 0; i < n_pages; ++i) hs[i] = i;
  cudaMalloc(&seq, n_pages * sizeof(int));
  cudaMemcpy(seq, hs.data(), n_pages * sizeof(int), cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d, pool %.1f GB, random 16 KB pages\n", sms, pool_bytes / 1e9);
  for (int i = 0; i < burn; ++i)
    run_tensor<5, 2, true>(pool, order, n_pages, sink, sms, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (burn) return 0;
  run_tma<4, 16384>(pool, order, n_pages, page_bytes, sink, sms, 1);
  run_tma<8, 16384>(pool, order, n_pages, page_bytes, sink, sms, 1);
  run_tma<12, 16384>(pool, order, n_pages, page_bytes, sink, sms, 1);
  run_tma<6, 32768>(pool, order, n_pages / 2, page_bytes * 2, sink, sms, 1);
  run_tma<8, 8192>(pool, order, n_pages, page_bytes, sink, sms, 1);
  run_tma<16, 8192>(pool, order, n_pages, page_bytes, sink, sms, 1);
  run_tma<4, 16384>(pool, order, n_pages, page_bytes, sink, sms, 2);
  run_tma<6, 16384>(pool, order, n_pages, page_bytes, sink, sms, 2);
  run_tma<4, 16384>(pool, order, n_pages, page_bytes, sink, sms, 4);
  run_multi<5, 16384, 2>(pool, order, n_pages, page_bytes, sink, sms);
  run_multi<3, 16384, 4>(pool, order, n_pages, page_bytes, sink, sms);
  run_multi<6, 8192, 4>(pool, order, n_pages, page_bytes, sink, sms);
  run_multi<3, 8192, 8>(pool, order, n_pages, page_bytes, sink, sms);
  run_tensor<5, 2, true>(pool, order, n_pages, sink, sms, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  run_tensor<5, 2, true>(pool, order, n_pages, sink, sms, CU_TENSOR_MAP_L2_PROMOTION_NONE);
  run_tensor<3, 4, true>(pool, order, n_pages, sink, sms, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  run_tensor<5, 2, false>(pool, order, n_pages, sink, sms, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  run_tensor<3, 4, false>(pool, order, n_pages, sink, sms, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  printf("sequential pages:\n");
  run_tma<8, 16384>(pool, seq, n_pages, page_bytes, sink, sms, 1);
  run_tma<4, 16384>(pool, seq, n_pages, page_bytes, sink, sms, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int tpb : {256, 512, 1024}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      ldg_probe<<<sms * (2048 / tpb), tpb>>>(reinterpret_cast<const uint4 *>(pool), order, n_pages,
                                              page_bytes, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128   threads/SM=2048 (%4d/CTA): %7.1f GB/s\n", tpb, pool_bytes / (ms * 1e-3) / 1e9);
  }
  // plain copy for reference (read+write)
  uint8_t *dst;
  cudaMalloc(&dst, pool_bytes / 2);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    cudaMemcpyAsync(dst, pool, pool_bytes / 2, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("memcpy D2D (read+write bytes): %7.1f GB/s\n", pool_bytes / (ms * 1e-3) / 1e9);
  return 0;
}
