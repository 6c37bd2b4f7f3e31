// Dev probe: cost of mbarrier.try_wait on an already-completed phase, and of a
// named-barrier bar.red.or, from one warp.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"
using namespace taper;

__global__ void probe(long long *out) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bar);
  __syncthreads();
  long long t0 = clock64();
  int ok = 0;
  for (int i = 0; i < 1000; ++i) ok += mbar_try_wait(&bar, 0);
  long long t1 = clock64();
  for (int i = 0; i < 1000; ++i) mbar_wait(&bar, 0);
  long long t2 = clock64();
  // dependent chain: each wait's result feeds the next address (forces serialisation)
  uint32_t a = 0;
  for (int i = 0; i < 1000; ++i) a += mbar_try_wait(&bar + (a & 0), 0);
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = ok + a; }
}

int main() {
  long long *d, h[4];
  cudaMalloc(&d, sizeof(h));
  probe<<<1, 32>>>(d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("try_wait x1000: %lld cycles (%.1f each); mbar_wait x1000: %lld (%.1f each); dependent: %.1f each; ok=%lld\n",
         h[0], h[0] / 1000.0, h[1], h[1] / 1000.0, h[2] / 1000.0, h[3]);
  return 0;
}
