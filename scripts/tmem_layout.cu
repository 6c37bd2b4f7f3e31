// Dev probe: which (TMEM lane, column) each thread receives for the 16-lane tcgen05.ld shapes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_layout tmem_layout.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

__global__ void probe(uint32_t *out) {
  __shared__ uint32_t slot;
  const int lane = threadIdx.x & 31;
  tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncwarp();
  tc_fence_after();
  const uint32_t t = slot;
  uint32_t v[32];
  for (int j = 0; j < 32; ++j) v[j] = (uint32_t(lane) << 8) | uint32_t(j);
  tmem_st32(t, v);
  tmem_st_wait();
  uint32_t a0, b0, b1, c0, c1, c2, c3, d0, d1, e[4];
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(a0) : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(c0), "=r"(c1), "=r"(c2), "=r"(c3) : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x2.b32 {%0,%1}, [%2], 16;" : "=r"(d0), "=r"(d1) : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3]) : "r"(t));
  tmem_ld_wait();
  uint32_t *o = out + lane * 16;
  o[0] = a0; o[1] = b0; o[2] = b1; o[3] = c0; o[4] = c1; o[5] = c2; o[6] = c3; o[7] = d0; o[8] = d1;
  for (int j = 0; j < 4; ++j) o[9 + j] = e[j];
  tc_fence_before();
  __syncwarp();
  tmem_dealloc<64>(t);
}

int main() {
  uint32_t *d, h[32 * 16];
  cudaMalloc(&d, sizeof(h));
  probe<<<1, 32>>>(d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  const char *names[] = {"16x64b.x1", "16x128b r0", "16x128b r1", "16x256b r0", "16x256b r1",
                         "16x256b r2", "16x256b r3", "16x32bx2 r0", "16x32bx2 r1", "16x64b.x4 r0",
                         "16x64b.x4 r1", "16x64b.x4 r2", "16x64b.x4 r3"};
  for (int k = 0; k < 13; ++k) {
    printf("%-14s", names[k]);
    for (int l = 0; l < 32; ++l) printf(" %d:%d", h[l * 16 + k] >> 8, h[l * 16 + k] & 255);
    printf("\n");
  }
  return 0;
}
