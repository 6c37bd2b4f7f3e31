// Dev probe: 16x256b.x2 register layout, and stmatrix.m8n8.x4.trans placement.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

__global__ void probe(uint32_t *out, uint16_t *sm_out) {
  __shared__ uint32_t slot;
  __shared__ __align__(16) uint16_t sm[4 * 64];
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
  uint32_t c[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]),
                 "=r"(c[6]), "=r"(c[7])
               : "r"(t));
  tmem_ld_wait();
  for (int j = 0; j < 8; ++j) out[lane * 8 + j] = c[j];
  // stmatrix: register i of thread t = (matrix i, row t/4, cols 2(t%4), +1) encoded as
  // value = i * 64 + row * 8 + col (16-bit each)
  uint32_t r[4];
  for (int i = 0; i < 4; ++i) {
    const int row = lane / 4, col = 2 * (lane % 4);
    r[i] = uint32_t(i * 64 + row * 8 + col) | (uint32_t(i * 64 + row * 8 + col + 1) << 16);
  }
  // lane 8i + k gives the address of stored row k of matrix i: sm + i * 64 + k * 8
  const uint32_t addr = smem_u32(sm + (lane / 8) * 64 + (lane % 8) * 8);
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
  __syncwarp();
  for (int i = lane; i < 256; i += 32) sm_out[i] = sm[i];
  tc_fence_before();
  __syncwarp();
  tmem_dealloc<64>(t);
}

int main() {
  uint32_t *d, h[32 * 8];
  uint16_t *ds, hs[256];
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&ds, sizeof(hs));
  probe<<<1, 32>>>(d, ds);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(hs, ds, sizeof(hs), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int j = 0; j < 8; ++j) {
    printf("16x256b.x2 r%d:", j);
    for (int l = 0; l < 32; ++l) printf(" %d:%d", h[l * 8 + j] >> 8, h[l * 8 + j] & 255);
    printf("\n");
  }
  printf("stmatrix.trans: stored row k of matrix i holds (i, orig row, orig col):\n");
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 8; ++k) {
      printf("m%d row%d:", i, k);
      for (int e = 0; e < 8; ++e) {
        int v = hs[i * 64 + k * 8 + e];
        printf(" (%d,%d,%d)", v / 64, (v % 64) / 8, v % 8);
      }
      printf("\n");
    }
  return 0;
}
