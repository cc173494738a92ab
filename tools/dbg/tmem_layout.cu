// Probe of the tcgen05.ld.16x256b fragment layout (debugging aid, not part of the product).
#include <cstdio>
#include <cstdint>
#include "../../paper_2508_18588_b200/csrc/hm_ptx.cuh"
using namespace hm;
__global__ void k(int* out) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<64>(&base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = base + ((uint32_t)(warp * 32) << 16);
  uint32_t v[32];
  for (int c = 0; c < 32; ++c) v[c] = (warp * 32 + lane) * 1000 + c;   // lane L, column c -> L*1000 + c
  tmem_st32(t, v);
  tmem_wait_st();
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 8; ++i) out[(warp * 32 + lane) * 8 + i] = r[i];
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<64>(base);
}
int main() {
  int* d; cudaMalloc(&d, 128 * 8 * 4);
  k<<<1, 128>>>(d);
  int h[128 * 8]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int th = 0; th < 32; th += 1) {
    printf("warp0 thread %2d:", th);
    for (int i = 0; i < 8; ++i) printf(" L%d.c%d", h[th * 8 + i] / 1000, h[th * 8 + i] % 1000);
    printf("\n");
  }
  printf("warp1 thread 0:"); for (int i = 0; i < 8; ++i) printf(" L%d.c%d", h[32*8 + i] / 1000, h[32*8 + i] % 1000); printf("\n");
}
