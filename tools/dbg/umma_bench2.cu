// Microbenchmark: the attention kernel's per-stage MMA issue pattern (debugging aid).
#include <cstdio>
#include <cstdint>
#include "../../paper_2508_18588_b200/csrc/hm_ptx.cuh"
using namespace hm;
template <int VARIANT>
__global__ void k(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t id_s = idesc_bf16(128, 64), id_pv = idesc_bf16(128, 144) | (1u << 16);
    const uint64_t kd = smem_desc_sw128(sm + 32768), vd = smem_desc_sw128_mn(sm, 8192);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) umma_f16_ts(base + 256, base + 192 + kk * 8, vd + kk * 128, id_pv, 1);
      if (VARIANT >= 1) { umma_commit(&bar[0]); umma_commit(&bar[1]); umma_commit(&bar[2]); }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) umma_f16_ts(base + (r % 3) * 64, base + 448 + kk * 8, kd + kk * 2, id_s, kk > 0);
      if (VARIANT >= 1) { umma_commit(&bar[3]); umma_commit(&bar[4]); }
    }
    long long t1 = clock64();
    umma_commit(&bar[5]);
    mbar_wait(&bar[5], 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(base);
}
template <int V>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int reps = 200;
  k<V><<<1, 128, 70 * 1024>>>(d, reps);
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-24s %.1f cycles per stage (issue), %.1f (complete) %s\n", name, h[0] / (double)reps, h[1] / (double)reps,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("PV4 + S8, no commits");
  run<1>("PV4 + S8 + 5 commits");
}
