// Microbenchmark: back-to-back tcgen05.mma issue throughput per shape/operand source (debugging aid).
#include <cstdio>
#include <cstdint>
#include "../../paper_2508_18588_b200/csrc/hm_ptx.cuh"
using namespace hm;
template <int M, int N, bool TS, bool BMN>
__global__ void k(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(M, N) | (BMN ? (1u << 16) : 0u);
    const uint64_t ad = smem_desc_sw128(sm), bd = BMN ? smem_desc_sw128_mn(sm + 32768, 8192) : smem_desc_sw128(sm + 32768);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (TS) umma_f16_ts(base + 256, base + 448 + kk * 8, bd + kk * 2, id, 1);
        else umma_f16(base + 256, ad + kk * 2, bd + kk * 2, id, 1);
      }
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(base);
}
template <int M, int N, bool TS, bool BMN>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<M, N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int reps = 200;
  k<M, N, TS, BMN><<<1, 128, 70 * 1024>>>(d, reps);
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-28s issue %.1f  complete %.1f cycles per MMA (%s)\n", name, h[0] / (8.0 * reps), h[1] / (8.0 * reps),
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<128, 64, false, false>("ss M128 N64");
  run<128, 64, true, false>("ts M128 N64");
  run<128, 128, true, false>("ts M128 N128");
  run<128, 256, true, false>("ts M128 N256");
  run<128, 256, false, false>("ss M128 N256");
  run<128, 144, true, true>("ts M128 N144 B-MN");
  run<128, 128, true, true>("ts M128 N128 B-MN");
  run<64, 64, true, false>("ts M64 N64");
  run<64, 144, true, true>("ts M64 N144 B-MN");
  run<64, 256, true, false>("ts M64 N256");
}
