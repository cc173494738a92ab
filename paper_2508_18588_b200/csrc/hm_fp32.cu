// fp32 parity path of the verify forward (tests only).
//
// The product forward runs bf16 operands with fp32 accumulation on tcgen05; its
// logits can only be compared with an fp32 reference within a documented bf16
// bound.  This file is the same forward with fp32 operands, fp32 accumulation
// and an fp32 KV cache, built from plain SIMT kernels, so the GPU logits can be
// held to 1e-3 relative of the fp32 restatement (oracle/model_ref.py).  Weights
// stay the bf16 tensors of model.Weights, widened to fp32 on load (exact).
// Nothing here is on the rollout hot path.
#include <cuda_bf16.h>

#include "../../include/hsmodel.h"

void hm_set_error(const char* msg);
void hm_count_launches(int64_t n);

namespace hm {
namespace f32 {

constexpr int TM = 64, TN = 64, TK = 16;

// Y[M, N] (+)= X[M, K] . W[N, K]^T (+ bias); 16 x 16 threads, 4 x 4 outputs each
__global__ void __launch_bounds__(256) k_gemm(const float* __restrict__ x, int64_t ldx,
                                              const __nv_bfloat16* __restrict__ w, int64_t ldw, int M, int N,
                                              int K, const __nv_bfloat16* __restrict__ bias, float* __restrict__ y,
                                              int64_t ldy, int accumulate) {
  __shared__ float xs[TK][TM + 1];
  __shared__ float ws[TK][TN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      const int r = i / TK, c = i % TK;
      const int m = m0 + r, k = k0 + c;
      xs[c][r] = (m < M && k < K) ? x[(int64_t)m * ldx + k] : 0.f;
      const int n = n0 + r;
      ws[c][r] = (n < N && k < K) ? __bfloat162float(w[(int64_t)n * ldw + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < TK; ++c) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = xs[c][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = ws[c][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v = acc[i][j] + (bias ? __bfloat162float(bias[n]) : 0.f);
      float* dst = y + (int64_t)m * ldy + n;
      *dst = accumulate ? *dst + v : v;
    }
  }
}

// out = x * rsqrt(mean(x^2) + eps) * w, block per row
__global__ void k_rmsnorm(const float* __restrict__ x, const __nv_bfloat16* __restrict__ w, int d, float eps,
                          float* __restrict__ out) {
  const float* xr = x + (int64_t)blockIdx.x * d;
  __shared__ float red[32];
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss += xr[i] * xr[i];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    out[(int64_t)blockIdx.x * d + i] = xr[i] * r * __bfloat162float(w[i]);
}

// rotate-half RoPE of the q and k heads, v copied; q -> [M][H][hd], k / v -> cache [slot][KVH][max_len][hd]
__global__ void k_rope_kv(const float* __restrict__ qkv, const int32_t* __restrict__ pos,
                          const int32_t* __restrict__ row_slot, const float* __restrict__ cos_t,
                          const float* __restrict__ sin_t, int H, int KVH, int hd, float* __restrict__ q,
                          float* __restrict__ kc, float* __restrict__ vc, int64_t slot_stride, int max_len) {
  const int row = blockIdx.x;
  const int p = pos[row];
  const int64_t slot = row_slot[row];
  const int half = hd / 2;
  const float* src = qkv + (int64_t)row * (H + 2 * KVH) * hd;
  for (int t = threadIdx.x; t < (H + 2 * KVH) * half; t += blockDim.x) {
    const int head = t / half, i = t % half;
    const float a = src[head * hd + i], b = src[head * hd + i + half];
    float ra = a, rb = b;
    if (head < H + KVH) {
      const float c = cos_t[(int64_t)p * half + i], s = sin_t[(int64_t)p * half + i];
      ra = a * c - b * s;
      rb = b * c + a * s;
    }
    float* dst;
    if (head < H) dst = q + ((int64_t)row * H + head) * hd;
    else if (head < H + KVH) dst = kc + slot * slot_stride + ((int64_t)(head - H) * max_len + p) * hd;
    else dst = vc + slot * slot_stride + ((int64_t)(head - H - KVH) * max_len + p) * hd;
    dst[i] = ra;
    dst[i + half] = rb;
  }
}

// causal attention of one (row, head) over keys 0..pos of the row's slot; scores staged in shared memory
__global__ void k_attention(const float* __restrict__ q, const float* __restrict__ kc, const float* __restrict__ vc,
                            int64_t slot_stride, const int32_t* __restrict__ pos,
                            const int32_t* __restrict__ row_slot, int H, int KVH, int hd, int max_len, float scale,
                            float* __restrict__ out) {
  extern __shared__ float sc[];   // [pos + 1] scores, then [hd] query
  __shared__ float red[32];
  const int row = blockIdx.x, h = blockIdx.y;
  const int n = pos[row] + 1;
  const int kvh = h / (H / KVH);
  const float* kb = kc + (int64_t)row_slot[row] * slot_stride + (int64_t)kvh * max_len * hd;
  const float* vb = vc + (int64_t)row_slot[row] * slot_stride + (int64_t)kvh * max_len * hd;
  float* qs = sc + max_len;
  for (int i = threadIdx.x; i < hd; i += blockDim.x) qs[i] = q[((int64_t)row * H + h) * hd + i];
  __syncthreads();
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    float s = 0.f;
    for (int i = 0; i < hd; ++i) s = fmaf(qs[i], kb[(int64_t)k * hd + i], s);
    s *= scale;
    sc[k] = s;
    mx = fmaxf(mx, s);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = -INFINITY;
    for (int i = 0; i < (int)blockDim.x / 32; ++i) v = fmaxf(v, red[i]);
    red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const float e = expf(sc[k] - mx);
    sc[k] = e;
    sum += e;
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = 0.f;
    for (int i = 0; i < (int)blockDim.x / 32; ++i) v += red[i];
    red[0] = v;
  }
  __syncthreads();
  const float inv = 1.f / red[0];
  for (int i = threadIdx.x; i < hd; i += blockDim.x) {
    float o = 0.f;
    for (int k = 0; k < n; ++k) o = fmaf(sc[k], vb[(int64_t)k * hd + i], o);
    out[(int64_t)row * H * hd + h * hd + i] = o * inv;
  }
}

// act[:, j * half + c] = silu(gu[:, 2 j half + c]) * gu[:, 2 j half + half + c] (model.interleave_gate_up)
__global__ void k_swiglu(const float* __restrict__ gu, int M, int F, int half, float* __restrict__ act) {
  const int64_t n = (int64_t)M * F;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = t / F;
    const int c = (int)(t % F);
    const int j = c / half, cc = c % half;
    const float g = gu[m * 2 * F + 2 * j * half + cc], u = gu[m * 2 * F + 2 * j * half + half + cc];
    act[t] = g / (1.f + expf(-g)) * u;
  }
}

}  // namespace f32
}  // namespace hm

#define F32_CHECK()                             \
  do {                                          \
    hm_count_launches(1);                       \
    cudaError_t _e = cudaGetLastError();        \
    if (_e != cudaSuccess) {                    \
      hm_set_error(cudaGetErrorString(_e));     \
      return HM_ERR_CUDA;                       \
    }                                           \
    return HM_OK;                               \
  } while (0)

extern "C" int hm_f32_gemm(const float* d_x, int64_t ldx, const void* d_w, int64_t ldw, int32_t M, int32_t N,
                           int32_t K, const void* d_bias, float* d_y, int64_t ldy, int32_t accumulate,
                           hm_stream_t stream) {
  if (M <= 0 || N <= 0) return HM_OK;
  if (K <= 0) { hm_set_error("hm_f32_gemm: K must be > 0"); return HM_ERR_INVALID; }
  const dim3 grid((N + hm::f32::TN - 1) / hm::f32::TN, (M + hm::f32::TM - 1) / hm::f32::TM);
  hm::f32::k_gemm<<<grid, 256, 0, (cudaStream_t)stream>>>(d_x, ldx, (const __nv_bfloat16*)d_w, ldw, M, N, K,
                                                          (const __nv_bfloat16*)d_bias, d_y, ldy, accumulate);
  F32_CHECK();
}

extern "C" int hm_f32_rmsnorm(const float* d_x, const void* d_w, int32_t M, int32_t d, float eps, float* d_out,
                              hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  hm::f32::k_rmsnorm<<<M, 256, 0, (cudaStream_t)stream>>>(d_x, (const __nv_bfloat16*)d_w, d, eps, d_out);
  F32_CHECK();
}

extern "C" int hm_f32_rope_kv_append(const float* d_qkv, const int32_t* d_pos, const int32_t* d_row_slot,
                                     const float* d_cos, const float* d_sin, int32_t M, int32_t H, int32_t KVH,
                                     int32_t hd, float* d_q, float* d_kcache, float* d_vcache, int64_t slot_stride,
                                     int32_t max_len, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (KVH <= 0 || H % KVH || hd % 2) { hm_set_error("hm_f32_rope_kv_append: H % KVH, even hd"); return HM_ERR_INVALID; }
  hm::f32::k_rope_kv<<<M, 256, 0, (cudaStream_t)stream>>>(d_qkv, d_pos, d_row_slot, d_cos, d_sin, H, KVH, hd, d_q,
                                                          d_kcache, d_vcache, slot_stride, max_len);
  F32_CHECK();
}

extern "C" int hm_f32_attention(const float* d_q, const float* d_kcache, const float* d_vcache, int64_t slot_stride,
                                const int32_t* d_pos, const int32_t* d_row_slot, int32_t M, int32_t H, int32_t KVH,
                                int32_t hd, int32_t max_len, float scale, float* d_out, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (KVH <= 0 || H % KVH) { hm_set_error("hm_f32_attention: H % KVH"); return HM_ERR_INVALID; }
  const size_t smem = (size_t)(max_len + hd) * sizeof(float);
  if (smem > 200 * 1024) { hm_set_error("hm_f32_attention: max_len too long for the staged scores"); return HM_ERR_INVALID; }
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(hm::f32::k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  hm::f32::k_attention<<<dim3(M, H), 128, smem, (cudaStream_t)stream>>>(d_q, d_kcache, d_vcache, slot_stride, d_pos,
                                                                       d_row_slot, H, KVH, hd, max_len, scale, d_out);
  F32_CHECK();
}

extern "C" int hm_f32_swiglu(const float* d_gu, int32_t M, int32_t F, int32_t half, float* d_act, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (half <= 0 || F % half) { hm_set_error("hm_f32_swiglu: F must be a multiple of the interleave half"); return HM_ERR_INVALID; }
  const int64_t n = (int64_t)M * F;
  const int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  hm::f32::k_swiglu<<<blocks, 256, 0, (cudaStream_t)stream>>>(d_gu, M, F, half, d_act);
  F32_CHECK();
}
