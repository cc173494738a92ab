// Memory-bound pieces of the verify forward: embedding gather, RMSNorm,
// RoPE + KV append (K5), verify-batch assembly.  All row-local with fixed
// reduction orders, so a row's bits do not depend on what else is batched.
#include <cuda_bf16.h>
#include <cstdio>

#include "../../include/hsmodel.h"

namespace {
thread_local char g_err[512];
int64_t g_launches = 0;
}  // namespace

void hm_set_error(const char* msg) { snprintf(g_err, sizeof(g_err), "%s", msg); }
void hm_count_launches(int64_t n) { __atomic_fetch_add(&g_launches, n, __ATOMIC_RELAXED); }
extern "C" const char* hm_last_error(void) { return g_err; }
extern "C" int64_t hm_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

// persistent-kernel CTA caps (hm_set_grid_caps); 0 = one CTA per SM
int g_cap_gemm = 0, g_cap_attn = 0;
extern "C" int hm_set_grid_caps(int32_t gemm_ctas, int32_t attn_ctas) {
  if (gemm_ctas < 0 || attn_ctas < 0) { hm_set_error("hm_set_grid_caps: caps must be >= 0"); return HM_ERR_INVALID; }
  g_cap_gemm = gemm_ctas;
  g_cap_attn = attn_ctas;
  return HM_OK;
}
int hm_cap(int n_sms, bool attn) {
  const int c = attn ? g_cap_attn : g_cap_gemm;
  return (c > 0 && c < n_sms) ? c : n_sms;
}

#define HM_LAUNCH_CHECK()                                 \
  do {                                                    \
    hm_count_launches(1);                                 \
    cudaError_t _e = cudaGetLastError();                  \
    if (_e != cudaSuccess) {                              \
      hm_set_error(cudaGetErrorString(_e));               \
      return HM_ERR_CUDA;                                 \
    }                                                     \
  } while (0)

namespace hm {

__global__ void k_embed(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ emb, int M, int d,
                        const int* m_dev, float* __restrict__ x) {
  const int m = m_dev ? *m_dev : M;
  for (int row = blockIdx.x; row < m; row += gridDim.x) {   // grid-stride: launches sized for max rows stay cheap
    const __nv_bfloat162* src = reinterpret_cast<const __nv_bfloat162*>(emb + (size_t)tok[row] * d);
    float2* dst = reinterpret_cast<float2*>(x + (size_t)row * d);
    for (int i = threadIdx.x; i < d / 2; i += blockDim.x) dst[i] = __bfloat1622float2(src[i]);
  }
}

// warp per row; each lane owns a fixed strided set of columns
__global__ void k_rmsnorm(const float* __restrict__ x, const __nv_bfloat16* __restrict__ w, int M, int d, float eps,
                          const int* m_dev, __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int m = m_dev ? *m_dev : M;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m;
       row += gridDim.x * (blockDim.x >> 5)) {
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * d);
  float ss = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    float4 v = xr[i];
    ss += v.x * v.x;
    ss += v.y * v.y;
    ss += v.z * v.z;
    ss += v.w * v.w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r = rsqrtf(ss / (float)d + eps);
  __nv_bfloat162* orow = reinterpret_cast<__nv_bfloat162*>(out + (size_t)row * d);
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(w);
  for (int i = lane; i < d / 4; i += 32) {
    float4 v = xr[i];
    float2 wa = __bfloat1622float2(w2[2 * i]), wb = __bfloat1622float2(w2[2 * i + 1]);
    orow[2 * i] = __floats2bfloat162_rn(v.x * r * wa.x, v.y * r * wa.y);
    orow[2 * i + 1] = __floats2bfloat162_rn(v.z * r * wb.x, v.w * r * wb.y);
  }
  }
}

// x += y (fp32), out = rmsnorm(x) * w; warp per row, same fixed reduction order as k_rmsnorm.
// MAXV = ceil(d / 128) float4 per lane, so the row stays in registers.
template <int MAXV>
__global__ void k_rmsnorm_residual(float* __restrict__ x, const float* __restrict__ y,
                                   const __nv_bfloat16* __restrict__ w, int M, int d, float eps, const int* m_dev,
                                   __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int m = m_dev ? *m_dev : M;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m;
       row += gridDim.x * (blockDim.x >> 5)) {
  float4* xr = reinterpret_cast<float4*>(x + (size_t)row * d);
  const float4* yr = reinterpret_cast<const float4*>(y + (size_t)row * d);
  float4 v[MAXV];
  float ss = 0.f;
  const int nv = d / 4;
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int i = lane + 32 * k;
    if (i < nv) {
      float4 a = xr[i];   // (an L2 evict-last policy on x measured slower: +0.01 / +0.11 ms per forward)
      const float4 b = yr[i];   // (an evict-first __ldcs here measured slower: +0.06 / +0.12 ms per forward)
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
      xr[i] = a;
      v[k] = a;
      ss += a.x * a.x;
      ss += a.y * a.y;
      ss += a.z * a.z;
      ss += a.w * a.w;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float r = rsqrtf(ss / (float)d + eps);
  __nv_bfloat162* orow = reinterpret_cast<__nv_bfloat162*>(out + (size_t)row * d);
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(w);
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int i = lane + 32 * k;
    if (i < nv) {
      float2 wa = __bfloat1622float2(w2[2 * i]), wb = __bfloat1622float2(w2[2 * i + 1]);
      orow[2 * i] = __floats2bfloat162_rn(v[k].x * r * wa.x, v[k].y * r * wa.y);
      orow[2 * i + 1] = __floats2bfloat162_rn(v[k].z * r * wb.x, v[k].w * r * wb.y);
    }
  }
  }
}

// Any d (two passes, the row is re-read from x instead of held in registers) and an optional second partial:
// x += (y + y2), the tensor-parallel all-reduce of the O / down projections folded into the norm -- y is this
// GPU's partial, y2 the peer's, read over NVLink from its symmetric buffer.  y + y2 is the same fp32 sum on
// both GPUs (commutative), so the replicated residual stream stays bit-identical across the pair.  Same
// per-lane reduction order as k_rmsnorm / k_rmsnorm_residual (column i = lane + 32 k).
__global__ void k_rmsnorm_residual_g(float* __restrict__ x, const float* __restrict__ y, const float* y2,
                                     const __nv_bfloat16* __restrict__ w, int M, int d, float eps, const int* m_dev,
                                     __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int m = m_dev ? *m_dev : M;
  const int nv = d / 4;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m;
       row += gridDim.x * (blockDim.x >> 5)) {
    float4* xr = reinterpret_cast<float4*>(x + (size_t)row * d);
    const float4* yr = y ? reinterpret_cast<const float4*>(y + (size_t)row * d) : nullptr;
    const float4* y2r = y2 ? reinterpret_cast<const float4*>(y2 + (size_t)row * d) : nullptr;
    float ss = 0.f;
    for (int i = lane; i < nv; i += 32) {
      float4 a = xr[i];
      if (yr) {
        float4 b = yr[i];
        if (y2r) {
          const float4 c = y2r[i];
          b.x += c.x;
          b.y += c.y;
          b.z += c.z;
          b.w += c.w;
        }
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
        xr[i] = a;
      }
      ss += a.x * a.x;
      ss += a.y * a.y;
      ss += a.z * a.z;
      ss += a.w * a.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float r = rsqrtf(ss / (float)d + eps);
    __nv_bfloat162* orow = reinterpret_cast<__nv_bfloat162*>(out + (size_t)row * d);
    const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(w);
    for (int i = lane; i < nv; i += 32) {
      const float4 v = xr[i];
      const float2 wa = __bfloat1622float2(w2[2 * i]), wb = __bfloat1622float2(w2[2 * i + 1]);
      orow[2 * i] = __floats2bfloat162_rn(v.x * r * wa.x, v.y * r * wa.y);
      orow[2 * i + 1] = __floats2bfloat162_rn(v.z * r * wb.x, v.w * r * wb.y);
    }
  }
}

// bf16 residual stream (the precision bf16 inference keeps it in): x = bf16(x + y [+ y2]) -- the projection
// output y (and, under TP, the peer's partial y2, read in place over NVLink) rounded to bf16 by its GEMM --
// then out = bf16(x * rsqrt(mean(x^2) + eps) * w).  Warp per row, lane-strided 8-element chunks held in
// registers (MAXV = ceil(d / 256)); the reduction order is fixed per lane, so a row's bits depend only on it.
template <int MAXV>
__global__ void k_rmsnorm_residual_bf16(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ y,
                                        const __nv_bfloat16* y2, const __nv_bfloat16* __restrict__ w, int M, int d,
                                        float eps, const int* m_dev, __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int m = m_dev ? *m_dev : M;
  const int nv = d / 8;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m;
       row += gridDim.x * (blockDim.x >> 5)) {
    uint4* xr = reinterpret_cast<uint4*>(x + (size_t)row * d);
    const uint4* yr = y ? reinterpret_cast<const uint4*>(y + (size_t)row * d) : nullptr;
    const uint4* y2r = y2 ? reinterpret_cast<const uint4*>(y2 + (size_t)row * d) : nullptr;
    uint4 v[MAXV];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
      const int i = lane + 32 * k;
      if (i < nv) {
        uint4 a = xr[i];
        if (yr) {
          const uint4 b = yr[i];
          uint4 c = make_uint4(0, 0, 0, 0);
          if (y2r) c = y2r[i];
          const uint32_t* pa = reinterpret_cast<const uint32_t*>(&a);
          const uint32_t* pb = reinterpret_cast<const uint32_t*>(&b);
          const uint32_t* pc = reinterpret_cast<const uint32_t*>(&c);
          uint4 r;
          uint32_t* pr = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pa[e]));
            float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pb[e]));
            if (y2r) {
              const float2 fc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pc[e]));
              fb.x += fc.x;
              fb.y += fc.y;
            }
            const __nv_bfloat162 o = __floats2bfloat162_rn(fa.x + fb.x, fa.y + fb.y);
            pr[e] = *reinterpret_cast<const uint32_t*>(&o);
          }
          a = r;
          xr[i] = a;
        }
        v[k] = a;
        const uint32_t* pv = reinterpret_cast<const uint32_t*>(&a);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv[e]));
          ss += f.x * f.x;
          ss += f.y * f.y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float r = rsqrtf(ss / (float)d + eps);
    uint4* orow = reinterpret_cast<uint4*>(out + (size_t)row * d);
    const uint4* w4 = reinterpret_cast<const uint4*>(w);
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
      const int i = lane + 32 * k;
      if (i < nv) {
        const uint4 ww = w4[i];
        const uint32_t* pv = reinterpret_cast<const uint32_t*>(&v[k]);
        const uint32_t* pw = reinterpret_cast<const uint32_t*>(&ww);
        uint4 o;
        uint32_t* po = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv[e]));
          const float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pw[e]));
          const __nv_bfloat162 h = __floats2bfloat162_rn(f.x * r * g.x, f.y * r * g.y);
          po[e] = *reinterpret_cast<const uint32_t*>(&h);
        }
        orow[i] = o;
      }
    }
  }
}

__global__ void k_embed_bf16(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ emb, int M, int d,
                             const int* m_dev, __nv_bfloat16* __restrict__ x) {
  const int m = m_dev ? *m_dev : M;
  for (int row = blockIdx.x; row < m; row += gridDim.x) {
    const uint4* src = reinterpret_cast<const uint4*>(emb + (size_t)tok[row] * d);
    uint4* dst = reinterpret_cast<uint4*>(x + (size_t)row * d);
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = src[i];
  }
}

// Two-GPU barrier over peer memory (tensor-parallel pair): bump this GPU's generation, publish it in the
// peer's flag word (system-scope release after a system fence: every write this stream made before -- the
// GEMM's partial in the symmetric buffer -- is visible to the peer first), then wait until the peer's
// generation reached ours.  Stream-ordered and graph-capturable (the generation lives in device memory).
__global__ void k_tp_barrier(int* my_flag, int* peer_flag, int* gen) {
  if (threadIdx.x != 0) return;
  const int g = *gen + 1;
  *gen = g;
  __threadfence_system();
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(peer_flag), "r"(g) : "memory");
  int v;
  const long long t0 = clock64();
  do {
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(my_flag) : "memory");
    // a peer that never arrives (diverged control flow) fails the launch loudly instead of hanging the GPU
    if (v < g && clock64() - t0 > (30ll << 30)) __trap();
  } while (v < g);
  __threadfence_system();
}

// block per row (grid-stride): threads cover the 16-byte chunks of q/k rotations and v copies
__global__ void k_rope_kv(const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ pos,
                          const int32_t* __restrict__ row_slot, const float* __restrict__ cosb,
                          const float* __restrict__ sinb, int M, int H, int KVH, int hd,
                          __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                          int64_t slot_stride, int max_len, const int* m_dev) {
  const int m = m_dev ? *m_dev : M;
  for (int row = blockIdx.x; row < m; row += gridDim.x) {
  // 8 elements (16 B) per work item: rotations pair chunk i of the first half with chunk i of the second
  const int half = hd / 2;
  const int hc = half / 8;                 // 16-byte chunks per half head
  const int p = pos[row];
  const int slot = row_slot[row];
  const __nv_bfloat16* src = qkv + (size_t)row * (H + 2 * KVH) * hd;
  const float* c = cosb + (size_t)p * half;
  const float* s = sinb + (size_t)p * half;
  const int n_rot = (H + KVH) * hc;
  const int G = H / KVH;
  for (int t = threadIdx.x; t < n_rot + KVH * 2 * hc; t += blockDim.x) {
    if (t < n_rot) {
      const int head = t / hc, i = (t % hc) * 8;
      const __nv_bfloat16* hsrc = src + head * hd;
      const uint4 ua = *reinterpret_cast<const uint4*>(hsrc + i);
      const uint4 ub = *reinterpret_cast<const uint4*>(hsrc + i + half);
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&ua);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&ub);
      const float4 c0 = *reinterpret_cast<const float4*>(c + i), c1 = *reinterpret_cast<const float4*>(c + i + 4);
      const float4 s0 = *reinterpret_cast<const float4*>(s + i), s1 = *reinterpret_cast<const float4*>(s + i + 4);
      const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      const float ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      uint4 ra, rb;
      __nv_bfloat162* ra2 = reinterpret_cast<__nv_bfloat162*>(&ra);
      __nv_bfloat162* rb2 = reinterpret_cast<__nv_bfloat162*>(&rb);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 a = __bfloat1622float2(a2[e]), b = __bfloat1622float2(b2[e]);
        // rounding pinned: the fused QKV + RoPE GEMM epilogue (hm_gemm_qkv_rope) computes the same bits
        ra2[e] = __floats2bfloat162_rn(__fsub_rn(__fmul_rn(a.x, cc[2 * e]), __fmul_rn(b.x, ss[2 * e])),
                                       __fsub_rn(__fmul_rn(a.y, cc[2 * e + 1]), __fmul_rn(b.y, ss[2 * e + 1])));
        rb2[e] = __floats2bfloat162_rn(__fadd_rn(__fmul_rn(b.x, cc[2 * e]), __fmul_rn(a.x, ss[2 * e])),
                                       __fadd_rn(__fmul_rn(b.y, cc[2 * e + 1]), __fmul_rn(a.y, ss[2 * e + 1])));
      }
      __nv_bfloat16* dst;
      if (head < H) dst = q + (((size_t)(head / G) * M + row) * G + head % G) * hd;   // [KVH][M][G][hd]
      else dst = kc + (size_t)slot * slot_stride + ((size_t)(head - H) * max_len + p) * hd;
      *reinterpret_cast<uint4*>(dst + i) = ra;
      *reinterpret_cast<uint4*>(dst + i + half) = rb;
    } else {
      const int u = t - n_rot;
      const int kh = u / (2 * hc), i = (u % (2 * hc)) * 8;
      const __nv_bfloat16* vsrc = src + (H + KVH + kh) * hd;
      __nv_bfloat16* dst = vc + (size_t)slot * slot_stride + ((size_t)kh * max_len + p) * hd;
      *reinterpret_cast<uint4*>(dst + i) = *reinterpret_cast<const uint4*>(vsrc + i);
    }
  }
  }
}

// single block: q_len = live ? 1 + draft_len : 0; exclusive scan -> q_off; rows
__global__ void k_build_verify(int n_seq, const int32_t* __restrict__ gen_tok, int gen_stride,
                               const int32_t* __restrict__ gen_len, const int32_t* __restrict__ target_len,
                               const int32_t* __restrict__ prompt_len, const int32_t* __restrict__ draft_tok,
                               int draft_stride, const int32_t* __restrict__ draft_len,
                               const int32_t* __restrict__ kv_slot, int32_t* __restrict__ tokens,
                               int32_t* __restrict__ pos, int32_t* __restrict__ row_slot, int32_t* __restrict__ q_off,
                               int32_t* __restrict__ q_len, int32_t* __restrict__ pos0, int32_t* __restrict__ m_out,
                               long long* __restrict__ acc, long long* __restrict__ qhist, int qhist_len,
                               const int32_t* __restrict__ seq_key, int32_t* __restrict__ row_key) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  __shared__ unsigned long long s_rows_pos, s_ctx;   // sum over rows of (pos + 1); over live seqs of ctx + q
  __shared__ unsigned int s_hist[64];
  if (threadIdx.x == 0) {
    carry = 0;
    s_rows_pos = 0;
    s_ctx = 0;
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  unsigned long long my_rows_pos = 0, my_ctx = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int base = 0; base < n_seq; base += blockDim.x) {
    const int s = base + threadIdx.x;
    int q = 0;
    if (s < n_seq) {
      const bool live = gen_len[s] < target_len[s] && gen_len[s] > 0;
      q = live ? 1 + draft_len[s] : 0;
    }
    // block-wide exclusive scan of q
    int incl = q;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? warp_sums[lane] : 0;
      int iv = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, iv, o);
        if (lane >= o) iv += y;
      }
      if (lane < nw) warp_sums[lane] = iv - v;
    }
    __syncthreads();
    const int off = carry + warp_sums[wid] + incl - q;
    if (s < n_seq) {
      q_off[s] = off;
      q_len[s] = q;
      const int g = gen_len[s];
      const int p0 = prompt_len[s] + g - 1;
      pos0[s] = p0;
      for (int i = 0; i < q; ++i) {
        tokens[off + i] = i == 0 ? gen_tok[(size_t)s * gen_stride + g - 1] : draft_tok[(size_t)s * draft_stride + i - 1];
        pos[off + i] = p0 + i;
        row_slot[off + i] = kv_slot[s];
        if (row_key) row_key[off + i] = seq_key[s];
      }
      if (q > 0) {
        // flop / KV-byte accounting of the forward (integers: order independent)
        my_rows_pos += (unsigned long long)q * (unsigned long long)(p0 + 1) + (unsigned long long)q * (q - 1) / 2;
        my_ctx += (unsigned long long)(p0 + q);
      }
      if (qhist) atomicAdd(&s_hist[q < qhist_len - 1 ? q : qhist_len - 1], 1u);
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = off + q;
    __syncthreads();
  }
  if (acc) {
    atomicAdd(&s_rows_pos, my_rows_pos);
    atomicAdd(&s_ctx, my_ctx);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    m_out[0] = carry;
    if (acc) {   // [rows, iterations with rows, sum (pos + 1) over rows, sum (ctx + q) over live sequences]
      acc[0] += carry;
      acc[1] += carry > 0;
      acc[2] += (long long)s_rows_pos;
      acc[3] += (long long)s_ctx;
    }
  }
  if (qhist)
    for (int i = threadIdx.x; i < qhist_len; i += blockDim.x) qhist[i] += s_hist[i];
}

}  // namespace hm

extern "C" int hm_embed(const int32_t* d_tokens, const void* d_emb, int32_t M, int32_t d, float* d_x,
                        const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  hm::k_embed<<<M < 2368 ? M : 2368, 128, 0, (cudaStream_t)stream>>>(d_tokens, (const __nv_bfloat16*)d_emb, M, d, d_m, d_x);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_rmsnorm(const float* d_x, const void* d_w, int32_t M, int32_t d, float eps, void* d_out,
                          const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (d % 4) { hm_set_error("rmsnorm: d % 4"); return HM_ERR_INVALID; }
  const int rows = 8;
  hm::k_rmsnorm<<<(M + rows - 1) / rows < 1184 ? (M + rows - 1) / rows : 1184, 32 * rows, 0, (cudaStream_t)stream>>>(
      d_x, (const __nv_bfloat16*)d_w, M, d, eps, d_m, (__nv_bfloat16*)d_out);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_rmsnorm_residual(float* d_x, const float* d_y, const void* d_w, int32_t M, int32_t d, float eps,
                                   void* d_out, const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (d % 4 || d > 4096) { hm_set_error("rmsnorm_residual: d % 4 == 0 and d <= 4096"); return HM_ERR_INVALID; }
  if (!d_y) return hm_rmsnorm(d_x, d_w, M, d, eps, d_out, d_m, stream);
  const int rows = 8;
  const dim3 grid((M + rows - 1) / rows < 1184 ? (M + rows - 1) / rows : 1184), block(32 * rows);
  cudaStream_t st = (cudaStream_t)stream;
  const __nv_bfloat16* w = (const __nv_bfloat16*)d_w;
  __nv_bfloat16* out = (__nv_bfloat16*)d_out;
  const int nv = (d + 127) / 128;
  if (nv <= 2) hm::k_rmsnorm_residual<2><<<grid, block, 0, st>>>(d_x, d_y, w, M, d, eps, d_m, out);
  else if (nv <= 4) hm::k_rmsnorm_residual<4><<<grid, block, 0, st>>>(d_x, d_y, w, M, d, eps, d_m, out);
  else if (nv <= 8) hm::k_rmsnorm_residual<8><<<grid, block, 0, st>>>(d_x, d_y, w, M, d, eps, d_m, out);
  else if (nv <= 12) hm::k_rmsnorm_residual<12><<<grid, block, 0, st>>>(d_x, d_y, w, M, d, eps, d_m, out);
  else if (nv <= 16) hm::k_rmsnorm_residual<16><<<grid, block, 0, st>>>(d_x, d_y, w, M, d, eps, d_m, out);
  else if (nv <= 24) hm::k_rmsnorm_residual<24><<<grid, block, 0, st>>>(d_x, d_y, w, M, d, eps, d_m, out);
  else hm::k_rmsnorm_residual<32><<<grid, block, 0, st>>>(d_x, d_y, w, M, d, eps, d_m, out);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_rmsnorm_residual2(float* d_x, const float* d_y, const float* d_y2, const void* d_w, int32_t M,
                                    int32_t d, float eps, void* d_out, const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (d % 4) { hm_set_error("rmsnorm_residual2: d % 4 == 0"); return HM_ERR_INVALID; }
  if (d_y2 && !d_y) { hm_set_error("rmsnorm_residual2: y2 needs y"); return HM_ERR_INVALID; }
  if (!d_y2 && d <= 4096) return hm_rmsnorm_residual(d_x, d_y, d_w, M, d, eps, d_out, d_m, stream);
  const int rows = 8;
  hm::k_rmsnorm_residual_g<<<(M + rows - 1) / rows < 1184 ? (M + rows - 1) / rows : 1184, 32 * rows, 0,
                             (cudaStream_t)stream>>>(d_x, d_y, d_y2, (const __nv_bfloat16*)d_w, M, d, eps, d_m,
                                                     (__nv_bfloat16*)d_out);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_rmsnorm_residual_bf16(void* d_x, const void* d_y, const void* d_y2, const void* d_w, int32_t M,
                                        int32_t d, float eps, void* d_out, const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (d % 8 || d > 8192) { hm_set_error("rmsnorm_residual_bf16: d % 8 == 0 and d <= 8192"); return HM_ERR_INVALID; }
  if (d_y2 && !d_y) { hm_set_error("rmsnorm_residual_bf16: y2 needs y"); return HM_ERR_INVALID; }
  const int rows = 8;
  const dim3 grid((M + rows - 1) / rows < 1184 ? (M + rows - 1) / rows : 1184), block(32 * rows);
  cudaStream_t st = (cudaStream_t)stream;
  auto* x = (__nv_bfloat16*)d_x;
  auto* y = (const __nv_bfloat16*)d_y;
  auto* y2 = (const __nv_bfloat16*)d_y2;
  auto* w = (const __nv_bfloat16*)d_w;
  auto* out = (__nv_bfloat16*)d_out;
  const int nv = (d + 255) / 256;
  if (nv <= 2) hm::k_rmsnorm_residual_bf16<2><<<grid, block, 0, st>>>(x, y, y2, w, M, d, eps, d_m, out);
  else if (nv <= 4) hm::k_rmsnorm_residual_bf16<4><<<grid, block, 0, st>>>(x, y, y2, w, M, d, eps, d_m, out);
  else if (nv <= 8) hm::k_rmsnorm_residual_bf16<8><<<grid, block, 0, st>>>(x, y, y2, w, M, d, eps, d_m, out);
  else if (nv <= 16) hm::k_rmsnorm_residual_bf16<16><<<grid, block, 0, st>>>(x, y, y2, w, M, d, eps, d_m, out);
  else hm::k_rmsnorm_residual_bf16<32><<<grid, block, 0, st>>>(x, y, y2, w, M, d, eps, d_m, out);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_embed_bf16(const int32_t* d_tok, const void* d_emb, int32_t M, int32_t d, void* d_x,
                             const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (d % 8) { hm_set_error("embed_bf16: d % 8 == 0"); return HM_ERR_INVALID; }
  hm::k_embed_bf16<<<M < 4096 ? M : 4096, 128, 0, (cudaStream_t)stream>>>(d_tok, (const __nv_bfloat16*)d_emb, M, d,
                                                                         d_m, (__nv_bfloat16*)d_x);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_tp_barrier(int32_t* d_my_flag, int32_t* d_peer_flag, int32_t* d_gen, hm_stream_t stream) {
  if (!d_my_flag || !d_peer_flag || !d_gen) { hm_set_error("hm_tp_barrier: null pointer"); return HM_ERR_INVALID; }
  hm::k_tp_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(d_my_flag, d_peer_flag, d_gen);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_rope_kv_append(const void* d_qkv, const int32_t* d_pos, const int32_t* d_row_slot,
                                 const float* d_cos, const float* d_sin, int32_t M, int32_t H, int32_t KVH,
                                 int32_t hd, void* d_q, void* d_kcache, void* d_vcache, int64_t slot_stride,
                                 int32_t max_len, const int32_t* d_m, hm_stream_t stream) {
  if (M <= 0) return HM_OK;
  if (hd % 16) { hm_set_error("rope: head_dim % 16"); return HM_ERR_INVALID; }
  hm::k_rope_kv<<<M < 2368 ? M : 2368, 128, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)d_qkv, d_pos, d_row_slot, d_cos, d_sin,
                                                     M, H, KVH, hd, (__nv_bfloat16*)d_q, (__nv_bfloat16*)d_kcache,
                                                     (__nv_bfloat16*)d_vcache, slot_stride, max_len, d_m);
  HM_LAUNCH_CHECK();
  return HM_OK;
}

extern "C" int hm_build_verify_batch(int32_t n_seq, const int32_t* d_gen_tok, int32_t gen_stride,
                                     const int32_t* d_gen_len, const int32_t* d_target_len,
                                     const int32_t* d_prompt_len, const int32_t* d_draft_tok, int32_t draft_stride,
                                     const int32_t* d_draft_len, const int32_t* d_kv_slot, int32_t* d_tokens,
                                     int32_t* d_pos, int32_t* d_row_slot, int32_t* d_q_off, int32_t* d_q_len,
                                     int32_t* d_pos0, int32_t* d_m, int64_t* d_acc, int64_t* d_qhist,
                                     int32_t qhist_len, const int32_t* d_seq_key, int32_t* d_row_key,
                                     hm_stream_t stream) {
  if (n_seq <= 0) return HM_OK;
  if ((d_seq_key == nullptr) != (d_row_key == nullptr)) {
    hm_set_error("hm_build_verify_batch: d_seq_key and d_row_key go together");
    return HM_ERR_INVALID;
  }
  if (d_qhist && (qhist_len < 2 || qhist_len > 64)) {
    hm_set_error("hm_build_verify_batch: qhist_len must be in [2, 64]");
    return HM_ERR_INVALID;
  }
  hm::k_build_verify<<<1, 1024, 0, (cudaStream_t)stream>>>(n_seq, d_gen_tok, gen_stride, d_gen_len, d_target_len,
                                                           d_prompt_len, d_draft_tok, draft_stride, d_draft_len,
                                                           d_kv_slot, d_tokens, d_pos, d_row_slot, d_q_off, d_q_len,
                                                           d_pos0, d_m, (long long*)d_acc, (long long*)d_qhist,
                                                           qhist_len, d_seq_key, d_row_key);
  HM_LAUNCH_CHECK();
  return HM_OK;
}
