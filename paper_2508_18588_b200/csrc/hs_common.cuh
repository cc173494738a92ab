// Shared device helpers for the HistoSpec kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/histospec.h"

#define HS_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) { hs_set_error(cudaGetErrorString(_e)); return HS_ERR_CUDA; } \
  } while (0)

void hs_set_error(const char* msg);
void hs_count_launches(int64_t n);

namespace hs {

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

// 64-bit hash of (slot, m, tokens[0..m)).  Same function is used at build and
// probe time; collisions are harmless because every hit is verified against
// the text.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27; x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// Polynomial gram hash: mix64(seed(slot, m) + sum_j (tok_j + 1) * P^(j+1)) mod 2^64.
// Each term depends on one token only, so a warp / lane group computes the terms
// in parallel and reduces them with shuffles (order independent mod 2^64).
constexpr uint64_t kHashP = 0x9E3779B97F4A7C15ULL;
struct PowTable {
  uint64_t v[HS_MAX_TABLE_PREFIX];
  constexpr PowTable() : v() {
    uint64_t p = kHashP;
    for (int i = 0; i < HS_MAX_TABLE_PREFIX; ++i) { v[i] = p; p *= kHashP; }
  }
};
static __constant__ PowTable kPow = PowTable();

// Linear in (slot, m): the final mix64 of gram_hash does the avalanche.  Hash
// collisions only lengthen probe sequences -- a lookup accepts an entry after
// the slot-range check and a text comparison, never on the hash alone.
__host__ __device__ __forceinline__ uint64_t gram_seed(int32_t slot, int32_t m) {
  return (uint64_t)((uint32_t)slot + 1u) * 0xD6E8FEB86659FD93ULL + (uint64_t)(uint32_t)m * 0xA0761D6478BD642FULL;
}
__device__ __forceinline__ uint64_t gram_term(int32_t tok, int j) {
  return (uint64_t)((uint32_t)tok + 1u) * kPow.v[j];
}
__device__ __forceinline__ uint64_t gram_hash(int32_t slot, int32_t m, const int32_t* tok) {
  uint64_t s = 0;
  for (int j = 0; j < m; ++j) s += gram_term(tok[j], j);
  return mix64(gram_seed(slot, m) + s);
}

// Hash-table tag: high bits of the hash with m in the low 6 bits.
__host__ __device__ __forceinline__ int32_t gram_tag(uint64_t h, int32_t m) {
  return (int32_t)(((uint32_t)(h >> 32) & ~0x3Fu) | (uint32_t)m);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace hs
