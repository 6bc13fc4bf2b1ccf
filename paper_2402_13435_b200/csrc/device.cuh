// Device-side data structures and helpers for the B200 hot path.
//
// HBM layout of one index shard:
//   emb_f32   N x dp fp32, row-major, dp = padded stride (16-byte chunks,
//             >= 8 chunks per row so a row maps onto 8/16/32 lanes)
//   emb_hi/lo N x dp bf16 (f32 index: RNE split x = hi + lo + O(2^-17 x);
//             bf16 index: emb_hi = RNE(x), no lo) -- TMA/tcgen05 operands
//   bitmaps   T_b x W u32: one eligibility bitmap per dense term
//             (slot, id) with df >= W/8; W = ceil(N/32) padded to 128 words
//   post_rows u32 postings sorted by (slot, id, row): CSR lists of the
//             sparse terms
//   sigs      N x words u64 sign-quant signatures (quantizer.hpp:34-44)
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>

#include <string>
#include <unordered_map>
#include <vector>

#include "host.hpp"

namespace hyreb {

#define HYRE_CUDA(x)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw ::hyreb::Error(e_ == cudaErrorMemoryAllocation ? HYRE_OUT_OF_MEMORY        \
                                                           : HYRE_CUDA_ERROR,          \
                           std::string(#x) + ": " + cudaGetErrorString(e_));           \
  } while (0)

constexpr uint32_t kChunkWords = 128;               // mask words per K1 CTA
constexpr uint32_t kChunkRows = kChunkWords * 32;   // 4096 rows
constexpr uint32_t kSegRows = 1024;                 // rows per scorer warp segment
constexpr uint32_t kMaxQG = 8;                      // queries per CUDA-core scorer pass
constexpr uint32_t kSelectMaxK = 4096;              // smem sort capacity of K4

// Query flags (QParam::flags)
enum : uint32_t {
  QF_ACTIVE = 1u,     // well-formed slot of the batch
  QF_EMB = 2u,        // has an embedding (hybrid); else term-only
  QF_MATCH_ALL = 4u,  // no clauses
  QF_EMPTY = 8u,      // a clause with no indexed term: matches nothing
  QF_QUANT = 16u,     // quant_enabled (decision n_elig > quant_k is made on device)
};

struct QParam {
  uint32_t flags;
  uint32_t k;         // min(k, shard rows)
  uint32_t prog_off;  // into the batch program
  uint32_t quant_k;   // effective quant_k (quant_k or 200 k)
};

struct Term {
  uint32_t bitmap;  // index into bitmaps, or UINT32_MAX if CSR
  uint32_t df;
  uint64_t begin;   // first posting in post_rows
};

struct DevIndex {
  int device = 0;
  uint32_t n_rows = 0, row_base = 0, dim = 0, dp = 0;
  uint32_t words = 0, n_chunks = 0;  // W and W / kChunkWords
  uint32_t emb_dtype = HYRE_EMB_F32;
  bool tensor_path = false;
  uint32_t num_clauses = 0, num_bits = 0, num_words = 0;
  uint64_t seed = 0;
  float* emb_f32 = nullptr;
  __nv_bfloat16* emb_hi = nullptr;
  __nv_bfloat16* emb_lo = nullptr;
  uint64_t* sigs = nullptr;
  uint32_t* bitmaps = nullptr;
  uint32_t n_bitmap_terms = 0;
  uint32_t* post_rows = nullptr;
  uint64_t n_postings = 0;
  std::unordered_map<uint64_t, Term> terms;  // key = (slot << 32) | id
  bool has_tmaps = false;                    // TMA descriptors of emb_hi / emb_lo (K3)
  CUtensorMap tm_hi{}, tm_lo{};
  Codec codec;
  hyre_index_stats stats{};
  ~DevIndex();
};

// Orderable 64-bit candidate key: larger key <=> (higher score, then lower
// global row) -- the reference's tie rule (types.hpp:28, knn.cpp:79-83).
__host__ __device__ __forceinline__ uint32_t f2ord(float f) {
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(f);
#else
  uint32_t u;
  std::memcpy(&u, &f, 4);
#endif
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float ord2f(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  std::memcpy(&f, &u, 4);
  return f;
#endif
}
__host__ __device__ __forceinline__ uint64_t make_key(float s, uint32_t global_row) {
  return (static_cast<uint64_t>(f2ord(s)) << 32) | static_cast<uint32_t>(~global_row);
}
__host__ __device__ __forceinline__ uint32_t key_row(uint64_t k) {
  return ~static_cast<uint32_t>(k);
}
__host__ __device__ __forceinline__ float key_score(uint64_t k) {
  return ord2f(static_cast<uint32_t>(k >> 32));
}

// clamp to [-1, 1] (knn.cpp:37) and fold -0 into +0 so that equal scores
// compare equal in key space exactly as they do as floats.
__device__ __forceinline__ float clamp_score(float s) {
  s = fminf(fmaxf(s, -1.0f), 1.0f);
  return s + 0.0f;
}

}  // namespace hyreb
