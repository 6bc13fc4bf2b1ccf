// Device-side data structures and helpers for the B200 hot path.
//
// HBM layout of one index shard:
//   emb_f32   N x dp fp32, row-major, dp = padded stride (16-byte chunks,
//             >= 8 chunks per row so a row maps onto 8/16/32 lanes)
//   tc_tiles  tensor-core tiles: bf16 RNE split x = hi + lo + O(2^-17 x)
//             (bf16 index: hi only), pre-swizzled 16 KB K-atoms per 128-row
//             tile, contiguous per tile (one bulk copy per pipeline stage)
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
#include <cstdlib>
#include <cstring>

#include <string>
#include <unordered_map>
#include <vector>

#include <atomic>

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

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// be scheduled while its stream predecessor is still running; it must call
// pdl_wait() before touching anything the predecessor (or earlier work)
// writes -- the wait returns once the predecessor grid has completed and its
// memory is visible.  pdl_trigger() lets the successor's CTAs be scheduled as
// soon as resources free up (its prologue then overlaps this kernel's tail).
// Both are no-ops for a normal launch.  HYRE_PDL=0 launches normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("HYRE_PDL");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  HYRE_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: set it once
// per (kernel, device), safe from several host threads (executor pools,
// sharded executors); `done` is a bitmask of devices already set.
inline void set_smem_limit(const void* fn, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  HYRE_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  HYRE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));  // idempotent
  done.fetch_or(bit, std::memory_order_acq_rel);
}

constexpr uint32_t kChunkWords = 128;               // mask words per K1 CTA
constexpr uint32_t kChunkRows = kChunkWords * 32;   // 4096 rows
constexpr uint32_t kSegRows = 1024;                 // rows per scorer warp segment
constexpr uint32_t kMaxQG = 8;                      // queries per CUDA-core scorer pass
constexpr uint32_t kSelectMaxK = 4096;              // smem sort capacity of K4
constexpr uint32_t kForwardMaxTerms = 8192;         // K1b users table must fit shared memory

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
  uint32_t id;      // term id (rank of (slot, id) among all index terms)
};

// Open-addressing term dictionary ((slot << 32) | id -> Term), linear
// probing at <= 50% load: the per-id lookup of every query clause on the
// host path (prepare) without unordered_map's node chasing.
struct TermDict {
  std::vector<uint64_t> keys;  // ~0 = empty
  std::vector<Term> vals;
  uint64_t mask = 0;
  void reserve(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    keys.assign(cap, ~0ull);
    vals.assign(cap, Term{});
    mask = cap - 1;
  }
  static uint64_t hash(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return k;
  }
  void emplace(uint64_t k, const Term& t) {
    for (uint64_t i = hash(k) & mask;; i = (i + 1) & mask)
      if (keys[i] == ~0ull || keys[i] == k) {
        keys[i] = k;
        vals[i] = t;
        return;
      }
  }
  const Term* find(uint64_t k) const {
    if (!dense.empty()) {  // direct (slot, id) table
      const uint64_t slot = k >> 32, id = k & 0xFFFFFFFFu;
      if (slot >= dense_base.size() - 1 || id >= dense_base[slot + 1] - dense_base[slot]) return nullptr;
      const uint32_t at = dense[dense_base[slot] + id];
      return at == UINT32_MAX ? nullptr : &vals[at];
    }
    if (keys.empty()) return nullptr;
    for (uint64_t i = hash(k) & mask;; i = (i + 1) & mask) {
      if (keys[i] == k) return &vals[i];
      if (keys[i] == ~0ull) return nullptr;
    }
  }
  // After the last emplace: when the ids of every slot are small enough
  // (sum over slots of max id + 1 <= 16M), a direct table replaces probing
  // on the per-query lookup path (one load per clause id).
  std::vector<uint64_t> dense_base;  // [slots + 1] offsets into dense
  std::vector<uint32_t> dense;       // slot table entry -> index into vals, or ~0
  void finalize() {
    uint64_t slots = 0;
    std::vector<uint64_t> max_id;
    for (uint64_t k : keys)
      if (k != ~0ull) {
        const uint64_t s = k >> 32;
        if (s >= max_id.size()) max_id.resize(s + 1, 0);
        max_id[s] = std::max<uint64_t>(max_id[s], k & 0xFFFFFFFFu);
        slots = std::max<uint64_t>(slots, s + 1);
      }
    uint64_t total = 0;
    for (uint64_t s = 0; s < slots; ++s) total += max_id[s] + 1;
    if (slots == 0 || slots > 1024 || total > (16u << 20)) return;
    dense_base.assign(slots + 1, 0);
    for (uint64_t s = 0; s < slots; ++s) dense_base[s + 1] = dense_base[s] + max_id[s] + 1;
    dense.assign(total, UINT32_MAX);
    for (uint64_t i = 0; i < keys.size(); ++i)
      if (keys[i] != ~0ull) dense[dense_base[keys[i] >> 32] + (keys[i] & 0xFFFFFFFFu)] = static_cast<uint32_t>(i);
  }
};

struct DevIndex {
  int device = 0;
  uint32_t n_rows = 0, row_base = 0, dim = 0, dp = 0;
  uint32_t words = 0, n_chunks = 0;  // W and W / kChunkWords
  uint32_t emb_dtype = HYRE_EMB_F32;
  float max_row_norm = 1.0f;  // largest row L2 norm (1 for frozen rows; scales the K3 prefilter bound)
  bool tensor_path = false;
  uint32_t num_clauses = 0, num_bits = 0, num_words = 0;
  uint64_t seed = 0;
  float* emb_f32 = nullptr;
  __nv_bfloat16* emb_hi = nullptr;  // bf16 index: RNE rows, row-major (K2 / gather path)
  // Tensor-core tiles (K3): plane o (0 = hi, 1 = lo for an fp32 index) at
  // o * tc_plane_bytes; within a plane, per 128-row tile t and K-atom k (64
  // elements) a 16 KB block at (t * kb + k) * 16 KB holding the 128 x 128-byte
  // atom in the UMMA canonical K-major SWIZZLE_128B layout (16-byte chunk c of
  // row r at chunk c ^ (r % 8)); tail rows zero.  A pipeline stage is one
  // cp.async.bulk per plane; the prefilter streams the hi plane alone
  // (contiguous, so its DRAM pattern is a plain sequential scan).
  uint8_t* tc_tiles = nullptr;
  uint64_t tc_plane_bytes = 0;
  // int8 prefilter plane (dp % 128 == 0): q = rint(x / i8_scale) in the same
  // tile layout (a K-atom = 128 int8 elements); i8_rmax = the largest row
  // residual ||x - i8_scale q||_2 (the row part of the prefilter bound)
  uint8_t* tc_i8 = nullptr;
  float i8_scale = 0.0f, i8_rmax = 0.0f;
  uint32_t tc_ops = 0;
  uint64_t* sigs = nullptr;
  uint32_t* bitmaps = nullptr;
  uint32_t n_bitmap_terms = 0;
  uint32_t* post_rows = nullptr;
  uint64_t n_postings = 0;
  TermDict terms;  // key = (slot << 32) | id
  bool has_tc = false;                       // tc_tiles present (dp % 64 == 0)
  // Forward term lists (K1b): row_terms[r * A + j] = term id of the row's j-th
  // attribute (slot order, 0xFFFF padding); slot_of[t] = clause slot of term t.
  uint16_t* row_terms = nullptr;
  uint8_t* slot_of = nullptr;
  uint32_t n_terms_fwd = 0, max_num_attr = 0, row_terms_width = 0;
  // Compact CNF rows (K3 fused evaluator): cnf_ids[r * cnf_row_bytes ..] =
  // the row's term ids as u8 (T <= 255) or u16, all-ones padded to
  // cnf_ids_per_row ids (row width an odd multiple of 8 B); cnf_masks[r] =
  // (slots present << 32) | segment starts (bit j: id j opens a new slot).
  uint8_t* cnf_ids = nullptr;
  uint64_t* cnf_masks = nullptr;
  uint32_t cnf_id_bytes = 0, cnf_ids_per_row = 0, cnf_row_bytes = 0;
  // Slot-grouped rows (cnf_group = W > 0, u8 ids, no masks): group g of W ids
  // = slot g's ids, PAD 0xFF, EMPTY_g = T + g for an empty slot, NONE 0xFE
  // leading the groups beyond the C slots (index.cu cnf_group_rows_kernel).
  uint32_t cnf_group = 0;
  uint64_t cnf_row_total() const { return cnf_row_bytes + (cnf_masks ? 8u : 0u); }  // HBM bytes per row
  // Learned per-row weights (north star: "learned link/attribute weights
  // applied in the epilogue"): score = w[r] x clamp(dot), w in [0, 1], local
  // rows; nullptr = identity (the reference's pure cosine, knn.cpp:36-37).
  float* row_w = nullptr;
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
// learned-weight epilogue: w x clamp(s), -0 folded to +0 (a zero weight times
// a negative score ties with every other zero score, ordered by row)
__device__ __forceinline__ float weighted_score(float s, float w) { return clamp_score(s) * w + 0.0f; }

}  // namespace hyreb
