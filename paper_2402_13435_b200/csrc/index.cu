// K0: device index build -- turns FrozenIndex's row-major arrays
// (corpus.hpp:114-123; freeze layout corpus.cpp:97-123) into the B200 column
// store described in device.cuh.  Build-time only (not on the query path);
// the one-off postings sort uses CUB from the CUDA toolkit.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>

#include "device.cuh"
#include "kernels.cuh"
#include "tc_score.cuh"

namespace hyreb {

namespace {

template <class T>
T* dmalloc(size_t n) {
  T* p = nullptr;
  if (n) HYRE_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

struct DFree {
  void operator()(void* p) const { cudaFree(p); }
};
template <class T>
using DPtr = std::unique_ptr<T, DFree>;

__global__ void count_kernel(const uint32_t* offsets, uint32_t C, uint32_t n, uint32_t* counts) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    counts[r] = offsets[static_cast<size_t>(r) * (C + 1) + C];
}

// One posting per (row, slot, attribute): key = (slot << 32) | id, value = local row.
__global__ void emit_kernel(const uint32_t* attributes, const uint32_t* offsets, uint32_t C,
                            uint32_t A, uint32_t n, const uint64_t* pos, uint64_t* keys,
                            uint32_t* vals) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const uint32_t* off = offsets + static_cast<size_t>(r) * (C + 1);
    const uint32_t* att = attributes + static_cast<size_t>(r) * A;
    uint64_t p = pos[r];
    for (uint32_t c = 0; c < C; ++c)
      for (uint32_t i = off[c]; i < off[c + 1]; ++i) {
        keys[p] = (static_cast<uint64_t>(c) << 32) | att[i];
        vals[p] = r;
        ++p;
      }
  }
}

// Forward index for the batched mask evaluator (K1b): per row, the term ids
// of its attributes in slot order, fixed width A, 0xFFFF padding.
__global__ void row_terms_kernel(const uint64_t* keys, const uint64_t* pos, uint32_t n, uint64_t P,
                                 const uint64_t* uniq, uint32_t T, uint32_t A, uint16_t* out) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const uint64_t b = pos[r], e = r + 1 < n ? pos[r + 1] : P;
    for (uint32_t j = 0; j < A; ++j) {
      uint16_t v = 0xFFFFu;
      if (b + j < e) {
        const uint64_t key = keys[b + j];
        uint32_t lo = 0, hi = T;  // first uniq >= key
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (uniq[mid] < key) lo = mid + 1; else hi = mid;
        }
        v = static_cast<uint16_t>(lo);
      }
      out[static_cast<size_t>(r) * A + j] = v;
    }
  }
}

// Compact CNF rows for K3's fused evaluator: per row the term ids as u8
// (T <= 255) or u16, padded with the all-ones sentinel to `wb` bytes, and a
// u64 of masks: low word = segment starts (bit j: id j opens a new slot
// segment, j >= 1), high word = slots present in the row.
__global__ void cnf_rows_kernel(const uint16_t* row_terms, const uint8_t* slot_of, uint32_t n, uint32_t A,
                                uint32_t tb, uint32_t wb, uint8_t* ids, uint64_t* masks) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const uint16_t* src = row_terms + static_cast<size_t>(r) * A;
    uint8_t* dst = ids + static_cast<size_t>(r) * wb;
    uint32_t starts = 0, pres = 0, prev = 0xFFFFFFFFu;
    for (uint32_t j = 0; j < wb / tb; ++j) {
      const uint32_t t = j < A ? src[j] : 0xFFFFu;
      if (t != 0xFFFFu) {
        const uint32_t sl = slot_of[t];
        if (j > 0 && sl != prev) starts |= 1u << j;
        pres |= 1u << sl;
        prev = sl;
      }
      if (tb == 1) dst[j] = static_cast<uint8_t>(t == 0xFFFFu ? 0xFFu : t);
      else reinterpret_cast<uint16_t*>(dst)[j] = static_cast<uint16_t>(t);
    }
    masks[r] = (static_cast<uint64_t>(pres) << 32) | starts;
  }
}

// HYRE_CNF_GROUPED=0 keeps the segmented CNF rows (A/B measurements).
bool cnf_grouped_enabled() {
  const char* e = std::getenv("HYRE_CNF_GROUPED");
  return !(e && std::string(e) == "0");
}

// Largest number of ids any row holds in one slot (the slot-grouped layout's
// group width W).
__global__ void slot_width_kernel(const uint16_t* row_terms, const uint8_t* slot_of, uint32_t n, uint32_t A,
                                  uint32_t* out) {
  uint32_t mx = 0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const uint16_t* src = row_terms + static_cast<size_t>(r) * A;
    uint32_t run = 0, prev = 0xFFFFFFFFu;
    for (uint32_t j = 0; j < A && src[j] != 0xFFFFu; ++j) {
      const uint32_t sl = slot_of[src[j]];
      run = sl == prev ? run + 1 : 1;
      prev = sl;
      mx = max(mx, run);
    }
  }
  atomicMax(out, mx);
}

// Slot-grouped compact CNF rows (u8 ids): group g (W ids) holds slot g's term
// ids padded with PAD (0xFF: the AND identity), EMPTY_g (T + g: every query
// constraining g fails) when the row has no id in slot g, and NONE (0xFE: no
// constraint) as the first id of the groups beyond the C slots.  The segment
// structure is then static: fail = OR over groups of AND over the group.
__global__ void cnf_group_rows_kernel(const uint16_t* row_terms, const uint8_t* slot_of, uint32_t n, uint32_t A,
                                      uint32_t C, uint32_t T, uint32_t W, uint32_t G, uint32_t wb, uint8_t* ids) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const uint16_t* src = row_terms + static_cast<size_t>(r) * A;
    uint8_t* dst = ids + static_cast<size_t>(r) * wb;
    uint32_t j = 0;
    for (uint32_t g = 0; g < G; ++g) {
      uint32_t k = 0;
      while (g < C && j < A && src[j] != 0xFFFFu && slot_of[src[j]] == g) dst[g * W + k++] = static_cast<uint8_t>(src[j++]);
      if (k == 0) dst[g * W + k++] = static_cast<uint8_t>(g < C ? T + g : 0xFEu);
      for (; k < W; ++k) dst[g * W + k] = 0xFFu;
    }
  }
}

__global__ void slot_of_kernel(const uint64_t* uniq, uint32_t T, uint8_t* slot_of) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x)
    slot_of[t] = static_cast<uint8_t>(uniq[t] >> 32);
}

// x = hi + lo with hi = RNE_bf16(x), lo = RNE_bf16(x - hi): |x - hi - lo| <= 2^-17 |x|.
// Largest squared row norm of the shard (positive floats order like their
// bit patterns): bounds the K3 prefilter error for rows that are not unit
// vectors (an index wrapped from external arrays).
__global__ void max_norm_kernel(const float* src, uint32_t n, uint32_t dp, uint32_t* out) {
  float mx = 0.0f;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (uint32_t e = 0; e < dp; ++e) s = fmaf(src[size_t{r} * dp + e], src[size_t{r} * dp + e], s);
    mx = fmaxf(mx, s);
  }
  atomicMax(out, __float_as_uint(mx));
}

// int8 prefilter plane (K3 "i8" prefilter): one global scale s = max|x| / 127
// (x = the row values the exact rescoring reads: fp32, or bf16 for a bf16
// index), q = clamp(rint(x / s), -127, 127), in the same pre-swizzled
// SWIZZLE_128B tile layout as the bf16 planes (a 128-byte K-atom = 128 int8
// elements).  The largest per-row residual ||x - s q||_2 bounds the prefilter
// error.
__device__ __forceinline__ float prefilter_src(const float* src, size_t i, bool bf16) {
  const float x = src[i];
  return bf16 ? __bfloat162float(__float2bfloat16_rn(x)) : x;
}

__global__ void max_abs_kernel(const float* src, size_t elems, bool bf16, uint32_t* out) {
  float mx = 0.0f;
  for (size_t i = blockIdx.x * size_t{blockDim.x} + threadIdx.x; i < elems; i += size_t{gridDim.x} * blockDim.x)
    mx = fmaxf(mx, fabsf(prefilter_src(src, i, bf16)));
  atomicMax(out, __float_as_uint(mx));
}

__device__ __forceinline__ int8_t quant_i8(float x, float inv) {
  return static_cast<int8_t>(fminf(fmaxf(rintf(x * inv), -127.0f), 127.0f));
}

__global__ void i8_tile_kernel(const float* src, uint32_t n, uint32_t dp, uint32_t kb8, float inv, bool bf16,
                               uint8_t* dst, uint64_t n_chunks) {
  for (uint64_t ci = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; ci < n_chunks;
       ci += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t atom = ci >> 10;  // 1024 chunks per 16 KB atom
    const uint32_t within = static_cast<uint32_t>(ci & 1023);
    const uint32_t rr = within >> 3, pc = within & 7;
    const uint32_t lc = pc ^ (rr & 7);  // logical 16-byte chunk (SWIZZLE_128B)
    const uint32_t k = static_cast<uint32_t>(atom % kb8);
    const uint64_t row = (atom / kb8) * 128 + rr;
    __align__(16) int8_t out[16];
#pragma unroll
    for (int e = 0; e < 16; ++e)
      out[e] = row < n ? quant_i8(prefilter_src(src, row * dp + k * 128 + lc * 16 + e, bf16), inv) : int8_t{0};
    *reinterpret_cast<uint4*>(dst + ci * 16) = *reinterpret_cast<const uint4*>(out);
  }
}

__global__ void i8_resid_kernel(const float* src, uint32_t n, uint32_t dp, float scale, float inv, bool bf16,
                                uint32_t* out) {
  float mx = 0.0f;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint32_t e = 0; e < dp; ++e) {
      const float x = prefilter_src(src, size_t{r} * dp + e, bf16);
      const double d = static_cast<double>(x) - static_cast<double>(scale) * quant_i8(x, inv);
      s += d * d;
    }
    mx = fmaxf(mx, static_cast<float>(sqrt(s)));
  }
  atomicMax(out, __float_as_uint(mx));
}

__global__ void split_kernel(const float* src, size_t n, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  for (size_t i = blockIdx.x * size_t{blockDim.x} + threadIdx.x; i < n; i += size_t{gridDim.x} * blockDim.x) {
    const float x = src[i];
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    hi[i] = h;
    if (lo) lo[i] = __float2bfloat16_rn(x - __bfloat162float(h));
  }
}

// Writes the pre-swizzled tensor-core tiles (see DevIndex::tc_tiles): one
// thread per 16-byte chunk (8 bf16) of the destination.
__global__ void tile_kernel(const float* src, uint32_t n, uint32_t dp, uint32_t kb, uint64_t plane_atoms, uint8_t* dst,
                            uint64_t n_chunks) {
  for (uint64_t ci = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; ci < n_chunks;
       ci += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t atom = ci >> 10;  // 1024 chunks per 16 KB atom
    const uint32_t within = static_cast<uint32_t>(ci & 1023);
    const uint32_t rr = within >> 3, pc = within & 7;  // physical chunk pc of row rr
    const uint32_t lc = pc ^ (rr & 7);                 // logical 16-byte chunk (SWIZZLE_128B)
    const uint32_t o = static_cast<uint32_t>(atom / plane_atoms);  // plane: 0 = hi, 1 = lo
    const uint64_t tk = atom % plane_atoms;
    const uint32_t k = static_cast<uint32_t>(tk % kb);
    const uint64_t row = (tk / kb) * 128 + rr;
    __align__(16) __nv_bfloat16 out[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float x = 0.0f;
      if (row < n) x = src[row * dp + k * 64 + lc * 8 + e];
      const __nv_bfloat16 h = __float2bfloat16_rn(x);
      out[e] = o == 0 ? h : __float2bfloat16_rn(x - __bfloat162float(h));
    }
    *reinterpret_cast<uint4*>(dst + ci * 16) = *reinterpret_cast<const uint4*>(out);
  }
}

uint32_t pad_dim(uint32_t d, bool bf16) {
  const uint32_t lo = bf16 ? 64 : 32, big = bf16 ? 256 : 128;
  if (d <= big) {
    uint32_t p = lo;
    while (p < d) p <<= 1;
    return p;
  }
  return (d + big - 1) / big * big;
}

}  // namespace

DevIndex::~DevIndex() {
  cudaSetDevice(device);
  cudaFree(emb_f32);
  cudaFree(emb_hi);
  cudaFree(tc_tiles);
  cudaFree(tc_i8);
  cudaFree(row_terms);
  cudaFree(cnf_ids);
  cudaFree(cnf_masks);
  cudaFree(slot_of);
  cudaFree(sigs);
  cudaFree(bitmaps);
  cudaFree(post_rows);
  cudaFree(row_w);
}

void set_row_weights(DevIndex& ix, const float* w, uint64_t n) {
  HYRE_CUDA(cudaSetDevice(ix.device));
  if (!w) {
    HYRE_CUDA(cudaDeviceSynchronize());
    cudaFree(ix.row_w);
    ix.row_w = nullptr;
    return;
  }
  if (n != ix.n_rows)
    validation("row weights: expected " + std::to_string(ix.n_rows) + " weights, got " + std::to_string(n));
  for (uint64_t i = 0; i < n; ++i)
    if (!(w[i] >= 0.0f && w[i] <= 1.0f))  // also rejects NaN
      validation("row weight " + std::to_string(i) + " = " + std::to_string(w[i]) + " outside [0, 1]");
  if (!ix.row_w) ix.row_w = dmalloc<float>(std::max<uint64_t>(n, 1));
  HYRE_CUDA(cudaMemcpy(ix.row_w, w, n * sizeof(float), cudaMemcpyHostToDevice));
}

DevIndex* build_device_index(const Frozen& f, const hyre_index_options& o) {
  const uint32_t rb = o.row_begin;
  const uint32_t re = o.row_end == 0 ? f.num_docs : o.row_end;
  if (rb >= re || re > f.num_docs) validation("index shard rows out of range");
  if (o.emb_dtype != HYRE_EMB_F32 && o.emb_dtype != HYRE_EMB_BF16) validation("unknown embedding dtype");
  HYRE_CUDA(cudaSetDevice(o.device));
  std::unique_ptr<DevIndex> ix(new DevIndex);
  ix->device = o.device;
  const uint32_t n = re - rb;
  const uint32_t C = f.num_clauses, A = f.max_num_attr, d = f.dim;
  ix->n_rows = n;
  ix->row_base = o.row_offset + rb;
  ix->dim = d;
  ix->emb_dtype = o.emb_dtype;
  ix->tensor_path = o.tensor_path != 0;
  ix->num_clauses = C;
  ix->max_num_attr = A;
  ix->num_bits = f.num_bits;
  ix->num_words = static_cast<uint32_t>(f.num_words());
  ix->seed = f.seed;
  ix->codec = make_codec(d, f.num_bits, f.seed);
  const bool bf16 = o.emb_dtype == HYRE_EMB_BF16;
  ix->dp = pad_dim(d, bf16);
  const uint32_t dp = ix->dp;
  const uint32_t w_raw = (n + 31) / 32;
  ix->words = (w_raw + kChunkWords - 1) / kChunkWords * kChunkWords;
  ix->n_chunks = ix->words / kChunkWords;
  cudaStream_t st = 0;

  // ---- embeddings --------------------------------------------------------
  {
    const size_t elems = size_t{n} * dp;
    float* f32 = dmalloc<float>(elems);
    HYRE_CUDA(cudaMemset(f32, 0, elems * sizeof(float)));
    HYRE_CUDA(cudaMemcpy2D(f32, dp * sizeof(float), f.embeddings.data() + size_t{rb} * d,
                           d * sizeof(float), d * sizeof(float), n, cudaMemcpyHostToDevice));
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((elems + 255) / 256, 148 * 64));
    {
      DPtr<uint32_t> mx(dmalloc<uint32_t>(1));
      HYRE_CUDA(cudaMemset(mx.get(), 0, 4));
      max_norm_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(f32, n, dp,
                                                                                                          mx.get());
      uint32_t bits = 0;
      HYRE_CUDA(cudaMemcpy(&bits, mx.get(), 4, cudaMemcpyDeviceToHost));
      float sq;
      std::memcpy(&sq, &bits, 4);
      ix->max_row_norm = std::sqrt(sq) * (1.0f + 1e-6f);
    }
    if (dp % 64 == 0 && (ix->tensor_path || bf16)) {
      const uint32_t kb = dp / 64, ops = bf16 ? 1 : 2;
      const uint64_t n_tiles = (n + 127) / 128;
      const uint64_t tc_bytes = n_tiles * kb * ops * 16384;
      ix->tc_tiles = dmalloc<uint8_t>(tc_bytes);
      const uint64_t n_chunks = tc_bytes / 16;
      tile_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n_chunks + 255) / 256, 148 * 64)), 256, 0, st>>>(
          f32, n, dp, kb, n_tiles * kb, ix->tc_tiles, n_chunks);
      HYRE_CUDA(cudaGetLastError());
      ix->tc_ops = ops;
      ix->tc_plane_bytes = n_tiles * kb * 16384;
      ix->has_tc = true;
      ix->stats.tensor_bytes = tc_bytes;
    }
    if (dp % 128 == 0 && (ix->tensor_path || bf16)) {
      DPtr<uint32_t> mx(dmalloc<uint32_t>(2));
      HYRE_CUDA(cudaMemset(mx.get(), 0, 8));
      max_abs_kernel<<<148 * 8, 256, 0, st>>>(f32, elems, bf16, mx.get());
      uint32_t bits = 0;
      HYRE_CUDA(cudaMemcpy(&bits, mx.get(), 4, cudaMemcpyDeviceToHost));
      float amax;
      std::memcpy(&amax, &bits, 4);
      if (amax > 0.0f) {
        const float scale = amax / 127.0f, inv = 127.0f / amax;
        const uint32_t kb8 = dp / 128;
        const uint64_t n_tiles = (n + 127) / 128, i8_bytes = n_tiles * kb8 * 16384, n_chunks = i8_bytes / 16;
        ix->tc_i8 = dmalloc<uint8_t>(i8_bytes);
        i8_tile_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n_chunks + 255) / 256, 148 * 64)), 256, 0, st>>>(
            f32, n, dp, kb8, inv, bf16, ix->tc_i8, n_chunks);
        i8_resid_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(
            f32, n, dp, scale, inv, bf16, mx.get() + 1);
        HYRE_CUDA(cudaGetLastError());
        HYRE_CUDA(cudaMemcpy(&bits, mx.get() + 1, 4, cudaMemcpyDeviceToHost));
        float rmax;
        std::memcpy(&rmax, &bits, 4);
        ix->i8_scale = scale;
        ix->i8_rmax = rmax * (1.0f + 1e-5f) + 1e-7f;
        ix->stats.tensor_bytes += i8_bytes;
      }
    }
    if (bf16) {
      ix->emb_hi = dmalloc<__nv_bfloat16>(elems);
      split_kernel<<<blocks, 256, 0, st>>>(f32, elems, ix->emb_hi, nullptr);
      HYRE_CUDA(cudaGetLastError());
      HYRE_CUDA(cudaDeviceSynchronize());
      cudaFree(f32);
    } else {
      ix->emb_f32 = f32;
    }
    ix->stats.embedding_bytes = elems * (bf16 ? 2 : 4);
  }

  // ---- signatures --------------------------------------------------------
  {
    const size_t nw = f.num_words();
    ix->sigs = dmalloc<uint64_t>(size_t{n} * nw);
    HYRE_CUDA(cudaMemcpy(ix->sigs, f.signatures.data() + size_t{rb} * nw, size_t{n} * nw * 8,
                         cudaMemcpyHostToDevice));
    ix->stats.signature_bytes = size_t{n} * nw * 8;
  }

  // ---- term postings -----------------------------------------------------
  {
    DPtr<uint32_t> att(dmalloc<uint32_t>(size_t{n} * A));
    DPtr<uint32_t> off(dmalloc<uint32_t>(size_t{n} * (C + 1)));
    HYRE_CUDA(cudaMemcpy(att.get(), f.attributes.data() + size_t{rb} * A, size_t{n} * A * 4,
                         cudaMemcpyHostToDevice));
    HYRE_CUDA(cudaMemcpy(off.get(), f.offsets.data() + size_t{rb} * (C + 1),
                         size_t{n} * (C + 1) * 4, cudaMemcpyHostToDevice));
    DPtr<uint32_t> cnt(dmalloc<uint32_t>(n));
    DPtr<uint64_t> pos(dmalloc<uint64_t>(size_t{n} + 1));
    const unsigned blocks = std::min(4096u, (n + 255) / 256);
    count_kernel<<<blocks, 256>>>(off.get(), C, n, cnt.get());
    HYRE_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.get(), pos.get(), n + 1);
    // scan over n+1 entries: the last entry reads cnt[n] -> use n and add total separately
    tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.get(), pos.get(), n);
    DPtr<uint8_t> tmp(dmalloc<uint8_t>(tmp_bytes));
    cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, cnt.get(), pos.get(), n);
    uint64_t last_pos = 0;
    uint32_t last_cnt = 0;
    HYRE_CUDA(cudaMemcpy(&last_pos, pos.get() + n - 1, 8, cudaMemcpyDeviceToHost));
    HYRE_CUDA(cudaMemcpy(&last_cnt, cnt.get() + n - 1, 4, cudaMemcpyDeviceToHost));
    const uint64_t P = last_pos + last_cnt;
    ix->n_postings = P;
    cnt.reset();
    if (P > 0) {
      DPtr<uint64_t> keys(dmalloc<uint64_t>(P)), keys2(dmalloc<uint64_t>(P));
      DPtr<uint32_t> vals(dmalloc<uint32_t>(P));
      ix->post_rows = dmalloc<uint32_t>(P);
      emit_kernel<<<blocks, 256>>>(att.get(), off.get(), C, A, n, pos.get(), keys.get(), vals.get());
      HYRE_CUDA(cudaGetLastError());
      att.reset();
      off.reset();
      int end_bit = 32;
      while ((uint64_t{1} << (end_bit - 32)) < C) ++end_bit;
      tmp_bytes = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.get(), keys2.get(), vals.get(),
                                      ix->post_rows, P, 0, end_bit);
      tmp.reset(dmalloc<uint8_t>(tmp_bytes));
      HYRE_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, keys.get(), keys2.get(),
                                                vals.get(), ix->post_rows, P, 0, end_bit));
      vals.reset();
      // unique (slot, id) runs
      DPtr<uint64_t> uniq(dmalloc<uint64_t>(P));
      DPtr<uint32_t> runs(dmalloc<uint32_t>(P));
      DPtr<uint32_t> n_runs(dmalloc<uint32_t>(1));
      tmp_bytes = 0;
      cub::DeviceRunLengthEncode::Encode(nullptr, tmp_bytes, keys2.get(), uniq.get(), runs.get(),
                                         n_runs.get(), P);
      tmp.reset(dmalloc<uint8_t>(tmp_bytes));
      HYRE_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), tmp_bytes, keys2.get(), uniq.get(),
                                                   runs.get(), n_runs.get(), P));
      uint32_t T = 0;
      HYRE_CUDA(cudaMemcpy(&T, n_runs.get(), 4, cudaMemcpyDeviceToHost));
      const uint32_t Ap = (A + 7) / 8 * 8;  // 16-byte rows
      if (T <= kForwardMaxTerms && C <= 32 && Ap <= 32) {
        ix->row_terms = dmalloc<uint16_t>(size_t{n} * Ap);
        ix->slot_of = dmalloc<uint8_t>(T);
        row_terms_kernel<<<blocks, 256>>>(keys.get(), pos.get(), n, P, uniq.get(), T, Ap, ix->row_terms);
        slot_of_kernel<<<(T + 255) / 256, 256>>>(uniq.get(), T, ix->slot_of);
        HYRE_CUDA(cudaGetLastError());
        HYRE_CUDA(cudaDeviceSynchronize());
        ix->n_terms_fwd = T;
        ix->stats.forward_bytes = size_t{n} * Ap * 2;
        ix->row_terms_width = Ap;
        // compact CNF rows (K3 fused): ids in as few bytes as T allows, row
        // width an odd multiple of 8 B (bank-conflict-free LDS.64 per row),
        // plus the per-row segment/present masks
        const uint32_t tb = T <= 255 ? 1u : 2u;
        uint32_t jw = A <= 8 ? 8u : (A <= 16 ? 16u : (A <= 24 ? 24u : 32u));
        if (tb == 2 && jw % 16) jw += 8;  // u16 variants: 16 or 32 ids
        // Slot-grouped layout (u8 ids, C <= 8 slots of <= 4 ids): J = W x G
        // with G = 4 or 8 groups; no per-row masks.  Preferred when it is no
        // wider than the segmented row + its 8-byte masks.
        uint32_t W = 0, G = 8;
        if (tb == 1 && C <= 8 && T + C <= 0xFEu && cnf_grouped_enabled()) {
          DPtr<uint32_t> d_w(dmalloc<uint32_t>(1));
          HYRE_CUDA(cudaMemset(d_w.get(), 0, 4));
          slot_width_kernel<<<blocks, 256>>>(ix->row_terms, ix->slot_of, n, Ap, d_w.get());
          HYRE_CUDA(cudaMemcpy(&W, d_w.get(), 4, cudaMemcpyDeviceToHost));
          W = std::max(W, 1u);
          if (C <= 4 && W >= 2) G = 4;  // K3 instantiates J = W x G in {8, 8|16, 12|24, 16|32}
          if (W > 4 || W * G > jw + 8 || W * G > 32) W = 0;
        }
        const uint32_t J = W ? W * G : jw;
        uint32_t wb = (J * tb + 7) / 8 * 8;
        if ((wb / 8) % 2 == 0) wb += 8;
        // whole 128-row tiles (K3 bulk-copies full tiles): sentinel ids, no masks in the tail
        const size_t n_pad = (size_t{n} + 127) / 128 * 128;
        ix->cnf_ids = dmalloc<uint8_t>(n_pad * wb);
        HYRE_CUDA(cudaMemset(ix->cnf_ids, 0xFF, n_pad * wb));
        if (W) {
          cnf_group_rows_kernel<<<blocks, 256>>>(ix->row_terms, ix->slot_of, n, Ap, C, T, W, G, wb, ix->cnf_ids);
        } else {
          ix->cnf_masks = dmalloc<uint64_t>(n_pad);
          HYRE_CUDA(cudaMemset(ix->cnf_masks, 0, n_pad * 8));
          cnf_rows_kernel<<<blocks, 256>>>(ix->row_terms, ix->slot_of, n, Ap, tb, wb, ix->cnf_ids, ix->cnf_masks);
        }
        HYRE_CUDA(cudaGetLastError());
        HYRE_CUDA(cudaDeviceSynchronize());
        ix->cnf_id_bytes = tb;
        ix->cnf_ids_per_row = J;
        ix->cnf_row_bytes = wb;
        ix->cnf_group = W;
        ix->stats.forward_bytes += size_t{n} * (wb + (W ? 0 : 8));
      }
      pos.reset();
      std::vector<uint64_t> hk(T);
      std::vector<uint32_t> hdf(T);
      HYRE_CUDA(cudaMemcpy(hk.data(), uniq.get(), T * 8ull, cudaMemcpyDeviceToHost));
      HYRE_CUDA(cudaMemcpy(hdf.data(), runs.get(), T * 4ull, cudaMemcpyDeviceToHost));
      // Dense terms (df >= W/8) become bitmaps: a bitmap costs W words, a CSR
      // list df words plus a scatter at query time.
      const uint64_t dense_df = std::max<uint64_t>(1, ix->words / 8);
      std::vector<ScatterItem> items;
      std::vector<uint64_t> prefix;
      uint64_t begin = 0, bsum = 0;
      ix->terms.reserve(T);
      for (uint32_t i = 0; i < T; ++i) {
        Term t{UINT32_MAX, hdf[i], begin, i};
        if (hdf[i] >= dense_df) {
          t.bitmap = ix->n_bitmap_terms++;
          items.push_back({begin, hdf[i], t.bitmap});
          prefix.push_back(bsum);
          bsum += hdf[i];
        } else {
          ix->stats.csr_terms++;
          ix->stats.csr_bytes += hdf[i] * 4ull;
        }
        ix->terms.emplace(hk[i], t);
        begin += hdf[i];
      }
      ix->terms.finalize();
      ix->stats.num_terms = T;
      ix->stats.bitmap_terms = ix->n_bitmap_terms;
      if (ix->n_bitmap_terms) {
        const size_t bm_words = size_t{ix->n_bitmap_terms} * ix->words;
        ix->bitmaps = dmalloc<uint32_t>(bm_words);
        HYRE_CUDA(cudaMemset(ix->bitmaps, 0, bm_words * 4));
        DPtr<ScatterItem> ditems(dmalloc<ScatterItem>(items.size()));
        DPtr<uint64_t> dprefix(dmalloc<uint64_t>(prefix.size()));
        HYRE_CUDA(cudaMemcpy(ditems.get(), items.data(), items.size() * sizeof(ScatterItem),
                             cudaMemcpyHostToDevice));
        HYRE_CUDA(cudaMemcpy(dprefix.get(), prefix.data(), prefix.size() * 8, cudaMemcpyHostToDevice));
        launch_scatter(ditems.get(), dprefix.get(), static_cast<uint32_t>(items.size()), bsum,
                       ix->post_rows, ix->bitmaps, ix->words, st);
        HYRE_CUDA(cudaGetLastError());
        HYRE_CUDA(cudaDeviceSynchronize());
        ix->stats.bitmap_bytes = bm_words * 4;
      }
    }
  }
  HYRE_CUDA(cudaDeviceSynchronize());
  ix->stats.num_rows = n;
  ix->stats.row_base = ix->row_base;
  ix->stats.dim = d;
  ix->stats.row_stride = dp;
  ix->stats.postings = ix->n_postings;
  return ix.release();
}

}  // namespace hyreb
