// GPU-side IndexBuilder::freeze (corpus.cpp:54-129) for large builds
// (SURVEY.md §8 f2).  The staged rows go to the device in chunks; per row the
// device performs exactly the host freeze's arithmetic, so the frozen arrays
// are bit-identical to Builder::freeze (and to the reference's):
//   * per clause sort + dedup of the staged ids, zero-padded attributes[N][A],
//     offsets[N][C+1] and the width check on the de-duplicated size
//     (corpus.cpp:61-107) -- one thread per row;
//   * L2 normalisation in double (corpus.cpp:109-119): the sum of squares is
//     sequential in dimension order with separate multiply and add (no FMA,
//     like the reference's x86-64 build), inv = 1 / sqrt(norm) correctly
//     rounded, x_d = float(e_d * inv); zero rows flagged -- one warp per row,
//     lane 0 summing;
//   * the sign-quant signature (quantizer.cpp:51-70): bit b = (sum over its
//     bin, in bin order, of double(sign) * x[perm]) >= 0 -- one lane per bit.
// The result is copied back into a host Frozen (the FrozenIndex the C-ABI
// hands out); rows whose staged slot holds more ids than the device sort
// buffer are canonicalised on the host with Builder::freeze's code.
#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "executor.cuh"

namespace hyreb {

namespace {

constexpr uint32_t kSlotBuf = 48;  // staged ids per slot sorted on the device (more: host fallback)

__global__ void canon_kernel(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ so, uint64_t id_base,
                             uint32_t n, uint32_t C, uint32_t A, uint32_t* __restrict__ attr,
                             uint32_t* __restrict__ offs, uint8_t* __restrict__ flags) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint32_t buf[kSlotBuf];
  uint32_t* a = attr + static_cast<size_t>(r) * A;
  uint32_t* o = offs + static_cast<size_t>(r) * (C + 1);
  uint32_t pos = 0;
  uint8_t fl = 0;  // bit 0: wider than A, bit 1: host fallback
  for (uint32_t c = 0; c < C; ++c) {
    const uint64_t s0 = so[static_cast<size_t>(r) * C + c] - id_base, s1 = so[static_cast<size_t>(r) * C + c + 1] - id_base;
    o[c] = pos;
    if (s1 - s0 > kSlotBuf) {
      fl |= 2u;
      continue;
    }
    const uint32_t m = static_cast<uint32_t>(s1 - s0);
    for (uint32_t i = 0; i < m; ++i) {  // insertion sort (a handful of ids per slot)
      const uint32_t v = ids[s0 + i];
      uint32_t j = i;
      while (j > 0 && buf[j - 1] > v) {
        buf[j] = buf[j - 1];
        --j;
      }
      buf[j] = v;
    }
    for (uint32_t i = 0; i < m; ++i) {
      if (i > 0 && buf[i] == buf[i - 1]) continue;  // dedup
      if (pos < A) a[pos] = buf[i];
      ++pos;
    }
    if (pos > A) fl |= 1u;
  }
  o[C] = min(pos, A);
  for (uint32_t p = pos; p < A; ++p) a[p] = 0u;  // zero padding
  flags[r] = fl;
}

// One warp per row: normalisation (lane 0 sums in dimension order) and the
// signature bits (one lane per bit, 32 bits per ballot).
__global__ void norm_encode_kernel(const float* __restrict__ emb, uint32_t n, uint32_t dim, float* __restrict__ out,
                                   uint8_t* __restrict__ zero, uint64_t* __restrict__ sigs, uint32_t num_bits,
                                   const uint32_t* __restrict__ bit_lo, const uint32_t* __restrict__ bit_hi,
                                   const uint32_t* __restrict__ perm, const float* __restrict__ signs) {
  extern __shared__ float xs[];  // [warps][dim]
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t r = blockIdx.x * (blockDim.x >> 5) + wib;
  if (r >= n) return;
  float* x = xs + static_cast<size_t>(wib) * dim;
  const float* e = emb + static_cast<size_t>(r) * dim;
  for (uint32_t d = lane; d < dim; d += 32) x[d] = e[d];
  __syncwarp();
  double inv = 0.0;
  if (lane == 0) {
    double nsq = 0.0;
    for (uint32_t d = 0; d < dim; ++d) {
      const double v = static_cast<double>(x[d]);
      nsq = __dadd_rn(nsq, __dmul_rn(v, v));
    }
    inv = nsq == 0.0 ? 0.0 : __ddiv_rn(1.0, __dsqrt_rn(nsq));
    zero[r] = nsq == 0.0 ? 1 : 0;
  }
  inv = __shfl_sync(0xffffffffu, inv, 0);
  __syncwarp();
  float* o = out + static_cast<size_t>(r) * dim;
  for (uint32_t d = lane; d < dim; d += 32) {
    const float v = inv == 0.0 ? 0.0f : __double2float_rn(__dmul_rn(static_cast<double>(x[d]), inv));
    x[d] = v;
    o[d] = v;
  }
  __syncwarp();
  uint32_t* sw = reinterpret_cast<uint32_t*>(sigs + static_cast<size_t>(r) * ((num_bits + 63) / 64));
  for (uint32_t b0 = 0; b0 < ((num_bits + 63) / 64) * 64; b0 += 32) {
    const uint32_t b = b0 + lane;
    bool on = false;
    if (b < num_bits) {
      double agg = 0.0;
      for (uint32_t i = bit_lo[b]; i < bit_hi[b]; ++i)  // flat (round x dim) index
        agg = __dadd_rn(agg, __dmul_rn(static_cast<double>(signs[i]), static_cast<double>(x[perm[i]])));
      on = agg >= 0.0;  // sign(0) = +1
    }
    const uint32_t m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) sw[b0 / 32] = m;
  }
}

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  HYRE_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

}  // namespace

Frozen* freeze_on_device(Builder& bld, uint32_t num_bits, uint64_t seed, int device) {
  if (bld.frozen) validation("builder already frozen");
  if (bld.doc_ids.empty()) validation("no documents staged");
  const Codec codec = make_codec(bld.dim, num_bits, seed);
  bld.frozen = true;  // consumed whatever the outcome (as Builder::freeze)
  HYRE_CUDA(cudaSetDevice(device));
  const uint32_t n = static_cast<uint32_t>(bld.doc_ids.size());
  const uint32_t C = bld.num_clauses, A = bld.max_num_attr, D = bld.dim;
  const size_t words = codec.num_words();

  std::unique_ptr<Frozen> f(new Frozen);  // released to the caller only on success
  f->num_docs = n;
  f->num_clauses = C;
  f->max_num_attr = A;
  f->dim = D;
  f->num_bits = num_bits;
  f->seed = seed;
  f->clause_names = bld.clause_names;
  f->attributes.resize(size_t{n} * A);
  f->offsets.resize(size_t{n} * (C + 1));
  f->embeddings.resize(size_t{n} * D);
  f->signatures.resize(size_t{n} * words);
  f->zero.resize(n);
  std::vector<uint8_t> flags(n);

  // codec tables: per bit its [lo, hi) range of the flat (round, position) arrays
  std::vector<uint32_t> lo(num_bits), hi(num_bits), perm;
  std::vector<float> sg;
  uint32_t bit = 0;
  for (size_t ri = 0; ri < codec.rounds.size(); ++ri) {
    const auto& rd = codec.rounds[ri];
    const uint32_t base = static_cast<uint32_t>(ri * D);
    for (size_t b = 0; b + 1 < rd.bounds.size() && bit < num_bits; ++b, ++bit) {
      lo[bit] = base + rd.bounds[b];
      hi[bit] = base + rd.bounds[b + 1];
    }
    perm.insert(perm.end(), rd.perm.begin(), rd.perm.end());
    sg.insert(sg.end(), rd.signs.begin(), rd.signs.end());
  }
  struct Bufs {  // device buffers freed on every exit
    std::vector<void*> p;
    ~Bufs() {
      for (void* x : p) cudaFree(x);
    }
  } bufs;
  auto keep = [&](auto* x) {
    bufs.p.push_back(x);
    return x;
  };
  uint32_t* d_lo = keep(dalloc<uint32_t>(num_bits));
  uint32_t* d_hi = keep(dalloc<uint32_t>(num_bits));
  uint32_t* d_perm = keep(dalloc<uint32_t>(perm.size()));
  float* d_sg = keep(dalloc<float>(sg.size()));
  HYRE_CUDA(cudaMemcpy(d_lo, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice));
  HYRE_CUDA(cudaMemcpy(d_hi, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
  HYRE_CUDA(cudaMemcpy(d_perm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice));
  HYRE_CUDA(cudaMemcpy(d_sg, sg.data(), sg.size() * 4, cudaMemcpyHostToDevice));

  // chunks of rows bound the device footprint (~1.3 GB per chunk at d = 128)
  const uint32_t chunk = std::max<uint32_t>(1, std::min<uint32_t>(n, static_cast<uint32_t>((1ull << 30) / (size_t{D} * 4 + 64))));
  uint64_t max_ids = 0;
  for (uint32_t r0 = 0; r0 < n; r0 += chunk) {
    const uint32_t r1 = std::min(n, r0 + chunk);
    max_ids = std::max(max_ids, bld.slot_offsets[size_t{r1} * C] - bld.slot_offsets[size_t{r0} * C]);
  }
  uint32_t* d_ids = keep(dalloc<uint32_t>(max_ids));
  uint64_t* d_so = keep(dalloc<uint64_t>(size_t{chunk} * C + 1));
  float* d_emb = keep(dalloc<float>(size_t{chunk} * D));
  float* d_out = keep(dalloc<float>(size_t{chunk} * D));
  uint32_t* d_attr = keep(dalloc<uint32_t>(size_t{chunk} * A));
  uint32_t* d_offs = keep(dalloc<uint32_t>(size_t{chunk} * (C + 1)));
  uint8_t* d_flags = keep(dalloc<uint8_t>(chunk));
  uint8_t* d_zero = keep(dalloc<uint8_t>(chunk));
  uint64_t* d_sig = keep(dalloc<uint64_t>(size_t{chunk} * words));
  const uint32_t warps = 8;
  const size_t smem = size_t{warps} * D * sizeof(float);
  if (smem > 48 * 1024)
    HYRE_CUDA(cudaFuncSetAttribute(norm_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  for (uint32_t r0 = 0; r0 < n; r0 += chunk) {
    const uint32_t m = std::min(chunk, n - r0);
    const uint64_t i0 = bld.slot_offsets[size_t{r0} * C], i1 = bld.slot_offsets[size_t{r0 + m} * C];
    if (i1 > i0) HYRE_CUDA(cudaMemcpy(d_ids, bld.ids.data() + i0, (i1 - i0) * 4, cudaMemcpyHostToDevice));
    HYRE_CUDA(cudaMemcpy(d_so, bld.slot_offsets.data() + size_t{r0} * C, (size_t{m} * C + 1) * 8,
                         cudaMemcpyHostToDevice));
    HYRE_CUDA(cudaMemcpy(d_emb, bld.embeddings.data() + size_t{r0} * D, size_t{m} * D * 4, cudaMemcpyHostToDevice));
    canon_kernel<<<(m + 127) / 128, 128>>>(d_ids, d_so, i0, m, C, A, d_attr, d_offs, d_flags);
    norm_encode_kernel<<<(m + warps - 1) / warps, 32 * warps, smem>>>(d_emb, m, D, d_out, d_zero, d_sig, num_bits,
                                                                     d_lo, d_hi, d_perm, d_sg);
    HYRE_CUDA(cudaGetLastError());
    HYRE_CUDA(cudaMemcpy(f->attributes.data() + size_t{r0} * A, d_attr, size_t{m} * A * 4, cudaMemcpyDeviceToHost));
    HYRE_CUDA(cudaMemcpy(f->offsets.data() + size_t{r0} * (C + 1), d_offs, size_t{m} * (C + 1) * 4,
                         cudaMemcpyDeviceToHost));
    HYRE_CUDA(cudaMemcpy(f->embeddings.data() + size_t{r0} * D, d_out, size_t{m} * D * 4, cudaMemcpyDeviceToHost));
    HYRE_CUDA(cudaMemcpy(f->signatures.data() + size_t{r0} * words, d_sig, size_t{m} * words * 8,
                         cudaMemcpyDeviceToHost));
    HYRE_CUDA(cudaMemcpy(f->zero.data() + r0, d_zero, m, cudaMemcpyDeviceToHost));
    HYRE_CUDA(cudaMemcpy(flags.data() + r0, d_flags, m, cudaMemcpyDeviceToHost));
  }

  // rows with a slot too long for the device sort buffer: the host freeze's
  // canonicalisation (corpus.cpp:61-107)
  std::string too;
  std::vector<uint32_t> tmp;
  for (uint32_t r = 0; r < n; ++r) {
    if (flags[r] & 2u) {
      uint32_t* attr = f->attributes.data() + size_t{r} * A;
      uint32_t* offs = f->offsets.data() + size_t{r} * (C + 1);
      std::fill(attr, attr + A, 0u);
      uint32_t pos = 0;
      flags[r] = 0;
      for (uint32_t c = 0; c < C; ++c) {
        const uint64_t s0 = bld.slot_offsets[size_t{r} * C + c], s1 = bld.slot_offsets[size_t{r} * C + c + 1];
        tmp.assign(bld.ids.begin() + s0, bld.ids.begin() + s1);
        std::sort(tmp.begin(), tmp.end());
        tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
        offs[c] = pos;
        for (auto id : tmp) {
          if (pos < A) attr[pos] = id;
          ++pos;
        }
        if (pos > A) flags[r] = 1;
      }
      offs[C] = std::min(pos, A);
    }
    if (flags[r] & 1u) too += " " + bld.doc_ids.at(r);
  }
  if (!too.empty()) validation("documents wider than maxNumAttr=" + std::to_string(A) + ":" + too);
  f->doc_ids = std::move(bld.doc_ids);
  std::vector<uint32_t>().swap(bld.ids);
  std::vector<float>().swap(bld.embeddings);
  std::vector<uint64_t>().swap(bld.slot_offsets);
  return f.release();
}

}  // namespace hyreb
