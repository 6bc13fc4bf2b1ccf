// Hot-path kernels for sm_100a (B200).  See DESIGN.md §4 for the roofline
// argument behind each one; reference functions are cited per kernel.
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <type_traits>
#include <vector>

#include "kernels.cuh"

namespace hyreb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Inclusive warp scan of a u32.
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Block-wide exclusive scan (blockDim.x multiple of 32, <= 1024).
// `tmp` needs 33 u32 of shared memory.  Returns exclusive prefix; total in *tot.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* tmp, uint32_t* tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = warp_incl_scan(v, lane);
  if (lane == 31) tmp[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t x = lane < nw ? tmp[lane] : 0;
    uint32_t xi = warp_incl_scan(x, lane);
    if (lane < nw) tmp[lane] = xi - x;
    if (lane == 31) tmp[32] = xi;
  }
  __syncthreads();
  uint32_t r = tmp[w] + inc - v;
  *tot = tmp[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint32_t tail_mask(uint32_t widx, uint32_t n_rows) {
  const uint64_t first = static_cast<uint64_t>(widx) * 32;
  if (first >= n_rows) return 0u;
  const uint64_t left = n_rows - first;
  return left >= 32 ? kFull : ((1u << left) - 1u);
}

}  // namespace

// ===========================================================================
// K1: CNF eligibility mask.  One CTA = one chunk of 128 mask words (4096
// rows), 128 threads, thread t owns word t.  All ref words of the chunk are
// staged once into shared memory (each term bitmap is read from HBM exactly
// once per batch), then every query's AND-of-ORs is evaluated from smem.
// Replaces full_scan_tbr (term_match.cpp:56-78) / batch_scan_tbr
// (pipeline.cpp:75-93): bit r of the mask <=> row r is a TBR match.
// ===========================================================================
__global__ void __launch_bounds__(128) mask_kernel(MaskArgs a, uint32_t staged) {
  extern __shared__ uint32_t st[];  // staged refs [n_refs][128] then warp sums [B][4]
  const uint32_t t = threadIdx.x, chunk = blockIdx.x;
  const uint32_t widx = chunk * kChunkWords + t;
  uint32_t* wsum = st + (staged ? a.n_refs * kChunkWords : 0);
  if (staged) {
    for (uint32_t r = 0; r < a.n_refs; ++r) st[r * kChunkWords + t] = __ldg(a.refs[r] + widx);
    __syncthreads();
  }
  const uint32_t tm = tail_mask(widx, a.n_rows);
  const int lane = t & 31, w = t >> 5;
  for (uint32_t q = 0; q < a.B; ++q) {
    const uint32_t flags = a.qp[q].flags;
    uint32_t word = 0;
    if ((flags & QF_ACTIVE) && !(flags & QF_EMPTY)) {
      if (flags & QF_MATCH_ALL) {
        word = tm;
      } else {
        const uint32_t* p = a.prog + a.qp[q].prog_off;
        const uint32_t nc = p[0];
        uint32_t pos = 1, acc = kFull;
        for (uint32_t c = 0; c < nc; ++c) {
          const uint32_t nr = p[pos++];
          uint32_t cw = 0;
          for (uint32_t r = 0; r < nr; ++r) {
            const uint32_t ref = p[pos + r];
            cw |= staged ? st[ref * kChunkWords + t] : __ldg(a.refs[ref] + widx);
          }
          pos += nr;
          acc &= cw;
        }
        word = acc & tm;
      }
    }
    a.mask[static_cast<size_t>(q) * a.words + widx] = word;
    const uint32_t c = __reduce_add_sync(kFull, __popc(word));
    if (lane == 0) wsum[q * 4 + w] = c;
  }
  __syncthreads();
  for (uint32_t q = t; q < a.B; q += blockDim.x) {
    const uint32_t c = wsum[q * 4] + wsum[q * 4 + 1] + wsum[q * 4 + 2] + wsum[q * 4 + 3];
    a.chunk_cnt[static_cast<size_t>(q) * a.n_chunks + chunk] = c;
    if (c) atomicAdd(a.n_elig + q, c);
  }
}

void launch_mask(const MaskArgs& a, cudaStream_t st) {
  if (a.B == 0 || a.n_chunks == 0) return;
  const size_t wsum_bytes = size_t{a.B} * 4 * sizeof(uint32_t);
  const size_t staged_bytes = size_t{a.n_refs} * kChunkWords * sizeof(uint32_t);
  constexpr size_t kSmemCap = 200 * 1024;
  const uint32_t staged = (a.n_refs > 0 && staged_bytes + wsum_bytes <= kSmemCap) ? 1u : 0u;
  const size_t smem = wsum_bytes + (staged ? staged_bytes : 0);
  static std::atomic<uint64_t> attr{0};
  set_smem_limit(reinterpret_cast<const void*>(mask_kernel), 227 * 1024, attr);
  mask_kernel<<<a.n_chunks, kChunkWords, smem, st>>>(a, staged);
}

// Term-major K1 (batched CNF evaluation).  Program layout in c_mask_prog:
//   [0] first group index of this launch, then per group g: [1+2g] offset,
//   [2+2g] live-query mask;
//   at offset: n_slots, then per slot: { constrained-query mask, n_refs,
//   n_refs x (ref pointer lo, ref pointer hi, using-query mask) }.
// Thread t of CTA (chunk, group) owns mask word chunk*128+t for the group's
// 32 queries: for every slot it ORs each ref word into the accumulators of
// the queries that use it (uniform predicates), then ANDs the slot into the
// result of the queries that constrain it.  Each ref word is loaded once per
// group (coalesced), nothing is staged in shared memory.
// The program travels as a __grid_constant__ kernel parameter (per launch,
// served by the constant cache) so concurrent executors never share it.
template <uint32_t N>
struct MaskProg {
  uint32_t w[N];
};

// QN = query slots evaluated per group (1, 8 or 32): single queries and small
// batches skip the unused accumulators (registers, predicated ORs, counts).
template <uint32_t N, int QN>
__global__ void __launch_bounds__(128) mask_tm_kernel(MaskArgs a, const __grid_constant__ MaskProg<N> prog) {
  const uint32_t* c_mask_prog = prog.w;
  __shared__ uint32_t wsum[QN][4];
  const uint32_t t = threadIdx.x, chunk = blockIdx.x, g = blockIdx.y;
  const uint32_t widx = chunk * kChunkWords + t;
  const uint32_t live = c_mask_prog[2 + 2 * g];
  uint32_t pos = c_mask_prog[1 + 2 * g];
  const uint32_t q0 = (c_mask_prog[0] + g) * 32;  // word 0 = first group of this launch
  const uint32_t tm = tail_mask(widx, a.n_rows);
  uint32_t res[QN];
#pragma unroll
  for (int q = 0; q < QN; ++q) res[q] = ((live >> q) & 1u) ? tm : 0u;
  const uint32_t n_slots = c_mask_prog[pos++];
  for (uint32_t s = 0; s < n_slots; ++s) {
    const uint32_t hc = c_mask_prog[pos], n_refs = c_mask_prog[pos + 1];
    pos += 2;
    uint32_t acc[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) acc[q] = 0u;
    // refs are (pointer lo, pointer hi, users) triples; 4 independent word
    // loads are issued before they are consumed.
    uint32_t r = 0;
    for (; r + 4 <= n_refs; r += 4, pos += 12) {
      uint32_t w[4], u[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ptr = (static_cast<uint64_t>(c_mask_prog[pos + 3 * k + 1]) << 32) | c_mask_prog[pos + 3 * k];
        w[k] = __ldg(reinterpret_cast<const uint32_t*>(ptr) + widx);
        u[k] = c_mask_prog[pos + 3 * k + 2];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int q = 0; q < QN; ++q) acc[q] |= ((u[k] >> q) & 1u) ? w[k] : 0u;
    }
    for (; r < n_refs; ++r, pos += 3) {
      const uint64_t ptr = (static_cast<uint64_t>(c_mask_prog[pos + 1]) << 32) | c_mask_prog[pos];
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(ptr) + widx);
      const uint32_t users = c_mask_prog[pos + 2];
#pragma unroll
      for (int q = 0; q < QN; ++q) acc[q] |= ((users >> q) & 1u) ? w : 0u;
    }
#pragma unroll
    for (int q = 0; q < QN; ++q)
      if ((hc >> q) & 1u) res[q] &= acc[q];
  }
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    if (q0 + q < a.B) a.mask[static_cast<size_t>(q0 + q) * a.words + widx] = res[q];
    const uint32_t c = __reduce_add_sync(0xffffffffu, __popc(res[q]));
    if (lane == 0) wsum[q][w] = c;
  }
  __syncthreads();
  if (t < QN && q0 + t < a.B) {
    const uint32_t c = wsum[t][0] + wsum[t][1] + wsum[t][2] + wsum[t][3];
    a.chunk_cnt[static_cast<size_t>(q0 + t) * a.n_chunks + chunk] = c;
    if (c) atomicAdd(a.n_elig + q0 + t, c);
  }
}

// The same for groups of <= 8 queries with four words per thread: one warp
// per 128-word chunk, every ref read as a 16-byte load, so a thread has a
// quarter of the load round trips in flight per byte and the grid fits one
// wave (the single-query mask over 10M rows is load-latency bound).
template <uint32_t N, int QN>
__global__ void __launch_bounds__(128) mask_tm4_kernel(MaskArgs a, const __grid_constant__ MaskProg<N> prog) {
  const uint32_t* c_mask_prog = prog.w;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, g = blockIdx.y;
  const uint32_t chunk = blockIdx.x * 4 + wib;
  if (chunk >= a.n_chunks) return;
  const uint32_t w0 = chunk * kChunkWords + lane * 4;  // this thread's four words
  const uint32_t live = c_mask_prog[2 + 2 * g];
  uint32_t pos = c_mask_prog[1 + 2 * g];
  const uint32_t q0 = (c_mask_prog[0] + g) * 32;
  uint32_t tm[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) tm[x] = tail_mask(w0 + x, a.n_rows);
  uint32_t res[QN][4];
#pragma unroll
  for (int q = 0; q < QN; ++q)
#pragma unroll
    for (int x = 0; x < 4; ++x) res[q][x] = ((live >> q) & 1u) ? tm[x] : 0u;
  const uint32_t n_slots = c_mask_prog[pos++];
  for (uint32_t s = 0; s < n_slots; ++s) {
    const uint32_t hc = c_mask_prog[pos], n_refs = c_mask_prog[pos + 1];
    pos += 2;
    uint32_t acc[QN][4];
#pragma unroll
    for (int q = 0; q < QN; ++q)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[q][x] = 0u;
    for (uint32_t r = 0; r < n_refs; r += 8, pos += 24) {  // up to 8 independent 16-byte loads in flight
      uint4 w[8];
      uint32_t u[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool on = r + k < n_refs;
        const uint64_t ptr = on ? (static_cast<uint64_t>(c_mask_prog[pos + 3 * k + 1]) << 32) | c_mask_prog[pos + 3 * k]
                                : 0ull;
        w[k] = on ? __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(ptr) + w0))
                  : make_uint4(0, 0, 0, 0);
        u[k] = on ? c_mask_prog[pos + 3 * k + 2] : 0u;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int q = 0; q < QN; ++q)
          if ((u[k] >> q) & 1u) {
            acc[q][0] |= w[k].x;
            acc[q][1] |= w[k].y;
            acc[q][2] |= w[k].z;
            acc[q][3] |= w[k].w;
          }
    }
    pos -= 24 * ((n_refs + 7) / 8) - 3 * n_refs;  // the loop advanced by whole batches of 8 refs
#pragma unroll
    for (int q = 0; q < QN; ++q)
      if ((hc >> q) & 1u)
#pragma unroll
        for (int x = 0; x < 4; ++x) res[q][x] &= acc[q][x];
  }
#pragma unroll
  for (int q = 0; q < QN; ++q) {
    if (q0 + q < a.B)
      *reinterpret_cast<uint4*>(a.mask + static_cast<size_t>(q0 + q) * a.words + w0) =
          make_uint4(res[q][0], res[q][1], res[q][2], res[q][3]);
    const uint32_t c = __reduce_add_sync(0xffffffffu, __popc(res[q][0]) + __popc(res[q][1]) + __popc(res[q][2]) +
                                                          __popc(res[q][3]));
    if (lane == 0 && q0 + q < a.B) {
      a.chunk_cnt[static_cast<size_t>(q0 + q) * a.n_chunks + chunk] = c;
      if (c) atomicAdd(a.n_elig + q0 + q, c);
    }
  }
}

template <uint32_t N>
void launch_mask_tm_n(const MaskArgs& a, const std::vector<uint32_t>& words, uint32_t n_groups, uint32_t live_or,
                      cudaStream_t st) {
  MaskProg<N> p;
  std::memcpy(p.w, words.data(), words.size() * 4);
  const dim3 grid(a.n_chunks, n_groups), grid4((a.n_chunks + 3) / 4, n_groups);
  if (live_or <= 1u) mask_tm4_kernel<N, 1><<<grid4, kChunkWords, 0, st>>>(a, p);
  else if (live_or <= 0xFFu) mask_tm4_kernel<N, 8><<<grid4, kChunkWords, 0, st>>>(a, p);
  else mask_tm_kernel<N, 32><<<grid, kChunkWords, 0, st>>>(a, p);
}

uint32_t launch_mask_tm(const MaskArgs& a, const std::vector<std::vector<uint32_t>>& groups,
                        const std::vector<uint32_t>& live, cudaStream_t st) {
  if (a.B == 0 || a.n_chunks == 0) return 0;
  uint32_t launches = 0;
  // pack consecutive groups into launches whose program fits the parameter
  for (size_t g0 = 0; g0 < groups.size();) {
    std::vector<uint32_t> w{static_cast<uint32_t>(g0)};
    size_t g1 = g0, body = 0;
    while (g1 < groups.size() && 1 + 2 * (g1 - g0 + 1) + body + groups[g1].size() <= kMaskProgWords)
      body += groups[g1++].size();
    if (g1 == g0) return launches | 0x80000000u;  // one group alone is too big
    const uint32_t n = static_cast<uint32_t>(g1 - g0);
    w.resize(1 + 2 * n);
    for (size_t g = g0; g < g1; ++g) {
      w[1 + 2 * (g - g0)] = static_cast<uint32_t>(w.size());
      w[2 + 2 * (g - g0)] = live[g];
      w.insert(w.end(), groups[g].begin(), groups[g].end());
    }
    uint32_t live_or = 0;
    for (size_t g = g0; g < g1; ++g) live_or |= live[g];
    if (w.size() <= 1024) launch_mask_tm_n<1024>(a, w, n, live_or, st);
    else launch_mask_tm_n<kMaskProgWords>(a, w, n, live_or, st);
    ++launches;
    g0 = g1;
  }
  return launches;
}

// ===========================================================================
// K1b: forward-index CNF evaluation (the paper's TBR direction, PAPER.md
// appendix: per row, its attributes against the query clauses).  For a batch
// it is the cheaper direction: each row's <= A term ids (2 B each) are read
// once and, per term, a 64-bit mask of the batch queries using that term is
// OR-ed into the row's clause accumulator; clauses are AND-ed across slots.
// All 64 (x NW) queries of the pass are evaluated together per row.  The
// per-query mask words are produced with warp ballots into a shared tile and
// written coalesced; per-chunk eligible counts feed K2/K3/K5 as before.
// CTA = one chunk (4096 rows = 128 mask words), 32 warps x 4 rounds of 32 rows.
// ===========================================================================
template <int NW>
__global__ void __launch_bounds__(1024) fwd_mask_kernel(FwdArgs a) {
  extern __shared__ __align__(16) uint8_t fsm[];
  uint32_t* tile = reinterpret_cast<uint32_t*>(fsm);                     // [64*NW][128]
  uint64_t* users = reinterpret_cast<uint64_t*>(tile + 64 * NW * 128);  // [T][NW]
  uint64_t* hc = users + static_cast<size_t>(a.T) * NW;                 // [C][NW]
  uint8_t* slot_of = reinterpret_cast<uint8_t*>(hc + a.C * NW);         // [T]
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, chunk = blockIdx.x;
  for (uint32_t i = tid; i < a.T * NW; i += blockDim.x) users[i] = 0ull;
  for (uint32_t i = tid; i < a.C * NW; i += blockDim.x) hc[i] = a.hc[i];
  for (uint32_t i = tid; i < a.T; i += blockDim.x) slot_of[i] = a.slot_of[i];
  __syncthreads();
  const uint32_t stride = 1 + 2 * NW;
  for (uint32_t e = tid; e < a.n_entries; e += blockDim.x) {
    const uint32_t* en = a.entries + static_cast<size_t>(e) * stride;
#pragma unroll
    for (int w = 0; w < NW; ++w)
      users[en[0] * NW + w] = (static_cast<uint64_t>(en[2 + 2 * w]) << 32) | en[1 + 2 * w];
  }
  uint64_t live[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) live[w] = a.live[w];
  __syncthreads();
  for (uint32_t rnd = 0; rnd < 4; ++rnd) {
    const uint32_t wl = rnd * 32 + warp;  // word within the chunk
    const uint32_t row = (chunk * kChunkWords + wl) * 32 + lane;
    uint64_t res[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) res[w] = row < a.n_rows ? live[w] : 0ull;
    if (row < a.n_rows) {
      // the row's term ids (slot-major, 0xFFFF padded) in registers: A <= 32
      uint32_t tw[16];
      const uint4* src = reinterpret_cast<const uint4*>(a.row_terms + static_cast<size_t>(row) * a.A);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint4 x = (v * 8 < static_cast<int>(a.A)) ? __ldg(src + v) : make_uint4(~0u, ~0u, ~0u, ~0u);
        tw[4 * v] = x.x;
        tw[4 * v + 1] = x.y;
        tw[4 * v + 2] = x.z;
        tw[4 * v + 3] = x.w;
      }
      uint64_t acc[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) acc[w] = 0ull;
      uint32_t present = 0, sprev = 0;
      // clause accumulators are closed (AND-ed into res) whenever the slot
      // changes; all lookups are independent, so they pipeline
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t t = (j < static_cast<int>(a.A)) ? ((tw[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu) : 0xFFFFu;
        if (t == 0xFFFFu) break;
        const uint32_t sl = slot_of[t];
        const bool change = j > 0 && sl != sprev;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint64_t close = change ? (acc[w] | ~hc[sprev * NW + w]) : ~0ull;
          res[w] &= close;
          acc[w] = (change ? 0ull : acc[w]) | users[t * NW + w];
        }
        present |= 1u << sl;
        sprev = sl;
      }
      if (present) {
#pragma unroll
        for (int w = 0; w < NW; ++w) res[w] &= acc[w] | ~hc[sprev * NW + w];
      }
      // constrained slots the row has no attribute in can never match
      for (uint32_t sl = 0; sl < a.C; ++sl)
        if (!((present >> sl) & 1u))
#pragma unroll
          for (int w = 0; w < NW; ++w) res[w] &= ~hc[sl * NW + w];
    }
    // transpose: query q's word for these 32 rows = ballot of bit q
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll 8
      for (int qb = 0; qb < 64; ++qb) {
        const unsigned bal = __ballot_sync(0xffffffffu, (res[w] >> qb) & 1ull);
        if (lane == (qb & 31)) tile[(w * 64 + qb) * kChunkWords + wl] = bal;
      }
    }
  }
  __syncthreads();
  // coalesced store of the tile + per-query chunk counts (warp w: queries w, w+32, ...)
  for (uint32_t q = warp; q < 64 * NW; q += 32) {
    const uint32_t gq = a.q0 + q;
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t word = tile[q * kChunkWords + i * 32 + lane];
      c += __popc(word);
      if (gq < a.B) a.mask[static_cast<size_t>(gq) * a.words + chunk * kChunkWords + i * 32 + lane] = word;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0 && gq < a.B) {
      a.chunk_cnt[static_cast<size_t>(gq) * a.n_chunks + chunk] = c;
      if (c) atomicAdd(a.n_elig + gq, c);
    }
  }
}

size_t fwd_mask_smem(uint32_t T, uint32_t C, uint32_t nw) {
  return size_t{64} * nw * kChunkWords * 4 + size_t{T} * nw * 8 + size_t{C} * nw * 8 + T + 16;
}

void launch_fwd_mask(const FwdArgs& a, cudaStream_t st) {
  const size_t smem = fwd_mask_smem(a.T, a.C, a.nw);
  static std::atomic<uint64_t> attr1{0}, attr2{0};
  set_smem_limit(reinterpret_cast<const void*>(fwd_mask_kernel<1>), 227 * 1024, attr1);
  set_smem_limit(reinterpret_cast<const void*>(fwd_mask_kernel<2>), 227 * 1024, attr2);
  if (a.nw == 2) fwd_mask_kernel<2><<<a.n_chunks, 1024, smem, st>>>(a);
  else fwd_mask_kernel<1><<<a.n_chunks, 1024, smem, st>>>(a);
}

// CSR postings -> scratch clause bitmaps (sparse terms, df < W/8).
__global__ void scatter_kernel(const ScatterItem* items, const uint64_t* prefix, uint32_t n_items,
                               uint64_t total, const uint32_t* post_rows, uint32_t* scratch,
                               uint32_t words) {
  for (uint64_t p = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; p < total;
       p += uint64_t{gridDim.x} * blockDim.x) {
    uint32_t lo = 0, hi = n_items;  // last item with prefix <= p
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (prefix[mid] <= p) lo = mid; else hi = mid;
    }
    const ScatterItem it = items[lo];
    const uint32_t row = post_rows[it.begin + (p - prefix[lo])];
    atomicOr(scratch + static_cast<size_t>(it.target) * words + (row >> 5), 1u << (row & 31));
  }
}

void launch_scatter(const ScatterItem* items, const uint64_t* item_prefix, uint32_t n_items,
                    uint64_t total, const uint32_t* post_rows, uint32_t* scratch, uint32_t words,
                    cudaStream_t st) {
  if (!total) return;
  const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, 148 * 16);
  scatter_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(items, item_prefix, n_items, total,
                                                                post_rows, scratch, words);
}

// ===========================================================================
// K2: streaming scorer on CUDA cores (single queries and small batches).
//
// Persistent grid of warps; a warp owns one 1024-row segment at a time.  The
// union of the group's mask words is compacted into a warp-private row list
// (ineligible rows are never loaded), then rows are scored 8*G at a time:
// every lane streams one 16-byte chunk of each of 8 rows with
// ld.global.nc.L1::no_allocate (8 independent LDG.128 in flight per lane),
// FMAs it against the query chunk held in registers, and a 3-level
// reduce-scatter butterfly leaves each leader lane with one finished dot.
// The epilogue clamps (knn.cpp:37), builds the orderable (score, ~row) key
// and appends it only if it beats the query's running lower bound `thr`
// (the K-th best key of a sampled subset, a provable lower bound on the
// global K-th key).  Replaces exact_scores (knn.cpp:8-40) and the gather
// half of bucket_top_k (knn.cpp:42-95).
// ===========================================================================
namespace {

template <typename RowT>
struct Chunk;

template <>
struct Chunk<float> {
  static constexpr int kElems = 4;
  __device__ static float dot(const uint4& v, const float* q) {
    float s = __uint_as_float(v.x) * q[0];
    s = fmaf(__uint_as_float(v.y), q[1], s);
    s = fmaf(__uint_as_float(v.z), q[2], s);
    s = fmaf(__uint_as_float(v.w), q[3], s);
    return s;
  }
};

template <>
struct Chunk<__nv_bfloat16> {
  static constexpr int kElems = 8;
  __device__ static float2 up(uint32_t w) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  }
  __device__ static float dot(const uint4& v, const float* q) {
    float2 a = up(v.x), b = up(v.y), c = up(v.z), d = up(v.w);
    float s = a.x * q[0];
    s = fmaf(a.y, q[1], s);
    s = fmaf(b.x, q[2], s);
    s = fmaf(b.y, q[3], s);
    s = fmaf(c.x, q[4], s);
    s = fmaf(c.y, q[5], s);
    s = fmaf(d.x, q[6], s);
    s = fmaf(d.y, q[7], s);
    return s;
  }
};

// int8 chunk: 16 elements; the lane's partial dot of 16 int8 products is
// exact (|sum| < 2^18) and exactly representable as a float, so the float
// butterfly below sums exact integers (< 2^24) -- the int8 dot is exact.
struct I8Chunk {
  static constexpr int kElems = 16;
  __device__ static float dot(const uint4& v, const uint4& q) {
    int acc = __dp4a(static_cast<int>(v.x), static_cast<int>(q.x), 0);
    acc = __dp4a(static_cast<int>(v.y), static_cast<int>(q.y), acc);
    acc = __dp4a(static_cast<int>(v.z), static_cast<int>(q.z), acc);
    acc = __dp4a(static_cast<int>(v.w), static_cast<int>(q.w), acc);
    return static_cast<float>(acc);
  }
};

__device__ __forceinline__ bool score_active(const ScoreArgs& a, uint32_t q) {
  if (q >= a.B) return false;
  const uint32_t f = a.qp[q].flags;
  if ((f & (QF_ACTIVE | QF_EMB)) != (QF_ACTIVE | QF_EMB)) return false;
  const uint32_t ne = a.n_elig[q];
  if (ne == 0) return false;
  if (a.mode == SCORE_SAMPLE) return ne > a.gate;
  if (a.mode == SCORE_RERUN) return a.rerun[q] != 0;
  return true;
}

}  // namespace

template <typename RowT>
struct ChunkElems {
  static constexpr int value = Chunk<RowT>::kElems;
};
template <>
struct ChunkElems<int8_t> {
  static constexpr int value = I8Chunk::kElems;
};

// RowT = int8_t: the int8 prefilter plane (DevIndex::tc_i8, swizzled 128-row
// tiles) with the int8 query; scores are prefilter scores (s' = acc x scale)
// and rows are admitted against score(thr) - delta_q for exact rescoring in K4p.
template <typename RowT, int LPR, int CPL, int QG>
__global__ void __launch_bounds__(256) score_kernel(ScoreArgs a) {
  constexpr bool kI8 = std::is_same<RowT, int8_t>::value;
  constexpr int G = 32 / LPR;                // row groups per warp load step
  constexpr int E = ChunkElems<RowT>::value;  // elements per 16-byte chunk
  constexpr int M1 = LPR / 2, M2 = LPR / 4, M3 = LPR / 8;
  __shared__ uint16_t lists[8][kSegRows];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int g = lane / LPR, li = lane % LPR;
  const uint32_t q0 = blockIdx.y * QG;

  uint32_t act = 0;
  uint64_t thr[QG];
  float ts8[QG], sc8[QG];  // int8: admission score bound and score scale per query
#pragma unroll
  for (int j = 0; j < QG; ++j) {
    const bool on = score_active(a, q0 + j);
    act |= on ? (1u << j) : 0u;
    thr[j] = (on && a.mode != SCORE_SAMPLE) ? a.thr[q0 + j] : 0ull;
    if (kI8) {
      sc8[j] = on ? a.qscale[q0 + j] : 0.0f;
      ts8[j] = thr[j] == 0ull ? -4.0f : key_score(thr[j]) - a.qdelta[q0 + j];
    }
  }
  if (!act) return;

  float qv[QG][CPL][kI8 ? 1 : E];
  uint4 qv8[QG][CPL];
#pragma unroll
  for (int j = 0; j < QG; ++j)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      if constexpr (kI8) {
        qv8[j][c] = (act >> j & 1u) ? *reinterpret_cast<const uint4*>(a.qi8 + static_cast<size_t>(q0 + j) * a.dp +
                                                                        (li + c * LPR) * E)
                                    : make_uint4(0, 0, 0, 0);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          qv[j][c][e] = (act >> j & 1u)
                            ? a.q[static_cast<size_t>(q0 + j) * a.dp + (li + c * LPR) * E + e]
                            : 0.0f;
      }
    }

  const uint32_t n_seg = (a.n_rows + kSegRows - 1) / kSegRows;
  // few segments: each is split into S parts of 32/S mask words so that
  // enough warps stream rows (the sample pass has its own split)
  const uint32_t S = a.mode == SCORE_SAMPLE ? a.split_sample : a.split;
  const uint32_t n_iter = (a.mode == SCORE_SAMPLE ? (n_seg + a.period - 1) / a.period : n_seg) * S;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const RowT* emb = static_cast<const RowT*>(a.emb);
  const int slot = ((lane & M1) ? 4 : 0) + ((lane & M2) ? 2 : 0) + ((lane & M3) ? 1 : 0);
  const bool leader = (lane & (M3 - 1)) == 0;

  for (uint32_t it = blockIdx.x * (blockDim.x >> 5) + wib; it < n_iter; it += warps) {
    const uint32_t seg = a.mode == SCORE_SAMPLE ? (it / S) * a.period : it / S;
    const uint32_t widx = seg * 32 + lane;
    const bool in_part = lane / (32u / S) == it % S;
    uint32_t wq[QG];
    uint32_t uni = 0;
#pragma unroll
    for (int j = 0; j < QG; ++j) {
      wq[j] = ((act >> j & 1u) && widx < a.words && in_part)
                  ? (a.match_all ? tail_mask(widx, a.n_rows) : a.mask[static_cast<size_t>(q0 + j) * a.words + widx])
                  : 0u;
      uni |= wq[j];
    }
    const uint32_t cnt = __popc(uni);
    const uint32_t incl = warp_incl_scan(cnt, lane);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (total == 0) continue;
    const bool full = total == kSegRows;
    if (!full) {
      uint32_t pos = incl - cnt, u = uni;
      while (u) {
        const int b = __ffs(u) - 1;
        u &= u - 1;
        lists[wib][pos++] = static_cast<uint16_t>(lane * 32 + b);
      }
    }
    __syncwarp();
    const size_t seg_row0 = static_cast<size_t>(seg) * kSegRows;
    for (uint32_t base = 0; base < total; base += 8 * G) {
      uint4 v[8][CPL];
      uint32_t roff[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint32_t idx = base + s * G + g;
        const bool ok = idx < total;
        roff[s] = ok ? (full ? idx : lists[wib][idx]) : 0u;
        if constexpr (kI8) {
          // tiled int8 row: tile lr / 128, K atom cidx / 8, physical chunk
          // (cidx % 8) ^ (row % 8) (SWIZZLE_128B), 16 KB per atom
          const uint32_t lr = static_cast<uint32_t>(seg_row0) + roff[s], rr = lr & 127u;
          const uint8_t* tile = reinterpret_cast<const uint8_t*>(emb) + size_t{lr >> 7} * (a.dp / 128) * 16384 + rr * 128;
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const uint32_t cidx = li + c * LPR;
            v[s][c] = ok ? ldg_stream(tile + (cidx >> 3) * 16384 + (((cidx & 7u) ^ (rr & 7u)) << 4)) : make_uint4(0, 0, 0, 0);
          }
        } else {
          const RowT* row = emb + (seg_row0 + roff[s]) * a.dp;
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            v[s][c] = ok ? ldg_stream(row + (li + c * LPR) * E) : make_uint4(0, 0, 0, 0);
        }
      }
      const uint32_t my_idx = base + slot * G + g;
      const bool my_ok = leader && my_idx < total;
      const uint32_t my_off = my_idx < total ? (full ? my_idx : lists[wib][my_idx]) : 0u;
      // learned row weight (identity without weights): scores are w x clamp(s)
      const float wr = (a.row_w && my_ok) ? __ldg(a.row_w + seg_row0 + my_off) : 1.0f;
#pragma unroll
      for (int j = 0; j < QG; ++j) {
        if (!(act >> j & 1u)) continue;
        float p[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          float acc = 0.0f;
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            if constexpr (kI8) acc += I8Chunk::dot(v[s][c], qv8[j][c]);
            else acc += Chunk<RowT>::dot(v[s][c], qv[j][c]);
          }
          p[s] = acc;
        }
        // reduce-scatter: 8 values over LPR lanes -> 1 value per lane.
        {
          const bool up = lane & M1;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float send = up ? p[i] : p[i + 4];
            const float recv = __shfl_xor_sync(kFull, send, M1);
            p[i] = (up ? p[i + 4] : p[i]) + recv;
          }
        }
        {
          const bool up = lane & M2;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const float send = up ? p[i] : p[i + 2];
            const float recv = __shfl_xor_sync(kFull, send, M2);
            p[i] = (up ? p[i + 2] : p[i]) + recv;
          }
        }
        {
          const bool up = lane & M3;
          const float send = up ? p[0] : p[1];
          const float recv = __shfl_xor_sync(kFull, send, M3);
          p[0] = (up ? p[1] : p[0]) + recv;
        }
#pragma unroll
        for (int m = M3 / 2; m >= 1; m >>= 1) p[0] += __shfl_xor_sync(kFull, p[0], m);

        const uint32_t src_word = __shfl_sync(kFull, wq[j], (my_off >> 5) & 31);
        const bool elig = (src_word >> (my_off & 31)) & 1u;
        const uint32_t grow = a.row_base + static_cast<uint32_t>(seg_row0) + my_off;
        if (kI8) p[0] *= sc8[j];  // exact int8 dot -> prefilter score
        // weighted: w x clamp(s) (|w s - w s'| <= w delta <= delta keeps the prefilter bound)
        const float ps = a.row_w ? weighted_score(p[0], wr) : clamp_score(p[0]);
        const uint64_t key = make_key(ps, grow);
        if (a.mode == SCORE_SAMPLE) {
          if (a.shist) {  // one increment in the query's score histogram
            if (my_ok && elig) {
              const uint32_t b = min(static_cast<uint32_t>((ps + 1.0f) * (0.5f * static_cast<float>(a.hbins))),
                                     a.hbins - 1u);
              atomicAdd(a.shist + static_cast<size_t>(q0 + j) * a.hbins + b, 1u);
            }
          } else if (my_ok && elig) {
            // dense sample slot: segment ordinal x 1024 + row in segment (no atomics)
            a.samp[static_cast<size_t>(q0 + j) * a.cap + (it / S) * kSegRows + my_off] = f2ord(ps);
          }
          continue;
        }
        const bool take = my_ok && elig && (kI8 ? (a.row_w ? ps : p[0]) >= ts8[j] : key >= thr[j]);
        const unsigned bal = __ballot_sync(kFull, take);
        if (bal) {
          const uint32_t q = q0 + j;
          uint32_t basei = 0;
          const int first = __ffs(bal) - 1;
          if (lane == first) basei = atomicAdd(a.cand_cnt + q, __popc(bal));
          basei = __shfl_sync(kFull, basei, first);
          if (take) {
            const uint32_t at = basei + __popc(bal & ((1u << lane) - 1u));
            if (at < a.cap) a.cand[static_cast<size_t>(q) * a.cap + at] = key;
          }
        }
      }
    }
    __syncwarp();
  }
}

namespace {
template <typename RowT, int QG>
void dispatch_score(const ScoreArgs& a, dim3 grid, cudaStream_t st) {
  const uint32_t cpr = a.dp_chunks;
  if (cpr == 8) score_kernel<RowT, 8, 1, QG><<<grid, 256, 0, st>>>(a);
  else if (cpr == 16) score_kernel<RowT, 16, 1, QG><<<grid, 256, 0, st>>>(a);
  else if (cpr == 32) score_kernel<RowT, 32, 1, QG><<<grid, 256, 0, st>>>(a);
  else if (cpr == 64) score_kernel<RowT, 32, 2, QG><<<grid, 256, 0, st>>>(a);
  else if (cpr == 128) score_kernel<RowT, 32, 4, QG><<<grid, 256, 0, st>>>(a);
  else if (cpr == 256) score_kernel<RowT, 32, 8, QG><<<grid, 256, 0, st>>>(a);
  else throw Error(HYRE_INTERNAL, "unsupported row stride (chunks per row " + std::to_string(cpr) + ")");
}
}  // namespace

void launch_score_i8(const ScoreArgs& a, cudaStream_t st) {
  if (a.B == 0) return;
  const uint32_t qg = a.B == 1 ? 1 : kMaxQG;
  const uint32_t groups = (a.B + qg - 1) / qg;
  const uint32_t n_seg = (a.n_rows + kSegRows - 1) / kSegRows;
  const uint32_t iters =
      a.mode == SCORE_SAMPLE ? (n_seg + a.period - 1) / a.period * a.split_sample : n_seg * a.split;
  const uint32_t blocks = std::max(1u, std::min((iters + 7) / 8, 148u * 8u));
  const dim3 grid(blocks, groups);
  const uint32_t cpr = a.dp / 16;  // 16-byte chunks of int8 per row
  if (qg == 1) {
    if (cpr == 8) score_kernel<int8_t, 8, 1, 1><<<grid, 256, 0, st>>>(a);
    else if (cpr == 16) score_kernel<int8_t, 16, 1, 1><<<grid, 256, 0, st>>>(a);
    else if (cpr == 32) score_kernel<int8_t, 32, 1, 1><<<grid, 256, 0, st>>>(a);
    else throw Error(HYRE_INTERNAL, "int8 K2: unsupported row width");
  } else {
    if (cpr == 8) score_kernel<int8_t, 8, 1, kMaxQG><<<grid, 256, 0, st>>>(a);
    else if (cpr == 16) score_kernel<int8_t, 16, 1, kMaxQG><<<grid, 256, 0, st>>>(a);
    else if (cpr == 32) score_kernel<int8_t, 32, 1, kMaxQG><<<grid, 256, 0, st>>>(a);
    else throw Error(HYRE_INTERNAL, "int8 K2: unsupported row width");
  }
}

void launch_score(const ScoreArgs& a, bool bf16, cudaStream_t st) {
  if (a.B == 0) return;
  const uint32_t qg = a.B == 1 ? 1 : kMaxQG;
  const uint32_t groups = (a.B + qg - 1) / qg;
  const uint32_t n_seg = (a.n_rows + kSegRows - 1) / kSegRows;
  const uint32_t iters =
      a.mode == SCORE_SAMPLE ? (n_seg + a.period - 1) / a.period * a.split_sample : n_seg * a.split;
  // Persistent grid: up to 148 SMs x 8 CTAs of 8 warps, no more warps than segments.
  const uint32_t blocks = std::max(1u, std::min((iters + 7) / 8, 148u * 8u));
  dim3 grid(blocks, groups);
  if (bf16) {
    if (qg == 1) dispatch_score<__nv_bfloat16, 1>(a, grid, st);
    else dispatch_score<__nv_bfloat16, kMaxQG>(a, grid, st);
  } else {
    if (qg == 1) dispatch_score<float, 1>(a, grid, st);
    else dispatch_score<float, kMaxQG>(a, grid, st);
  }
}

// ===========================================================================
// K4: exact per-query selection over candidate keys (one CTA per query).
// Radix select (12-bit digits from the top) finds the K-th largest key, the
// keys >= it are gathered into shared memory and bitonic-sorted descending.
// Keys are unique (they embed the row), so exactly min(K, n) survive and the
// order is (score desc, row asc) -- identical to the full sort the reference
// performs (knn.cpp:79-92; "Result == full sort for every G").
// ===========================================================================
namespace {
constexpr int kSelThreads = 512;

// Returns the k-th largest key among keys[0..n) (1 <= k <= n).
__device__ uint64_t kth_largest(const uint64_t* keys, uint32_t n, uint32_t k, uint32_t* hist,
                                uint32_t* tmp) {
  __shared__ uint32_t sel_digit, sel_unique, sel_kk;
  __shared__ uint64_t found;
  uint64_t prefix = 0, pmask = 0;
  uint32_t kk = k;
  const int shifts[6] = {52, 40, 28, 16, 4, 0};
  for (int pass = 0; pass < 6; ++pass) {
    const int sh = shifts[pass];
    const uint32_t dm = pass == 5 ? 0xfu : 0xfffu;
    for (uint32_t i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    // Candidate scores cluster in a few digits, so aggregate equal digits
    // within the warp first (one smem atomic per distinct digit); each thread
    // keeps 4 independent key loads in flight.
    for (uint32_t base = 0; base < n; base += 4 * blockDim.x) {
      uint64_t kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        kv[u] = i < n ? keys[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        uint32_t digit = 0xffffffffu;
        if (i < n && (kv[u] & pmask) == prefix) digit = static_cast<uint32_t>((kv[u] >> sh) & dm);
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        if (digit != 0xffffffffu && (threadIdx.x & 31) == static_cast<uint32_t>(__ffs(peers) - 1))
          atomicAdd(hist + digit, static_cast<uint32_t>(__popc(peers)));
      }
    }
    __syncthreads();
    // Position t of the scan owns bins [8*o, 8*o+8) with o = T-1-t, so the
    // exclusive prefix at t counts every key in bins above o's range.
    // (per = 4096 / blockDim.x bins per scan position: 8 at 512 threads, 4 at 1024)
    const uint32_t owner = blockDim.x - 1 - threadIdx.x, per = 4096 / blockDim.x;
    uint32_t mine = 0;
    for (uint32_t b = 0; b < per; ++b) mine += hist[owner * per + b];
    uint32_t tot;
    uint32_t above = block_excl_scan(mine, tmp, &tot);
    for (int b = static_cast<int>(per) - 1; b >= 0; --b) {
      const uint32_t h = hist[owner * per + b];
      if (above < kk && kk <= above + h) {
        sel_digit = owner * per + b;
        sel_unique = h == 1;
        sel_kk = kk - above;
      }
      above += h;
    }
    __syncthreads();
    kk = sel_kk;
    prefix |= static_cast<uint64_t>(sel_digit) << sh;
    pmask |= static_cast<uint64_t>(dm) << sh;
    const bool uniq = sel_unique;
    __syncthreads();
    if (uniq && pass < 5) {
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
        if ((keys[i] & pmask) == prefix) found = keys[i];
      __syncthreads();
      return found;
    }
  }
  return prefix;
}

__device__ void bitonic_desc(uint64_t* s, uint32_t m) {  // m power of two
  for (uint32_t size = 2; size <= m; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < m / 2; i += blockDim.x) {
        const uint32_t lo = 2 * stride * (i / stride) + (i % stride);
        const uint32_t hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const uint64_t x = s[lo], y = s[hi];
        if ((x < y) == desc) {
          s[lo] = y;
          s[hi] = x;
        }
      }
      __syncthreads();
    }
  }
}
}  // namespace

namespace {
constexpr int kSampleVec = 8;  // uint4 of sample scores per thread: 8 x 4 x 512 = 16K slots

__device__ __forceinline__ uint32_t kth_m(uint32_t k, uint32_t period) {
  return min(k, max(8u, (4 * k + period - 1) / period));
}
// bins [per*o, per*o + per) belong to scan position t, o = T-1-t; returns
// nnz; s_sel = {bin of the k-th key, keys at/above it, same for the m-th}
__device__ __forceinline__ uint32_t kth_bins(const uint32_t* hist, uint32_t k, uint32_t m, uint32_t* tmp,
                                             uint32_t* s_sel) {
  const uint32_t per = 4096 / blockDim.x;
  const uint32_t owner = blockDim.x - 1 - threadIdx.x;
  uint32_t mine = 0;
  for (uint32_t b = 0; b < per; ++b) mine += hist[owner * per + b];
  uint32_t nnz;
  uint32_t above = block_excl_scan(mine, tmp, &nnz);
  for (int b = static_cast<int>(per) - 1; b >= 0; --b) {
    const uint32_t h = hist[owner * per + b];
    if (above < k && k <= above + h) {
      s_sel[0] = owner * per + b;
      s_sel[1] = above + h;
    }
    if (above < m && m <= above + h) {
      s_sel[2] = owner * per + b;
      s_sel[3] = above + h;
    }
    above += h;
  }
  __syncthreads();
  return nnz;
}
// warp-aggregated shared-memory histogram increment (equal digits of a warp
// cost one atomic); 0xffffffff = no value
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t digit) {
  const unsigned peers = __match_any_sync(0xffffffffu, digit);
  if (digit != 0xffffffffu && (threadIdx.x & 31) == static_cast<uint32_t>(__ffs(peers) - 1))
    atomicAdd(hist + digit, static_cast<uint32_t>(__popc(peers)));
}
// Number of keys in s[0, m) greater than key: two keys per 16-byte shared
// load and four independent counters (the serial add chain was the K4p
// ranking's latency).
__device__ __forceinline__ uint32_t count_greater(const uint64_t* s, uint32_t m, uint64_t key) {
  uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0, j = 0;
  for (; j + 4 <= m; j += 4) {
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(s + j);
    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(s + j + 2);
    r0 += a.x > key ? 1u : 0u;
    r1 += a.y > key ? 1u : 0u;
    r2 += b.x > key ? 1u : 0u;
    r3 += b.y > key ? 1u : 0u;
  }
  for (; j < m; ++j) r0 += s[j] > key ? 1u : 0u;
  return r0 + r1 + r2 + r3;
}
// 12-bit histogram bin of an orderable score (f2ord): linear in the score
// over [-1, 1] (2^-11 wide bins), monotone in the key order.  The top 12 key
// bits would give one bin per (exponent, 3 mantissa bits): cosines in
// [0.25, 0.5) share 8 bins, so the K-th key's bin held thousands of keys.
__device__ __forceinline__ uint32_t score_bin(uint32_t ord) {
  const float sc = ord2f(ord);
  return static_cast<uint32_t>(fminf(fmaxf((sc + 1.0f) * 2048.0f, 0.0f), 4095.0f));
}
// warp-aggregated append of `key` (if take) to dst[*cnt++] (capacity dcap)
__device__ __forceinline__ void warp_append(bool take, uint64_t key, uint64_t* dst, uint32_t* cnt, uint32_t dcap) {
  const unsigned bal = __ballot_sync(0xffffffffu, take);
  if (!bal) return;
  uint32_t at = 0;
  if ((threadIdx.x & 31) == 0) at = atomicAdd(cnt, static_cast<uint32_t>(__popc(bal)));
  at = __shfl_sync(0xffffffffu, at, 0) + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
  if (take && at < dcap) dst[at] = key;
}
}  // namespace

constexpr uint32_t kSelResident = 8192;  // FINAL: candidates sorted from shared memory

__global__ void __launch_bounds__(kSelThreads) select_kernel(SelectArgs a) {
  extern __shared__ uint64_t sel_smem[];
  uint64_t* sortbuf = sel_smem;                                        // kSelectMaxK keys
  uint32_t* hist = reinterpret_cast<uint32_t*>(sel_smem + kSelectMaxK);  // 4096
  uint32_t* tmp = hist + 4096;                                         // 33
  __shared__ uint32_t gathered;
  const uint32_t q = blockIdx.x;
  const QParam qp = a.qp[q];
  if ((qp.flags & a.require_flags) != a.require_flags) return;
  if (a.mode == SELECT_FINAL_RERUN && !a.rerun[q]) return;
  const uint32_t total = (a.mode == SELECT_KTH && a.dense_n) ? a.dense_n : a.cnt[q];
  const uint32_t n = min(total, a.cap);
  const uint64_t* keys = a.buf + static_cast<size_t>(q) * a.cap;
  const uint32_t k = qp.k;

  if (a.mode == SELECT_KTH) {
    // Only queries that were sampled (n_elig > cap) get a threshold.
    if (!(a.n_elig[q] > a.gate)) {
      if (threadIdx.x == 0) a.thr[q] = 0;
      return;
    }
    uint64_t t_safe = 0;
    if (n >= k && k > 0) t_safe = kth_largest(keys, n, k, hist, tmp);
    const uint32_t m = min(k, max(8u, (4 * k + a.period - 1) / a.period));
    uint64_t t_est = t_safe;
    if (m < k && n >= m) {
      if (t_safe != 0ull) {
        // the m-th key is among the k keys >= t_safe: sort those in smem
        if (threadIdx.x == 0) gathered = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
          const uint64_t key = keys[i];
          if (key >= t_safe) {
            const uint32_t at = atomicAdd(&gathered, 1u);
            if (at < kSelectMaxK) sortbuf[at] = key;
          }
        }
        __syncthreads();
        const uint32_t g = min(gathered, kSelectMaxK);
        uint32_t g2 = 1;
        while (g2 < g) g2 <<= 1;
        for (uint32_t i = g + threadIdx.x; i < g2; i += blockDim.x) sortbuf[i] = 0ull;
        __syncthreads();
        bitonic_desc(sortbuf, g2);
        t_est = sortbuf[m - 1];
      } else {
        t_est = kth_largest(keys, n, m, hist, tmp);
      }
    }
    if (threadIdx.x == 0) {
      a.thr[q] = t_est;
      const float dl = a.qdelta ? a.qdelta[q] : a.delta;
      if (a.thr_safe) a.thr_safe[q] = dl > 0.0f ? key_minus_delta(t_safe, dl) : t_safe;
    }
    return;
  }
  // FINAL
  if (a.n_elig[q] == 0 || (total == 0 && !(a.thr_safe && a.thr[q] != a.thr_safe[q]))) {
    if (threadIdx.x == 0) {
      a.out_cnt[q] = 0;
      if (a.rerun) a.rerun[q] = 0;
    }
    return;
  }
  if (total > a.cap) {
    // Candidate buffer overflowed: the first `cap` candidates are a subset of
    // the eligible rows, so their K-th key is a valid, tighter lower bound.
    const uint64_t t = kth_largest(keys, n, k, hist, tmp);
    if (threadIdx.x == 0) {
      a.thr[q] = t;
      a.rerun[q] = 1;
    }
    return;
  }
  if (a.thr_safe && total < min(k, a.n_elig[q]) && a.thr[q] != a.thr_safe[q]) {
    // The estimated threshold admitted fewer than K rows: rescore with the
    // guaranteed bound.
    if (threadIdx.x == 0) {
      a.thr[q] = a.thr_safe[q];
      a.rerun[q] = 1;
    }
    return;
  }
  uint32_t m = 0;
  bool done = false;
  if (n <= k) {  // every candidate is a hit (n <= k <= kSelectMaxK)
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sortbuf[i] = keys[i];
    m = n;
    done = true;
  } else if (n <= kSelResident) {
    // the common case: one coalesced pass into shared memory, a histogram of
    // the top 12 key bits there finds the K-th key's bin, and only the keys
    // at or above it (about K + one bin) are sorted -- no passes over global
    // memory
    uint64_t* res = reinterpret_cast<uint64_t*>(tmp + 40);
    __shared__ uint32_t s_sel[4];
    for (uint32_t i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) gathered = 0;
    __syncthreads();
    for (uint32_t base = 0; base < n; base += 4 * blockDim.x) {  // four independent loads in flight
      uint64_t kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        kv[u] = i < n ? keys[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        if (i < n) res[i] = kv[u];
        hist_add(hist, i < n ? score_bin(static_cast<uint32_t>(kv[u] >> 32)) : 0xffffffffu);
      }
    }
    __syncthreads();
    kth_bins(hist, k, k, tmp, s_sel);
    if (s_sel[1] <= kSelectMaxK) {
      const uint32_t dk = s_sel[0];
      for (uint32_t base = 0; base < n; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const uint64_t key = i < n ? res[i] : 0ull;
        warp_append(i < n && score_bin(static_cast<uint32_t>(key >> 32)) >= dk, key, sortbuf, &gathered, kSelectMaxK);
      }
      __syncthreads();
      m = gathered;
      done = true;
    }
  }
  if (!done) {
    const uint64_t t = kth_largest(keys, n, k, hist, tmp);
    if (threadIdx.x == 0) gathered = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t key = keys[i];
      if (key >= t) {
        const uint32_t at = atomicAdd(&gathered, 1u);
        if (at < kSelectMaxK) sortbuf[at] = key;
      }
    }
    __syncthreads();
    m = min(gathered, kSelectMaxK);
  }
  const uint32_t take = min(m, k);
  hyre_hit* out = a.hits + a.hit_off[q];
  __syncthreads();  // sortbuf complete (the n <= k path fills it without a barrier)
  if (m <= 1024) {
    // rank by counting (keys are unique): no sort stages, one pass over the
    // gathered keys per key (broadcast shared reads)
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint64_t key = sortbuf[i];
      const uint32_t rank = count_greater(sortbuf, m, key);
      if (rank < take) {
        out[rank].row = key_row(key);
        out[rank].score = key_score(key);
      }
    }
  } else {
    uint32_t m2 = 1;
    while (m2 < m) m2 <<= 1;
    for (uint32_t i = m + threadIdx.x; i < m2; i += blockDim.x) sortbuf[i] = 0ull;
    __syncthreads();
    bitonic_desc(sortbuf, m2);
    for (uint32_t i = threadIdx.x; i < take; i += blockDim.x) {
      const uint64_t key = sortbuf[i];
      out[i].row = key_row(key);
      out[i].score = key_score(key);
    }
  }
  if (threadIdx.x == 0) {
    a.out_cnt[q] = take;
    if (a.rerun) a.rerun[q] = 0;
  }
}

// K4 over the dense sample (SELECT_KTH with dense_n): the thresholds need
// the K-th and m-th largest keys among the sample's eligible slots (slot
// value = f2ord(score), 0 = ineligible; the slot index gives the row, so the
// key (score, ~row) is rebuilt on the fly).  Two kernels:
//   slice: each CTA holds one 16K-slot slice of a query's sample in
//          registers, finds (4096-bin histogram of the top 12 score bits) the
//          bin of its local r-th key, r = max(m, ceil(K / slices)), and
//          appends the keys at or above it (its top r plus bin-mates) to the
//          query's union buffer;
//   union: one CTA per query sorts the union (a few hundred keys) in shared
//          memory.  The union holds every slice's top m, so its m-th key is
//          exactly the sample's m-th (t_est); it is a subset of the sample, so
//          its K-th key is a valid lower bound on the global K-th (t_safe).
__global__ void __launch_bounds__(kSelThreads) sample_slice_kernel(SelectArgs a, uint32_t* ucnt) {
  __shared__ uint32_t hist[4096];
  __shared__ uint32_t tmp[40], s_sel[4];
  const uint32_t q = blockIdx.y;
  const QParam qp = a.qp[q];
  if ((qp.flags & a.require_flags) != a.require_flags || !(a.n_elig[q] > a.gate)) return;
  const uint32_t k = qp.k, m = kth_m(k, a.period);
  const uint32_t r = min(kSelectMaxK, max(m, (k + gridDim.x - 1) / gridDim.x));
  const uint32_t n = a.dense_n, s0 = blockIdx.x * (kSampleVec * 4 * kSelThreads);
  const uint32_t* sc = a.samp + static_cast<size_t>(q) * a.cap;
  uint4 v[kSampleVec];
#pragma unroll
  for (int u = 0; u < kSampleVec; ++u) {
    const uint32_t slot = s0 + 4 * (u * blockDim.x + threadIdx.x);
    v[u] = slot + 3 < n ? *reinterpret_cast<const uint4*>(sc + slot)
                        : make_uint4(slot < n ? sc[slot] : 0u, slot + 1 < n ? sc[slot + 1] : 0u,
                                     slot + 2 < n ? sc[slot + 2] : 0u, 0u);
  }
  for (uint32_t i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kSampleVec; ++u) {
    hist_add(hist, v[u].x ? score_bin(v[u].x) : 0xffffffffu);
    hist_add(hist, v[u].y ? score_bin(v[u].y) : 0xffffffffu);
    hist_add(hist, v[u].z ? score_bin(v[u].z) : 0xffffffffu);
    hist_add(hist, v[u].w ? score_bin(v[u].w) : 0xffffffffu);
  }
  __syncthreads();
  const uint32_t nnz = kth_bins(hist, r, r, tmp, s_sel);
  if (nnz == 0) return;
  const uint32_t dsel = nnz >= r ? s_sel[0] : 0u;  // fewer than r: the whole slice
  uint64_t* dst = a.fb + static_cast<size_t>(q) * a.fb_cap;
#pragma unroll
  for (int u = 0; u < kSampleVec; ++u) {
    const uint32_t b0 = s0 + 4 * (u * blockDim.x + threadIdx.x);
    const uint32_t o[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t slot = b0 + e, local = (slot >> 10) * a.period * 1024u + (slot & 1023u);
      warp_append(o[e] != 0u && score_bin(o[e]) >= dsel,
                  (static_cast<uint64_t>(o[e]) << 32) | static_cast<uint32_t>(~(a.row_base + local)), dst, ucnt + q,
                  a.fb_cap);
    }
  }
}

__global__ void __launch_bounds__(kSelThreads) sample_union_kernel(SelectArgs a, const uint32_t* ucnt) {
  extern __shared__ uint64_t sel_smem[];
  uint64_t* sortbuf = sel_smem;                                          // kSelectMaxK keys
  uint32_t* hist = reinterpret_cast<uint32_t*>(sel_smem + kSelectMaxK);  // 4096
  uint32_t* tmp = hist + 4096;                                           // 33
  const uint32_t q = blockIdx.x;
  const QParam qp = a.qp[q];
  if ((qp.flags & a.require_flags) != a.require_flags) return;
  uint64_t t_safe = 0, t_est = 0;
  if (a.n_elig[q] > a.gate) {
    const uint32_t k = qp.k, m = kth_m(k, a.period);
    const uint32_t n = min(ucnt[q], a.fb_cap);
    const uint64_t* keys = a.fb + static_cast<size_t>(q) * a.fb_cap;
    if (n <= kSelectMaxK) {
      uint32_t c2 = 1;
      while (c2 < n) c2 <<= 1;
      for (uint32_t i = threadIdx.x; i < c2; i += blockDim.x) sortbuf[i] = i < n ? keys[i] : 0ull;
      __syncthreads();
      bitonic_desc(sortbuf, c2);
      t_safe = n >= k ? sortbuf[k - 1] : 0ull;
      t_est = n >= m ? sortbuf[m - 1] : 0ull;
    } else {
      t_safe = n >= k ? kth_largest(keys, n, k, hist, tmp) : 0ull;
      t_est = m < k ? kth_largest(keys, n, m, hist, tmp) : t_safe;
    }
  }
  if (threadIdx.x == 0) {
    a.thr[q] = t_est;
    const float dl = a.qdelta ? a.qdelta[q] : a.delta;
    if (a.thr_safe) a.thr_safe[q] = dl > 0.0f ? key_minus_delta(t_safe, dl) : t_safe;
  }
}

void launch_sample_kth(const SelectArgs& a, uint32_t* ucnt, cudaStream_t st) {
  if (a.B == 0) return;
  constexpr uint32_t slice = kSampleVec * 4 * kSelThreads;
  const dim3 grid((a.dense_n + slice - 1) / slice, a.B);
  sample_slice_kernel<<<grid, kSelThreads, 0, st>>>(a, ucnt);
  const size_t smem = kSelectMaxK * sizeof(uint64_t) + (4096 + 40) * sizeof(uint32_t);
  static std::atomic<uint64_t> attr{0};
  set_smem_limit(reinterpret_cast<const void*>(sample_union_kernel), static_cast<int>(smem), attr);
  sample_union_kernel<<<a.B, kSelThreads, smem, st>>>(a, ucnt);
}

__global__ void __launch_bounds__(256) hist_thr_kernel(HistThrArgs a) {
  __shared__ uint32_t tmp[40];
  __shared__ uint32_t s_bin[2];
  pdl_trigger();
  pdl_wait();  // the sample pass's histograms
  const uint32_t q = blockIdx.x;
  const QParam qp = a.qp[q];
  const bool on = (qp.flags & a.require_flags) == a.require_flags && a.n_elig[q] > a.gate;
  if (!on) {
    if (threadIdx.x == 0) {
      a.thr[q] = 0ull;
      a.thr_safe[q] = 0ull;
    }
    return;
  }
  const uint32_t k = qp.k, m = kth_m(k, a.period);
  // thread t owns bins [nb - (t + 1) per, nb - t per): scan positions run
  // from the top score down, so the exclusive prefix counts the rows above
  const uint32_t per = a.nb / blockDim.x, hi = a.nb - threadIdx.x * per;
  const uint32_t* h = a.hist + static_cast<size_t>(q) * a.nb;
  // the thread's 16 bins (nb = 4096, 256 threads) in four vector loads, kept
  // in registers for both passes
  uint32_t c16[16];
  if (per == 16) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint4 x = *reinterpret_cast<const uint4*>(h + hi - 16 + 4 * v);
      c16[4 * v] = x.x;
      c16[4 * v + 1] = x.y;
      c16[4 * v + 2] = x.z;
      c16[4 * v + 3] = x.w;
    }
  }
  uint32_t mine = 0;
  if (per == 16) {
#pragma unroll
    for (int v = 0; v < 16; ++v) mine += c16[v];
  } else {
    for (uint32_t b = hi - per; b < hi; ++b) mine += h[b];
  }
  if (threadIdx.x == 0) s_bin[0] = s_bin[1] = UINT32_MAX;
  uint32_t total;
  uint32_t above = block_excl_scan(mine, tmp, &total);
  if (per == 16) {
#pragma unroll
    for (int v = 15; v >= 0; --v) {
      const uint32_t b = hi - 16 + v, c = c16[v];
      if (above < k && k <= above + c) s_bin[0] = b;
      if (above < m && m <= above + c) s_bin[1] = b;
      above += c;
    }
  } else {
    for (uint32_t b = hi; b-- > hi - per;) {
      const uint32_t c = h[b];
      if (above < k && k <= above + c) s_bin[0] = b;
      if (above < m && m <= above + c) s_bin[1] = b;
      above += c;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // lower bin edge, a hair lower so float rounding of the binning can never
    // leave a binned score below it; the key of (edge, last row) is below every
    // key with a score >= edge
    auto edge_key = [&](uint32_t b) {
      const float e = -1.0f + 2.0f * static_cast<float>(b) / static_cast<float>(a.nb) - 1e-6f;
      return make_key(fmaxf(e, -1.0f), 0xFFFFFFFFu);
    };
    const uint64_t t_safe = s_bin[0] == UINT32_MAX ? 0ull : edge_key(s_bin[0]);
    a.thr[q] = s_bin[1] == UINT32_MAX ? 0ull : edge_key(s_bin[1]);
    const float dl = a.qdelta ? a.qdelta[q] : a.delta;
    a.thr_safe[q] = dl > 0.0f ? key_minus_delta(t_safe, dl) : t_safe;
  }
}

__global__ void run_init_kernel(uint32_t* counters, uint32_t n_counters, uint32_t B, uint4* hist, size_t hist_vec) {
  pdl_trigger();  // the K3 sample pass may set up while the counters are zeroed
  const size_t stride = size_t{gridDim.x} * blockDim.x;
  const size_t t0 = size_t{blockIdx.x} * blockDim.x + threadIdx.x;
  for (size_t i = t0; i < n_counters; i += stride) counters[i] = i < B ? 0xFFFFFFFFu : 0u;
  for (size_t i = t0; i < hist_vec; i += stride) hist[i] = make_uint4(0, 0, 0, 0);
}

void launch_run_init(uint32_t* counters, uint32_t n_counters, uint32_t B, uint32_t* hist, size_t hist_words,
                     cudaStream_t st) {
  const size_t hv = hist ? hist_words / 4 : 0;  // hist_words is a multiple of 4096
  const uint32_t blocks = static_cast<uint32_t>(std::min<size_t>(592, (std::max<size_t>(hv, n_counters) + 255) / 256));
  run_init_kernel<<<std::max(1u, blocks), 256, 0, st>>>(counters, n_counters, B, reinterpret_cast<uint4*>(hist), hv);
}

void launch_hist_thr(const HistThrArgs& a, cudaStream_t st) {
  if (a.B == 0) return;
  launch_pdl(hist_thr_kernel, dim3(a.B), dim3(256), 0, st, a);
}

void launch_select(const SelectArgs& a, cudaStream_t st) {
  if (a.B == 0) return;
  // sort buffer | histogram + scan scratch | resident candidates (FINAL)
  const size_t smem = kSelectMaxK * sizeof(uint64_t) + (4096 + 40) * sizeof(uint32_t) + kSelResident * sizeof(uint64_t);
  static std::atomic<uint64_t> attr{0};
  set_smem_limit(reinterpret_cast<const void*>(select_kernel), static_cast<int>(smem), attr);
  select_kernel<<<a.B, kSelThreads, smem, st>>>(a);
}

// ---------------------------------------------------------------------------
// K4 for the K3 prefilter (SELECT_FINAL / SELECT_FINAL_RERUN): candidates
// carry prefilter keys (|exact - prefilter| <= delta).  One CTA per query:
//   1. tau = K-th largest prefilter key of the candidates.  K candidates have
//      exact scores >= score(tau) - delta, so the exact K-th score is too, and
//      every row of the exact top K has prefilter score >= score(tau) - 2 delta:
//      only those survivors (about K + the rows in a 2-delta band) are rescored;
//   2. survivors are rescored exactly with K2's arithmetic (the fp32 or bf16
//      row and the fp32 unit query; LPR lanes per row, the butterfly of
//      score_kernel), so batch scores equal single-query scores bit for bit;
//   3. the threshold was valid if K rows are known to score >= score(thr)
//      (score(tau) - delta >= score(thr), or K rescored keys above it); else
//      the query reruns with thr_safe, exactly as in select_kernel;
//   4. the survivors' exact keys are sorted; the first K are the hits.
// Overflowing candidate buffers rerun with the delta-lowered K-th prefilter
// key of the kept subset (a valid bound).  More than kSelectMaxK survivors
// (near-duplicate rows; adversarial) fall back to rescoring every candidate
// in place and an exact radix select.
// ---------------------------------------------------------------------------
namespace {
template <typename RowT, int LPR, int CPL>
__device__ void rescore_list(const PrefSelectArgs& a, uint32_t q, uint64_t* keys, uint32_t n, float thr_s,
                             uint32_t* above) {
  constexpr int G = 32 / LPR, E = Chunk<RowT>::kElems, U = CPL >= 8 ? 1 : (CPL >= 4 ? 2 : (CPL >= 2 ? 4 : 8));  // rows in flight per lane group
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane / LPR, li = lane % LPR;
  float qv[CPL][E];
#pragma unroll
  for (int c = 0; c < CPL; ++c)
#pragma unroll
    for (int e = 0; e < E; ++e) qv[c][e] = a.q[static_cast<size_t>(q) * a.dp + (li + c * LPR) * E + e];
  const RowT* emb = static_cast<const RowT*>(a.emb);
  uint32_t mine = 0;
  for (uint32_t base = wib * U * G; base < n; base += nw * U * G) {
    uint4 v[U][CPL];
    uint32_t idx[U], grow[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      idx[u] = base + u * G + g;
      const bool ok = idx[u] < n;
      grow[u] = ok ? key_row(keys[idx[u]]) : a.row_base;
      const RowT* r = emb + static_cast<size_t>(grow[u] - a.row_base) * a.dp;
#pragma unroll
      for (int c = 0; c < CPL; ++c) v[u][c] = ok ? ldg_stream(r + (li + c * LPR) * E) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float acc = 0.0f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc += Chunk<RowT>::dot(v[u][c], qv[c]);
#pragma unroll
      for (int m = LPR / 2; m >= 1; m >>= 1) acc += __shfl_xor_sync(kFull, acc, m);
      if (li == 0 && idx[u] < n) {
        const float sc = a.row_w ? weighted_score(acc, __ldg(a.row_w + (grow[u] - a.row_base))) : clamp_score(acc);
        keys[idx[u]] = make_key(sc, grow[u]);
        mine += sc >= thr_s ? 1u : 0u;
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) mine += __shfl_xor_sync(kFull, mine, m);
  if (lane == 0 && mine) atomicAdd(above, mine);
}
}  // namespace

// K4p block size: 1024 threads (more warps -> more survivor rows in flight)
// while the batch fits one wave of one CTA per SM; 512 threads and two CTAs
// per SM for larger batches (one CTA per query: B = 256 is then one wave,
// not two)
constexpr int kSelPThreads = 1024;
constexpr uint32_t kSelPWide = 148;  // batches above this use the 512-thread variant
template <typename RowT, int LPR, int CPL, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) select_prefilter_kernel(PrefSelectArgs pa) {
  pdl_wait();  // the main pass's candidates
  const SelectArgs& a = pa.s;
  extern __shared__ uint64_t sel_smem[];
  uint64_t* sortbuf = sel_smem;                                          // kSelectMaxK keys
  uint32_t* hist = reinterpret_cast<uint32_t*>(sel_smem + kSelectMaxK);  // 4096
  uint32_t* tmp = hist + 4096;                                           // 33
  uint64_t* res = reinterpret_cast<uint64_t*>(tmp + 40);                 // kSelResident keys
  __shared__ uint32_t gathered, above;
  const uint32_t q = blockIdx.x;
  const QParam qp = a.qp[q];
  if ((qp.flags & a.require_flags) != a.require_flags) return;
  if (a.mode == SELECT_FINAL_RERUN && !a.rerun[q]) return;
  const uint32_t total = a.cnt[q], n = min(total, a.cap), k = qp.k;
  uint64_t* keys = const_cast<uint64_t*>(a.buf) + static_cast<size_t>(q) * a.cap;  // the candidate buffer (rescored in place on spill)
  const uint64_t thr = a.thr[q];
  const bool has_safe = a.thr_safe && thr != a.thr_safe[q];
  if (a.n_elig[q] == 0 || (total == 0 && !has_safe)) {
    if (threadIdx.x == 0) {
      a.out_cnt[q] = 0;
      a.rerun[q] = 0;
    }
    return;
  }
  const float dl = a.qdelta ? a.qdelta[q] : a.delta;  // this query's prefilter bound
  if (total > a.cap) {  // overflow: the kept subset's K-th prefilter key, lowered by delta, bounds the exact K-th
    const uint64_t t = kth_largest(keys, n, k, hist, tmp);
    if (threadIdx.x == 0) {
      a.thr[q] = key_minus_delta(t, dl);
      a.rerun[q] = 1;
    }
    return;
  }
  const float thr_s = thr == 0ull ? -2.0f : key_score(thr);
  // 1. tau: K-th largest prefilter key (no pruning when n <= K)
  const bool resident = n <= kSelResident;
  if (resident) {
    for (uint32_t base = 0; base < n; base += 4 * blockDim.x) {  // four independent loads in flight
      uint64_t kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        kv[u] = i < n ? keys[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = base + u * blockDim.x + threadIdx.x;
        if (i < n) res[i] = kv[u];
      }
    }
    __syncthreads();
  }
  const uint64_t* src = resident ? res : keys;
  // tau_s: a lower bound on the K-th largest prefilter score, the lower edge
  // of its bin in a 4096-bin linear histogram over [-1, 1] (bin width 4.9e-4,
  // one pass; K candidates lie at or above the edge, which is all steps 1-3
  // need -- a lower tau only admits a few more survivors)
  float tau_s = -4.0f;
  if (n > k) {
    __shared__ uint32_t s_sel[4];
    for (uint32_t i = threadIdx.x; i < 4096; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t base = 0; base < n; base += blockDim.x) {
      const uint32_t i = base + threadIdx.x;
      uint32_t b = 0xffffffffu;
      if (i < n) b = min(static_cast<uint32_t>((key_score(src[i]) + 1.0f) * 2048.0f), 4095u);
      hist_add(hist, b);
    }
    __syncthreads();
    kth_bins(hist, k, k, tmp, s_sel);
    tau_s = -1.0f + static_cast<float>(s_sel[0]) / 2048.0f - 1e-6f;
  }
  const float prune = tau_s - 2.0f * dl;
  // 2. survivors -> sortbuf, rescored in place
  if (threadIdx.x == 0) {
    gathered = 0;
    above = 0;
  }
  __syncthreads();
  for (uint32_t base = 0; base < n; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint64_t key = i < n ? src[i] : 0ull;
    warp_append(i < n && key_score(key) >= prune, key, sortbuf, &gathered, kSelectMaxK);
  }
  __syncthreads();
  const uint32_t g = gathered;
  const bool spill = g > kSelectMaxK;
  if (!spill) {
    rescore_list<RowT, LPR, CPL>(pa, q, sortbuf, g, thr_s, &above);
  } else {  // adversarial: rescore every candidate in place in global memory
    rescore_list<RowT, LPR, CPL>(pa, q, keys, n, thr_s, &above);
  }
  __syncthreads();
  // 3. threshold validity (select_kernel's rule with the prefilter bound)
  const bool valid = (n >= k && tau_s - dl >= thr_s) || above >= min(k, a.n_elig[q]);
  if (!valid && has_safe) {
    if (threadIdx.x == 0) {
      a.thr[q] = a.thr_safe[q];
      a.rerun[q] = 1;
    }
    return;
  }
  // 4. exact order
  uint32_t m = g;
  if (spill) {
    const uint64_t t = kth_largest(keys, n, k, hist, tmp);
    if (threadIdx.x == 0) gathered = 0;
    __syncthreads();
    for (uint32_t base = 0; base < n; base += blockDim.x) {
      const uint32_t i = base + threadIdx.x;
      const uint64_t key = i < n ? keys[i] : 0ull;
      warp_append(i < n && key >= t, key, sortbuf, &gathered, kSelectMaxK);
    }
    __syncthreads();
    m = min(gathered, kSelectMaxK);
  }
  const uint32_t take = min(m, k);
  hyre_hit* out = a.hits + a.hit_off[q];
  if (m <= 1024) {
    // rank by counting (keys are unique): no sort stages, one pass over the
    // survivors per key in shared memory (broadcast reads)
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint64_t key = sortbuf[i];
      const uint32_t rank = count_greater(sortbuf, m, key);
      if (rank < take) {
        out[rank].row = key_row(key);
        out[rank].score = key_score(key);
      }
    }
  } else {
    uint32_t m2 = 1;
    while (m2 < m) m2 <<= 1;
    for (uint32_t i = m + threadIdx.x; i < m2; i += blockDim.x) sortbuf[i] = 0ull;
    __syncthreads();
    bitonic_desc(sortbuf, m2);
    for (uint32_t i = threadIdx.x; i < take; i += blockDim.x) {
      const uint64_t key = sortbuf[i];
      out[i].row = key_row(key);
      out[i].score = key_score(key);
    }
  }
  if (threadIdx.x == 0) {
    a.out_cnt[q] = take;
    a.rerun[q] = 0;
  }
}

namespace {
template <typename RowT>
void dispatch_select_prefilter(const PrefSelectArgs& a, size_t smem, cudaStream_t st) {
  using KFn = void (*)(PrefSelectArgs);
  KFn k = nullptr;
  const uint32_t cpr = a.dp_chunks;
  const bool wide = a.s.B > kSelPWide;
#define HYRE_K4P(LPR, CPL) (wide ? select_prefilter_kernel<RowT, LPR, CPL, 512> : select_prefilter_kernel<RowT, LPR, CPL, kSelPThreads>)
  if (cpr == 8) k = HYRE_K4P(8, 1);
  else if (cpr == 16) k = HYRE_K4P(16, 1);
  else if (cpr == 32) k = HYRE_K4P(32, 1);
  else if (cpr == 64) k = HYRE_K4P(32, 2);
  else if (cpr == 128) k = HYRE_K4P(32, 4);
  else if (cpr == 256) k = HYRE_K4P(32, 8);
  else throw Error(HYRE_INTERNAL, "unsupported row stride (chunks per row " + std::to_string(cpr) + ")");
#undef HYRE_K4P
  static std::atomic<uint64_t> attr_set[2][2][6];  // [bf16][wide][row-width variant]: device bitmask per kernel
  const int vi = cpr == 8 ? 0 : cpr == 16 ? 1 : cpr == 32 ? 2 : cpr == 64 ? 3 : cpr == 128 ? 4 : 5;
  set_smem_limit(reinterpret_cast<const void*>(k), static_cast<int>(smem),
                 attr_set[std::is_same<RowT, float>::value ? 0 : 1][wide ? 1 : 0][vi]);
  if (wide) {  // two 112 KB CTAs per SM need the largest shared-memory carveout
    static std::atomic<uint64_t> carve[2][6];
    std::atomic<uint64_t>& c = carve[std::is_same<RowT, float>::value ? 0 : 1][vi];
    int dev = 0;
    HYRE_CUDA(cudaGetDevice(&dev));
    if (!(c.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
      HYRE_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k), cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      c.fetch_or(1ull << (dev & 63), std::memory_order_acq_rel);
    }
  }
  launch_pdl(k, dim3(a.s.B), dim3(wide ? 512 : kSelPThreads), smem, st, a);
}
}  // namespace

void launch_select_prefilter(const PrefSelectArgs& a, bool bf16, cudaStream_t st) {
  if (a.s.B == 0) return;
  const size_t smem = kSelectMaxK * sizeof(uint64_t) + (4096 + 40) * sizeof(uint32_t) + kSelResident * sizeof(uint64_t);
  if (bf16) dispatch_select_prefilter<__nv_bfloat16>(a, smem, st);
  else dispatch_select_prefilter<float>(a, smem, st);
}

// ===========================================================================
// K5: first-K eligible rows in ascending row order (term-only queries,
// pipeline.cpp:30-40; with all_rows it is full_scan_tbr's row list).
// One CTA per query: scan the per-chunk counts K1 produced, then extract only
// the chunks that hold output rows.
// ===========================================================================
// Grid (G, B): CTA g of query q owns a contiguous range of chunks.  It sums
// the per-chunk counts before its range (the rows that precede it), exits if
// those already fill the output, scans its own counts, and its warps extract
// the non-empty chunks that hold output rows in parallel -- one chunk per
// warp, four mask words per lane, a warp scan for the output positions.
// (A single CTA per query walking the chunks one at a time took 1.8 ms for a
// sparse low-selectivity query over 50M rows: one dependent mask load per
// non-empty chunk.)
__global__ void __launch_bounds__(256) first_k_kernel(FirstKArgs a) {
  __shared__ uint32_t tmp[40];
  __shared__ uint32_t s_list[256], s_start[256], s_n;
  const uint32_t q = blockIdx.y;
  const QParam qp = a.qp[q];
  if (!a.all_rows && (qp.flags & (QF_ACTIVE | QF_EMB)) != QF_ACTIVE) return;
  const uint32_t ne = a.n_elig[q];
  const uint64_t want64 = a.all_rows ? a.rows_cap : qp.k;
  const uint32_t want = static_cast<uint32_t>(min(static_cast<uint64_t>(ne), want64));
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.out_cnt) a.out_cnt[q] = want;
  if (want == 0) return;
  const uint32_t per = (a.n_chunks + gridDim.x - 1) / gridDim.x;
  const uint32_t c0 = blockIdx.x * per, c1 = min(c0 + per, a.n_chunks);
  if (c0 >= c1) return;
  const uint32_t* cc = a.chunk_cnt + static_cast<size_t>(q) * a.n_chunks;
  const uint32_t* mk = a.mask + static_cast<size_t>(q) * a.words;
  hyre_hit* hits = a.hits ? a.hits + a.hit_off[q] : nullptr;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // rows in the chunks before this CTA's range, 8 counts per thread per
  // step; stop as soon as they fill the output (dense queries: one step)
  uint32_t base = 0;
  for (uint32_t i0 = 0; i0 < c0 && base < want; i0 += 8 * blockDim.x) {
    uint32_t part = 0;
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u) {
      const uint32_t i = i0 + u * blockDim.x + threadIdx.x;
      part += i < c0 ? cc[i] : 0u;
    }
    uint32_t tot;
    block_excl_scan(part, tmp, &tot);
    base += tot;
  }
  if (base >= want) return;
  for (uint32_t t0 = c0; t0 < c1 && base < want; t0 += blockDim.x) {
    const uint32_t ch = t0 + threadIdx.x;
    const uint32_t c = ch < c1 ? cc[ch] : 0u;
    uint32_t tot;
    const uint32_t pre = block_excl_scan(c, tmp, &tot);
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    if (c && base + pre < want) {  // a chunk holding output rows
      const uint32_t e = atomicAdd(&s_n, 1u);
      s_list[e] = ch;
      s_start[e] = base + pre;
    }
    __syncthreads();
    const uint32_t n = s_n;
    for (uint32_t e = warp; e < n; e += nwarps) {
      const uint32_t chunk = s_list[e];
      const uint32_t w0 = chunk * kChunkWords + lane * 4;
      uint32_t w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = w0 + u < a.words ? mk[w0 + u] : 0u;
      const uint32_t p = __popc(w[0]) + __popc(w[1]) + __popc(w[2]) + __popc(w[3]);
      uint32_t out = s_start[e] + warp_incl_scan(p, lane) - p;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t x = w[u];
        while (x && out < want) {
          const int b = __ffs(x) - 1;
          x &= x - 1;
          const uint32_t row = a.row_base + (w0 + u) * 32 + b;
          if (hits) {
            hits[out].row = row;
            hits[out].score = 0.0f;
          }
          if (a.rows_out) a.rows_out[out] = row;
          ++out;
        }
      }
    }
    base += tot;
    __syncthreads();  // s_list / s_n reuse
  }
}

void launch_first_k(const FirstKArgs& a, cudaStream_t st) {
  if (a.B == 0 || a.n_chunks == 0) return;
  // ~4 CTAs per SM over the batch, at least 32 chunks (128K rows) per CTA
  const uint32_t want_g = std::max(1u, 592u / a.B), max_g = (a.n_chunks + 31) / 32;
  const uint32_t G = std::max(1u, std::min(want_g, max_g));
  first_k_kernel<<<dim3(G, a.B), 256, 0, st>>>(a);
}

// ===========================================================================
// K6: sign-quant pre-selection (quantizer.cpp:72-138, batched form
// pipeline.cpp:184-242).  For each query with quant on and more than quant_k
// eligible rows: Q1 histograms popcount(~(q ^ sig)) over eligible rows, Q2
// picks the threshold score t and how many score==t rows survive (lowest
// rows first), Q3 counts ==t rows per chunk, Q4 scans those counts and Q5
// rewrites the mask so exactly quant_k rows stay eligible.  Integer work, so
// the survivor set is bit-exact with the reference's nth_element selection.
// ===========================================================================
namespace {
__device__ __forceinline__ uint32_t qscore(const uint64_t* sig, const uint64_t* qs, uint32_t nw,
                                           uint32_t num_bits) {
  uint32_t s = 0;
  for (uint32_t w = 0; w < nw; ++w) {
    uint64_t same = ~(sig[w] ^ qs[w]);
    if (w + 1 == nw && (num_bits & 63)) same &= (1ull << (num_bits & 63)) - 1ull;
    s += __popcll(same);
  }
  return s;
}
__device__ __forceinline__ bool quant_needed(const QuantArgs& a, uint32_t q) {
  const uint32_t f = a.qp[q].flags;
  // sharded: every shard histograms its rows; the global count decides (thresh)
  return (f & (QF_ACTIVE | QF_EMB | QF_QUANT)) == (QF_ACTIVE | QF_EMB | QF_QUANT) &&
         (a.shard_mode || a.n_elig[q] > a.qp[q].quant_k);
}
}  // namespace

__global__ void __launch_bounds__(128) quant_hist_kernel(QuantArgs a) {
  extern __shared__ uint32_t h[];
  const uint32_t q = blockIdx.y, chunk = blockIdx.x;
  if (!quant_needed(a, q)) return;
  for (uint32_t i = threadIdx.x; i <= a.num_bits; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t widx = chunk * kChunkWords + threadIdx.x;
  uint32_t w = a.mask[static_cast<size_t>(q) * a.words + widx];
  const uint64_t* qs = a.qsig + static_cast<size_t>(q) * a.nw;
  while (w) {
    const int b = __ffs(w) - 1;
    w &= w - 1;
    const uint32_t row = widx * 32 + b;
    atomicAdd(h + qscore(a.sigs + static_cast<size_t>(row) * a.nw, qs, a.nw, a.num_bits), 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i <= a.num_bits; i += blockDim.x)
    if (h[i]) atomicAdd(a.hist + static_cast<size_t>(q) * (a.num_bits + 1) + i, h[i]);
}

__global__ void quant_thresh_kernel(QuantArgs a) {
  const uint32_t q = blockIdx.x;
  if (threadIdx.x != 0) return;
  uint32_t* ts = a.tsel + q * 4;
  ts[2] = 0;
  ts[3] = 0;
  if (!quant_needed(a, q)) return;
  const uint32_t qk = a.qp[q].quant_k;
  const uint32_t* h = (a.hist_total ? a.hist_total : a.hist) + static_cast<size_t>(q) * (a.num_bits + 1);
  if (a.shard_mode) {  // global eligible count = sum of the global histogram
    uint64_t total = 0;
    for (uint32_t s = 0; s <= a.num_bits; ++s) total += h[s];
    if (total <= qk) return;
  }
  uint32_t above = 0;
  for (int s = static_cast<int>(a.num_bits); s >= 0; --s) {
    if (above + h[s] >= qk) {
      ts[0] = static_cast<uint32_t>(s);
      ts[1] = qk - above;  // rows with score == s to keep (lowest rows first)
      ts[2] = 1;
      break;
    }
    above += h[s];
  }
  a.n_elig[q] = a.shard_mode ? 0u : qk;  // sharded: quant_apply counts the local survivors
}

__global__ void __launch_bounds__(128) quant_eq_kernel(QuantArgs a) {
  const uint32_t q = blockIdx.y, chunk = blockIdx.x;
  const uint32_t* ts = a.tsel + q * 4;
  if (!ts[2]) return;
  const uint32_t widx = chunk * kChunkWords + threadIdx.x;
  uint32_t w = a.mask[static_cast<size_t>(q) * a.words + widx];
  const uint64_t* qs = a.qsig + static_cast<size_t>(q) * a.nw;
  uint32_t c = 0;
  while (w) {
    const int b = __ffs(w) - 1;
    w &= w - 1;
    c += qscore(a.sigs + static_cast<size_t>(widx * 32 + b) * a.nw, qs, a.nw, a.num_bits) == ts[0];
  }
  c = __reduce_add_sync(kFull, c);
  __shared__ uint32_t ws[4];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0)
    a.eq_cnt[static_cast<size_t>(q) * a.n_chunks + chunk] = ws[0] + ws[1] + ws[2] + ws[3];
}

__global__ void __launch_bounds__(1024) quant_scan_kernel(QuantArgs a) {
  __shared__ uint32_t tmp[40];
  const uint32_t q = blockIdx.x;
  if (!a.tsel[q * 4 + 2]) return;
  uint32_t* e = a.eq_cnt + static_cast<size_t>(q) * a.n_chunks;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < a.n_chunks; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < a.n_chunks ? e[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, tmp, &tot);
    if (i < a.n_chunks) e[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) a.tsel[q * 4 + 3] = carry;  // this shard's ==t rows
}

__global__ void __launch_bounds__(128) quant_apply_kernel(QuantArgs a) {
  __shared__ uint32_t tmp[40];
  __shared__ uint32_t ws[4];
  const uint32_t q = blockIdx.y, chunk = blockIdx.x;
  const uint32_t* ts = a.tsel + q * 4;
  if (!ts[2]) return;
  const uint32_t t = ts[0], keep_eq = ts[1];
  const uint32_t widx = chunk * kChunkWords + threadIdx.x;
  uint32_t* mp = a.mask + static_cast<size_t>(q) * a.words + widx;
  const uint32_t w = *mp;
  const uint64_t* qs = a.qsig + static_cast<size_t>(q) * a.nw;
  uint32_t gt = 0, eq = 0;
  uint32_t u = w;
  while (u) {
    const int b = __ffs(u) - 1;
    u &= u - 1;
    const uint32_t s = qscore(a.sigs + static_cast<size_t>(widx * 32 + b) * a.nw, qs, a.nw, a.num_bits);
    if (s > t) gt |= 1u << b;
    else if (s == t) eq |= 1u << b;
  }
  uint32_t tot;
  uint32_t rank = a.eq_cnt[static_cast<size_t>(q) * a.n_chunks + chunk] +
                  block_excl_scan(__popc(eq), tmp, &tot);
  uint32_t keep = gt;
  u = eq;
  while (u) {
    const int b = __ffs(u) - 1;
    u &= u - 1;
    if (rank < keep_eq) keep |= 1u << b;
    ++rank;
  }
  *mp = keep;
  const uint32_t c = __reduce_add_sync(kFull, __popc(keep));
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t tot4 = ws[0] + ws[1] + ws[2] + ws[3];
    a.chunk_cnt[static_cast<size_t>(q) * a.n_chunks + chunk] = tot4;
    if (a.shard_mode && tot4) atomicAdd(a.n_elig + q, tot4);
  }
}

void launch_quant_hist(const QuantArgs& a, cudaStream_t st) {
  if (a.B == 0) return;
  dim3 grid(a.n_chunks, a.B);
  quant_hist_kernel<<<grid, kChunkWords, (a.num_bits + 1) * sizeof(uint32_t), st>>>(a);
}
void launch_quant_select(const QuantArgs& a, cudaStream_t st) {
  if (a.B == 0) return;
  dim3 grid(a.n_chunks, a.B);
  quant_thresh_kernel<<<a.B, 32, 0, st>>>(a);
  quant_eq_kernel<<<grid, kChunkWords, 0, st>>>(a);
  quant_scan_kernel<<<a.B, 1024, 0, st>>>(a);
}
void launch_quant_apply(const QuantArgs& a, cudaStream_t st) {
  if (a.B == 0) return;
  dim3 grid(a.n_chunks, a.B);
  quant_apply_kernel<<<grid, kChunkWords, 0, st>>>(a);
}
void launch_quant(const QuantArgs& a, cudaStream_t st) {
  launch_quant_hist(a, st);
  launch_quant_select(a, st);
  launch_quant_apply(a, st);
}

// ---- peer-memory exchanges of a sharded batch (ShardCtx) ----
namespace {
__global__ void sum_peers_kernel(PeerPtrs src, uint32_t G, size_t n, uint32_t* dst) {
  for (size_t i = blockIdx.x * size_t{blockDim.x} + threadIdx.x; i < n; i += size_t{gridDim.x} * blockDim.x) {
    uint32_t s = 0;
    for (uint32_t g = 0; g < G; ++g) s += src.p[g][i];
    dst[i] = s;
  }
}
__global__ void quant_offset_kernel(PeerPtrs tsel, uint32_t g, uint32_t B, uint32_t* my) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= B || !my[q * 4 + 2]) return;
  uint32_t below = 0;  // ==t rows of the lower shards (lower global rows keep ties first)
  for (uint32_t h = 0; h < g; ++h) below += tsel.p[h][q * 4 + 3];
  const uint32_t budget = my[q * 4 + 1];
  my[q * 4 + 1] = budget > below ? budget - below : 0u;
}
}  // namespace

void launch_sum_peers(const PeerPtrs& src, uint32_t G, size_t n, uint32_t* dst, cudaStream_t st) {
  if (!n) return;
  sum_peers_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 1024)), 256, 0, st>>>(src, G, n, dst);
}
void launch_quant_offset(const PeerPtrs& tsel, uint32_t g, uint32_t B, uint32_t* my_tsel, cudaStream_t st) {
  if (!B) return;
  quant_offset_kernel<<<(B + 127) / 128, 128, 0, st>>>(tsel, g, B, my_tsel);
}

// ===========================================================================
// Stage helpers
// ===========================================================================
template <typename RowT>
__global__ void gather_scores_kernel(const RowT* emb, uint32_t dp, uint32_t row_base,
                                     const float* q, const uint32_t* rows, uint64_t n, float* out) {
  const uint64_t warp = (blockIdx.x * uint64_t{blockDim.x} + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const RowT* row = emb + static_cast<size_t>(rows[warp] - row_base) * dp;
  float s = 0.0f;
  for (uint32_t e = lane; e < dp; e += 32) s = fmaf(static_cast<float>(row[e]), q[e], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0) out[warp] = clamp_score(s);
}

void launch_gather_scores(const void* emb, bool bf16, uint32_t dp, uint32_t row_base,
                          const float* q, const uint32_t* rows, uint64_t n, float* out,
                          cudaStream_t st) {
  if (!n) return;
  const unsigned blocks = static_cast<unsigned>((n * 32 + 255) / 256);
  if (bf16)
    gather_scores_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(emb), dp, row_base, q, rows, n, out);
  else
    gather_scores_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(emb), dp,
                                                          row_base, q, rows, n, out);
}

__global__ void make_keys_kernel(const uint32_t* rows, const float* scores, uint64_t n, uint64_t* keys) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x)
    keys[i] = make_key(scores[i] + 0.0f, rows[i]);
}

void launch_make_keys(const uint32_t* rows, const float* scores, uint64_t n, uint64_t* keys,
                      cudaStream_t st) {
  if (!n) return;
  make_keys_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096)), 256, 0, st>>>(
      rows, scores, n, keys);
}

// Quant keys: (agreement << 32) | ~row, so "larger key" = (score desc, row asc).
__global__ void quant_keys_kernel(const uint64_t* sigs, uint32_t nw, uint32_t num_bits, uint32_t row_base,
                                  const uint64_t* qsig, const uint32_t* rows, uint64_t n, uint64_t* keys) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x) {
    const uint32_t r = rows[i];
    const uint32_t s = qscore(sigs + static_cast<size_t>(r - row_base) * nw, qsig, nw, num_bits);
    keys[i] = (static_cast<uint64_t>(s) << 32) | static_cast<uint32_t>(~r);
  }
}

void launch_quant_keys(const uint64_t* sigs, uint32_t nw, uint32_t num_bits, uint32_t row_base,
                       const uint64_t* qsig, const uint32_t* rows, uint64_t n, uint64_t* keys,
                       cudaStream_t st) {
  if (!n) return;
  quant_keys_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096)), 256, 0, st>>>(
      sigs, nw, num_bits, row_base, qsig, rows, n, keys);
}

// ===========================================================================
// Multi-GPU merge: the global top-K is a subset of the union of
// the shard top-Ks, so the exact answer is K4 over the gathered keys.
// g_hits: [G][hits_stride] hyre_hit, g_off: [G][B] u64, g_cnt: [G][B] u32.
// ===========================================================================
__global__ void gather_keys_kernel(const hyre_hit* g_hits, uint64_t hits_stride, const uint64_t* g_off,
                                   uint64_t off_stride, const uint32_t* g_cnt, uint64_t cnt_stride, uint32_t G,
                                   uint32_t cap, uint64_t* keys, uint32_t* cnt) {
  const uint32_t q = blockIdx.x;
  uint32_t base = 0;
  for (uint32_t g = 0; g < G; ++g) {
    const uint32_t c = g_cnt[g * cnt_stride + q];
    const hyre_hit* h = g_hits + g * hits_stride + g_off[g * off_stride + q];
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x)
      if (base + i < cap) keys[static_cast<size_t>(q) * cap + base + i] = make_key(h[i].score + 0.0f, h[i].row);
    base += c;
  }
  if (threadIdx.x == 0) cnt[q] = base;
}

void launch_gather_keys(const hyre_hit* g_hits, uint64_t hits_stride, const uint64_t* g_off, uint64_t off_stride,
                        const uint32_t* g_cnt, uint64_t cnt_stride, uint32_t G, uint32_t B, uint32_t cap,
                        uint64_t* keys, uint32_t* cnt, cudaStream_t st) {
  if (B == 0) return;
  gather_keys_kernel<<<B, 256, 0, st>>>(g_hits, hits_stride, g_off, off_stride, g_cnt, cnt_stride, G, cap, keys, cnt);
}

// Sharded merge, one CTA per query, reading every shard's results in place
// through peer memory (NVLink loads on a multi-GPU node): the gather and the
// merge's key build in one pass, no staging copy.
namespace {
__global__ void gather_peer_keys_kernel(PeerHits ph, uint32_t G, const uint64_t* hit_off, const QParam* qp,
                                        uint32_t cap, uint64_t* keys, uint32_t* cnt) {
  const uint32_t q = blockIdx.x;
  if ((qp[q].flags & (QF_ACTIVE | QF_EMB)) != (QF_ACTIVE | QF_EMB)) return;
  const uint64_t off = hit_off[q];
  uint32_t base = 0;
  for (uint32_t g = 0; g < G; ++g) {
    const uint32_t c = ph.cnt[g][q];
    const hyre_hit* h = ph.hits[g] + off;
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x)
      if (base + i < cap) keys[static_cast<size_t>(q) * cap + base + i] = make_key(h[i].score + 0.0f, h[i].row);
    base += c;
  }
  if (threadIdx.x == 0) cnt[q] = min(base, cap);
}
// term-only (pipeline.cpp:30-40): shard row lists are ascending and the
// shards are contiguous row ranges, so the global first K is their
// concatenation in shard order
__global__ void concat_term_only_kernel(PeerHits ph, uint32_t G, const uint64_t* hit_off, const QParam* qp,
                                        const uint32_t* true_k, hyre_hit* out, uint32_t* out_cnt) {
  const uint32_t q = blockIdx.x;
  if ((qp[q].flags & (QF_ACTIVE | QF_EMB)) != QF_ACTIVE) return;
  const uint64_t off = hit_off[q];
  const uint32_t k = true_k[q];
  uint32_t base = 0;
  for (uint32_t g = 0; g < G && base < k; ++g) {
    const uint32_t c = min(ph.cnt[g][q], k - base);
    const hyre_hit* h = ph.hits[g] + off;
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) out[off + base + i] = h[i];
    base += c;
  }
  if (threadIdx.x == 0) out_cnt[q] = base;
}
__global__ void gather_peer_keys_one_kernel(PeerHits ph, uint32_t G, uint64_t off, uint32_t q, uint64_t cap,
                                            uint64_t* keys, uint32_t* cnt) {
  uint64_t base = 0;
  for (uint32_t g = 0; g < G; ++g) {
    const uint32_t c = ph.cnt[g][q];
    const hyre_hit* h = ph.hits[g] + off;
    for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < c; i += uint64_t{gridDim.x} * blockDim.x)
      if (base + i < cap) keys[base + i] = make_key(h[i].score + 0.0f, h[i].row);
    base += c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = static_cast<uint32_t>(min(base, cap));
}
}  // namespace

void launch_gather_peer_keys(const PeerHits& ph, uint32_t G, const uint64_t* hit_off, const QParam* qp, uint32_t B,
                             uint32_t cap, uint64_t* keys, uint32_t* cnt, cudaStream_t st) {
  if (B) gather_peer_keys_kernel<<<B, 256, 0, st>>>(ph, G, hit_off, qp, cap, keys, cnt);
}
void launch_concat_term_only(const PeerHits& ph, uint32_t G, const uint64_t* hit_off, const QParam* qp,
                             const uint32_t* true_k, uint32_t B, hyre_hit* out, uint32_t* out_cnt, cudaStream_t st) {
  if (B) concat_term_only_kernel<<<B, 256, 0, st>>>(ph, G, hit_off, qp, true_k, out, out_cnt);
}
void launch_gather_peer_keys_one(const PeerHits& ph, uint32_t G, uint64_t off, uint32_t q, uint64_t cap,
                                 uint64_t* keys, uint32_t* cnt, cudaStream_t st) {
  gather_peer_keys_one_kernel<<<148, 256, 0, st>>>(ph, G, off, q, cap, keys, cnt);
}


// ===========================================================================
// Exhaustive exact top-K (Executor::exhaustive): every eligible row of one
// query scored exactly, all keys sorted.  Runs for hybrid queries with
// k > kSelectMaxK (bucket_top_k returns min(k, n) for any k,
// proj/src/knn.cpp:42-95) and for a query whose threshold recovery rounds
// did not converge (more than the candidate capacity of rows tied within the
// prefilter band).  The scores use rescore_list's arithmetic -- the one every
// other returned score uses -- so a query's hits do not depend on the path.
// ===========================================================================
namespace {
__global__ void rows_to_keys_kernel(const uint32_t* rows, uint64_t n, uint64_t* keys) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x)
    keys[i] = make_key(0.0f, rows[i]);
}
// quant keys (agreement << 32 | ~row) -> score keys of the same rows
__global__ void quant_to_keys_kernel(const uint64_t* qkeys, uint64_t n, uint64_t* keys) {
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n; i += uint64_t{gridDim.x} * blockDim.x)
    keys[i] = make_key(0.0f, ~static_cast<uint32_t>(qkeys[i]));
}
__global__ void keys_to_hits_kernel(const uint64_t* keys, uint64_t n, hyre_hit* out, uint32_t* out_cnt,
                                    uint32_t* rerun) {
  const uint64_t t = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
  if (t == 0) {
    if (out_cnt) *out_cnt = static_cast<uint32_t>(n);
    if (rerun) *rerun = 0;
  }
  for (uint64_t i = t; i < n; i += uint64_t{gridDim.x} * blockDim.x) {
    out[i].row = key_row(keys[i]);
    out[i].score = key_score(keys[i]);
  }
}
constexpr uint32_t kRescoreSlice = 2048;  // keys per CTA step
template <typename RowT, int LPR, int CPL>
__global__ void __launch_bounds__(256) rescore_keys_kernel(PrefSelectArgs pa, uint32_t q, uint64_t* keys,
                                                           uint64_t n) {
  __shared__ uint32_t above;  // rescore_list's threshold count (threshold 2: never incremented)
  for (uint64_t b0 = uint64_t{blockIdx.x} * kRescoreSlice; b0 < n; b0 += uint64_t{gridDim.x} * kRescoreSlice)
    rescore_list<RowT, LPR, CPL>(pa, q, keys + b0, static_cast<uint32_t>(n - b0 < kRescoreSlice ? n - b0 : kRescoreSlice), 2.0f,
                                 &above);
}
template <typename RowT>
void dispatch_rescore_keys(const PrefSelectArgs& a, uint32_t q, uint64_t* keys, uint64_t n, cudaStream_t st) {
  using KFn = void (*)(PrefSelectArgs, uint32_t, uint64_t*, uint64_t);
  KFn k = nullptr;
  const uint32_t cpr = a.dp_chunks;
  if (cpr == 8) k = rescore_keys_kernel<RowT, 8, 1>;
  else if (cpr == 16) k = rescore_keys_kernel<RowT, 16, 1>;
  else if (cpr == 32) k = rescore_keys_kernel<RowT, 32, 1>;
  else if (cpr == 64) k = rescore_keys_kernel<RowT, 32, 2>;
  else if (cpr == 128) k = rescore_keys_kernel<RowT, 32, 4>;
  else if (cpr == 256) k = rescore_keys_kernel<RowT, 32, 8>;
  else throw Error(HYRE_INTERNAL, "unsupported row stride (chunks per row " + std::to_string(cpr) + ")");
  const uint64_t slices = (n + kRescoreSlice - 1) / kRescoreSlice;
  k<<<static_cast<unsigned>(std::min<uint64_t>(slices, 148 * 8)), 256, 0, st>>>(a, q, keys, n);
}
unsigned grid_for(uint64_t n) { return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16))); }
}  // namespace

void launch_rows_to_keys(const uint32_t* rows, uint64_t n, uint64_t* keys, cudaStream_t st) {
  if (n) rows_to_keys_kernel<<<grid_for(n), 256, 0, st>>>(rows, n, keys);
}
void launch_quant_to_keys(const uint64_t* qkeys, uint64_t n, uint64_t* keys, cudaStream_t st) {
  if (n) quant_to_keys_kernel<<<grid_for(n), 256, 0, st>>>(qkeys, n, keys);
}
void launch_keys_to_hits(const uint64_t* keys, uint64_t n, hyre_hit* out, uint32_t* out_cnt, uint32_t* rerun,
                         cudaStream_t st) {
  keys_to_hits_kernel<<<grid_for(n), 256, 0, st>>>(keys, n, out, out_cnt, rerun);
}
void launch_rescore_keys(const PrefSelectArgs& a, bool bf16, uint32_t q, uint64_t* keys, uint64_t n,
                         cudaStream_t st) {
  if (!n) return;
  if (bf16) dispatch_rescore_keys<__nv_bfloat16>(a, q, keys, n, st);
  else dispatch_rescore_keys<float>(a, q, keys, n, st);
}
// ---------------------------------------------------------------------------
// batch_scan_tbr (pipeline.cpp:75-93): the (row, batchId) messenger stream of
// a term-only batch, ordered by row then by query position, from the batch's
// eligibility masks.  Pass 1 counts each 32-row word's matches over every
// active query; an exclusive scan places each word; pass 2 (one warp per
// word, lane = row) writes the word's messengers in (row, query) order.
// ---------------------------------------------------------------------------
__global__ void scan_count_kernel(const uint32_t* __restrict__ mask, const QParam* __restrict__ qp, uint32_t B,
                                  uint32_t W, uint64_t* __restrict__ cnt) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w > W) return;
  uint64_t c = 0;
  if (w < W)
    for (uint32_t b = 0; b < B; ++b)
      if (qp[b].flags & QF_ACTIVE) c += __popc(mask[static_cast<size_t>(b) * W + w]);
  cnt[w] = c;  // cnt[W] = 0: the scan's total lands in off[W]
}

__global__ void scan_emit_kernel(const uint32_t* __restrict__ mask, const QParam* __restrict__ qp, uint32_t B,
                                 uint32_t W, uint32_t row_base, const uint64_t* __restrict__ off,
                                 const uint32_t* __restrict__ batch_ids, hyre_messenger* __restrict__ out,
                                 uint64_t cap) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= W) return;
  const uint64_t base = off[w];
  if (base >= cap || off[w + 1] == base) return;
  uint32_t mine = 0;
  for (uint32_t b = 0; b < B; ++b)
    if (qp[b].flags & QF_ACTIVE) mine += (mask[static_cast<size_t>(b) * W + w] >> lane) & 1u;
  uint32_t incl = mine;  // inclusive warp scan over the rows of this word
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  uint64_t pos = base + incl - mine;
  const uint32_t row = row_base + w * 32 + lane;
  for (uint32_t b = 0; b < B && pos < cap; ++b) {
    if (!(qp[b].flags & QF_ACTIVE)) continue;
    if ((mask[static_cast<size_t>(b) * W + w] >> lane) & 1u) out[pos++] = hyre_messenger{row, batch_ids[b], 0.0f};
  }
}

void launch_scan_count(const uint32_t* mask, const QParam* qp, uint32_t B, uint32_t W, uint64_t* cnt,
                       cudaStream_t st) {
  scan_count_kernel<<<(W + 1 + 255) / 256, 256, 0, st>>>(mask, qp, B, W, cnt);
}

void launch_scan_emit(const uint32_t* mask, const QParam* qp, uint32_t B, uint32_t W, uint32_t row_base,
                      const uint64_t* off, const uint32_t* batch_ids, hyre_messenger* out, uint64_t cap,
                      cudaStream_t st) {
  if (W) scan_emit_kernel<<<(W + 7) / 8, 256, 0, st>>>(mask, qp, B, W, row_base, off, batch_ids, out, cap);
}

// ---------------------------------------------------------------------------
// K7: single-launch scorer for small indexes (latency-bound
// single queries).  One CTA per 1024-row segment evaluates the query's CNF
// words for its segment from the K1 program (dense bitmaps only), compacts the
// eligible rows, scores them exactly with K2's arithmetic (the lane layout and
// xor butterfly of rescore_list, so scores equal every other path's bit for
// bit), keeps its segment's top min(k, n) keys (bitonic sort in shared memory)
// and appends them to the query's candidate buffer; K4 selects the final top
// K.  No sample, no thresholds, no recovery: the candidates are exact.
// ---------------------------------------------------------------------------
namespace {
template <typename RowT, int LPR, int CPL>
__global__ void __launch_bounds__(512) small_topk_kernel(SmallArgs a) {
  __shared__ uint16_t list[kSegRows];
  __shared__ uint64_t keys[kSegRows];
  __shared__ uint32_t s_n, s_base, s_nc;
  __shared__ uint32_t s_prog[kSmallProg];
  __shared__ const uint32_t* s_refs[kSmallRefs];
  __shared__ uint32_t s_cl[kSmallClauses];
  __shared__ uint32_t s_cw[kSmallClauses][32];
  constexpr int G = 32 / LPR, E = Chunk<RowT>::kElems;
  const uint32_t seg = blockIdx.x, lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane / LPR, li = lane % LPR;
  const RowT* emb = static_cast<const RowT*>(a.emb);
  for (uint32_t qi = 0; qi < a.B; ++qi) {
    const QParam qp = a.qp[qi];
    if ((qp.flags & (QF_ACTIVE | QF_EMB)) != (QF_ACTIVE | QF_EMB)) continue;  // uniform
    // this segment's 32 mask words (mask_kernel's AND of ORs over the refs):
    // the query's program and the batch's ref pointers are staged in shared
    // memory, then one warp per clause ORs its refs' words (independent
    // loads in flight) and warp 0 ANDs the clauses
    const uint32_t widx = seg * 32 + lane;
    const bool constrained = !(qp.flags & (QF_EMPTY | QF_MATCH_ALL));
    if (constrained) {
      const uint32_t L = min(kSmallProg, a.prog_words - qp.prog_off);
      for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) s_prog[i] = a.prog[qp.prog_off + i];
      for (uint32_t i = threadIdx.x; i < min(a.n_refs, kSmallRefs); i += blockDim.x) s_refs[i] = a.refs[i];
      __syncthreads();
      if (threadIdx.x == 0) {  // clause layout: first ref index and ref count
        const uint32_t nc = min(s_prog[0], kSmallClauses);
        uint32_t pos = 1;
        for (uint32_t c = 0; c < nc; ++c) {
          const uint32_t nr = pos < L ? s_prog[pos] : 0u;
          s_cl[c] = (pos + 1) | (min(nr, L - min(L, pos + 1)) << 16);
          pos += 1 + nr;
        }
        s_nc = nc;
      }
      __syncthreads();
      for (uint32_t c = wib; c < s_nc; c += nw) {
        const uint32_t first = s_cl[c] & 0xFFFFu, nr = s_cl[c] >> 16;
        uint32_t cw = 0;
        if (widx < a.words)
          for (uint32_t r = 0; r < nr; ++r) {
            const uint32_t ref = s_prog[first + r];
            cw |= __ldg((ref < kSmallRefs ? s_refs[ref] : a.refs[ref]) + widx);
          }
        s_cw[c][lane] = cw;
      }
      __syncthreads();
    }
    if (wib == 0) {
      uint32_t word = 0;
      if (widx < a.words && !(qp.flags & QF_EMPTY)) {
        if (qp.flags & QF_MATCH_ALL) {
          word = tail_mask(widx, a.n_rows);
        } else {
          uint32_t acc = kFull;
          for (uint32_t c = 0; c < s_nc; ++c) acc &= s_cw[c][lane];
          word = acc & tail_mask(widx, a.n_rows);
        }
      }
      const uint32_t c = __popc(word), incl = warp_incl_scan(c, lane);
      uint32_t pos = incl - c;
      for (uint32_t u = word; u; u &= u - 1u) list[pos++] = static_cast<uint16_t>(lane * 32 + __ffs(u) - 1);
      if (lane == 31) s_n = incl;
    }
    __syncthreads();
    const uint32_t n = s_n;
    if (n == 0) {
      __syncthreads();
      continue;
    }
    float qv[CPL][E];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
      for (int e = 0; e < E; ++e) qv[c][e] = a.q[static_cast<size_t>(qi) * a.dp + (li + c * LPR) * E + e];
    const size_t row0 = static_cast<size_t>(seg) * kSegRows;
    for (uint32_t base = 0; base < n; base += nw * G) {
      const uint32_t idx = base + wib * G + g;
      const bool ok = idx < n;
      const uint32_t lr = ok ? static_cast<uint32_t>(row0) + list[idx] : static_cast<uint32_t>(row0);
      const RowT* r = emb + static_cast<size_t>(lr) * a.dp;
      uint4 v[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) v[c] = ok ? ldg_stream(r + (li + c * LPR) * E) : make_uint4(0, 0, 0, 0);
      float acc = 0.0f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc += Chunk<RowT>::dot(v[c], qv[c]);
#pragma unroll
      for (int m = LPR / 2; m >= 1; m >>= 1) acc += __shfl_xor_sync(kFull, acc, m);
      if (li == 0 && ok) {
        const float sc = a.row_w ? weighted_score(acc, __ldg(a.row_w + lr)) : clamp_score(acc);
        keys[idx] = make_key(sc, a.row_base + lr);
      }
    }
    __syncthreads();
    uint32_t m = n;
    if (n > qp.k) {  // the segment's top k keys (score desc, row asc)
      uint32_t p2 = 1;
      while (p2 < n) p2 <<= 1;
      for (uint32_t i = n + threadIdx.x; i < p2; i += blockDim.x) keys[i] = 0ull;
      __syncthreads();
      bitonic_desc(keys, p2);
      m = qp.k;
    }
    if (threadIdx.x == 0) {
      s_base = atomicAdd(a.cand_cnt + qi, m);
      atomicAdd(a.n_elig + qi, n);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
      if (s_base + i < a.cap) a.cand[static_cast<size_t>(qi) * a.cap + s_base + i] = keys[i];
    __syncthreads();
  }
}
}  // namespace

bool small_supported(uint32_t dp_chunks) {
  return dp_chunks == 8 || dp_chunks == 16 || dp_chunks == 32 || dp_chunks == 64 || dp_chunks == 128;
}

void launch_small(const SmallArgs& a, bool bf16, cudaStream_t st) {
  const uint32_t n_seg = (a.n_rows + kSegRows - 1) / kSegRows;
  if (a.B == 0 || n_seg == 0) return;
  using KFn = void (*)(SmallArgs);
  KFn k = nullptr;
  const uint32_t cpr = a.dp_chunks;
#define HYRE_SMALL_PICK(T)                          \
  k = cpr == 8     ? small_topk_kernel<T, 8, 1>     \
      : cpr == 16  ? small_topk_kernel<T, 16, 1>    \
      : cpr == 32  ? small_topk_kernel<T, 32, 1>    \
      : cpr == 64  ? small_topk_kernel<T, 32, 2>    \
      : cpr == 128 ? small_topk_kernel<T, 32, 4>    \
                   : nullptr;
  if (bf16) {
    HYRE_SMALL_PICK(__nv_bfloat16)
  } else {
    HYRE_SMALL_PICK(float)
  }
#undef HYRE_SMALL_PICK
  if (!k) throw Error(HYRE_INTERNAL, "K7: unsupported row stride");
  k<<<n_seg, 512, 0, st>>>(a);
}

}  // namespace hyreb
