// K3: batched scorer on the 5th-gen tensor cores (tcgen05 + TMEM + bulk copies).
//
// Scoring B queries against N jobs is the dense contraction
//   S[N x B] = E[N x d] . Q[B x d]^T
// (Executor::execute_batch's scoring loop, pipeline.cpp:246-256) fused with
// the CNF term match (term_match.cpp:56-78).  One persistent CTA per SM
// streams 128-row tiles through a bulk-copy -> shared-memory ring; one elected
// thread issues tcgen05.mma into TMEM accumulators; CNF warps evaluate each
// row's clauses from its compact term list; epilogue warps pull the
// accumulator tile out of TMEM with tcgen05.ld, compare every score with its
// query's threshold in registers and append only the (eligible, passing)
// (score, row) keys.  Ineligible / sub-threshold jobs never leave registers.
//
// Operand planes:
//  * prefilter (default): the int8 plane, one kind::i8 MMA per K step
//    (K = 32, s32 accumulation; s' = acc x scale_q), or the bf16 hi plane
//    (kind::f16, K = 16, fp32); rows are admitted at s' >= thr - delta_q and
//    rescored exactly afterwards (select_prefilter_kernel), so K3's scores are
//    never returned;
//  * exact (HYRE_PREFILTER=0): hi + lo bf16 planes of the fp32 rows and of the
//    query, E_hi.Q_hi + E_hi.Q_lo + E_lo.Q_hi (the dropped E_lo.Q_lo term is
//    O(2^-16)); a bf16 index scores E.Q_hi + E.Q_lo.
//
// Warp roles: w0 bulk-copy producer, w1 TMEM owner + MMA issuer, 8 epilogue
// warps (16 in the mask / match-all variant; TMEM lane quadrant = warp % 4),
// then 4 or 8 CNF warps in the fused variants.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.cuh"
#include "tc_score.cuh"

namespace hyreb {

namespace {

constexpr uint32_t kTileRows = 128;
constexpr uint32_t kAtomBytes = kTileRows * 128;  // one 128-row x 128-B swizzle-128 box (16 KB)
// per-CTA candidate staging: 16 KB for groups of <= 64 queries (32 keys per
// query), 8 KB for 128-query groups (8 keys per query; overflow goes straight
// to the global buffer) so that their larger query tile still leaves >= 4 ring
// stages in flight
__host__ __device__ constexpr uint32_t stage_bytes_for(uint32_t Np) { return Np <= 64 ? 16384u : 8192u; }
// epilogue warps: 8 (2 per TMEM lane quadrant) next to the fused CNF warps;
// 16 for the mask / match-all variant, whose only per-tile work is the
// epilogue (large query groups need the extra warps to hide TMEM-load and
// compare-chain latency)
__host__ __device__ constexpr uint32_t epi_warps(bool fused) { return fused ? 8u : 16u; }
// fused CNF warps: one thread per tile row and query-chunk share (4 warps
// for one 32-query chunk, 8 -- two chunk halves per row -- for 2 or 4 chunks)
__host__ __device__ constexpr uint32_t cnf_warps(int nch) { return nch <= 2 ? 4u : 8u; }
constexpr uint32_t kAccBufs = 4;                  // max TMEM accumulators (MMA runs up to 4 tiles ahead of the epilogue)
constexpr uint32_t kMaxWarpChunks = 4;            // 32-query chunks per epilogue warp (Np <= 256)
constexpr uint32_t kEligSlots = 4;                // fused CNF: tiles of eligibility words in flight
__host__ __device__ constexpr uint32_t threads_for(bool fused, int nch) {
  return 64 + 32 * epi_warps(fused) + (fused ? 32 * cnf_warps(nch) : 0);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in the barrier
// (woken when the phase completes) instead of re-polling, so idle roles do
// not steal issue slots from the CNF / epilogue warps on the same SMSP
// (without the hint ~20% of K3's issued instructions were poll loops).
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity), "r"(20000u)
        : "memory");
  } while (!done);
}

// Wait for the many-warp roles (epilogue, CNF): after a failed try_wait the
// warp sleeps briefly before re-testing.  try_wait's own suspension ends after
// ~100 cycles whatever the hint, so without the back-off waiting warps re-poll
// continuously and their spin instructions (measured: up to 25% of K3's issued
// instructions) take issue slots from the warps doing work on the same SMSP.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* b, uint32_t parity, uint32_t ns) {
  uint32_t done = 0;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  while (!done) {
    if (ns) __nanosleep(ns);
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// K-major, 128-byte swizzle canonical layout: 8-row core groups 1024 B apart
// (SBO = 64 x 16 B), LBO unused (1), descriptor version 1, layout type 2.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(
          d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// The same with descriptors given as their low words (high word constant:
// SBO = 1024 B, descriptor version 1, SWIZZLE_128B).
__device__ __forceinline__ void mma_bf16w(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n .reg .b64 da, db;\n setp.ne.b32 p, %4, 0;\n"
      " mov.b64 da, {%1, %5};\n mov.b64 db, {%2, %5};\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate), "n"(0x40004040));
}

__device__ __forceinline__ void mma_i8w(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n .reg .b64 da, db;\n setp.ne.b32 p, %4, 0;\n"
      " mov.b64 da, {%1, %5};\n mov.b64 db, {%2, %5};\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate), "n"(0x40004040));
}

// int8 MMA with explicit 64-bit descriptors (the bias K-step's SWIZZLE_NONE
// operands: lo = start >> 4 | LBO >> 4 << 16, hi = SBO >> 4 | version 1)
__device__ __forceinline__ void mma_i8d(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                        uint32_t idesc) {
  asm volatile(
      "{\n .reg .b64 da, db;\n mov.b64 da, {%1, %2};\n mov.b64 db, {%3, %4};\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, 1;\n}" ::"r"(d_tmem),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// v[j] for a lane-varying j without local memory: a 5-level select tree
__device__ __forceinline__ uint32_t pick32(const uint32_t (&v)[32], uint32_t j) {
  uint32_t a[16], b[8], c[4], d[2];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = (j & 16u) ? v[i + 16] : v[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = (j & 8u) ? a[i + 8] : a[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (j & 4u) ? b[i + 4] : b[i];
#pragma unroll
  for (int i = 0; i < 2; ++i) d[i] = (j & 2u) ? c[i + 2] : c[i];
  return (j & 1u) ? d[1] : d[0];
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ bool tc_active(const TcArgs& a, uint32_t q) {
  if (q >= a.B) return false;
  const uint32_t f = a.qp[q].flags;
  if ((f & (QF_ACTIVE | QF_EMB)) != (QF_ACTIVE | QF_EMB)) return false;
  const uint32_t ne = a.n_elig[q];
  if (ne == 0) return false;
  if (a.mode == SCORE_SAMPLE) return ne > a.gate;
  if (a.mode == SCORE_RERUN) return a.rerun[q] != 0;
  return true;
}

// i-th tile this CTA processes in the given mode, or UINT32_MAX.
__device__ __forceinline__ uint32_t tile_of(const TcArgs& a, uint32_t i) {
  const uint32_t j = blockIdx.x + i * gridDim.x;
  if (a.mode != SCORE_SAMPLE) return j < a.n_tiles ? j : UINT32_MAX;
  // sampled 1024-row segments (8 tiles) every `period` segments, like K2
  const uint32_t seg = (j / 8) * a.period, t = seg * 8 + (j % 8);
  return t < a.n_tiles ? t : UINT32_MAX;
}

// Eligibility of one row for all NCH 32-query chunks of the group
// (term_match.cpp:34-78: a query matches iff every slot it constrains holds a
// row term listed in its clause).  The table holds, per term t,
//   v(t) = hc(slot(t)) & ~users(t)
// (the group's queries that constrain t's slot but do not list t; sentinel:
// all ones).  A constrained slot s fails a query iff EVERY row term in s
// fails it, i.e. fail_s = AND over the slot's segment of v(t), so
//   fail = OR over present slots of AND over the segment of v  |  hc of the
//          constrained slots the row has no term in
// (an empty doc slice never matches, term_match.cpp:45-46).  The row's ids are
// slot-major, and its segment-start mask (bit j: id j opens a new slot) makes
// the whole evaluation two LOP3s per id and chunk, after J independent table
// loads issued back to back.
template <int J, int TB, int NCH, int NT>
__device__ __forceinline__ void cnf_row(const uint32_t (&tw)[J * TB / 4], uint64_t masks, uint32_t T, uint32_t tbl,
                                        uint32_t hc, uint32_t live, uint32_t cslots, uint32_t c0,
                                        uint32_t (&out)[NT]) {
  uint32_t v[J][NT];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const uint32_t id = TB == 1 ? (tw[j >> 2] >> ((j & 3) * 8)) & 0xFFu : (tw[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
    // u8 ids index a 256-entry table directly (entries T..255 are sentinels)
    const uint32_t e = tbl + ((TB == 1 ? id : min(id, T)) * NCH + c0) * 4;
    // explicit ld.shared (32-bit shared addresses): generic loads would cost
    // long-scoreboard waits
    if (NT == 1) {
      asm("ld.shared.u32 %0, [%1];" : "=r"(v[j][0]) : "r"(e));
    } else if (NT == 2) {
      asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v[j][0]), "=r"(v[j][NT - 1]) : "r"(e));
    } else {
      asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
          : "=r"(v[j][0]), "=r"(v[j][1 % NT]), "=r"(v[j][2 % NT]), "=r"(v[j][3 % NT])
          : "r"(e));
    }
  }
  const uint32_t starts = static_cast<uint32_t>(masks), pres = static_cast<uint32_t>(masks >> 32);
  // segment masks: bit j of starts lands on a byte's sign bit in starts << s,
  // s = (7 - j) mod 8, and prmt replicates that sign across the word -- one
  // instruction per id plus 7 shifts per row
  uint32_t sh[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) sh[k] = starts << k;
  uint32_t seg[NT], fail[NT];
#pragma unroll
  for (int c = 0; c < NT; ++c) {
    seg[c] = v[0][c];
    fail[c] = 0u;
  }
#pragma unroll
  for (int j = 1; j < J; ++j) {
    uint32_t m;  // all ones where id j opens a new slot segment
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(m) : "r"(sh[(7 - j) & 7]), "r"(((j >> 3) | 8) * 0x1111));
#pragma unroll
    for (int c = 0; c < NT; ++c) {
      fail[c] |= seg[c] & m;
      seg[c] = (seg[c] | m) & v[j][c];
    }
  }
#pragma unroll
  for (int c = 0; c < NT; ++c) fail[c] |= pres ? seg[c] : 0u;
  for (uint32_t miss = cslots & ~pres; miss; miss &= miss - 1u) {
    const uint32_t sl = __ffs(miss) - 1;
#pragma unroll
    for (int c = 0; c < NT; ++c) {
      uint32_t x;
      asm("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(hc + (sl * NCH + c0 + c) * 4));
      fail[c] |= x;
    }
  }
#pragma unroll
  for (int c = 0; c < NT; ++c) {
    uint32_t lv;
    asm("ld.shared.u32 %0, [%1];" : "=r"(lv) : "r"(live + (c0 + c) * 4));
    out[c] = lv & ~fail[c];
  }
}

// Slot-grouped rows (W ids per group, static segments; index.cu
// cnf_group_rows_kernel): fail = OR over groups of AND over the group's
// table words -- one LOP3 per id after the first and one OR per group and
// chunk, no segment masks, no missing-slot loop (EMPTY_g entries carry hc_g).
template <int J, int W, int NCH, int NT, int JWN>
__device__ __forceinline__ void cnf_row_grouped(const uint32_t (&tw)[JWN], const uint32_t* __restrict__ tbl8,
                                                uint32_t live, uint32_t c0, uint32_t (&out)[NT]) {
  // entry byte offset id x (NCH x 4) straight from the packed id word: one
  // shift and one mask per id; the static table's address folds into the
  // load's immediate (c0 = 0 whenever a thread owns every chunk)
  constexpr int kSh = NCH == 1 ? 2 : (NCH == 2 ? 3 : (NCH == 4 ? 4 : 5));
  constexpr uint32_t kMask = 0xFFu << kSh;
  const uint32_t* base = NT == NCH ? tbl8 : tbl8 + c0;
  uint32_t v[J][NT];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int sh = (j & 3) * 8 - kSh;
    const uint32_t off = (sh >= 0 ? (tw[j >> 2] >> sh) : (tw[j >> 2] << -sh)) & kMask;  // bytes
    const uint32_t* e = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(base) + off);
    if (NT == 1) {
      v[j][0] = e[0];
    } else if (NT == 2) {
      const uint2 x = *reinterpret_cast<const uint2*>(e);
      v[j][0] = x.x;
      v[j][NT - 1] = x.y;
    } else {
      const uint4 x = *reinterpret_cast<const uint4*>(e);
      v[j][0] = x.x;
      v[j][1 % NT] = x.y;
      v[j][2 % NT] = x.z;
      v[j][3 % NT] = x.w;
    }
  }
  uint32_t fail[NT];
#pragma unroll
  for (int c = 0; c < NT; ++c) fail[c] = 0u;
#pragma unroll
  for (int g = 0; g < J / W; ++g) {
#pragma unroll
    for (int c = 0; c < NT; ++c) {
      uint32_t a = v[g * W][c];
#pragma unroll
      for (int p = 1; p < W; ++p) a &= v[g * W + p][c];
      fail[c] |= a;
    }
  }
#pragma unroll
  for (int c = 0; c < NT; ++c) {
    uint32_t lv;
    asm("ld.shared.u32 %0, [%1];" : "=r"(lv) : "r"(live + (c0 + c) * 4));
    out[c] = lv & ~fail[c];
  }
}

}  // namespace

// J > 0: fused CNF over compact CNF rows of J ids of TB bytes for NCH
// 32-query chunks, evaluated by cnf_warps(NCH) dedicated warps one tile ahead of
// the epilogue; J == 0: eligibility from the K1 mask.  One instantiation per
// variant keeps each kernel's code (and instruction-cache footprint) small.
// Fused groups of <= 64 queries run two CTAs per SM (tc_ctas_per_sm): twice
// the CNF / epilogue warps to hide their latency chains, each CTA with half
// the shared-memory ring and 256 TMEM columns (67 registers, no spills).
// W > 0: slot-grouped rows (u8 ids, W ids per slot group, no masks).
template <int J, int TB, int NCH, int W>
__global__ void __launch_bounds__(threads_for(J > 0, NCH), (J > 0 && NCH <= 2) ? 2 : 1)
    tc_score_kernel(const __grid_constant__ CUtensorMap tm_qhi, const __grid_constant__ CUtensorMap tm_qlo, TcArgs a) {
  constexpr bool kFused = J > 0;
  constexpr uint32_t kEW = epi_warps(kFused);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array so every derived pointer
  // stays in the shared window (LDS/STS, not generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t Np = a.Np, kb = a.kblocks, S = a.stages;
  const uint32_t AB = a.acc_bufs;  // TMEM accumulator buffers (4, or 2 for Np > 128): a power of two
  const uint32_t ab_shift = AB == 4 ? 2u : (AB == 2 ? 1u : 0u);
  const uint32_t q_box = Np * 128;  // bytes of one K-atom of the query tile
  const uint32_t q_bytes = q_box * kb;
  const uint32_t a_bytes = kAtomBytes;  // one 128-byte K atom of 128 rows of one plane
  const uint32_t aps = a.aps;           // K atoms per pipeline stage (kb % aps == 0)
  const uint32_t n_ops = a.split ? 2 : 1;
  const uint32_t st_bytes = n_ops * aps * a_bytes;  // stage: [hi atoms][lo atoms]
  const uint32_t TS = a.term_slots;  // fused CNF: tiles of row term lists in flight
  // smem carve-up (the prefilter uses Q_hi only: no Q_lo tile)
  uint8_t* s_qhi = smem;
  uint8_t* s_qlo = s_qhi + q_bytes;
  uint8_t* s_stage = s_qlo + (a.prefilter ? 0u : q_bytes);  // [S][n_ops][aps][16 KB]: ring of stages, kb / aps per tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_stage + size_t{S} * st_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = tfull + kAccBufs;
  uint64_t* qbar = tempty + kAccBufs;
  float* s_ts = reinterpret_cast<float*>(bars + ((2 * S + 2 * kAccBufs + 2) & ~1u));  // [Np] threshold score (16-B aligned)
  uint32_t* s_tr = reinterpret_cast<uint32_t*>(s_ts + Np);     // [Np] threshold row
  float* s_sc = reinterpret_cast<float*>(s_tr + Np);           // [Np] i8: score = accumulator x s_sc
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_sc + Np);   // TMEM base
  uint32_t* s_act = s_tmem + 1;                                // [Np / 32] active bitmasks
  // per-CTA candidate staging shared by the epilogue warps: [Np][kst] keys + [Np] counts
  const uint32_t kst = stage_bytes_for(Np) / (8 * Np);
  uint32_t* s_scnt = s_act + 8;
  uint8_t* after_cnt = reinterpret_cast<uint8_t*>(s_scnt + Np);
  uint64_t* s_skey = reinterpret_cast<uint64_t*>(after_cnt + ((16u - (smem_u32(after_cnt) & 15u)) & 15u));
  // fused CNF: a ring of TS tiles of row term lists (bulk-copied by
  // the producer; 128 rows x A u16 each), a ring of kEligSlots tiles of
  // eligibility words ([NCH][128 rows] u32, written by the CNF warps), their
  // barriers, then the tables: per term entry {users[NCH], hc of its
  // slot[NCH]} for T terms + sentinel, hc [C][NCH], live [NCH] + constrained
  // slots, slot of term [T + 1]
  uint8_t* after_skey = reinterpret_cast<uint8_t*>(s_skey) + stage_bytes_for(Np);
  uint8_t* s_terms = after_skey + ((128u - (smem_u32(after_skey) & 127u)) & 127u);
  // term slot: [128 rows x wb id bytes][128 x u64 masks]
  const uint32_t term_ids_bytes = kTileRows * a.wb, term_tile_bytes = term_ids_bytes + (W ? 0u : kTileRows * 8);
  uint32_t* s_elig = reinterpret_cast<uint32_t*>(s_terms + (kFused ? TS * term_tile_bytes : 0u));
  uint64_t* s_tbar = reinterpret_cast<uint64_t*>(s_elig + (kFused ? kEligSlots * NCH * kTileRows : 0u));
  uint64_t* ttfull = s_tbar;
  uint64_t* ttempty = s_tbar + TS;
  uint64_t* efull = s_tbar + 2 * TS;
  uint64_t* eempty = efull + kEligSlots;
  // u8 ids: a static 256-entry table (its address folds into the loads'
  // immediate offset); u16 ids: the table follows in dynamic memory
  __shared__ __align__(16) uint32_t s_tbl8[(kFused && TB == 1) ? 256 * NCH : 4];
  uint32_t* s_ftbl = (kFused && TB == 1) ? s_tbl8 : reinterpret_cast<uint32_t*>(eempty + kEligSlots);
  const uint32_t n_tbl = TB == 1 ? 256u : a.T + 1;  // table entries (u8 ids: direct index, sentinels above T)
  uint32_t* s_fhc = (kFused && TB == 1) ? reinterpret_cast<uint32_t*>(eempty + kEligSlots)
                                        : s_ftbl + static_cast<size_t>(n_tbl) * NCH;
  uint32_t* s_flive = s_fhc + a.C * NCH;
  uint8_t* s_fslot = reinterpret_cast<uint8_t*>(s_flive + NCH + 1);
  // int8 threshold bias (one extra K step adds -T_q to every accumulator, so
  // the epilogue tests the sign directly): A' = 256 B (one row pattern, every
  // 8-row group aliased: SBO 0), B' = Np x 32 B (K-major, SWIZZLE_NONE), then
  // the per-query bias S_q = -T_q (int)
  uint8_t* bias_base = kFused ? s_fslot + a.T + 1 : s_terms;
  uint8_t* s_bias_a = bias_base + ((128u - (smem_u32(bias_base) & 127u)) & 127u);
  uint8_t* s_bias_b = s_bias_a + 256;
  int32_t* s_bias_s = reinterpret_cast<int32_t*>(s_bias_b + Np * 32);

  pdl_trigger();  // the next kernel of the run may set up while this one streams
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (uint32_t i = 0; i < kAccBufs; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, kEW);
    }
    mbar_init(qbar, 1);
    if (kFused) {
      for (uint32_t i = 0; i < TS; ++i) {
        mbar_init(ttfull + i, 1);
        mbar_init(ttempty + i, cnf_warps(NCH));
      }
      for (uint32_t i = 0; i < kEligSlots; ++i) {
        mbar_init(efull + i, cnf_warps(NCH));
        mbar_init(eempty + i, kEW);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (kFused) {
    for (uint32_t i = threadIdx.x; i < (a.C + 1) * NCH + 1; i += blockDim.x) s_fhc[i] = a.fz[a.hc_off + i];
    for (uint32_t i = threadIdx.x; i <= a.T; i += blockDim.x) s_fslot[i] = i < a.T ? a.slot_of[i] : a.C;
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < n_tbl; t += blockDim.x) {  // unlisted term: v = hc of its slot
      uint32_t* e = s_ftbl + t * NCH;
#pragma unroll
      for (uint32_t c = 0; c < NCH; ++c) {
        uint32_t x = t < a.T ? s_fhc[s_fslot[t] * NCH + c] : 0xFFFFFFFFu;  // sentinel / PAD: AND identity
        if (W && t >= a.T && t < a.T + a.C) x = s_fhc[(t - a.T) * NCH + c];  // EMPTY_g: queries constraining g
        if (W && t == 0xFEu) x = 0u;                                          // NONE: no constraint
        e[c] = x;
      }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < a.n_entries; e += blockDim.x) {  // listed terms: v = hc & ~users
      const uint32_t* en = a.fz + static_cast<size_t>(e) * (1 + NCH);
#pragma unroll
      for (uint32_t c = 0; c < NCH; ++c) s_ftbl[en[0] * NCH + c] = en[1 + c];
    }
  }
  pdl_wait();  // everything below reads what earlier kernels of the run wrote
  const uint32_t q0 = a.q0;
  // Any active query in this group?  One query per thread, then a block vote
  // (uniform early exit before TMEM allocation; keeps no-op rerun launches cheap).
  bool mine = false;
  for (uint32_t j = threadIdx.x; j < Np; j += blockDim.x) mine |= tc_active(a, q0 + j);
  if (!__syncthreads_or(mine)) return;

  // key >= thr  <=>  score > ts || (score == ts && row <= tr)   (make_key order)
  for (uint32_t j = threadIdx.x; j < Np; j += blockDim.x) {
    const bool on = tc_active(a, q0 + j);
    const uint64_t thr = (on && a.mode != SCORE_SAMPLE) ? a.thr[q0 + j] : 0ull;
    if (!on) {
      s_ts[j] = 2.0f;  // above any clamped score: never taken
      s_tr[j] = 0u;
    } else if (thr == 0ull) {
      s_ts[j] = -2.0f;  // no threshold
      s_tr[j] = 0u;
    } else {
      // prefilter: admit s' >= ts - delta (a superset of exact score >= ts)
      const float dl = a.prefilter ? (a.qdelta ? a.qdelta[q0 + j] : a.delta) : 0.0f;
      const float ts = key_score(thr) - dl;
      s_ts[j] = ts <= -1.0f ? -2.0f : ts;
      s_tr[j] = a.prefilter ? 0xFFFFFFFFu : key_row(thr);
    }
    if (a.i8) {
      // int8 prefilter: s' = acc x scale_q, so s' >= ts  <=  acc >= floor(ts / scale_q) - 1
      // (an integer threshold one below the exact bound absorbs the division's rounding)
      const float sc = q0 + j < a.B ? a.qscale[q0 + j] : 1.0f, ts = s_ts[j];
      s_sc[j] = sc;
      int32_t T;
      if (a.row_w) {
        // weighted: admit acc x W_r >= 256 T with W_r = ceil(256 w_r) >= 256 w_r,
        // a superset of w_r s' >= ts when ts > 0 (then s' > 0); ts <= 0 takes
        // every row.  |acc| < 2^21 and W_r <= 256 keep the IMAD inside s32.
        if (ts >= 2.0f) T = 1 << 30;  // inactive: never taken
        else if (ts <= 0.0f) T = -(1 << 30);  // no threshold
        else T = static_cast<int32_t>(fminf(fmaxf((floorf(ts / sc) - 1.0f) * 256.0f, -1.0e9f), 1.0e9f));
      } else if (ts >= 2.0f) T = INT32_MAX;  // inactive: never taken
      else if (ts <= -1.0f) T = INT32_MIN / 2;  // no threshold
      else T = static_cast<int32_t>(fmaxf(floorf(ts / sc) - 1.0f, -1.0e9f));
      s_ts[j] = __int_as_float(T);
    }
  }
  // threshold bias: S_q = -T_q as b0 + 127 (b1 + ... + b31) against the row
  // pattern (1, 127, ..., 127); |S| <= 500062.  "No threshold" needs S above
  // every possible -acc (|acc| <= (1 + delta_q) / scale_q).  Main / rerun
  // passes of the unweighted int8 prefilter only; otherwise the IADD compare.
  bool bias_ok = a.i8 && !a.row_w && a.mode != SCORE_SAMPLE && !(a.debug & (1u | 128u | 256u | 0x200u));
  constexpr int32_t kBiasMax = 3937 * 127 + 63;
  for (uint32_t j = threadIdx.x; j < Np && bias_ok; j += blockDim.x) {
    const int32_t T = __float_as_int(s_ts[j]);
    int32_t S = 0;
    if (T == INT32_MAX) {
      S = 0;  // inactive: never eligible
    } else if (T == INT32_MIN / 2) {
      const float dl = a.qdelta ? a.qdelta[q0 + j] : a.delta;
      if ((1.0f + dl) / s_sc[j] + 2.0f > static_cast<float>(kBiasMax)) bias_ok = false;
      S = kBiasMax;
    } else if (T > kBiasMax || T < -kBiasMax) {
      bias_ok = false;
    } else {
      S = -T;
    }
    s_bias_s[j] = S;
    // B' row j: b0 = r, b1..b31 carry m (S = 127 m + r, |r| <= 63)
    const int32_t m = (S >= 0 ? S + 63 : S - 63) / 127, r = S - 127 * m;
    int8_t b[32];
    b[0] = static_cast<int8_t>(r);
    int32_t left = m;
    for (int k = 1; k < 32; ++k) {
      const int32_t x = left > 127 ? 127 : (left < -127 ? -127 : left);
      b[k] = static_cast<int8_t>(x);
      left -= x;
    }
    uint8_t* row = s_bias_b + (j / 8) * 256 + (j % 8) * 16;
    for (int k = 0; k < 16; ++k) {
      row[k] = static_cast<uint8_t>(b[k]);
      row[128 + k] = static_cast<uint8_t>(b[16 + k]);
    }
  }
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x)  // A': rows (1, 127, ..., 127)
    s_bias_a[i] = (i < 128u && (i & 15u) == 0u) ? 1u : 127u;
  const uint32_t bias_on = __syncthreads_and(bias_ok) ? 1u : 0u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared operands -> the tensor core
  for (uint32_t j = threadIdx.x; j < Np; j += blockDim.x) s_scnt[j] = 0;
  if (warp < Np / 32) {  // one ballot per 32-query chunk (parallel loads, not 32 serial ones)
    const uint32_t m = __ballot_sync(0xffffffffu, tc_active(a, q0 + warp * 32 + lane));
    if (lane == 0) s_act[warp] = m;
  }
  const uint32_t tmem_cols = a.tmem_cols;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      mbar_expect_tx(qbar, (a.prefilter ? 1 : 2) * q_bytes);
      for (uint32_t k = 0; k < kb; ++k) {
        tma_load_2d(s_qhi + k * q_box, &tm_qhi, qbar, static_cast<int>(k * (a.i8 ? 128 : 64)),
                    static_cast<int>(a.q_row0));
        if (!a.prefilter)
          tma_load_2d(s_qlo + k * q_box, &tm_qlo, qbar, static_cast<int>(k * 64), static_cast<int>(a.q_row0));
      }
      uint32_t s = 0, ph = 0, ts = 0, tph = 0;  // ring slots and phases (no runtime modulo)
      for (uint32_t i = 0;; ++i) {
        const uint32_t t = tile_of(a, i);
        if (t == UINT32_MAX) break;
        if (kFused) {  // the tile's compact CNF rows (ids, masks; padded to whole tiles) into the term ring
          if (i > 0 && ++ts == TS) {
            ts = 0;
            tph ^= 1;
          }
          mbar_wait(ttempty + ts, tph ^ 1);
          mbar_expect_tx(ttfull + ts, term_tile_bytes);
          bulk_load(s_terms + ts * term_tile_bytes, a.cnf_ids + static_cast<size_t>(t) * term_ids_bytes,
                    term_ids_bytes, ttfull + ts);
          if (!W)
            bulk_load(s_terms + ts * term_tile_bytes + term_ids_bytes,
                      a.cnf_masks + static_cast<size_t>(t) * kTileRows, kTileRows * 8, ttfull + ts);
        }
        for (uint32_t k = 0; k < kb; k += aps) {
          mbar_wait(empty + s, ph ^ 1);
          mbar_expect_tx(full + s, st_bytes);
          // aps pre-swizzled K-atoms per plane (hi [+ lo]) per stage, one
          // bulk copy per plane (a tile's atoms are contiguous in a plane)
          const uint8_t* src = a.tiles + (static_cast<size_t>(t) * kb + k) * a_bytes;
          bulk_load(s_stage + size_t{s} * st_bytes, src, aps * a_bytes, full + s);
          if (n_ops == 2)
            bulk_load(s_stage + size_t{s} * st_bytes + aps * a_bytes, src + a.plane_bytes, aps * a_bytes, full + s);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: the whole warp walks the rings, one elected lane
    // issues.  Descriptors are built from warp-uniform 32-bit words (low word
    // = start address >> 4 | LBO 1; high word = SBO 64 | version 1 | SW128),
    // so a K-step is one add per operand and the tcgen05.mma itself.
    // instruction descriptor: D type (bits 4-5: 1 = f32, 2 = s32), A/B types
    // (bits 7-9 / 10-12: bf16 = 1 for kind::f16, signed int8 = 1 for
    // kind::i8), K-major A and B, N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t idesc = ((a.i8 ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) | ((Np >> 3) << 17) |
                           ((kTileRows >> 4) << 24);
    const uint32_t a_lo0 = (smem_u32(s_stage) >> 4) | 0x10000u;
    const uint32_t qh_lo0 = (smem_u32(s_qhi) >> 4) | 0x10000u, ql_lo0 = (smem_u32(s_qlo) >> 4) | 0x10000u;
    const uint32_t nkk = (a.debug & 16u) ? 1u : 4u;  // debug bit4: one K16 step per atom (timing only)
    // (non-fused variants only: the fused ones run two CTAs per SM under a
    // 72-register cap, where the second body spills, and are HBM-bound)
    const bool i8_only = !kFused && a.i8 && a.prefilter && !a.split && !(a.debug & (1u | 16u | 0x2000u));  // 0x2000: generic body
    mbar_wait(qbar, 0);
    fence_after();
    uint32_t s = 0, ph = 0;
    for (uint32_t i = 0;; ++i) {
      const uint32_t t = tile_of(a, i);
      if (t == UINT32_MAX) break;
      const uint32_t acc = i & (AB - 1), aph = (i >> ab_shift) & 1;
      if (!(a.debug & 8u)) mbar_wait(tempty + acc, aph ^ 1);  // debug bit3: ignore the accumulator ring
      fence_after();
      const uint32_t d = tmem + acc * Np;
      for (uint32_t k0 = 0; k0 < kb; k0 += aps) {
        mbar_wait(full + s, ph);
        fence_after();
        if (elect_one()) {
          const uint32_t st_lo = a_lo0 + ((s * st_bytes) >> 4);
          if (i8_only) {
            // the int8 prefilter: straight-line kind::i8 MMAs only.  (The
            // generic body below compiles to four predicated tensor
            // instructions per K step -- i8, f16 hi, f16 lo, split -- and
            // the predicated-off ones still cost issue time: ~190 instead of
            // 128 cycles per N = 256 K step.)
            for (uint32_t k = 0; k < aps; ++k) {
              const uint32_t ka = st_lo + ((k * a_bytes) >> 4), kq = qh_lo0 + (((k0 + k) * q_box) >> 4);
              mma_i8w(d, ka, kq, idesc, (k0 + k) != 0);
              mma_i8w(d, ka + 2, kq + 2, idesc, 1u);
              mma_i8w(d, ka + 4, kq + 4, idesc, 1u);
              mma_i8w(d, ka + 6, kq + 6, idesc, 1u);
            }
          }
          for (uint32_t k = 0; k < aps && !i8_only && !(a.debug & 1u); ++k) {
            const uint32_t ka = st_lo + ((k * a_bytes) >> 4), kq = ((k0 + k) * q_box) >> 4;
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk) {  // 4 x K16 per 128-byte atom (+32 B = +2 per step)
              if (kk >= nkk) break;
              const uint32_t acc_in = (k0 + k + kk) != 0;
              // one K step = 32 bytes of every row (16 bf16 or 32 int8 elements)
              if (a.i8) mma_i8w(d, ka + 2 * kk, qh_lo0 + kq + 2 * kk, idesc, acc_in);
              else mma_bf16w(d, ka + 2 * kk, qh_lo0 + kq + 2 * kk, idesc, acc_in);
              if (!a.prefilter) mma_bf16w(d, ka + 2 * kk, ql_lo0 + kq + 2 * kk, idesc, 1u);
              if (a.split) mma_bf16w(d, ka + ((aps * a_bytes) >> 4) + 2 * kk, qh_lo0 + kq + 2 * kk, idesc, 1u);
            }
          }
          if (bias_on && k0 + aps >= kb)  // + (-T_q): the accumulator's sign is the threshold test
            mma_i8d(d, (smem_u32(s_bias_a) >> 4) | (8u << 16), 0x4000u, (smem_u32(s_bias_b) >> 4) | (8u << 16),
                    0x4000u | 16u, idesc);
          mma_commit(empty + s);  // this stage is free once its MMAs retire
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) mma_commit(tfull + acc);  // accumulator ready for the epilogue
      __syncwarp();
    }
  } else if (warp < 2 + kEW) {
    // ===== epilogue: TMEM -> registers -> mask / clamp / threshold -> candidates =====
    // 8 warps: lane quadrant = warp % 4 (TMEM access rule), column half =
    // (warp - 2) / 4; each warp owns chunks c = half, half + 2, ... (32
    // queries each; up to 4 chunks at Np = 256).
    // warp = 2 + 4 part + quad: chunks c = part, part + P, ... (P = kEW / 4)
    constexpr uint32_t P = kEW / 4;
    const uint32_t quad = warp & 3, ewarp = warp - 2, half = ewarp >> 2;
    const uint32_t nq32 = Np / 32;
    // chunks per warp: NCH / 2 for a fused group (compile time), up to 4 otherwise
    constexpr uint32_t WC = kFused ? (NCH >= 2 ? NCH / 2 : 1) : (kMaxWarpChunks * 2 + P - 1) / P;
    uint32_t mw[WC] = {};  // mask words of the current tile (lane l: query 32c + l)
    auto load_mask = [&](uint32_t t, uint32_t (&out)[WC]) {
      if (kFused || a.match_all) return;
#pragma unroll
      for (uint32_t cc = 0; cc < WC; ++cc) {
        const uint32_t c = half + P * cc;
        const uint32_t qq = c * 32 + lane;
        out[cc] = (c < nq32 && t != UINT32_MAX && ((s_act[c] >> lane) & 1u))
                      ? __ldg(a.mask + static_cast<size_t>(q0 + qq) * a.words + t * (kTileRows / 32) + quad)
                      : 0u;
      }
    };
    // the main pass of the unweighted int8 prefilter with the threshold bias:
    // one uniform test per chunk selects the lean body (sign bits, survivors)
    const bool fast = bias_on && !a.row_w && a.mode != SCORE_SAMPLE && !(a.debug & (2u | 128u | 256u));
    uint32_t t = tile_of(a, 0);
    load_mask(t, mw);
    for (uint32_t i = 0; t != UINT32_MAX; ++i) {
      const uint32_t acc = i & (AB - 1), aph = (i >> ab_shift) & 1;
      const uint32_t t_next = tile_of(a, i + 1);
      uint32_t mw_next[WC];
      load_mask(t_next, mw_next);  // in flight while this tile is processed
      const uint32_t grow = a.row_base + t * kTileRows + quad * 32 + lane;
      // learned row weight of this lane's row (weighted index only)
      float wr = 1.0f;
      int32_t wi = 256;
      if (a.row_w) {
        const uint32_t lr = t * kTileRows + quad * 32 + lane;
        wr = lr < a.n_rows ? __ldg(a.row_w + lr) : 0.0f;
        wi = static_cast<int32_t>(ceilf(wr * 256.0f));
      }
      uint32_t fel[WC] = {};  // fused: bit j = row `lane` eligible for query 32c + j
      if (kFused) {
        // this row's eligibility words for chunks half, half + 2, ... (CNF warps)
        const uint32_t es = i % kEligSlots, eph = (i / kEligSlots) & 1;
        mbar_wait_backoff(efull + es, eph, a.backoff_ns);
#pragma unroll
        for (uint32_t cc = 0; cc < WC; ++cc) {
          const uint32_t c = half + P * cc;
          if (c < NCH)
            asm volatile("ld.shared.u32 %0, [%1];"
                         : "=r"(fel[cc])
                         : "r"(smem_u32(s_elig) + ((es * NCH + c) * kTileRows + quad * 32 + lane) * 4));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(eempty + es);
      }
      mbar_wait_backoff(tfull + acc, aph, a.backoff_ns);
      fence_after();
      // not unrolled: one copy of the (large) chunk body keeps the
      // instruction-cache footprint small when a warp owns two chunks
#pragma unroll 1
      for (uint32_t cc = 0; cc < WC; ++cc) {
        const uint32_t c = half + P * cc;
        if (c >= nq32 || (a.debug & 2u)) break;
        uint32_t v[32];
        tmem_ld32(tmem + ((quad * 32) << 16) + acc * Np + c * 32, v);
        if (a.debug & 128u) {  // diagnostics: TMEM loads only (results invalid)
          if (v[0] == 0x7fffffffu && v[31] == 0x7fffffffu) a.cand_cnt[0] = 1;
          continue;
        }
        // 32x32 bit transpose: lane l held query (32c+l)'s word over this
        // warp's 32 rows; afterwards bit j of `elig` = row `lane`, query 32c+j.
        // (register arrays indexed by a runtime cc: select, no local memory)
        uint32_t elig = mw[0], fe = fel[0];
#pragma unroll
        for (uint32_t x = 1; x < WC; ++x) {
          elig = cc == x ? mw[x] : elig;
          fe = cc == x ? fel[x] : fe;
        }
        if (kFused) {
          elig = fe;
        } else if (a.match_all) {  // every active query, every row inside the shard
          elig = (t * kTileRows + quad * 32 + lane < a.n_rows) ? s_act[c] : 0u;
        } else {
#pragma unroll
          for (uint32_t j = 16, m = 0x0000FFFFu; j > 0; j >>= 1, m ^= m << j) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, elig, j);
            elig = (lane & j) ? ((elig & ~m) | ((y & ~m) >> j)) : ((elig & m) | ((y & m) << j));
          }
        }
        // threshold test for all 32 queries: one compare of the raw
        // accumulator against the query's threshold score.  `>=` admits a
        // superset of the exact key test (ties with the threshold row, values
        // clamped later); K4 resolves it exactly.  Thresholds at or below -1
        // are stored as -2 so clamping can never hide a candidate.
        // Two instructions per score: d = v - ts (>= 0 exactly when v >= ts,
        // monotone rounding) and a funnel shift collecting d's sign bit.
        uint32_t below = 0;  // bit 31 - j: query 32c + j scored below its threshold
        if (fast) {
          // the MMA added -T_q: one funnel shift per score collects the sign;
          // survivors (rare) rebuild their prefilter score from acc = v + T_q
#pragma unroll
          for (uint32_t j = 0; j < 32; ++j) below = __funnelshift_l(v[j], below, 1);
          for (uint32_t tk = __brev(~below) & elig; tk; tk &= tk - 1u) {
            const uint32_t j = __ffs(tk) - 1, qq = c * 32 + j;
            const int32_t accv = static_cast<int32_t>(pick32(v, j)) - s_bias_s[qq];
            const uint64_t key = make_key(clamp_score(static_cast<float>(accv) * s_sc[qq]), grow);
            const uint32_t slot = atomicAdd(s_scnt + qq, 1u);
            if (slot < kst) {
              s_skey[qq * kst + slot] = key;
            } else {
              const uint32_t at = atomicAdd(a.cand_cnt + q0 + qq, 1u);
              if (at < a.cap) a.cand[static_cast<size_t>(q0 + qq) * a.cap + at] = key;
            }
          }
          continue;
        }
        const float4* ts4 = reinterpret_cast<const float4*>(s_ts + c * 32);
        if (bias_on) {  // the MMA added -T_q: one funnel shift per score collects the sign
#pragma unroll
          for (uint32_t j = 0; j < 32; ++j) below = __funnelshift_l(v[j], below, 1);
        } else if (a.i8 && a.row_w) {  // weighted: acc x W_r - 256 T (one IMAD per score)
#pragma unroll
          for (uint32_t j4 = 0; j4 < 8; ++j4) {
            const int4 t4 = *reinterpret_cast<const int4*>(ts4 + j4);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 0]) * wi - t4.x), below, 1);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 1]) * wi - t4.y), below, 1);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 2]) * wi - t4.z), below, 1);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 3]) * wi - t4.w), below, 1);
          }
        } else if (a.row_w) {  // weighted bf16 prefilter: sign of fma(s', w_r, -ts) (exact sign)
#pragma unroll
          for (uint32_t j4 = 0; j4 < 8; ++j4) {
            const float4 t4 = ts4[j4];
            below = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(v[4 * j4 + 0]), wr, -t4.x)), below, 1);
            below = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(v[4 * j4 + 1]), wr, -t4.y)), below, 1);
            below = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(v[4 * j4 + 2]), wr, -t4.z)), below, 1);
            below = __funnelshift_l(__float_as_uint(fmaf(__uint_as_float(v[4 * j4 + 3]), wr, -t4.w)), below, 1);
          }
        } else if (a.i8) {  // int32 accumulators against integer thresholds (no overflow: |acc|, |T| < 2^30)
#pragma unroll
          for (uint32_t j4 = 0; j4 < 8; ++j4) {
            const int4 t4 = *reinterpret_cast<const int4*>(ts4 + j4);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 0]) - t4.x), below, 1);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 1]) - t4.y), below, 1);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 2]) - t4.z), below, 1);
            below = __funnelshift_l(static_cast<uint32_t>(static_cast<int32_t>(v[4 * j4 + 3]) - t4.w), below, 1);
          }
        } else {
#pragma unroll
          for (uint32_t j4 = 0; j4 < 8; ++j4) {
            const float4 t4 = ts4[j4];
            below = __funnelshift_l(__float_as_uint(__uint_as_float(v[4 * j4 + 0]) - t4.x), below, 1);
            below = __funnelshift_l(__float_as_uint(__uint_as_float(v[4 * j4 + 1]) - t4.y), below, 1);
            below = __funnelshift_l(__float_as_uint(__uint_as_float(v[4 * j4 + 2]) - t4.z), below, 1);
            below = __funnelshift_l(__float_as_uint(__uint_as_float(v[4 * j4 + 3]) - t4.w), below, 1);
          }
        }
        const uint32_t take = (a.debug & 256u) ? ((__brev(~below) & elig) == 0x12345u ? 1u : 0u)  // diagnostics: no survivors
                                               : (__brev(~below) & elig);
        // prefilter score of (row lane, query 32c + j) from the accumulator word
        auto score_of = [&](uint32_t w, uint32_t j) {
          const int32_t acc = static_cast<int32_t>(w) - (bias_on ? s_bias_s[c * 32 + j] : 0);
          return a.i8 ? static_cast<float>(acc) * s_sc[c * 32 + j] : __uint_as_float(w);
        };
        // clamped (and weighted: w_r x clamp(s')) score of (row lane, query 32c + j)
        auto final_of = [&](uint32_t w, uint32_t j) {
          return a.row_w ? weighted_score(score_of(w, j), wr) : clamp_score(score_of(w, j));
        };
        if (a.mode == SCORE_SAMPLE && a.shist) {
          // sample pass, histogram form: one global increment per eligible
          // sampled (row, query) in the query's score histogram
          const float scale = 0.5f * static_cast<float>(a.hbins);
          uint32_t keep = elig;
          if (a.sample_floor) {  // match-all samples: only scores >= 0 (the top K lie far above)
            uint32_t neg = 0;
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) neg = __funnelshift_l(v[j], neg, 1);  // sign of acc / fp32 score
            keep &= __brev(~neg);
          }
          if constexpr (J < 0) {
            // match-all: about half of the 32 scores are kept, so one
            // unrolled pass over all 32 (no per-bit loop with a select tree
            // per score: measured ~60 instructions per kept score).  (CTA-local
            // floors -- shared-memory level counts that let scores below the
            // CTA's own k-th largest skip the global histogram -- measured
            // slower: the 32 lanes of a query collide on a few counters.)
            uint32_t* hq = a.shist + static_cast<size_t>(q0 + c * 32) * a.hbins;
#pragma unroll
            for (uint32_t j4 = 0; j4 < 8; ++j4) {
              const float4 s4 = reinterpret_cast<const float4*>(s_sc + c * 32)[j4];
              const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
              for (uint32_t u = 0; u < 4; ++u) {
                const uint32_t j = 4 * j4 + u;
                if ((keep >> j) & 1u) {
                  const float sc = clamp_score(a.i8 ? static_cast<float>(static_cast<int32_t>(v[j])) * sv[u]
                                                    : __uint_as_float(v[j]));
                  const uint32_t b = min(static_cast<uint32_t>((sc + 1.0f) * scale), a.hbins - 1u);
                  atomicAdd(hq + j * a.hbins + b, 1u);
                }
              }
            }
            continue;
          }
          // (J >= 0: eligible pairs are sparse; a per-bit loop)
          for (uint32_t el = keep; el; el &= el - 1u) {
            const uint32_t j = __ffs(el) - 1;
            const float sc = final_of(pick32(v, j), j);
            const uint32_t b = min(static_cast<uint32_t>((sc + 1.0f) * scale), a.hbins - 1u);
            atomicAdd(a.shist + static_cast<size_t>(q0 + c * 32 + j) * a.hbins + b, 1u);
          }
          continue;
        }
        if (a.mode == SCORE_SAMPLE) {
          // sample pass: every eligible sampled row goes to its fixed slot
          // (segment ordinal x 1024 + row in segment) -- no threshold, no atomics
          const uint32_t local = t * kTileRows + quad * 32 + lane;
          const uint32_t sidx = (local / 1024) / a.period * 1024 + (local & 1023);
#pragma unroll
          for (uint32_t j = 0; j < 32; ++j)
            if ((elig >> j) & 1u)
              a.samp[static_cast<size_t>(q0 + c * 32 + j) * a.cap + sidx] = f2ord(final_of(v[j], j));
          continue;
        }
        // survivors (rare): each lane walks its own set bits; the score is
        // picked out of the register array by a select tree, so no
        // 32-way-unrolled body sits in the hot loop's instruction footprint.
        // Keys are staged per CTA in shared memory and spill to the global
        // candidate buffer only when a query's slots are full.
        for (uint32_t tk = take; tk; tk &= tk - 1u) {
          const uint32_t j = __ffs(tk) - 1, qq = c * 32 + j;
          const uint64_t key = make_key(final_of(pick32(v, j), j), grow);
          if (key_score(key) == s_ts[qq] && grow > s_tr[qq]) continue;  // exact tie rule: below the threshold key
                                                                        // (prefilter: s_tr = ~0, never)
          const uint32_t slot = atomicAdd(s_scnt + qq, 1u);
          if (slot < kst) {
            s_skey[qq * kst + slot] = key;
          } else {
            const uint32_t at = atomicAdd(a.cand_cnt + q0 + qq, 1u);
            if (at < a.cap) a.cand[static_cast<size_t>(q0 + qq) * a.cap + at] = key;
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
#pragma unroll
      for (uint32_t cc = 0; cc < WC; ++cc) mw[cc] = mw_next[cc];
      t = t_next;
    }
    // final flush of the CTA's staged keys once every epilogue warp is done:
    // warp w owns queries w, w + 8, ...; one global reservation per query
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kEW) : "memory");
    for (uint32_t qq = ewarp; qq < Np; qq += kEW) {
      const uint32_t ns = min(s_scnt[qq], kst);
      if (ns == 0) continue;
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(a.cand_cnt + q0 + qq, ns);
      base = __shfl_sync(0xffffffffu, base, 0);
      uint64_t* dst = a.cand + static_cast<size_t>(q0 + qq) * a.cap;
      for (uint32_t k = lane; k < ns; k += 32)
        if (base + k < a.cap) dst[base + k] = s_skey[qq * kst + k];
    }
  } else if (kFused) {
    // ===== CNF warps: thread r evaluates tile row r % 128 for its share
    // of the NCH query chunks (all of them with 4 CNF warps, half with 8) =====
    constexpr int JW = kFused ? (J * TB + 7) / 8 * 2 : 2;  // u32 words of a row's ids (whole 8-byte loads)
    constexpr int NT = kFused ? NCH * 4 / static_cast<int>(cnf_warps(NCH)) : 1;  // chunks per thread
    const uint32_t rr = threadIdx.x - 32 * (2 + kEW);
    const uint32_t r = rr & (kTileRows - 1), c0 = (rr / kTileRows) * NT;
    const uint32_t cslots = s_flive[NCH];
    uint32_t ts = TS - 1, tph = 1;  // term ring slot / phase of tile i (advanced at the top)
    for (uint32_t i = 0;; ++i) {
      const uint32_t t = tile_of(a, i);
      if (t == UINT32_MAX) break;
      if (++ts == TS) {
        ts = 0;
        tph ^= 1;
      }
      mbar_wait_backoff(ttfull + ts, tph, a.backoff_ns);
      uint32_t tw[JW];
      const uint32_t src = smem_u32(s_terms) + ts * term_tile_bytes + r * a.wb;
#pragma unroll
      for (int v = 0; v < JW / 2; ++v)
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(tw[2 * v]), "=r"(tw[2 * v + 1]) : "r"(src + 8 * v));
      uint64_t masks = 0;
      if (!W)
        asm volatile("ld.shared.u64 %0, [%1];"
                     : "=l"(masks)
                     : "r"(smem_u32(s_terms) + ts * term_tile_bytes + term_ids_bytes + r * 8));
      __syncwarp();
      if (lane == 0) mbar_arrive(ttempty + ts);
      uint32_t el[NT];
      if (a.debug & 4u) {  // diagnostics: no CNF evaluation (every live query eligible)
#pragma unroll
        for (int c = 0; c < NT; ++c) el[c] = s_flive[c0 + c] ^ (tw[0] & 1u) ^ static_cast<uint32_t>(masks & 2u);
      } else if constexpr (W > 0) {
        cnf_row_grouped<J, W, NCH, NT, JW>(tw, s_tbl8, smem_u32(s_flive), c0, el);
      } else {
        cnf_row<(kFused ? J : 8), (kFused ? TB : 1), NCH, NT>(tw, masks, a.T, smem_u32(s_ftbl), smem_u32(s_fhc),
                                                             smem_u32(s_flive), cslots, c0, el);
      }
      if (t * kTileRows + r >= a.n_rows) {  // tail of the last tile
#pragma unroll
        for (int c = 0; c < NT; ++c) el[c] = 0u;
      }
      const uint32_t es = i % kEligSlots, eph = (i / kEligSlots) & 1;
      mbar_wait_backoff(eempty + es, eph ^ 1, a.backoff_ns);
#pragma unroll
      for (int c = 0; c < NT; ++c)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(s_elig) + ((es * NCH + c0 + c) * kTileRows + r) * 4),
                     "r"(el[c])
                     : "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(efull + es);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    HYRE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw Error(HYRE_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
}  // namespace

void make_bf16_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t dp, uint32_t box_rows) {
  const cuuint64_t dims[2] = {dp, rows};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(dp) * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(HYRE_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

void make_i8_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t dp, uint32_t box_rows) {
  const cuuint64_t dims[2] = {dp, rows};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(dp)};
  const cuuint32_t box[2] = {128, box_rows};  // one 128-byte K atom of box_rows queries
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(HYRE_CUDA_ERROR, "cuTensorMapEncodeTiled (int8) failed: " + std::to_string(r));
}

uint32_t tc_acc_bufs(uint32_t Np) { return Np <= 128 ? kAccBufs : 2u; }  // 512 TMEM columns

uint32_t tc_tmem_cols(uint32_t Np) {
  uint32_t cols = 32;
  while (cols < tc_acc_bufs(Np) * Np) cols <<= 1;
  return cols;
}

size_t tc_smem_bytes(uint32_t Np, uint32_t kb, uint32_t n_ops, uint32_t stages, size_t fused_bytes, uint32_t q_planes,
                     uint32_t aps) {
  return 1024 + size_t{q_planes} * Np * 128 * kb + size_t{stages} * aps * n_ops * kAtomBytes + (2 * stages + 2 * kAccBufs + 2) * 8 + Np * 12 +
         4 + 32 + Np * 4 + 16 + stage_bytes_for(Np) + 64 + fused_bytes + (128 + 256 + size_t{Np} * 36);  // + bias operands
}

uint32_t tc_fused_chunks(uint32_t Np) { return Np <= 32 ? 1u : (Np <= 64 ? 2u : (Np <= 128 ? 4u : 8u)); }

uint32_t tc_ctas_per_sm(bool fused, uint32_t Np) {
  static const int forced = [] {
    const char* e = std::getenv("HYRE_TC_CTAS");  // profiling: 1 forces one CTA per SM
    return e ? std::atoi(e) : 0;
  }();
  const uint32_t two = (fused && tc_fused_chunks(Np) <= 2 && tc_tmem_cols(Np) <= 256) ? 2u : 1u;
  return forced == 1 ? 1u : two;
}

size_t tc_smem_cap(bool fused, uint32_t Np) {
  // per SM: 228 KB shared memory, 1 KB reserved per resident CTA; the fused
  // variants' static table is 256 entries x chunks x 4 B
  const size_t stat = fused ? 256 * 4 * size_t{tc_fused_chunks(Np)} + 64 : 64;
  if (tc_ctas_per_sm(fused, Np) == 2) return (228 * 1024 - 2 * 1024) / 2 - stat;
  return 227 * 1024 - (fused ? kTcStaticSmem : 64);
}

size_t tc_fused_bytes(uint32_t Np, uint32_t T, uint32_t C, uint32_t row_bytes, uint32_t term_slots) {
  const size_t nch = tc_fused_chunks(Np);
  const size_t n_tbl = T <= 255 ? 0 : T + 1;  // u8 ids: static 256-entry table (kTcStaticSmem)
  return 128 + size_t{term_slots} * kTileRows * row_bytes + size_t{kEligSlots} * nch * kTileRows * 4 +
         16 * (term_slots + kEligSlots) + 4 * (n_tbl * nch + C * nch + nch + 1) + T + 1 + 16;
}

void launch_tc_score(const CUtensorMap& qhi, const CUtensorMap& qlo, const TcArgs& a, uint32_t grid, size_t smem,
                     cudaStream_t st) {
  using KFn = void (*)(const CUtensorMap, const CUtensorMap, TcArgs);
  // segmented rows [id width: u8 J = 8/16/24/32, u16 J = 16/32][query chunks 1/2/4/8];
  // slot-grouped rows [(J, W) = (8,1) (8,2) (16,2) (12,3) (24,3) (16,4) (32,4)][chunks]
#define HYRE_TC_ROW(J, TB, W)                                                                     \
  {tc_score_kernel<J, TB, 1, W>, tc_score_kernel<J, TB, 2, W>, tc_score_kernel<J, TB, 4, W>, \
   tc_score_kernel<J, TB, 8, W>}
  static const KFn fused[13][4] = {HYRE_TC_ROW(8, 1, 0),  HYRE_TC_ROW(16, 1, 0), HYRE_TC_ROW(24, 1, 0),
                                   HYRE_TC_ROW(32, 1, 0), HYRE_TC_ROW(16, 2, 0), HYRE_TC_ROW(32, 2, 0),
                                   HYRE_TC_ROW(8, 1, 1),  HYRE_TC_ROW(8, 1, 2),  HYRE_TC_ROW(16, 1, 2),
                                   HYRE_TC_ROW(12, 1, 3), HYRE_TC_ROW(24, 1, 3), HYRE_TC_ROW(16, 1, 4),
                                   HYRE_TC_ROW(32, 1, 4)};
#undef HYRE_TC_ROW
  static std::atomic<uint64_t> attr{0};  // devices whose limits are set (every variant at once)
  int dev = 0;
  HYRE_CUDA(cudaGetDevice(&dev));
  if (!(attr.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
    HYRE_CUDA(cudaFuncSetAttribute(tc_score_kernel<0, 1, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   227 * 1024 - 64));
    HYRE_CUDA(cudaFuncSetAttribute(tc_score_kernel<-1, 1, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   227 * 1024 - 64));
    for (auto& row : fused)
      for (KFn k : row)
        HYRE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - kTcStaticSmem));
    attr.fetch_or(1ull << (dev & 63), std::memory_order_acq_rel);
  }
  // J = -1: the match-all variant's instance for sample passes (their
  // unrolled histogram body stays out of the main pass's instruction footprint)
  KFn k = (a.sample_floor && a.mode == SCORE_SAMPLE) ? tc_score_kernel<-1, 1, 1, 0> : tc_score_kernel<0, 1, 1, 0>;
  if (a.fused) {
    const uint32_t nch = tc_fused_chunks(a.Np), ci = nch == 1 ? 0 : (nch == 2 ? 1 : (nch == 4 ? 2 : 3));
    int ri = -1;
    if (a.W) {
      const uint32_t J = a.J, W = a.W;
      ri = W == 1 && J == 8 ? 6 : W == 2 && J == 8 ? 7 : W == 2 && J == 16 ? 8 : W == 3 && J == 12 ? 9
         : W == 3 && J == 24 ? 10 : W == 4 && J == 16 ? 11 : W == 4 && J == 32 ? 12 : -1;
    } else if (a.tb == 1) {
      ri = a.J == 8 ? 0 : a.J == 16 ? 1 : a.J == 24 ? 2 : a.J == 32 ? 3 : -1;
    } else if (a.tb == 2) {
      ri = a.J == 16 ? 4 : a.J == 32 ? 5 : -1;
    }
    if (ri < 0) throw Error(HYRE_INTERNAL, "fused CNF: unsupported compact row shape");
    k = fused[ri][ci];
  }
  launch_pdl(k, dim3(grid), dim3(threads_for(a.fused != 0, static_cast<int>(tc_fused_chunks(a.Np)))), smem, st, qhi,
             qlo, a);
}

}  // namespace hyreb
