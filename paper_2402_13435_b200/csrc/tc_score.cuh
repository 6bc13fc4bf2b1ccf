// K3 launch interface (tcgen05 batched scorer, tc_score.cu).
#pragma once

#include <cuda.h>

#include "device.cuh"

namespace hyreb {

struct TcArgs {
  const uint8_t* tiles;  // DevIndex::tc_tiles
  uint32_t n_rows, row_base, words, n_tiles;
  uint32_t B;        // queries in the batch
  uint32_t q0;       // first query of this group
  uint32_t q_row0;   // its row in the padded bf16 query matrix
  uint32_t Np;       // queries per group (multiple of 32, <= 256)
  uint32_t kblocks;  // dp / 64 (128-byte K atoms per row)
  uint32_t stages, tmem_cols, split;
  const uint32_t* mask;
  const QParam* qp;
  const uint32_t* n_elig;
  const uint64_t* thr;
  uint64_t* cand;
  uint32_t* cand_cnt;
  uint32_t cap, mode, period, gate;
  const uint32_t* rerun;
  uint32_t* samp;  // SCORE_SAMPLE: dense [B][cap] orderable scores (0 = ineligible)
  // SCORE_SAMPLE with shist: per-query histograms [B][hbins] of the sampled
  // eligible rows' clamped scores (linear bins over [-1, 1]) instead of samp
  uint32_t* shist;
  uint32_t hbins;
  uint32_t debug;  // diagnostics: bit0 skip MMAs, bit1 skip epilogue work, bit2 skip CNF (results invalid)
  // Fused CNF (fused != 0, mask unused): dedicated warps evaluate each row's
  // eligibility from its compact CNF row (DevIndex::cnf_ids / cnf_masks: J
  // ids of tb bytes in wb-byte rows, slot-major, segment/present masks)
  // against this group's program, scattered into shared memory:
  //   fz[0 .. n_entries*(1+W))  (term id, W words v = hc(slot) & ~users)
  //                             per term some query of the group lists
  //   fz + hc_off: hc[C][W]     queries constraining each slot
  //   fz + live_off: live[W], then the constrained-slot bitmask
  // with W = tc_fused_chunks(Np) words (word c = queries 32c .. 32c+31).
  uint32_t fused;
  const uint8_t* cnf_ids;
  const uint64_t* cnf_masks;
  const uint8_t* slot_of;
  uint32_t J, tb, wb, T, C;
  uint32_t W;  // slot-grouped rows: ids per slot group (0: segmented rows + masks)
  const uint32_t* fz;
  uint32_t n_entries, hc_off, live_off;
  // Prefilter mode (prefilter != 0): only the hi plane of each K-atom is
  // loaded and one MMA E_hi.Q_hi
  // per K-step computes s' with |s - s'| <= delta for unit rows and queries
  // (bf16 RNE of both operands: 2^-8 relative, Cauchy-Schwarz); rows are
  // admitted when s' >= thr_score - delta and rescored exactly afterwards
  // (launch_rescore), so no row whose exact score passes the threshold is lost.
  uint32_t prefilter;
  // int8 prefilter (i8 != 0; tiles = DevIndex::tc_i8, kblocks = dp / 128):
  // kind::i8 MMAs into s32 accumulators, score s' = acc x qscale[q];
  // per-query bounds qdelta[q] replace delta when given (bf16 prefilter too)
  uint32_t i8;
  const float* qscale;
  const float* qdelta;
  // learned per-row weights (local rows; nullptr = identity; prefilter mode
  // only): admission w x s' >= ts, keys and sample scores w x clamp(s')
  const float* row_w;
  uint64_t plane_bytes;  // DevIndex::tc_plane_bytes (offset of the lo plane)
  float delta;
  uint32_t acc_bufs;    // TMEM accumulator buffers (tc_acc_bufs(Np))
  uint32_t backoff_ns;  // sleep between failed barrier tests of the epilogue / CNF warps (0 = spin)
  uint32_t match_all;   // non-fused: every query of the batch is match-all (no mask; all rows eligible)
  // sample pass of a match-all batch: histogram only scores >= 0 (a query's
  // sampled K-th score below 0 leaves it without a threshold: correct, slower)
  uint32_t sample_floor;
  uint32_t aps;         // K atoms per pipeline stage (divides kblocks; one MMA commit per stage)
  uint32_t term_slots;  // fused CNF: tiles of row term lists in flight (ring depth, <= kMaxTermSlots)
};

constexpr uint32_t kTcMinBatch = 9;  // batches above 8 queries use the tensor-core scorer
constexpr uint32_t kTcMaxGroup = 256;

void make_bf16_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t dp, uint32_t box_rows);
void make_i8_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t dp, uint32_t box_rows);
size_t tc_smem_bytes(uint32_t Np, uint32_t kb, uint32_t n_ops, uint32_t stages, size_t fused_bytes = 0,
                     uint32_t q_planes = 2, uint32_t aps = 1);
// shared memory of the fused CNF tables (term users, slot of term, hc, live)
// row_bytes: a row's compact CNF bytes in the term ring (ids [+ 8 B masks])
size_t tc_fused_bytes(uint32_t Np, uint32_t T, uint32_t C, uint32_t row_bytes, uint32_t term_slots);
constexpr uint32_t kMaxTermSlots = 8;
// static shared memory of the fused variants (the u8-id term table, <= 256 x 8 words)
constexpr uint32_t kTcStaticSmem = 8 * 1024 + 64;
// TMEM accumulator buffers / columns for a group of Np queries (512 columns)
uint32_t tc_acc_bufs(uint32_t Np);
uint32_t tc_tmem_cols(uint32_t Np);
// query chunks of a fused group as laid out in its program (1, 2, 4 or 8)
uint32_t tc_fused_chunks(uint32_t Np);
// CTAs per SM of the K3 variant (2 for fused groups of <= 64 queries) and the
// dynamic shared memory one CTA may use
uint32_t tc_ctas_per_sm(bool fused, uint32_t Np);
size_t tc_smem_cap(bool fused, uint32_t Np);
void launch_tc_score(const CUtensorMap& qhi, const CUtensorMap& qlo, const TcArgs& a, uint32_t grid, size_t smem,
                     cudaStream_t st);

}  // namespace hyreb
