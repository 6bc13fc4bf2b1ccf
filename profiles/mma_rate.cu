// Tensor-pipe issue rate of the MMA shapes K3 uses (profiling aid, not product
// code): one CTA per SM, one elected thread issues R back-to-back
// tcgen05.mma (cta_group::1, M = 128, K-major SWIZZLE_128B operands in shared
// memory, accumulator in TMEM) and the CTA times them with clock64 until the
// commit barrier fires.  Prints cycles per MMA and the implied dense rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/mma_rate profiles/mma_rate.cu
//   ./profiles/mma_rate          (on a B200)
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// CH: independent accumulator chains the MMAs rotate over (1 = every MMA
// accumulates onto the previous one's result, as within one K3 tile)
// CE: a tcgen05.commit after every CE MMAs (0: none); CB: with CE, a second
// commit to another barrier right after it (K3's stage-release + accumulator-ready pair)
template <int KIND, int N, int CH, int CE = 0, int CB = 0, int BC = 0, int RND = 0>  // RND: random operand bytes (else a sparse 0/1/2/3 pattern); BC: warp 1 streams 16 KB bulk copies from HBM into 4 other shared-memory stages meanwhile; KIND 0: kind::f16 (bf16, K = 16), 1: kind::i8 (K = 32)
__global__ void __launch_bounds__(128) mma_rate(int reps, unsigned long long* cycles, const uint8_t* src, size_t src_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* a = sm;                    // 128 rows x 128 B
  uint8_t* b = sm + 128 * 128;        // N rows x 128 B
  __shared__ uint64_t bar, bar2, bar3, cbar[4];
  __shared__ volatile uint32_t stop;
  uint8_t* cst = sm + (128 + N) * 128;  // 4 x 16 KB copy stages
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) {
    uint32_t x = static_cast<uint32_t>(i) * 2654435761u + blockIdx.x * 97u;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    // RND: random int8 (|v| <= 127) or random bf16 pairs of magnitude ~1
    const uint32_t r = KIND ? (x & 0x7f7f7f7fu) ^ (x & 0x80808080u) : ((x & 0x007f007fu) | 0x3f003f00u) ^ (x & 0x80008000u);
    reinterpret_cast<uint32_t*>(sm)[i] = RND ? r : 0x01010101u * (i & 3);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar3)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar[i])));
    stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = ((KIND ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
  const uint32_t a_lo = (su32(a) >> 4) | 0x10000u, b_lo = (su32(b) >> 4) | 0x10000u;
  if (threadIdx.x == 0) {
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t kk = r & 3, d = tmem + (r % CH) * N;
      if (KIND)
        asm volatile(
            "{\n .reg .b64 da, db;\n mov.b64 da, {%1, %4};\n mov.b64 db, {%2, %4};\n"
            " tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %3, 1;\n}" ::"r"(d),
            "r"(a_lo + 2 * kk), "r"(b_lo + 2 * kk), "r"(idesc), "n"(0x40004040));
      else
        asm volatile(
            "{\n .reg .b64 da, db;\n mov.b64 da, {%1, %4};\n mov.b64 db, {%2, %4};\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %3, 1;\n}" ::"r"(d),
            "r"(a_lo + 2 * kk), "r"(b_lo + 2 * kk), "r"(idesc), "n"(0x40004040));
      if (CE && (r % CE) == CE - 1) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2))
                     : "memory");
        if (CB)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar3))
                       : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(su32(&bar))
          : "memory");
    cycles[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  if (BC && threadIdx.x == 32) {  // bulk-copy stream: 16 KB per copy, 4 stages in flight
    size_t off = static_cast<size_t>(blockIdx.x) * 16384 * 64;
    uint32_t ph[4] = {0, 0, 0, 0};
    for (uint32_t i = 0; !stop; ++i) {
      const uint32_t st = i & 3;
      if (i >= 4) {  // wait for this stage's previous copy
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
              : "=r"(done)
              : "r"(su32(&cbar[st])), "r"(ph[st])
              : "memory");
        ph[st] ^= 1;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&cbar[st])), "r"(16384) : "memory");
      if (off + 16384 > src_bytes) off = 0;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(cst + st * 16384)), "l"(src + off), "r"(16384), "r"(su32(&cbar[st]))
                   : "memory");
      off += 16384 * 148;
    }
    for (uint32_t st = 0; st < 4; ++st) {  // drain
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(su32(&cbar[st])), "r"(ph[st])
            : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int KIND, int N, int CH, int CE = 0, int CB = 0, int BC = 0, int RND = 0>
void run(const char* name, int sms, int clock_khz) {
  const int reps = 20000;
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = 1024 + (128 + N) * 128 + 4 * 16384;
  static uint8_t* src = nullptr;
  const size_t src_bytes = size_t{2} << 30;
  if (!src) cudaMalloc(&src, src_bytes);
  cudaFuncSetAttribute(mma_rate<KIND, N, CH, CE, CB, BC, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate<KIND, N, CH, CE, CB, BC, RND><<<sms, 128, smem>>>(200, d, src, src_bytes);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_rate<KIND, N, CH, CE, CB, BC, RND><<<sms, 128, smem>>>(reps, d, src, src_bytes);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double kdim = KIND ? 32 : 16, ops = 2.0 * 128 * N * kdim * reps * sms;
  std::printf("{\"mma\": \"%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"chains\": %d, \"commit_every\": %d, \"second_commit\": %d, \"bulk_copies\": %d, \"random_operands\": %d, \"cycles_per_mma\": %.1f, \"event_ms\": %.3f, "
              "\"dense_tops\": %.1f, \"sm_clock_mhz_attr\": %d, \"error\": \"%s\"}\n",
              name, N, KIND ? 32 : 16, CH, CE, CB, BC, RND, mx / reps, ms, ops / (ms * 1e-3) / 1e12, clock_khz / 1000,
              cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  run<1, 256, 1>("kind::i8", sms, clk);
  run<1, 256, 1, 0, 0, 0, 1>("kind::i8", sms, clk);
  run<1, 256, 1, 5, 1, 1, 1>("kind::i8", sms, clk);
  run<1, 128, 1, 0, 0, 0, 1>("kind::i8", sms, clk);
  run<0, 256, 1>("kind::f16 (bf16)", sms, clk);
  run<0, 256, 1, 0, 0, 0, 1>("kind::f16 (bf16)", sms, clk);
  run<1, 256, 1, 0, 0, 1>("kind::i8", sms, clk);
  return 0;
}
