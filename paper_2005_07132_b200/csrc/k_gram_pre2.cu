// Gram matrix G0 = A0^T A0 (F2) on CTA PAIRS fed by the pre-split MMA image of A0
// (written by logratio_pre_kernel, k_gram_tc.cu): tcgen05.mma.cta_group::2 kind::tf32, 3xTF32
// (reading A22), one 256 x 256 tile of G per cluster of two CTAs, no producer threads.
//
// Each CTA of the pair bulk-copies (cp.async.bulk) its 128-channel halves of the A block and the B
// block from the image (the B operand is split by N across the pair, D by M: tools/micro/tc2.cu), so
// per SM the tensor core reads 8 KB of operands per 128-clock instruction (64 B/clk) and the copy
// engine writes 66 KB per 32-pixel stage (43 B/clk): ~105 B/clk of the 128 B/clk smem bandwidth,
// against 128 B/clk for the MMA reads alone in the 1-CTA 128 x 128 kernel.
//
// STATUS: parity-green; the default when ceil(M/128) is even (no extra channel padding).  Measured at
// cfg3: 3.50 ms vs 3.61 ms for the 1-CTA image-fed kernel, once the fp64 flush of the register sums
// was batched (before: 3.89 vs 3.88 ms, both MMA warps waiting on the epilogue ~18% of the time).
//
// Accuracy: hi*hi and the cross terms share one TMEM accumulator per
// buffer (256 columns, double-buffered = the 512 TMEM columns), drained every 64 pixels (24
// truncating accumulator adds per drain, ~7e-7 relative bias) into fp32 register sums (round to
// nearest), flushed to fp64 partials every 16384 pixels (5.2e-7 max-norm relative error vs fp64 at
// N = 300,000, tools/gram_acc.py; the flush was 8192 before, 3% slower).
//   warps 0-7 : epilogue (TMEM lane group warp % 4, columns 128 (warp / 4) .. +127 in registers)
//   warp 8    : TMEM alloc (both CTAs); MMA issue (leader)
//   warp 9    : bulk loader (both CTAs)
//   warp 10   : peer only -- forwards the completion of each of its stages to the leader
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fkk_internal.h"
#include "tc_common.cuh"

namespace fkk {

namespace {

constexpr int H = 128;                      // channels per CTA half
constexpr int T2 = 256;                     // tile edge
constexpr int KC = 32;                      // pixels per stage (= image stage)
constexpr int NSTG = 3;
constexpr int PERIOD = 64;                  // pixels per TMEM drain
constexpr int SPP = PERIOD / KC;            // stages per period
constexpr int FLUSH = 16384;
constexpr int LBO = 128;
constexpr int SBO = (KC / 4) * LBO + 16;    // 1040 B (the image's padded layout)
constexpr int OPB = (H / 8) * SBO;          // 16640 B per operand part (hi or lo)
constexpr int HALF = 2 * OPB;               // hi + lo of one 128-channel half
constexpr int STB = 2 * HALF;               // A half, B half
constexpr int SMEM = NSTG * STB + 256;
constexpr int NTHR = 352;
constexpr int NEPI = 256;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arrive_on(uint64_t* bar, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(tc::smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
// relaxed remote arrive (no MEMBAR.ALL.GPU): for signals that order no memory, e.g. "TMEM drained"
// after tcgen05.wait::ld + tcgen05.fence::before_thread_sync
__device__ __forceinline__ void arrive_on_relaxed(uint64_t* bar, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(tc::smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WP_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WP_%=;\n\t}" ::"r"(tc::smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   tc::smem_u32(bar)),
               "h"((unsigned short)3)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(NTHR, 1) gram_pre2_kernel(const unsigned char* __restrict__ Apre, int64_t nq,
                                                            const int2* __restrict__ tiles, int ntiles,
                                                            double* __restrict__ partials,
                                                            unsigned long long* __restrict__ dbg) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSTG * STB);
  uint64_t* full = bars;                    // [NSTG] local: this CTA's bulk copies (tx)
  uint64_t* pfull = bars + NSTG;            // [NSTG] leader: the peer's stage completed (forwarded)
  uint64_t* empty = bars + 2 * NSTG;        // [NSTG] local: MMA commit (multicast)
  uint64_t* acc_full = bars + 3 * NSTG;     // [2] local: MMA commit (multicast)
  uint64_t* acc_empty = acc_full + 2;       // [2] leader: epilogues of both CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const int pair = blockIdx.x >> 1;
  const int t = pair % ntiles, split = pair / ntiles, nsplit = (gridDim.x >> 1) / ntiles;
  const int bi = tiles[t].x, bj = tiles[t].y;
  const bool diag = bi == bj;
  const int64_t qb = nq * split / nsplit, qe = nq * (split + 1) / nsplit;
  const int64_t nper = qe > qb ? (qe - qb + SPP - 1) / SPP : 0;

  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&pfull[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&acc_full[b], 1); tc::mbar_init(&acc_empty[b], 2 * (NEPI / 32)); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3, chalf = warp >> 2;
    const int i = (int)rank * H + lg * 32 + lane;          // tile row
    double* part = partials + (int64_t)pair * (T2 * T2);  // [j][i]
    float S[128];
#pragma unroll
    for (int q = 0; q < 128; ++q) S[q] = 0.f;
    uint32_t ph = 0;   // bit b: phase of accumulator b (bit mask, not an indexed array)
    bool first = true;
    for (int64_t pidx = 0; pidx < nper; ++pidx) {
      const int b = (int)(pidx & 1);
      tc::mbar_wait(&acc_full[b], ((ph >> b) & 1u));
      ph ^= 1u << b;
      tc::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(256 * b + 128 * chalf);
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float h[16];
        tc::tmem_ld16(tb + c0, h);
#pragma unroll
        for (int q = 0; q < 16; ++q) S[c0 + q] += h[q];
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_on_relaxed(&acc_empty[b], 0);   // TMEM drained: orders no memory
      const bool last = pidx == nper - 1;
      if (last || ((pidx + 1) * PERIOD) % FLUSH == 0) {
        // fp64 flush in batches of 16 (one L2 round trip per batch, as gram_pre_kernel)
#pragma unroll
        for (int q0 = 0; q0 < 128; q0 += 16) {
          double old[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) old[u] = first ? 0.0 : part[(int64_t)(128 * chalf + q0 + u) * T2 + i];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            part[(int64_t)(128 * chalf + q0 + u) * T2 + i] = old[u] + (double)S[q0 + u];
            S[q0 + u] = 0.f;
          }
        }
        first = false;
      }
    }
    if (nper == 0)
      for (int q = 0; q < 128; ++q) part[(int64_t)(128 * chalf + q) * T2 + i] = 0.0;
  } else if (warp == 8) {
    if (rank == 0) {
      // ---------------------------------------------------------- MMA issue (leader)
      constexpr uint32_t idesc = tc::make_idesc_tf32(T2, T2, false, false);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t eph = 0;   // bit b: phase of acc_empty[b]
      const uint64_t d00 = tc::make_sdesc(tc::smem_u32(smem), LBO, SBO);
      unsigned long long w_full = 0, w_peer = 0, w_acc = 0;   // dbg cycle split
      const unsigned long long t_start = clock64();
      for (int64_t pidx = 0; pidx < nper; ++pidx) {
        const int b = (int)(pidx & 1);
        if (pidx >= 2) {
          const unsigned long long c0 = dbg ? clock64() : 0;
          wait_cluster(&acc_empty[b], ((eph >> b) & 1u));
          if (dbg) w_acc += clock64() - c0;
          eph ^= 1u << b;
          tc::tc_fence_after();
        }
        const uint32_t d = tmem + 256 * b;
        const int64_t q0 = qb + pidx * SPP, q1 = (qe < q0 + SPP) ? qe : (q0 + SPP);
        uint32_t acc = 0;
        for (int64_t q = q0; q < q1; ++q) {
          const unsigned long long c0 = dbg ? clock64() : 0;
          tc::mbar_wait(&full[stage], phase);
          const unsigned long long c1 = dbg ? clock64() : 0;
          wait_cluster(&pfull[stage], phase);
          if (dbg) { w_full += c1 - c0; w_peer += clock64() - c1; }
          tc::tc_fence_after();
          const uint64_t dah = tc::sdesc_add(d00, (uint32_t)(stage * STB)), dal = tc::sdesc_add(dah, OPB);
          const uint64_t dbh = diag ? dah : tc::sdesc_add(dah, HALF);
          const uint64_t dbl = diag ? dal : tc::sdesc_add(dah, HALF + OPB);
          if (tc::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
              const uint32_t ko = ks * 2 * LBO;
              mma2(d, tc::sdesc_add(dal, ko), tc::sdesc_add(dbh, ko), idesc, acc);   // lo_i * hi_j
              mma2(d, tc::sdesc_add(dah, ko), tc::sdesc_add(dbl, ko), idesc, 1);     // hi_i * lo_j
              mma2(d, tc::sdesc_add(dah, ko), tc::sdesc_add(dbh, ko), idesc, 1);     // hi_i * hi_j
              acc = 1;
            }
            commit2(&empty[stage]);
          }
          acc = 1;
          __syncwarp();
          if (++stage == NSTG) { stage = 0; phase ^= 1; }
        }
        if (tc::elect_one()) commit2(&acc_full[b]);
        __syncwarp();
      }
      if (dbg && lane == 0) {
        dbg[pair * 4 + 0] = clock64() - t_start;
        dbg[pair * 4 + 1] = w_full;
        dbg[pair * 4 + 2] = w_peer;
        dbg[pair * 4 + 3] = w_acc;
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      // ---------------------------------------------------------- bulk loader (both CTAs)
      const uint32_t sbase = tc::smem_u32(smem);
      const uint32_t bytes = (diag ? 1u : 2u) * HALF;
      const int cA = 2 * bi + (int)rank, cB = 2 * bj + (int)rank;     // 128-channel image blocks
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t q = qb; q < qe; ++q) {
        tc::mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t st = sbase + stage * STB;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&full[stage])),
                     "r"(bytes)
                     : "memory");
        bulk_g2s(st, Apre + (size_t)(cA * nq + q) * HALF, HALF, &full[stage]);
        if (!diag) bulk_g2s(st + HALF, Apre + (size_t)(cB * nq + q) * HALF, HALF, &full[stage]);
        if (++stage == NSTG) { stage = 0; phase ^= 1; }
      }
    }
  } else if (rank == 1 && lane == 0) {
    // ------------------------------------------------------------ forwarder (peer): stage landed -> leader
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t q = qb; q < qe; ++q) {
      tc::mbar_wait(&full[stage], phase);
      arrive_on(&pfull[stage], 0);
      if (++stage == NSTG) { stage = 0; phase ^= 1; }
    }
  } else if (rank == 0 && lane == 0) {
    // leader: its own stages need no forwarding; complete pfull for the single-CTA degenerate case
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc::tc_fence_after();
  if (warp == 8)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

}  // namespace

int gram_pre2_image_blocks(int M) { return 2 * ((M + T2 - 1) / T2); }

void launch_gram_pre2(const unsigned char* Apre, int64_t n, const int2* d_tiles, int ntiles, int nsplit,
                      double* partials, cudaStream_t s) {
  const int64_t nq = (n + KC - 1) / KC;
  FKK_CUDA_CHECK(cudaFuncSetAttribute(gram_pre2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * ntiles * nsplit);
  cfg.blockDim = dim3(NTHR);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // FKK_GRAM_DBG (debug only): leader MMA-warp cycle split per pair, printed to stderr; synchronises
  static const bool gdbg = getenv("FKK_GRAM_DBG") != nullptr;
  unsigned long long* dbg = nullptr;
  const int npair = ntiles * nsplit;
  if (gdbg) FKK_CUDA_CHECK(cudaMalloc(&dbg, (size_t)npair * 4 * sizeof(unsigned long long)));
  FKK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gram_pre2_kernel, Apre, nq, d_tiles, ntiles, partials, dbg));
  check_launch("gram_pre2");
  if (gdbg) {
    std::vector<unsigned long long> h((size_t)npair * 4);
    FKK_CUDA_CHECK(cudaMemcpyAsync(h.data(), dbg, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    FKK_CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFree(dbg);
    double tot[4] = {0, 0, 0, 0};
    for (int b = 0; b < npair; ++b)
      for (int q = 0; q < 4; ++q) tot[q] += (double)h[b * 4 + q] / npair;
    fprintf(stderr, "gram_pre2 dbg: %d pairs, mean cycles total %.0f, wait own stage %.0f, wait peer %.0f, wait epilogue %.0f\n",
            npair, tot[0], tot[1], tot[2], tot[3]);
  }
}

}  // namespace fkk
