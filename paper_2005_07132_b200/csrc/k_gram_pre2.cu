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

// Work schedule: the ntiles x nq (tile, 32-pixel stage) units in tile-major order are cut into one
// contiguous range per pair (as many pairs as the SMs hold, not a multiple of the tile count), so a
// pair runs up to MAXSEG segments (tile, [qb, qe)), each into its own fp64 partial slot.
constexpr int MAXSEG = 4;

__global__ void __launch_bounds__(NTHR, 1) gram_pre2_kernel(const unsigned char* __restrict__ Apre, int64_t nq,
                                                            const int2* __restrict__ tiles,
                                                            const int4* __restrict__ sched,
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
  const int4* seg = sched + (size_t)pair * MAXSEG;   // (tile, qb, qe, slot); tile < 0 ends the list

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
    float S[128];
#pragma unroll
    for (int q = 0; q < 128; ++q) S[q] = 0.f;
    uint32_t ph[2] = {0, 0};
    int64_t gp = 0;   // periods over all segments (accumulator buffer parity)
    for (int sg = 0; sg < MAXSEG; ++sg) {
      const int4 sd = seg[sg];
      if (sd.x < 0) break;
      double* part = partials + (int64_t)sd.w * (T2 * T2);  // [j][i]
      const int64_t nper = ((int64_t)sd.z - sd.y + SPP - 1) / SPP;
      bool first = true;
      for (int64_t pidx = 0; pidx < nper; ++pidx, ++gp) {
        const int b = (int)(gp & 1);
        tc::mbar_wait(&acc_full[b], ph[b]);
        ph[b] ^= 1;
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
    }
  } else if (warp == 8) {
    if (rank == 0) {
      // ---------------------------------------------------------- MMA issue (leader)
      constexpr uint32_t idesc = tc::make_idesc_tf32(T2, T2, false, false);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t eph[2] = {0, 0};
      const uint64_t d00 = tc::make_sdesc(tc::smem_u32(smem), LBO, SBO);
      unsigned long long w_full = 0, w_peer = 0, w_acc = 0;   // dbg cycle split
      const unsigned long long t_start = clock64();
      int64_t gp = 0;
      for (int sg = 0; sg < MAXSEG; ++sg) {
        const int4 sd = seg[sg];
        if (sd.x < 0) break;
        const bool diag = tiles[sd.x].x == tiles[sd.x].y;
        const int64_t nper = ((int64_t)sd.z - sd.y + SPP - 1) / SPP;
        for (int64_t pidx = 0; pidx < nper; ++pidx, ++gp) {
          const int b = (int)(gp & 1);
          if (gp >= 2) {
            const unsigned long long c0 = dbg ? clock64() : 0;
            wait_cluster(&acc_empty[b], eph[b]);
            if (dbg) w_acc += clock64() - c0;
            eph[b] ^= 1;
            tc::tc_fence_after();
          }
          const uint32_t d = tmem + 256 * b;
          const int64_t q0 = sd.y + pidx * SPP, q1 = ((int64_t)sd.z < q0 + SPP) ? (int64_t)sd.z : (q0 + SPP);
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
      int stage = 0;
      uint32_t phase = 0;
      for (int sg = 0; sg < MAXSEG; ++sg) {
        const int4 sd = seg[sg];
        if (sd.x < 0) break;
        const int bi = tiles[sd.x].x, bj = tiles[sd.x].y;
        const bool diag = bi == bj;
        const uint32_t bytes = (diag ? 1u : 2u) * HALF;
        const int cA = 2 * bi + (int)rank, cB = 2 * bj + (int)rank;     // 128-channel image blocks
        for (int64_t q = sd.y; q < sd.z; ++q) {
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
    }
  } else if (rank == 1 && lane == 0) {
    // ------------------------------------------------------------ forwarder (peer): stage landed -> leader
    int stage = 0;
    uint32_t phase = 0;
    for (int sg = 0; sg < MAXSEG; ++sg) {
      const int4 sd = seg[sg];
      if (sd.x < 0) break;
      for (int64_t q = sd.y; q < sd.z; ++q) {
        tc::mbar_wait(&full[stage], phase);
        arrive_on(&pfull[stage], 0);
        if (++stage == NSTG) { stage = 0; phase ^= 1; }
      }
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

namespace {
// G[r][c] from the partial slots of the tile holding (min(r,c), max(r,c)): slots tile_ptr[t] .. tile_ptr[t+1]
__global__ void gram_pre2_reduce_kernel(const double* __restrict__ partials, int M, const int* __restrict__ tile_of,
                                        int nT, const int* __restrict__ tile_ptr, const int* __restrict__ slots,
                                        double* __restrict__ G, int accumulate) {
  const int64_t total = (int64_t)M * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / M), c = (int)(e % M);
    const int i = min(r, c), j = max(r, c);
    const int ti = i / T2, tj = j / T2;
    const int t = tile_of[ti * nT + tj];
    const int64_t off = (int64_t)(j - tj * T2) * T2 + (i - ti * T2);
    double sum = 0.0;
    for (int k = tile_ptr[t]; k < tile_ptr[t + 1]; ++k) sum += partials[(int64_t)slots[k] * (T2 * T2) + off];
    G[e] = accumulate ? G[e] + sum : sum;
  }
}
}  // namespace

// pairs: cudaOccupancyMaxActiveClusters reports all 74 SM pairs of a B200, but 72 or 74 pairs run the
// cfg3 Gram in 4.0 ms against 3.34 ms for 70 (FKK_GRAM_PAIRS A/B, the MMA warp's own-stage waits +40%),
// so the schedule takes at most 70
int gram_pre2_pairs() {
  static int cached = 0;
  if (cached) return cached;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  FKK_CUDA_CHECK(cudaFuncSetAttribute(gram_pre2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * (sms / 2));
  cfg.blockDim = dim3(NTHR);
  cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, gram_pre2_kernel, &cfg) != cudaSuccess || nc < 1) {
    cudaGetLastError();
    nc = sms / 2;
  }
  cached = std::min(std::min(nc, sms / 2), 70);
  return cached;
}
size_t gram_pre2_partial_doubles(int ntiles) { return (size_t)(gram_pre2_pairs() + ntiles) * T2 * T2; }
size_t gram_pre2_sched_ints(int ntiles) {
  const int P = gram_pre2_pairs();
  return (size_t)4 * P * MAXSEG + (ntiles + 1) + (P + ntiles);
}

void launch_gram_pre2(const unsigned char* Apre, int64_t n, int M, const int2* d_tiles, const int* d_tile_of, int nT,
                      int ntiles, int* d_sched, int64_t* sched_key, double* partials, double* G, int accumulate,
                      cudaStream_t s) {
  const int64_t nq = (n + KC - 1) / KC;
  // schedule: W = ntiles x nq units, P contiguous ranges (at least 8 stages each)
  const int64_t W = (int64_t)ntiles * nq;
  int Pcap = gram_pre2_pairs();
  if (const char* ev = getenv("FKK_GRAM_PAIRS")) Pcap = std::max(1, std::min(Pcap, atoi(ev)));   // A/B only
  const int P = (int)std::max<int64_t>(1, std::min<int64_t>(Pcap, W / 8));
  std::vector<int> h((size_t)4 * P * MAXSEG + (ntiles + 1) + (P + ntiles), -1);
  std::vector<std::vector<int>> tslots(ntiles);
  int nslot = 0;
  for (int p = 0; p < P; ++p) {
    const int64_t L0 = W * p / P, L1 = W * (p + 1) / P;
    int sg = 0;
    for (int64_t t = L0 / std::max<int64_t>(nq, 1); L1 > L0 && t <= (L1 - 1) / nq; ++t) {
      const int64_t qb = std::max(L0, t * nq) - t * nq, qe = std::min(L1, (t + 1) * nq) - t * nq;
      if (qe <= qb) continue;
      if (sg == MAXSEG) throw Status(10, "gram_pre2: more tiles per pair than the schedule holds");
      int* e = &h[(size_t)4 * (p * MAXSEG + sg)];
      e[0] = (int)t; e[1] = (int)qb; e[2] = (int)qe; e[3] = nslot;
      tslots[t].push_back(nslot++);
      ++sg;
    }
  }
  int* tp = &h[(size_t)4 * P * MAXSEG];
  int* sl = tp + (ntiles + 1);
  int k = 0;
  for (int t = 0; t < ntiles; ++t) {
    tp[t] = k;
    for (int v : tslots[t]) sl[k++] = v;
  }
  tp[ntiles] = k;
  // uploaded once per (rows, tiles) of the owning plan (*sched_key): a copy in the stream ahead of every
  // Gram cost ~40 us (pageable source: staged before the call returns, no device synchronisation)
  const int64_t key = n * 65536 + ntiles;
  if (!sched_key || *sched_key != key) {
    FKK_CUDA_CHECK(cudaMemcpyAsync(d_sched, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    if (sched_key) *sched_key = key;
  }
  FKK_CUDA_CHECK(cudaFuncSetAttribute(gram_pre2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * P);
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
  if (gdbg) FKK_CUDA_CHECK(cudaMalloc(&dbg, (size_t)P * 4 * sizeof(unsigned long long)));
  FKK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gram_pre2_kernel, Apre, nq, d_tiles,
                                    reinterpret_cast<const int4*>(d_sched), partials, dbg));
  check_launch("gram_pre2");
  if (gdbg) {
    std::vector<unsigned long long> hd((size_t)P * 4);
    FKK_CUDA_CHECK(cudaMemcpyAsync(hd.data(), dbg, hd.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    FKK_CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFree(dbg);
    double tot[4] = {0, 0, 0, 0};
    for (int b = 0; b < P; ++b)
      for (int q = 0; q < 4; ++q) tot[q] += (double)hd[b * 4 + q] / P;
    fprintf(stderr, "gram_pre2 dbg: %d pairs, mean cycles total %.0f, wait own stage %.0f, wait peer %.0f, wait epilogue %.0f\n",
            P, tot[0], tot[1], tot[2], tot[3]);
  }
  gram_pre2_reduce_kernel<<<1024, 256, 0, s>>>(partials, M, d_tile_of, nT, d_sched + 4 * P * MAXSEG,
                                                d_sched + 4 * P * MAXSEG + (ntiles + 1), G, accumulate);
  check_launch("gram_pre2_reduce");
}

}  // namespace fkk
