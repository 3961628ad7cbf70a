// Gram matrix G0 = A0^T A0 (F2) on a CTA PAIR: tcgen05.mma.cta_group::2 kind::tf32,
// 3xTF32 (reading A22), one 256 x 256 tile of G per cluster of two CTAs.
// STATUS: parity-green but measured slower than the 1-CTA kernel at cfg3 (7.9 vs 6.1 ms, tensor pipe
// 31% active in both): the producers' register-prefetched global loads remain the bottleneck.  Opt-in
// (FKK_GRAM_PAIR=1); the next step is TMA staging of the raw A0 tiles (kind::tf32 operands must be
// K-major, so a register transpose stays -- tools/micro/tcmn.cu shows MN-major tf32 reads zeros).
//
// Why a pair: with 1-CTA 128 x 128 tiles the tensor core reads 8 KB of smem operands per 64-clock
// MMA (128 B/clk, the whole smem bandwidth) before the producers write a byte, and each SM must
// stream 32 KB of A0 per stage.  The pair computes 256 x 256 x 8 per instruction with each CTA
// holding 128 rows of the A block and 128 rows of the B block (the B operand is split by N across
// the pair, D by M; verified by tools/micro/tc2.cu), so per SM the operand reads and the A0
// stream per flop halve.
//
// Tile (bi <= bj) of 256-channel blocks; CTA rank r holds A channels 256 bi + 128 r .. and B channels
// 256 bj + 128 r .. (K-major core matrices as in k_gram_tc.cu; the diagonal tiles share one operand).
// Accuracy: hi*hi and the cross terms accumulate in separate TMEM
// accumulators (256 columns each: the 512 TMEM columns, single-buffered), drained every 128 pixels
// into fp32 register sums (round to nearest), flushed to fp64 partials every 8192 pixels.  The MMA
// waits for the drain (~5% of a period).
//   warps 0-7  : producers (register lookahead, tf32 split, st.shared; arrive on the LEADER's
//                full barrier through the cluster)                        setmaxnreg 64
//   warps 8-15 : epilogue (128 columns per thread in registers)           setmaxnreg 152
//   warps 16-19: warp 16 allocates TMEM (both CTAs) and, in the leader, issues the MMAs    48
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "fkk_internal.h"
#include "tc_common.cuh"

namespace fkk {

namespace {

constexpr int H = 128;                      // rows per CTA of the 256-tile (A half / B half)
constexpr int T2 = 256;                     // tile edge
constexpr int KC = 32;                      // pixels per stage
constexpr int NSTG = 3;
constexpr int PERIOD = 128;                 // pixels per TMEM drain
constexpr int FLUSH = 8192;                 // pixels per fp64 flush
constexpr int LBO = 128;
constexpr int SBO = (KC / 4) * LBO + 16;    // 1040 B
constexpr int OPB = (H / 8) * SBO;          // 16640 B per operand (hi or lo)
constexpr int STB = 4 * OPB;                // A hi, A lo, B hi, B lo
constexpr int SMEM = NSTG * STB + 256;
constexpr int NTHR = 640;
constexpr int NPROD = 256, NEPI = 256;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive (release, cluster scope) on the mbarrier at the same smem offset in CTA `rank`
__device__ __forceinline__ void arrive_on(uint64_t* bar, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(tc::smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
// wait with cluster-scope acquire (arrivals come from the peer CTA too)
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W2_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra W2_%=;\n\t}" ::"r"(tc::smem_u32(bar)),
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
__device__ __forceinline__ void commit2(uint64_t* bar) {   // arrive on `bar` in both CTAs of the pair
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   tc::smem_u32(bar)),
               "h"((unsigned short)3)
               : "memory");
}

__device__ __forceinline__ void load_block(const float* __restrict__ A, int M, int64_t px0, int64_t pend, int col,
                                           float4 (&x)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    x[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (px0 + q < pend && col < M) x[q] = __ldg(reinterpret_cast<const float4*>(A + (px0 + q) * (int64_t)M + col));
  }
}
__device__ __forceinline__ void store_block(const float4 (&x)[4], unsigned char* hi_base, unsigned char* lo_base, int c4,
                                            int p4) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int r = c4 * 4 + e;
    const int off = (r >> 3) * SBO + p4 * LBO + (r & 7) * 16;
    const float v0 = e == 0 ? x[0].x : e == 1 ? x[0].y : e == 2 ? x[0].z : x[0].w;
    const float v1 = e == 0 ? x[1].x : e == 1 ? x[1].y : e == 2 ? x[1].z : x[1].w;
    const float v2 = e == 0 ? x[2].x : e == 1 ? x[2].y : e == 2 ? x[2].z : x[2].w;
    const float v3 = e == 0 ? x[3].x : e == 1 ? x[3].y : e == 2 ? x[3].z : x[3].w;
    float4 h, l;
    tc::split_fast(v0, h.x, l.x);
    tc::split_fast(v1, h.y, l.y);
    tc::split_fast(v2, h.z, l.z);
    tc::split_fast(v3, h.w, l.w);
    *reinterpret_cast<float4*>(hi_base + off) = h;
    *reinterpret_cast<float4*>(lo_base + off) = l;
  }
}

__global__ void __launch_bounds__(NTHR, 1) gram_tc2_kernel(const float* __restrict__ A, int64_t n, int M,
                                                           const int2* __restrict__ tiles, int ntiles,
                                                           double* __restrict__ partials) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSTG * STB);
  uint64_t* full = bars;                    // [NSTG]  leader: producers of both CTAs (2 x 256)
  uint64_t* empty = bars + NSTG;            // [NSTG]  MMA commit (multicast) -> producers
  uint64_t* acc_full = bars + 2 * NSTG;     // MMA commit (multicast) -> epilogues
  uint64_t* acc_empty = acc_full + 1;       // leader: epilogues of both CTAs (2 x 256)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const int pair = blockIdx.x >> 1;
  const int t = pair % ntiles, split = pair / ntiles, nsplit = (gridDim.x >> 1) / ntiles;
  const int bi = tiles[t].x, bj = tiles[t].y;
  const bool diag = bi == bj;
  const int ca = bi * T2 + (int)rank * H, cb = bj * T2 + (int)rank * H;   // first A / B channel of this CTA
  const int64_t rb = n * split / nsplit, re = n * (split + 1) / nsplit;
  const int64_t nper = re > rb ? (re - rb + PERIOD - 1) / PERIOD : 0;

  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) { tc::mbar_init(&full[s], 2 * NPROD); tc::mbar_init(&empty[s], 1); }
    tc::mbar_init(acc_full, 1);
    tc::mbar_init(acc_empty, 2 * NEPI);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 16) {
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
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");
    // ------------------------------------------------------------ producers
    const int c4 = tid & 31, p4 = tid >> 5;     // channel quad, pixel quad
    float4 xa[4], xb[4];
    int64_t k0 = rb;
    if (k0 < re) {
      load_block(A, M, k0 + 4 * p4, re, ca + 4 * c4, xa);
      if (!diag) load_block(A, M, k0 + 4 * p4, re, cb + 4 * c4, xb);
    }
    int stage = 0;
    uint32_t phase = 0;
    for (; k0 < re; k0 += KC) {
      tc::mbar_wait(&empty[stage], phase ^ 1);
      unsigned char* st = smem + stage * STB;
      store_block(xa, st, st + OPB, c4, p4);
      if (!diag) store_block(xb, st + 2 * OPB, st + 3 * OPB, c4, p4);
      tc::fence_proxy_async_smem();
      arrive_on(&full[stage], 0);
      if (++stage == NSTG) { stage = 0; phase ^= 1; }
      const int64_t kn = k0 + KC;               // prefetch the next stage into registers
      if (kn < re) {
        load_block(A, M, kn + 4 * p4, re, ca + 4 * c4, xa);
        if (!diag) load_block(A, M, kn + 4 * p4, re, cb + 4 * c4, xb);
      }
    }
  } else if (warp < 16) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;" ::: "memory");
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3;                    // TMEM lane group
    const int chalf = (warp - 8) >> 2;          // columns 128 chalf .. +127 of the tile
    const int i = (int)rank * H + lg * 32 + lane;   // tile row
    double* part = partials + (int64_t)pair * (T2 * T2);   // [j][i]
    float S[128];
#pragma unroll
    for (int q = 0; q < 128; ++q) S[q] = 0.f;
    bool first = true;
    for (int64_t pidx = 0; pidx < nper; ++pidx) {
      tc::mbar_wait(acc_full, (uint32_t)(pidx & 1));
      tc::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(128 * chalf);
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float h[16];
        tc::tmem_ld16(tb + c0, h);               // hi * hi
#pragma unroll
        for (int q = 0; q < 16; ++q) S[c0 + q] += h[q];
        tc::tmem_ld16(tb + 256 + c0, h);         // cross terms
#pragma unroll
        for (int q = 0; q < 16; ++q) S[c0 + q] += h[q];
      }
      tc::tc_fence_before();
      arrive_on(acc_empty, 0);
      const bool last = pidx == nper - 1;
      if (last || ((pidx + 1) * PERIOD) % FLUSH == 0) {
#pragma unroll
        for (int q = 0; q < 128; ++q) {
          double* p = part + (int64_t)(128 * chalf + q) * T2 + i;
          *p = (first ? 0.0 : *p) + (double)S[q];
          S[q] = 0.f;
        }
        first = false;
      }
    }
    if (nper == 0)
      for (int q = 0; q < 128; ++q) part[(int64_t)(128 * chalf + q) * T2 + i] = 0.0;
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;" ::: "memory");
    if (warp == 16 && rank == 0) {
      // ---------------------------------------------------------- MMA issue (leader CTA only)
      constexpr uint32_t idesc = tc::make_idesc_tf32(T2, T2, false, false);
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t d00 = tc::make_sdesc(tc::smem_u32(smem), LBO, SBO);
      const uint32_t d_hi = tmem, d_mid = tmem + 256;
      for (int64_t pidx = 0; pidx < nper; ++pidx) {
        if (pidx >= 1) {
          wait_cluster(acc_empty, (uint32_t)((pidx - 1) & 1));
          tc::tc_fence_after();
        }
        const int64_t p0 = rb + pidx * PERIOD, p1 = (re < p0 + PERIOD) ? re : (p0 + PERIOD);
        uint32_t acc = 0;
        for (int64_t k0 = p0; k0 < p1; k0 += KC) {
          wait_cluster(&full[stage], phase);
          tc::tc_fence_after();
          const uint64_t dah = tc::sdesc_add(d00, (uint32_t)(stage * STB)), dal = tc::sdesc_add(dah, OPB);
          const uint64_t dbh = diag ? dah : tc::sdesc_add(dah, 2 * OPB);
          const uint64_t dbl = diag ? dal : tc::sdesc_add(dah, 3 * OPB);
          if (tc::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
              const uint32_t ko = ks * 2 * LBO;   // 8 pixels = 2 K-core matrices
              mma2(d_mid, tc::sdesc_add(dal, ko), tc::sdesc_add(dbh, ko), idesc, acc);   // lo_i * hi_j
              mma2(d_mid, tc::sdesc_add(dah, ko), tc::sdesc_add(dbl, ko), idesc, 1);     // hi_i * lo_j
              mma2(d_hi, tc::sdesc_add(dah, ko), tc::sdesc_add(dbh, ko), idesc, acc);    // hi_i * hi_j
              acc = 1;
            }
            commit2(&empty[stage]);
          }
          acc = 1;
          __syncwarp();
          if (++stage == NSTG) { stage = 0; phase ^= 1; }
        }
        if (tc::elect_one()) commit2(acc_full);
        __syncwarp();
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc::tc_fence_after();
  if (warp == 16)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

__global__ void gram_tc2_reduce_kernel(const double* __restrict__ partials, int ntiles, int nsplit, int M,
                                       const int* __restrict__ tile_of, int nT, double* __restrict__ G, int accumulate) {
  const int64_t total = (int64_t)M * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / M), c = (int)(e % M);
    const int i = min(r, c), j = max(r, c);
    const int ti = i / T2, tj = j / T2;
    const int t = tile_of[ti * nT + tj];
    const int64_t off = (int64_t)(j - tj * T2) * T2 + (i - ti * T2);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += partials[((int64_t)sp * ntiles + t) * (T2 * T2) + off];
    G[e] = accumulate ? G[e] + s : s;
  }
}

}  // namespace

void gram_tc2_tiles(int M, std::vector<int2>& tiles, std::vector<int>& tile_of, int& nT) {
  nT = (M + T2 - 1) / T2;
  tiles.clear();
  tile_of.assign((size_t)nT * nT, -1);
  for (int ti = 0; ti < nT; ++ti)
    for (int tj = ti; tj < nT; ++tj) {
      tile_of[ti * nT + tj] = (int)tiles.size();
      tiles.push_back(make_int2(ti, tj));
    }
}

int gram_tc2_splits(int ntiles, int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ns = std::max(1, sms / std::max(1, 2 * ntiles));
  const int64_t by_rows = std::max<int64_t>(1, n / 1024);
  return (int)std::min<int64_t>(ns, by_rows);
}

size_t gram_tc2_partial_doubles(int ntiles, int nsplit) { return (size_t)ntiles * nsplit * T2 * T2; }

void launch_gram_tc2(const float* A, int64_t n, int M, const int2* d_tiles, int ntiles, int nsplit, double* partials,
                     cudaStream_t s) {
  FKK_CUDA_CHECK(cudaFuncSetAttribute(gram_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
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
  FKK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gram_tc2_kernel, A, n, M, d_tiles, ntiles, partials));
  check_launch("gram_tc2");
}

void launch_gram_tc2_reduce(const double* partials, int ntiles, int nsplit, int M, const int* d_tile_of, int nT,
                            double* G, int accumulate, cudaStream_t s) {
  gram_tc2_reduce_kernel<<<1024, 256, 0, s>>>(partials, ntiles, nsplit, M, d_tile_of, nT, G, accumulate);
  check_launch("gram_tc2_reduce");
}

}  // namespace fkk
