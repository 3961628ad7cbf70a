// Gram matrix G0 = A0^T A0 (F2, the normal matrix of the truncated SVD) on the
// 5th-generation tensor cores: tcgen05.mma kind::tf32, 3xTF32 (hi*hi + hi*lo + lo*hi, reading A22),
// fp32 accumulation in TMEM over <= 8192 pixels, then an fp64 flush into this CTA's own partial tile
// (deterministic; summed over the row splits by gram_tc_reduce).
//
// Tiles of G: 128 (i) x 256 (j) covering the upper triangle; the CTA for (tile, split) streams the
// pixels of its split.  Both operands are MN-major in smem (the channel index is contiguous in A0):
// a core matrix is 8 pixels (K) x 16 B (4 channels); a 4-channel column strip holds the KC pixels of
// a stage contiguously and strips are SBO = 16*KC + 16 bytes apart (the 16-B pad makes the producer's
// 128-bit smem stores bank-conflict free).
//   warps 0-3 : producers (global fp32 loads, tf32 hi/lo split, st.shared) and the TMEM epilogue
//   warp 4    : TMEM allocation and the single-thread MMA issue
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "fkk_internal.h"
#include "tc_common.cuh"

namespace fkk {

namespace {

constexpr int GB_M = 128;                 // tile rows (i)
constexpr int GB_N = 256;                 // tile cols (j)
constexpr int GKC = 32;                   // pixels per stage
constexpr int GSTAGES = 2;
constexpr int GFLUSH = 8192;              // fp32 accumulation span in pixels
constexpr int GSTRIP = GKC * 16 + 16;     // bytes per 4-channel strip (SBO)
constexpr int GA_BYTES = (GB_M / 4) * GSTRIP;   // 16896
constexpr int GB_BYTES = (GB_N / 4) * GSTRIP;   // 33792
constexpr int GSTAGE_BYTES = 2 * GA_BYTES + 2 * GB_BYTES;
constexpr int GSMEM = GSTAGES * GSTAGE_BYTES + 256;
constexpr int GTHREADS = 160;

__global__ void __launch_bounds__(GTHREADS, 1)
gram_tc_kernel(const float* __restrict__ A, int64_t n, int M, const int2* __restrict__ tiles, int ntiles,
               double* __restrict__ partials) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GSTAGES * GSTAGE_BYTES);
  uint64_t* full = bars;                  // [GSTAGES]
  uint64_t* empty = bars + GSTAGES;       // [GSTAGES]
  uint64_t* acc_full = bars + 2 * GSTAGES;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = blockIdx.x % ntiles, split = blockIdx.x / ntiles, nsplit = gridDim.x / ntiles;
  const int ti = tiles[t].x, tj = tiles[t].y;
  const int64_t rb = n * split / nsplit, re = n * (split + 1) / nsplit;
  double* part = partials + (int64_t)blockIdx.x * (GB_M * GB_N);   // [j][i] layout

  if (tid == 0) {
    for (int s = 0; s < GSTAGES; ++s) { tc::mbar_init(&full[s], 128); tc::mbar_init(&empty[s], 1); }
    tc::mbar_init(acc_full, 1);
    tc::mbar_init(acc_empty, 128);
    tc::fence_mbar_init();
  }
  if (warp == 4) tc::tmem_alloc(tmem_slot, GB_N);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t nchunks = re > rb ? (re - rb + GFLUSH - 1) / GFLUSH : 0;
  if (warp < 4) {
    // ------------------------------------------------------------ producers + epilogue
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t c0 = rb + ch * GFLUSH, c1 = (re < c0 + GFLUSH) ? re : (c0 + GFLUSH);
      for (int64_t k0 = c0; k0 < c1; k0 += GKC) {
        tc::mbar_wait(&empty[stage], phase ^ 1);
        unsigned char* st = smem + stage * GSTAGE_BYTES;
        unsigned char* ahi = st;
        unsigned char* alo = st + GA_BYTES;
        unsigned char* bhi = st + 2 * GA_BYTES;
        unsigned char* blo = bhi + GB_BYTES;
        // A block: 32 pixels x 128 channels (i = ti*128 ..), 8 float4 per thread
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int idx = tid + h * 128;
          const int row = idx >> 5, c4 = idx & 31;
          const int64_t px = k0 + row;
          const int col = ti * GB_M + c4 * 4;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (px < c1 && col < M) v = __ldg(reinterpret_cast<const float4*>(A + px * (int64_t)M + col));
          float4 hi, lo;
          tc::split4(v, hi, lo);
          const int off = c4 * GSTRIP + row * 16;
          *reinterpret_cast<float4*>(ahi + off) = hi;
          *reinterpret_cast<float4*>(alo + off) = lo;
        }
        // B block: 32 pixels x 256 channels (j = tj*256 ..), 16 float4 per thread
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          const int idx = tid + h * 128;
          const int row = idx >> 6, c4 = idx & 63;
          const int64_t px = k0 + row;
          const int col = tj * GB_N + c4 * 4;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (px < c1 && col < M) v = __ldg(reinterpret_cast<const float4*>(A + px * (int64_t)M + col));
          float4 hi, lo;
          tc::split4(v, hi, lo);
          const int off = c4 * GSTRIP + row * 16;
          *reinterpret_cast<float4*>(bhi + off) = hi;
          *reinterpret_cast<float4*>(blo + off) = lo;
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&full[stage]);
        stage ^= 1;
        if (stage == 0) phase ^= 1;
      }
      // flush the fp32 accumulator: TMEM lane = i (row), column = j; partial layout [j][i]
      tc::mbar_wait(acc_full, acc_phase);
      acc_phase ^= 1;
      tc::tc_fence_after();
      const int i = warp * 32 + lane;
#pragma unroll 1
      for (int cb = 0; cb < GB_N / 16; ++cb) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cb * 16), v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          double* p = part + (int64_t)(cb * 16 + q) * GB_M + i;
          *p = (ch == 0 ? 0.0 : *p) + (double)v[q];
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(acc_empty);
    }
    if (nchunks == 0) {
      for (int e = tid; e < GB_M * GB_N; e += 128) part[e] = 0.0;
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------ single-thread MMA issue
    constexpr uint32_t idesc = tc::make_idesc_tf32(GB_M, GB_N, true, true);
    int stage = 0;
    uint32_t phase = 0, acc_empty_phase = 0;
    const uint32_t sbase = tc::smem_u32(smem);
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int64_t c0 = rb + ch * GFLUSH, c1 = (re < c0 + GFLUSH) ? re : (c0 + GFLUSH);
      if (ch > 0) {
        tc::mbar_wait(acc_empty, acc_empty_phase);
        acc_empty_phase ^= 1;
        tc::tc_fence_after();
      }
      uint32_t acc = 0;
      for (int64_t k0 = c0; k0 < c1; k0 += GKC) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t st = sbase + stage * GSTAGE_BYTES;
        const uint32_t ahi = st, alo = st + GA_BYTES, bhi = st + 2 * GA_BYTES, blo = bhi + GB_BYTES;
#pragma unroll
        for (int ks = 0; ks < GKC / 8; ++ks) {
          const uint32_t ko = ks * 128;   // 8 pixels x 16 B
          const uint64_t dah = tc::make_sdesc(ahi + ko, 128, GSTRIP), dal = tc::make_sdesc(alo + ko, 128, GSTRIP);
          const uint64_t dbh = tc::make_sdesc(bhi + ko, 128, GSTRIP), dbl = tc::make_sdesc(blo + ko, 128, GSTRIP);
          tc::mma_tf32(tmem, dal, dbh, idesc, acc);   // lo * hi
          acc = 1;
          tc::mma_tf32(tmem, dah, dbl, idesc, 1);     // hi * lo
          tc::mma_tf32(tmem, dah, dbh, idesc, 1);     // hi * hi
        }
        tc::mma_commit(&empty[stage]);
        stage ^= 1;
        if (stage == 0) phase ^= 1;
      }
      tc::mma_commit(acc_full);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 4) tc::tmem_dealloc(tmem, GB_N);
}

__global__ void gram_tc_reduce_kernel(const double* __restrict__ partials, int ntiles, int nsplit, int M,
                                      const int* __restrict__ tile_of, int nTj, double* __restrict__ G, int accumulate) {
  const int64_t total = (int64_t)M * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / M), c = (int)(e % M);
    const int i = min(r, c), j = max(r, c);
    const int ti = i / GB_M, tj = j / GB_N;
    const int t = tile_of[ti * nTj + tj];
    const int64_t off = (int64_t)(j - tj * GB_N) * GB_M + (i - ti * GB_M);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += partials[((int64_t)sp * ntiles + t) * (GB_M * GB_N) + off];
    G[e] = accumulate ? G[e] + s : s;
  }
}

}  // namespace

// Tile list of the upper triangle: (ti, tj) with tj*256 + 255 >= ti*128.
void gram_tc_tiles(int M, std::vector<int2>& tiles, std::vector<int>& tile_of, int& nTj) {
  const int nTi = (M + GB_M - 1) / GB_M;
  nTj = (M + GB_N - 1) / GB_N;
  tiles.clear();
  tile_of.assign((size_t)nTi * nTj, -1);
  for (int ti = 0; ti < nTi; ++ti)
    for (int tj = 0; tj < nTj; ++tj)
      if (tj * GB_N + GB_N - 1 >= ti * GB_M) {
        tile_of[ti * nTj + tj] = (int)tiles.size();
        tiles.push_back(make_int2(ti, tj));
      }
}

int gram_tc_splits(int ntiles, int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int ns = std::max(1, sms / std::max(1, ntiles));
  const int64_t by_rows = std::max<int64_t>(1, n / 1024);
  return (int)std::min<int64_t>(ns, by_rows);
}

size_t gram_tc_partial_doubles(int ntiles, int nsplit) { return (size_t)ntiles * nsplit * GB_M * GB_N; }

void launch_gram_tc(const float* A, int64_t n, int M, const int2* d_tiles, int ntiles, int nsplit, double* partials,
                    cudaStream_t s) {
  FKK_CUDA_CHECK(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GSMEM));
  gram_tc_kernel<<<ntiles * nsplit, GTHREADS, GSMEM, s>>>(A, n, M, d_tiles, ntiles, partials);
  check_launch("gram_tc");
}

void launch_gram_tc_reduce(const double* partials, int ntiles, int nsplit, int M, const int* d_tile_of, int nTj,
                           double* G, int accumulate, cudaStream_t s) {
  gram_tc_reduce_kernel<<<1024, 256, 0, s>>>(partials, ntiles, nsplit, M, d_tile_of, nTj, G, accumulate);
  check_launch("gram_tc_reduce");
}

}  // namespace fkk
