// Gram matrix G0 = A0^T A0 of the log-ratio matrix (F2; the normal matrix of the truncated SVD,
// PAPER.md:64-70), CUDA-core fp32 variant (FKK_GEMM_FP32_SIMT): 128 x 128 tiles of the upper
// triangle, 8 x 8 register blocks per thread, fp32 accumulation over <= 8192 pixels, then an fp64
// read-modify-write into this CTA's own partial slot (deterministic; summed by gram_reduce).
#include <cuda_runtime.h>

#include <algorithm>

#include "fkk_internal.h"

namespace fkk {

namespace {

constexpr int TB = 128;      // tile edge
constexpr int KC = 16;       // pixels per smem chunk
constexpr int FLUSH = 8192;  // fp32 accumulation span (pixels) before the fp64 flush

__device__ __forceinline__ void tile_coords(int t, int nT, int& ti, int& tj) {
  int r = 0, base = 0;
  while (t >= base + (nT - r)) { base += nT - r; ++r; }
  ti = r;
  tj = r + (t - base);
}

__global__ void __launch_bounds__(256, 2) gram_simt_kernel(const float* __restrict__ A, int64_t n, int M, int nT,
                                                        double* __restrict__ partials, int ntiles) {
  __shared__ __align__(16) float As[KC][TB + 4];
  __shared__ __align__(16) float Bs[KC][TB + 4];
  int ti, tj;
  tile_coords(blockIdx.x, nT, ti, tj);
  const bool diag = ti == tj;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int64_t rb = n * split / nsplit, re = n * (split + 1) / nsplit;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double* part = partials + ((int64_t)split * ntiles + blockIdx.x) * (TB * TB);
  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
  bool first_flush = true;
  int64_t since = 0;
  for (int64_t r0 = rb; r0 < re; r0 += KC) {
    // load KC pixels x 128 channels for column blocks ti and tj
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int idx = tid + h * 256;        // 0..511
      const int row = idx >> 5, c4 = (idx & 31) * 4;
      const int64_t r = r0 + row;
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      if (r < re) {
        const int ca = ti * TB + c4, cb = tj * TB + c4;
        if (ca < M) va = __ldg(reinterpret_cast<const float4*>(A + r * (int64_t)M + ca));
        if (!diag && cb < M) vb = __ldg(reinterpret_cast<const float4*>(A + r * (int64_t)M + cb));
      }
      *reinterpret_cast<float4*>(&As[row][c4]) = va;
      if (!diag) *reinterpret_cast<float4*>(&Bs[row][c4]) = vb;
    }
    __syncthreads();
    const float(*Bp)[TB + 4] = diag ? As : Bs;
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      float a[8], b[8];
      *reinterpret_cast<float4*>(&a[0]) = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      *reinterpret_cast<float4*>(&a[4]) = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      *reinterpret_cast<float4*>(&b[0]) = *reinterpret_cast<const float4*>(&Bp[kk][tx * 8]);
      *reinterpret_cast<float4*>(&b[4]) = *reinterpret_cast<const float4*>(&Bp[kk][tx * 8 + 4]);
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y] = fmaf(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
    since += KC;
    if (since >= FLUSH || r0 + KC >= re) {
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          double* d = part + (ty * 8 + x) * TB + tx * 8 + y;
          *d = (first_flush ? 0.0 : *d) + (double)acc[x][y];
          acc[x][y] = 0.f;
        }
      first_flush = false;
      since = 0;
    }
  }
  if (first_flush) {   // empty row range: still define the slot
    for (int x = 0; x < 8; ++x)
      for (int y = 0; y < 8; ++y) part[(ty * 8 + x) * TB + tx * 8 + y] = 0.0;
  }
}

__global__ void gram_reduce_kernel(const double* __restrict__ partials, int nsplit, int ntiles, int nT, int M,
                                   double* __restrict__ G, int accumulate) {
  const int64_t total = (int64_t)M * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e / M), j = (int)(e % M);
    int a = min(i, j), b = max(i, j);
    const int ti = a / TB, tj = b / TB;
    // index of tile (ti, tj) in the row-major upper-triangle enumeration
    const int t = ti * nT - ti * (ti - 1) / 2 + (tj - ti);
    const int li = a - ti * TB, lj = b - tj * TB;
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += partials[((int64_t)sp * ntiles + t) * (TB * TB) + li * TB + lj];
    G[e] = accumulate ? G[e] + s : s;
  }
}

}  // namespace

int gram_num_tiles(int M) {
  const int nT = (M + TB - 1) / TB;
  return nT * (nT + 1) / 2;
}

int gram_num_splits(int64_t n, int M) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntiles = gram_num_tiles(M);
  int64_t ns = (2LL * sms + ntiles - 1) / ntiles;
  const int64_t max_by_rows = std::max<int64_t>(1, n / 256);
  ns = std::max<int64_t>(1, std::min(ns, max_by_rows));
  return (int)ns;
}

void launch_gram_simt(const float* A, int64_t n, int M, double* partials, int nsplit, cudaStream_t s) {
  const int nT = (M + TB - 1) / TB;
  const int ntiles = nT * (nT + 1) / 2;
  dim3 grid(ntiles, nsplit);
  gram_simt_kernel<<<grid, 256, 0, s>>>(A, n, M, nT, partials, ntiles);
  check_launch("gram_simt");
}

void launch_gram_reduce(const double* partials, int nsplit, int M, double* G, int accumulate, cudaStream_t s) {
  const int nT = (M + TB - 1) / TB;
  gram_reduce_kernel<<<1024, 256, 0, s>>>(partials, nsplit, nT * (nT + 1) / 2, nT, M, G, accumulate);
  check_launch("gram_reduce");
}

}  // namespace fkk
