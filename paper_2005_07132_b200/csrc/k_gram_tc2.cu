// Tile list, split count and fp64 split reduction of the CTA-PAIR Gram (256 x 256 tiles of G over the
// upper triangle of 256-channel blocks), shared by gram_pre2_kernel (k_gram_pre2.cu), the default
// Gram at cfg3.  (This file also held an fp32-A pair kernel fed by register-prefetched global loads:
// parity-green but measured slower than the 1-CTA kernel, 7.9 vs 6.1 ms at cfg3, and reachable only
// through an A/B switch; removed.)
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "fkk_internal.h"

namespace fkk {

namespace {

constexpr int T2 = 256;                     // tile edge

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

void launch_gram_tc2_reduce(const double* partials, int ntiles, int nsplit, int M, const int* d_tile_of, int nT,
                            double* G, int accumulate, cudaStream_t s) {
  gram_tc2_reduce_kernel<<<1024, 256, 0, s>>>(partials, ntiles, nsplit, M, d_tile_of, nT, G, accumulate);
  check_launch("gram_tc2_reduce");
}

}  // namespace fkk
