// Randomized range finder ("random sampling ('randomized') SVD ...
// [Halko 2011]"): the pieces of F2-F4 that are specific to it.  The heavy passes reuse the hot kernels:
//   Y = A W          : the TMA projection (raw cube -> A0 in its converter warps), W = Omega or orth(Z);
//   A^T Y and Y^T Y  : the image Gram kernel (gram_pre) on tiles (A0 block cb, Y block) and (Y, Y), Y
//                      written as one extra 128-"channel" block of the pre-split tf32 hi/lo image;
//   orth(.)          : CholQR (gram_rows / chol_inv / apply_rinv of the eigensolver);
//   the l x l eig    : the GPU eigensolver.
// Here: the test matrix (SplitMix64 + Box-Muller, the same counter-based generator as the oracle's
// range_finder_omega), the reduction of the tile partials into A^T Y (with D_f) and Y^T Y, and the
// final V = Z_q U_k diag(1/sigma) with the sign rule.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fkk_internal.h"

namespace fkk {

namespace {

constexpr int GT = 128;   // image block / Gram tile edge

inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Zraw[c][j] = f_j sum_splits P[(sp nt + j / GT)][c][j % GT]   (c < l, j < M): (A^T Y)^T with A = A0 D_f
// SY[c1][c2] = sum_splits P[(sp nt + nT)][c1][c2]               (Y^T Y)
__global__ void rf_reduce_kernel(const double* __restrict__ P, int nT, int nsplit, int M, int l,
                                 const double* __restrict__ f, double* __restrict__ Zraw, double* __restrict__ SY) {
  const int nt = nT + 1;
  const int64_t nz = (int64_t)l * M, total = nz + (int64_t)l * l;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (e < nz) {
      const int c = (int)(e / M), j = (int)(e % M);
      const int cb = j / GT, i = j % GT;
      for (int sp = 0; sp < nsplit; ++sp) acc += P[((int64_t)sp * nt + cb) * (GT * GT) + (int64_t)c * GT + i];
      Zraw[e] = acc * f[j];
    } else {
      const int64_t r = e - nz;
      const int c1 = (int)(r / l), c2 = (int)(r % l);
      for (int sp = 0; sp < nsplit; ++sp) acc += P[((int64_t)sp * nt + nT) * (GT * GT) + (int64_t)c1 * GT + c2];
      SY[r] = acc;
    }
  }
}

// V[c][j] = sum_b Zq[b][j] U[c][b] / sqrt(lam_c), then the sign rule (largest |entry| positive, ties ->
// lowest index; as oracle/eig_topk): one CTA per vector
__global__ void __launch_bounds__(256) rf_combine_kernel(const double* __restrict__ Zq, int M, int l,
                                                         const double* __restrict__ U, const double* __restrict__ lam,
                                                         double* __restrict__ V) {
  __shared__ double red_v[256];
  __shared__ int red_i[256];
  const int c = blockIdx.x, tid = threadIdx.x;
  const double inv = lam[c] > 0.0 ? 1.0 / sqrt(lam[c]) : 0.0;
  double* v = V + (int64_t)c * M;
  double best = -1.0;
  int bi = M;
  for (int j = tid; j < M; j += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < l; ++b) acc = fma(Zq[(int64_t)b * M + j], U[(int64_t)c * l + b], acc);
    acc *= inv;
    v[j] = acc;
    if (fabs(acc) > best) { best = fabs(acc); bi = j; }
  }
  red_v[tid] = best;
  red_i[tid] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (tid < o) {
      const double a = red_v[tid], b2 = red_v[tid + o];
      const int ia = red_i[tid], ib = red_i[tid + o];
      if (b2 > a || (b2 == a && ib < ia)) { red_v[tid] = b2; red_i[tid] = ib; }
    }
    __syncthreads();
  }
  const bool flip = red_i[0] < M && v[red_i[0]] < 0.0;
  __syncthreads();
  if (flip)
    for (int j = tid; j < M; j += blockDim.x) v[j] = -v[j];
}

}  // namespace

// Omega (stored l x M: vector i contiguous) = the oracle's range_finder_omega(seed, M, l) transposed:
// entry (j, i) from counter c = seed 2^40 + j l + i, u1 = ((h(2c) >> 11) + 1) / 2^53,
// u2 = (h(2c+1) >> 11) / 2^53, sqrt(-2 ln u1) cos(2 pi u2)
void rf_omega_host(uint64_t seed, int M, int l, double* omega_lxM) {
  const double two53 = 9007199254740992.0;
  for (int j = 0; j < M; ++j)
    for (int i = 0; i < l; ++i) {
      const uint64_t c = seed * (1ull << 40) + (uint64_t)j * (uint64_t)l + (uint64_t)i;
      const double u1 = ((double)(splitmix64(2 * c) >> 11) + 1.0) / two53;
      const double u2 = (double)(splitmix64(2 * c + 1) >> 11) / two53;
      omega_lxM[(size_t)i * M + j] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
}

void launch_rf_reduce(const double* partials, int nT, int nsplit, int M, int l, const double* f, double* Zraw,
                      double* SY, cudaStream_t s) {
  rf_reduce_kernel<<<512, 256, 0, s>>>(partials, nT, nsplit, M, l, f, Zraw, SY);
  check_launch("rf_reduce");
}

void launch_rf_combine(const double* Zq, int M, int l, const double* U, const double* lam, int k, double* V,
                       cudaStream_t s) {
  rf_combine_kernel<<<k, 256, 0, s>>>(Zq, M, l, U, lam, V);
  check_launch("rf_combine");
}

}  // namespace fkk

extern "C" {
// Host helper (test hook): the range finder's test matrix Omega, M x l row-major (as the oracle).
int32_t fkk_range_finder_omega(uint64_t seed, int32_t M, int32_t l, double* out_Mxl) {
  if (!out_Mxl || M < 1 || l < 1) return 1;
  std::vector<double> t((size_t)M * l);
  fkk::rf_omega_host(seed, M, l, t.data());
  for (int j = 0; j < M; ++j)
    for (int i = 0; i < l; ++i) out_Mxl[(size_t)j * l + i] = t[(size_t)i * M + j];
  return 0;
}
}
