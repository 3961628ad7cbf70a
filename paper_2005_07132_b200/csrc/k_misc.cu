// Small streaming / bookkeeping kernels of the factorized path:
//   prep_ref   : reference checks and reciprocals (Eq. 3 needs I_ref > 0)
//   logratio   : A0 = 1/2 ln(max(I/I_ref, floor)) (Eq. 6), float4 streaming, fp32 out
//   colsum     : <I>(omega) for f(omega) of Eq. 9
//   scale_gram : G = D_f G0 D_f (Eq. 10 applied to the Gram: A = A0 D_f)
//   cast_w     : W (M x kp fp32, row-major) = D_f V diag(c) for the projection GEMM
//   gather     : X = US[q, :] (Eq. 15), fp64
//   extremes   : merge per-block column (max, argmax, min, argmin), ties -> lowest index (A12)
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "fkk_internal.h"

namespace fkk {

thread_local int64_t g_launches = 0;

namespace {

__global__ void prep_ref_kernel(const void* iref, int in_f64, int M, float* inv_ref, double* ref64, int* flags) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < M; j += gridDim.x * blockDim.x) {
    double r = in_f64 ? reinterpret_cast<const double*>(iref)[j] : (double)reinterpret_cast<const float*>(iref)[j];
    if (!(r > 0.0) || !isfinite(r)) { atomicOr(flags, 1); r = 1.0; }
    ref64[j] = r;
    inv_ref[j] = (float)(1.0 / r);
  }
}

template <typename TIn>
__global__ void logratio_kernel(const TIn* __restrict__ I, int64_t n, int M, const float* __restrict__ inv_ref,
                                const double* __restrict__ ref64, float floor, float* __restrict__ A,
                                int* __restrict__ flags) {
  const int64_t total4 = n * (int64_t)M / 4;   // M % 4 == 0
  const int M4 = M / 4;
  int bad = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total4; e += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(e % M4) * 4;
    float4 o;
    if constexpr (sizeof(TIn) == 8) {
      const double2* p = reinterpret_cast<const double2*>(I) + 2 * e;
      double2 u = p[0], v = p[1];
      double vals[4] = {u.x, u.y, v.x, v.y};
      float r[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        bad |= !isfinite(vals[t]);
        r[t] = (float)(0.5 * log(fmax(vals[t] / ref64[c4 + t], (double)floor)));
      }
      o = make_float4(r[0], r[1], r[2], r[3]);
    } else {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(I) + e);
      const float4 ir = *reinterpret_cast<const float4*>(inv_ref + c4);
      bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
      o.x = 0.5f * logf(fmaxf(v.x * ir.x, floor));
      o.y = 0.5f * logf(fmaxf(v.y * ir.y, floor));
      o.z = 0.5f * logf(fmaxf(v.z * ir.z, floor));
      o.w = 0.5f * logf(fmaxf(v.w * ir.w, floor));
    }
    reinterpret_cast<float4*>(A)[e] = o;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, 2);
}

template <typename TIn>
__global__ void colsum_kernel(const TIn* __restrict__ I, int64_t n, int M, double* __restrict__ colsum) {
  // grid.x tiles columns by blockDim.x, grid.y splits rows; atomics in fp64 (Eq. 9 option only)
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const int64_t r0 = n * blockIdx.y / gridDim.y, r1 = n * (blockIdx.y + 1) / gridDim.y;
  double s = 0.0;
  for (int64_t r = r0; r < r1; ++r) s += (double)I[r * (int64_t)M + j];
  atomicAdd(colsum + j, s);
}

__global__ void noise_scale_kernel(const double* colsum, int M, double inv_n, double alpha, double sg, double* f64,
                                   float* f32) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const double m = colsum[j] * inv_n;
  const double f = 2.0 * m / sqrt(alpha * m + sg * sg);
  f64[j] = f;
  f32[j] = (float)f;
}

__global__ void fill_kernel(double* p, double v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void fill_f_kernel(float* p, float v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void scale_gram_kernel(double* G, const double* f, int M) {
  const int64_t total = (int64_t)M * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / M), j = (int)(e % M);
    G[e] *= f[i] * f[j];
  }
}

__global__ void cast_w_kernel(const double* V, const double* fscale, const double* cscale, int M, int k, int kp,
                              float* W) {
  const int64_t total = (int64_t)M * kp;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / kp), c = (int)(e % kp);
    double v = 0.0;
    if (c < k) {
      v = V[(int64_t)c * M + j];
      if (fscale) v *= fscale[j];
      if (cscale) v *= cscale[c];
    }
    W[e] = (float)v;
  }
}

__global__ void gather_kernel(const float* US, int k, int ldus, const int64_t* q, int nq, double* X) {
  const int r = blockIdx.x;
  if (r >= nq) return;
  const int64_t row = q[r];
  for (int c = threadIdx.x; c < k; c += blockDim.x) X[(int64_t)r * k + c] = row >= 0 ? (double)US[row * ldus + c] : 0.0;
}

__global__ void extremes_reduce_kernel(const float* val, const int64_t* idx, int nblk, int k, float* oval,
                                       int64_t* oidx) {
  // one block per column c; val/idx layout [blk][c][2] (0 = max, 1 = min)
  const int c = blockIdx.x;
  __shared__ float sv[2][256];
  __shared__ int64_t si[2][256];
  float bmax = -INFINITY, bmin = INFINITY;
  int64_t imax = INT64_MAX, imin = INT64_MAX;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    const int64_t o = ((int64_t)b * k + c) * 2;
    const float vM = val[o], vm = val[o + 1];
    const int64_t iM = idx[o], im = idx[o + 1];
    if (vM > bmax || (vM == bmax && iM < imax)) { bmax = vM; imax = iM; }
    if (vm < bmin || (vm == bmin && im < imin)) { bmin = vm; imin = im; }
  }
  sv[0][threadIdx.x] = bmax; si[0][threadIdx.x] = imax;
  sv[1][threadIdx.x] = bmin; si[1][threadIdx.x] = imin;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const int o = threadIdx.x + s;
      if (sv[0][o] > sv[0][threadIdx.x] || (sv[0][o] == sv[0][threadIdx.x] && si[0][o] < si[0][threadIdx.x])) {
        sv[0][threadIdx.x] = sv[0][o]; si[0][threadIdx.x] = si[0][o];
      }
      if (sv[1][o] < sv[1][threadIdx.x] || (sv[1][o] == sv[1][threadIdx.x] && si[1][o] < si[1][threadIdx.x])) {
        sv[1][threadIdx.x] = sv[1][o]; si[1][threadIdx.x] = si[1][o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    oval[c * 2] = sv[0][0]; oidx[c * 2] = si[0][0];
    oval[c * 2 + 1] = sv[1][0]; oidx[c * 2 + 1] = si[1][0];
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

void launch_prep_ref(const void* d_iref, int in_f64, int M, float* inv_ref, double* ref64, int* flags, cudaStream_t s) {
  prep_ref_kernel<<<(M + 255) / 256, 256, 0, s>>>(d_iref, in_f64, M, inv_ref, ref64, flags);
  check_launch("prep_ref");
}

void launch_logratio(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                     float floor, float* A, int* flags, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t total4 = n * (int64_t)M / 4;
  int64_t grid = (total4 + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (grid > cap) grid = cap;
  if (in_f64)
    logratio_kernel<double><<<(int)grid, 256, 0, s>>>((const double*)I, n, M, inv_ref, ref64, floor, A, flags);
  else
    logratio_kernel<float><<<(int)grid, 256, 0, s>>>((const float*)I, n, M, inv_ref, ref64, floor, A, flags);
  check_launch("logratio");
}

void launch_colsum(const void* I, int in_f64, int64_t n, int M, double* colsum, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid((M + 127) / 128, (unsigned)std::min<int64_t>(n, 512));
  if (in_f64) colsum_kernel<double><<<grid, 128, 0, s>>>((const double*)I, n, M, colsum);
  else colsum_kernel<float><<<grid, 128, 0, s>>>((const float*)I, n, M, colsum);
  check_launch("colsum");
}

void launch_noise_scale_from_sums(const double* colsum, int M, double inv_n, double alpha, double sg, double* f64,
                                  float* f32, cudaStream_t s) {
  noise_scale_kernel<<<(M + 255) / 256, 256, 0, s>>>(colsum, M, inv_n, alpha, sg, f64, f32);
  check_launch("noise_scale");
}

// B for the linear reconstruction I_k = US . V^T (conventional SVD denoise, reading A26): amp row i =
// column i of V (M x k column-major), phase rows zero
__global__ void bi_linear_kernel(const double* __restrict__ V, int k, int M, float* __restrict__ Bi) {
  const int64_t total = (int64_t)k * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    Bi[2 * e] = (float)V[e];
    Bi[2 * e + 1] = 0.f;
  }
}
void launch_bi_linear(const double* V, int k, int M, float* Bi, cudaStream_t s) {
  bi_linear_kernel<<<256, 256, 0, s>>>(V, k, M, Bi);
  check_launch("bi_linear");
}

void launch_fill(double* p, double v, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  fill_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(p, v, n);
  check_launch("fill");
}
void launch_fill_f(float* p, float v, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  fill_f_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(p, v, n);
  check_launch("fill_f");
}

void launch_scale_gram(double* G, const double* f, int M, cudaStream_t s) {
  scale_gram_kernel<<<512, 256, 0, s>>>(G, f, M);
  check_launch("scale_gram");
}

void launch_cast_w(const double* V, const double* fscale, const double* cscale, int M, int k, int kp, float* W,
                   cudaStream_t s) {
  cast_w_kernel<<<(int)std::min<int64_t>(((int64_t)M * kp + 255) / 256, 2048), 256, 0, s>>>(V, fscale, cscale, M, k, kp, W);
  check_launch("cast_w");
}

void launch_gather_rows(const float* US, int k, int ldus, const int64_t* q_local, int nq, double* X, cudaStream_t s) {
  if (nq <= 0) return;
  gather_kernel<<<nq, 128, 0, s>>>(US, k, ldus, q_local, nq, X);
  check_launch("gather");
}

void launch_extremes_reduce(const float* ext_val, const int64_t* ext_idx, int nblk, int k, float* out_val,
                            int64_t* out_idx, cudaStream_t s) {
  extremes_reduce_kernel<<<k, 256, 0, s>>>(ext_val, ext_idx, nblk, k, out_val, out_idx);
  check_launch("extremes_reduce");
}

}  // namespace fkk

namespace fkk {
namespace {
__global__ void add_f64_kernel(const double* a, const double* b, double* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}
}  // namespace
void launch_add_f64(const double* a, const double* b, double* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  add_f64_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(a, b, out, n);
  check_launch("add_f64");
}
}  // namespace fkk
