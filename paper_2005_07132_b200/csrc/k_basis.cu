// Basis-level steps F6..F10 of fKK-EC, all fp64 (k <= 128 rows of length M; latency-bound, tiny):
//   hilbert_rows : H{.} row-wise (Eq. 11 H{V^T/f}, Eq. 18 H{Phi_PEC}), fp64 FFT in smem
//   sg_rows      : trendline M{.} row-wise (Eq. 22), fp64 moment prefix sums
//   dgemm_small  : P = X H{V^T/f} (Eq. 16), X^T X and X^T Phi_err (Eq. 17)
//   ridge        : Phi_PEC^T = (X^T X + lam I)^{-1} X^T Phi_err, lam = ridge_rel lambda_max(X^T X)
//                  (Eq. 17, reading A11); lambda_max by normalised repeated squaring, Cholesky solve
//   assemble_B   : B_amp = V^T/f + H{Phi_PEC} - V_SEC^T, B_ph = H{V^T/f} - Phi_PEC^T (Eq. 23)
#include <cuda_runtime.h>
#include <math.h>

#include "device_common.cuh"
#include <algorithm>

#include "fkk_internal.h"

namespace fkk {

namespace {

__global__ void __launch_bounds__(256) hilbert_rows_f64_kernel(const double* __restrict__ X, int rows, int M, int ldx,
                                                               double* __restrict__ out, int L, int log2L,
                                                               int pad_zero, const double2* __restrict__ tw_g) {
  extern __shared__ __align__(16) unsigned char smem[];
  cplx<double>* tw = reinterpret_cast<cplx<double>*>(smem);
  cplx<double>* x = tw + (L >> 1);
  for (int j = threadIdx.x; j < (L >> 1); j += blockDim.x) { double2 t = tw_g[j]; tw[j].x = t.x; tw[j].y = t.y; }
  const int r0 = 2 * blockIdx.x, r1 = r0 + 1;
  const double* x0 = X + (int64_t)r0 * ldx;
  const double* x1 = (r1 < rows) ? X + (int64_t)r1 * ldx : x0;
  __syncthreads();
  pad_pair<double, double>(x, x0, x1, M, L, pad_zero);
  hilbert_pair_inplace<double>(x, tw, L, log2L);
  const int pl = (L - M) >> 1;
  const double invL = 1.0 / (double)L;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    out[(int64_t)r0 * M + j] = x[pl + j].x * invL;
    if (r1 < rows) out[(int64_t)r1 * M + j] = x[pl + j].y * invL;
  }
}

__global__ void __launch_bounds__(256) sg_rows_f64_kernel(const double* __restrict__ X, int M, int h,
                                                          double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* P0 = reinterpret_cast<double*>(smem);
  double* P1 = P0 + (M + 1);
  double* P2 = P1 + (M + 1);
  double* wsum = P2 + (M + 1);
  const double* y = X + (int64_t)blockIdx.x * M;
  block_prefix3(y, M, P0, P1, P2, wsum);
  for (int j = threadIdx.x; j < M; j += blockDim.x) out[(int64_t)blockIdx.x * M + j] = sg_point(P0, P1, P2, M, h, j);
}

__global__ void dgemm_small_kernel(int m, int n, int kk, const double* __restrict__ A, int lda, int ta,
                                   const double* __restrict__ B, int ldb, int tb, double* __restrict__ C, int ldc,
                                   double beta) {
  const int64_t total = (int64_t)m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    double s = 0.0;
    for (int t = 0; t < kk; ++t) {
      const double a = ta ? A[(int64_t)t * lda + i] : A[(int64_t)i * lda + t];
      const double b = tb ? B[(int64_t)j * ldb + t] : B[(int64_t)t * ldb + j];
      s = fma(a, b, s);
    }
    C[(int64_t)i * ldc + j] = (beta == 0.0 ? 0.0 : beta * C[(int64_t)i * ldc + j]) + s;
  }
}

// Single CTA: lambda_max(C) by normalised repeated squaring, then the Cholesky factor of C + lam I
// in Lw (lower, row-major k x k).  The squarings run in shared memory when 2 k^2 doubles fit
// (k <= 80), else in the global work buffers.  24 squarings: the final term log lambda_max(B_T) is
// bracketed within log(k) and weighted 2^-24, i.e. lambda_max to ~3e-7 relative -- far below
// anything the ridge weight (reading A11) is sensitive to.
constexpr int kRidgeSquarings = 24;

// lambda_max estimate of the fPEC ridge (squarings, see ridge_factor_kernel) on ONE cluster of CL CTAs:
// every CTA keeps B in shared memory, computes its block of rows of B^2 and pushes it (and its partial
// trace) into the other CTAs' shared memory (st.shared::cluster), one cluster barrier per squaring.  The
// single-CTA version is FP64-throughput bound on one SM (24 x k^3 FMAs).  Same arithmetic, the traces
// summed in a different order.
template <int CL>
__global__ void __launch_bounds__(256) ridge_lmax_kernel(const double* __restrict__ C, int k, double ridge_rel,
                                                         double* __restrict__ lam_out) {
  extern __shared__ __align__(16) double lm[];
  double* B0 = lm;                    // k x k
  double* B1 = lm + k * k;            // [2][k x k] (parity: a peer's next push never hits a buffer still read)
  double* trp = B1 + 2 * k * k;       // [2][CL] partial traces
  __shared__ double red[8];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int kk = k * k, rb = (k + CL - 1) / CL, r0 = min(k, (int)rank * rb), r1 = min(k, r0 + rb);
  double t = 0.0;
  for (int i = lane; i < k; i += 32) t += C[i * k + i];
  t = warp_sum(t);                    // every warp holds the full trace
  const double tr = t;
  double loglam = log(tr > 0 ? tr : 1e-300);
  for (int e = tid; e < kk; e += nt) B0[e] = C[e] / tr;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  double wgt = 0.5;
  for (int it = 0; it < kRidgeSquarings; ++it) {
    double* B1p = B1 + (it & 1) * kk;
    double* trq = trp + (it & 1) * CL;
    double tl = 0.0;
    for (int e = tid; e < (r1 - r0) * k; e += nt) {
      const int i = r0 + e / k, j = e - (e / k) * k;
      double s0 = 0.0, s1 = 0.0;
      int q = 0;
      for (; q + 1 < k; q += 2) {
        s0 = fma(B0[i * k + q], B0[q * k + j], s0);
        s1 = fma(B0[i * k + q + 1], B0[(q + 1) * k + j], s1);
      }
      if (q < k) s0 = fma(B0[i * k + q], B0[q * k + j], s0);
      const double v = s0 + s1;
      if (i == j) tl += v;
      // own copy + every peer's copy of this entry
#pragma unroll
      for (int d = 0; d < CL; ++d) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((uint32_t)__cvta_generic_to_shared(B1p + i * k + j)), "r"(d));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
      }
    }
    tl = warp_sum(tl);
    if (lane == 0) red[wid] = tl;
    __syncthreads();
    if (tid < CL) {
      double ps = 0.0;
      for (int w2 = 0; w2 < nt / 32; ++w2) ps += red[w2];
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((uint32_t)__cvta_generic_to_shared(trq + rank)), "r"(tid));
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(ps) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    double c = 0.0;
    for (int d = 0; d < CL; ++d) c += trq[d];
    c = c > 0 ? c : 1e-300;
    loglam += wgt * log(c);
    wgt *= 0.5;
    for (int e = tid; e < kk; e += nt) B0[e] = B1p[e] / c;
    __syncthreads();
  }
  double fr = 0.0;
  for (int e = tid; e < kk; e += nt) fr += B0[e] * B0[e];
  fr = warp_sum(fr);
  if (lane == 0) red[wid] = fr;
  __syncthreads();
  if (tid == 0 && rank == 0) {
    double sfr = 0;
    for (int w2 = 0; w2 < nt / 32; ++w2) sfr += red[w2];
    const double lmax = exp(loglam + 2.0 * wgt * log(sqrt(sfr > 0 ? sfr : 1e-300)));
    lam_out[0] = ridge_rel * lmax;
  }
  // no CTA leaves while a peer may still push into it (the last pushes precede the last barrier)
}

template <bool SMEM>   // SMEM: the k x k work matrices in shared memory (typed shared pointers: LDS, not generic loads)
__global__ void __launch_bounds__(1024) ridge_factor_kernel(const double* __restrict__ C, int k, double ridge_rel,
                                                            double* __restrict__ Lw, double* __restrict__ work,
                                                            double* __restrict__ lam_out, int* __restrict__ flags,
                                                            int have_lam) {
  extern __shared__ __align__(16) double shm[];
  __shared__ double red[32];
  __shared__ double sh_scal[2];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int kk = k * k;
  constexpr bool in_smem = SMEM;
  double* B0 = SMEM ? shm : work;
  double* B1 = SMEM ? shm + kk : work + kk;
  if (!have_lam) {
  // trace
  double t = 0.0;
  for (int i = tid; i < k; i += nt) t += C[i * k + i];
  t = warp_sum(t);
  if (lane == 0) red[wid] = t;
  __syncthreads();
  if (tid == 0) { double s = 0; for (int w2 = 0; w2 < nt / 32; ++w2) s += red[w2]; sh_scal[0] = s; }
  __syncthreads();
  const double tr = sh_scal[0];
  double loglam = log(tr > 0 ? tr : 1e-300);
  for (int e = tid; e < kk; e += nt) B0[e] = C[e] / tr;
  __syncthreads();
  double wgt = 0.5;
  const int kh = (k + 1) >> 1;   // 2 x 2 output blocks: four independent accumulator chains per thread
  for (int it = 0; it < kRidgeSquarings; ++it) {
    for (int e = tid; e < kh * kh; e += nt) {
      const int i = 2 * (e / kh), j = 2 * (e % kh);
      const bool i1 = i + 1 < k, j1 = j + 1 < k;
      double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
      for (int q = 0; q < k; ++q) {
        const double a0 = B0[i * k + q], a1 = i1 ? B0[(i + 1) * k + q] : 0.0;
        const double b0 = B0[q * k + j], b1 = j1 ? B0[q * k + j + 1] : 0.0;
        s00 = fma(a0, b0, s00);
        s01 = fma(a0, b1, s01);
        s10 = fma(a1, b0, s10);
        s11 = fma(a1, b1, s11);
      }
      B1[i * k + j] = s00;
      if (j1) B1[i * k + j + 1] = s01;
      if (i1) B1[(i + 1) * k + j] = s10;
      if (i1 && j1) B1[(i + 1) * k + j + 1] = s11;
    }
    __syncthreads();
    double tl = 0.0;
    for (int i = tid; i < k; i += nt) tl += B1[i * k + i];
    tl = warp_sum(tl);
    if (lane == 0) red[wid] = tl;
    __syncthreads();
    if (tid == 0) { double s = 0; for (int w2 = 0; w2 < nt / 32; ++w2) s += red[w2]; sh_scal[1] = s; }
    __syncthreads();
    const double c = sh_scal[1] > 0 ? sh_scal[1] : 1e-300;
    loglam += wgt * log(c);
    wgt *= 0.5;
    for (int e = tid; e < kk; e += nt) B0[e] = B1[e] / c;
    __syncthreads();
  }
  // lambda_max(B_T) ~ ||B_T||_F (between lambda_max and sqrt(rank) lambda_max); weight 2^-T
  double fr = 0.0;
  for (int e = tid; e < kk; e += nt) fr += B0[e] * B0[e];
  fr = warp_sum(fr);
  if (lane == 0) red[wid] = fr;
  __syncthreads();
  if (tid == 0) {
    double s = 0; for (int w2 = 0; w2 < nt / 32; ++w2) s += red[w2];
    const double lmax = exp(loglam + 2.0 * wgt * log(sqrt(s > 0 ? s : 1e-300)));
    sh_scal[0] = ridge_rel * lmax;
    lam_out[0] = sh_scal[0];
  }
  __syncthreads();
  } else {
    if (tid == 0) sh_scal[0] = lam_out[0];
    __syncthreads();
  }
  const double lam = sh_scal[0];
  double* L = in_smem ? shm : Lw;   // factor in smem when it fits, copied out at the end
  for (int e = tid; e < kk; e += nt) { const int i = e / k, j = e % k; L[e] = (j <= i) ? C[e] + (i == j ? lam : 0.0) : 0.0; }
  __syncthreads();
  // right-looking Cholesky, lower triangle, one barrier per column: every thread reads the pivot,
  // column j of L is written from the (not yet scaled) column, and the trailing update uses the
  // unscaled column over the pivot (column j is only read in this phase)
  for (int j = 0; j < k; ++j) {
    const double d = L[j * k + j];
    const bool ok = d > 0.0;
    const double ljj = ok ? sqrt(d) : 1e-300, il = ok ? 1.0 / ljj : 0.0, id = ok ? 1.0 / d : 0.0;
    if (tid == 0 && !ok) atomicOr(flags, 4);
    const int rem = k - j - 1;
    // trailing update L[i][c] -= L[i][j] L[c][j] / d for j < c <= i (2-D: rows by tid / 32, cols by lane)
    for (int i = j + 1 + (tid >> 5); i < k; i += nt >> 5) {
      const double lij = L[i * k + j] * id;
      for (int c = j + 1 + lane; c <= i; c += 32) L[i * k + c] -= lij * L[c * k + j];
    }
    (void)rem;
    __syncthreads();
    for (int i = j + tid; i < k; i += nt) L[i * k + j] = i == j ? ljj : L[i * k + j] * il;
    // (column j is written after the barrier above and read by no later phase before the next barrier
    //  except as L[c][j'] with j' > j)
  }
  __syncthreads();
  if (in_smem)
    for (int e = tid; e < kk; e += nt) Lw[e] = L[e];
}

// ncol independent right-hand sides, one per thread; L and the thread block's columns in shared
// memory ([k][blockDim] layout: a warp's accesses are consecutive), reciprocal diagonal precomputed
__global__ void ridge_solve_kernel(const double* __restrict__ Lw, int k, const double* __restrict__ R, int ncol,
                                   double* __restrict__ Phi) {
  extern __shared__ __align__(16) double rs[];
  double* Ls = rs;               // k x k
  double* rd = Ls + k * k;       // k
  double* X = rd + k;            // [k][nt]
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < k * k; e += nt) Ls[e] = Lw[e];
  __syncthreads();
  for (int i = tid; i < k; i += nt) rd[i] = 1.0 / Ls[i * k + i];
  const int j = blockIdx.x * nt + tid;
  const bool act = j < ncol;
  for (int i = 0; i < k; ++i) X[i * nt + tid] = act ? R[(int64_t)i * ncol + j] : 0.0;
  __syncthreads();
  // forward L y = r (two partial sums per row: half the dependent chain)
  for (int i = 0; i < k; ++i) {
    double s0 = X[i * nt + tid], s1 = 0.0;
    int q = 0;
    for (; q + 1 < i; q += 2) {
      s0 = fma(-Ls[i * k + q], X[q * nt + tid], s0);
      s1 = fma(-Ls[i * k + q + 1], X[(q + 1) * nt + tid], s1);
    }
    if (q < i) s0 = fma(-Ls[i * k + q], X[q * nt + tid], s0);
    X[i * nt + tid] = (s0 + s1) * rd[i];
  }
  // backward L^T x = y
  for (int i = k - 1; i >= 0; --i) {
    double s0 = X[i * nt + tid], s1 = 0.0;
    int q = i + 1;
    for (; q + 1 < k; q += 2) {
      s0 = fma(-Ls[q * k + i], X[q * nt + tid], s0);
      s1 = fma(-Ls[(q + 1) * k + i], X[(q + 1) * nt + tid], s1);
    }
    if (q < k) s0 = fma(-Ls[q * k + i], X[q * nt + tid], s0);
    X[i * nt + tid] = (s0 + s1) * rd[i];
  }
  if (act)
    for (int i = 0; i < k; ++i) Phi[(int64_t)i * ncol + j] = X[i * nt + tid];
}

__global__ void assemble_B_kernel(const double* Vt_f, const double* HPhi, const double* Vsec, const double* Hv,
                                  const double* Phi, int k, int M, float* Bi) {
  const int64_t total = (int64_t)k * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    Bi[2 * e] = (float)(Vt_f[e] + HPhi[e] - Vsec[e]);
    Bi[2 * e + 1] = (float)(Hv[e] - Phi[e]);
  }
}

__global__ void vt_over_f_kernel(const double* V, const double* f, int M, int k, double* Vt_f) {
  const int64_t total = (int64_t)k * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % M);
    Vt_f[e] = V[e] / f[j];
  }
}

inline int ilog2(int L) { int r = 0; while ((1 << r) < L) ++r; return r; }

}  // namespace

void launch_hilbert_rows_f64(const double* X, int rows, int M, int ldx, double* out, int L, int pad_zero,
                             const double2* tw, cudaStream_t s) {
  if (rows <= 0) return;
  const size_t smem = (size_t)(L / 2 + L) * sizeof(double2);
  cudaFuncSetAttribute(hilbert_rows_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  hilbert_rows_f64_kernel<<<(rows + 1) / 2, 256, smem, s>>>(X, rows, M, ldx, out, L, ilog2(L), pad_zero, tw);
  check_launch("hilbert_rows_f64");
}

void launch_sg_rows_f64(const double* X, int rows, int M, int h, double* out, cudaStream_t s) {
  if (rows <= 0) return;
  const size_t smem = (size_t)(3 * (M + 1) + 96) * sizeof(double);
  cudaFuncSetAttribute(sg_rows_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  sg_rows_f64_kernel<<<rows, 256, smem, s>>>(X, M, h, out);
  check_launch("sg_rows_f64");
}

void launch_dgemm_small(int m, int n, int kk, const double* A, int lda, int ta, const double* B, int ldb, int tb,
                        double* C, int ldc, double beta, cudaStream_t s) {
  if (m <= 0 || n <= 0) return;
  const int64_t total = (int64_t)m * n;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 4096);
  dgemm_small_kernel<<<grid, 256, 0, s>>>(m, n, kk, A, lda, ta, B, ldb, tb, C, ldc, beta);
  check_launch("dgemm_small");
}

void launch_ridge(const double* C, int k, const double* R, int ncol, double ridge_rel, double* Phi, double* lam_out,
                  double* work, int* flags, cudaStream_t s) {
  double* Lw = work;
  // squarings and factor in shared memory up to 200 KB (k <= 114; k = 100 ran them in global memory: 1.5 ms)
  const size_t sm = (size_t)2 * k * k * sizeof(double) <= 200 * 1024 ? (size_t)2 * k * k * sizeof(double) : 0;
  int have_lam = 0;
  constexpr int CL = 8;
  const size_t lsm = (3 * (size_t)k * k + 2 * CL) * sizeof(double);
  if (k >= CL && lsm <= 200 * 1024) {
    FKK_CUDA_CHECK(cudaFuncSetAttribute(ridge_lmax_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = lsm;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FKK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, ridge_lmax_kernel<CL>, C, k, ridge_rel, lam_out));
    have_lam = 1;
  }
  if (sm) {
    cudaFuncSetAttribute(ridge_factor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    ridge_factor_kernel<true><<<1, 1024, sm, s>>>(C, k, ridge_rel, Lw, work + (int64_t)k * k, lam_out, flags, have_lam);
  } else {
    ridge_factor_kernel<false><<<1, 1024, 0, s>>>(C, k, ridge_rel, Lw, work + (int64_t)k * k, lam_out, flags, have_lam);
  }
  check_launch("ridge_factor");
  const int nts = 32;   // 32 columns per CTA: ncol / 32 CTAs spread over the SMs
  const size_t ssm = ((size_t)k * k + k + (size_t)k * nts) * sizeof(double);
  FKK_CUDA_CHECK(cudaFuncSetAttribute(ridge_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
  ridge_solve_kernel<<<(ncol + nts - 1) / nts, nts, ssm, s>>>(Lw, k, R, ncol, Phi);
  check_launch("ridge_solve");
}

void launch_assemble_B(const double* Vt_f, const double* HPhi, const double* Vsec, const double* Hv,
                       const double* Phi_pec, int k, int M, float* Bi, cudaStream_t s) {
  assemble_B_kernel<<<256, 256, 0, s>>>(Vt_f, HPhi, Vsec, Hv, Phi_pec, k, M, Bi);
  check_launch("assemble_B");
}

void launch_vt_over_f(const double* V, const double* f, int M, int k, double* Vt_f, cudaStream_t s) {
  vt_over_f_kernel<<<256, 256, 0, s>>>(V, f, M, k, Vt_f);
  check_launch("vt_over_f");
}

}  // namespace fkk
