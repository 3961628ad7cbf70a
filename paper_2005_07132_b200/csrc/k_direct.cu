// Direct (conventional) per-spectrum KK + PEC + SEC (Eqs. 3-5), K7 in DESIGN.md.
//   direct_phase  : a = 1/2 ln(max(I/I_ref, floor)); phi = H{a}         (D1-D2, fp32 FFT in smem)
//   als_rows      : phi_err = ALS baseline of phi, fp64 banded LDL^T     (D3, reading A6/A7)
//   direct_finish : a' = a + H{phi_err}; phi' = phi - phi_err; K' = e^{a'} e^{i phi'};
//                   T = SG trend(Re K') (fp64 moments; scalar mean if min T <= 0); K = K'/T  (D4-D5)
#include <cuda_runtime.h>
#include <math.h>

#include "device_common.cuh"
#include "fkk_internal.h"

namespace fkk {

namespace {

template <typename TIn>
__device__ __forceinline__ float log_ratio_elem(const TIn v, const float inv_ref, const double ref64, float floor) {
  if constexpr (sizeof(TIn) == 8) {
    double r = (double)v / ref64;
    return (float)(0.5 * log(fmax(r, (double)floor)));
  } else {
    float r = (float)v * inv_ref;
    return 0.5f * __logf(fmaxf(r, floor));   // hardware log (<= 2 ulp; the direct path only)
  }
}

template <typename TIn>
__device__ __forceinline__ bool finite_elem(const TIn v) { return isfinite(v); }

constexpr int kDirectThreads = 256;

// fp64 reciprocal: MUFU seed + two Newton steps (~1 ulp; keeps the IEEE-division slow path off the
// ALS recurrence's critical path)
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <typename TIn, int MAXB>
__global__ void __launch_bounds__(kDirectThreads, 2)
direct_phase_kernel(const TIn* __restrict__ I, int64_t n, int M, const float* __restrict__ inv_ref,
                    const double* __restrict__ ref64, float floor, int L, int log2L, int pad_zero,
                    const float2* __restrict__ tw_g, float* __restrict__ phi, int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char smem[];
  cplx<float>* tw = reinterpret_cast<cplx<float>*>(smem);
  cplx<float>* x = tw + (L >> 1);
  float* a0 = reinterpret_cast<float*>(x + L);
  float* a1 = a0 + M;
  for (int j = threadIdx.x; j < (L >> 1); j += blockDim.x) { float2 t = tw_g[j]; tw[j].x = t.x; tw[j].y = t.y; }
  const int64_t npairs = (n + 1) >> 1;
  const int pl = (L - M) >> 1;
  const float invL = 1.0f / (float)L;
  int bad = 0;
  // f32 rows with M % 4 == 0 (M <= 4 x 4 x blockDim): the next pair's rows are loaded as float4 into
  // registers while this pair's FFTs run (the row loads' latency was the kernel's largest stall)
  constexpr int kPF = 2;   // float4 per thread and row (M <= 2048; larger M takes the scalar loop)
  const bool vec = sizeof(TIn) == 4 && (M & 3) == 0 && M <= 4 * kPF * (int)blockDim.x;
  float4 nx0[kPF], nx1[kPF];
  auto prefetch = [&](int64_t pr) {
#pragma unroll
    for (int u = 0; u < kPF; ++u) { nx0[u] = make_float4(0.f, 0.f, 0.f, 0.f); nx1[u] = nx0[u]; }
    if (pr >= npairs) return;
    const int64_t r0 = 2 * pr, r1 = r0 + 1;
    const float4* p0 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(I) + r0 * (int64_t)M);
    const float4* p1 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(I) + r1 * (int64_t)M);
#pragma unroll
    for (int u = 0; u < kPF; ++u) {
      const int q = threadIdx.x + u * blockDim.x;
      if (4 * q < M) {
        nx0[u] = __ldcs(p0 + q);
        if (r1 < n) nx1[u] = __ldcs(p1 + q);
      }
    }
  };
  if (vec) prefetch(blockIdx.x);
  for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int64_t r0 = 2 * pr, r1 = r0 + 1;
    const TIn* i0 = I + r0 * (int64_t)M;
    const TIn* i1 = I + r1 * (int64_t)M;
    const bool has1 = r1 < n;
    if (vec) {
#pragma unroll
      for (int u = 0; u < kPF; ++u) {
        const int q = threadIdx.x + u * blockDim.x;
        if (4 * q < M) {
          const float4 ir = *reinterpret_cast<const float4*>(inv_ref + 4 * q);
          const float4 v0 = nx0[u], v1 = nx1[u];
          bad |= !isfinite(v0.x) | !isfinite(v0.y) | !isfinite(v0.z) | !isfinite(v0.w);
          a0[4 * q] = 0.5f * __logf(fmaxf(v0.x * ir.x, floor));
          a0[4 * q + 1] = 0.5f * __logf(fmaxf(v0.y * ir.y, floor));
          a0[4 * q + 2] = 0.5f * __logf(fmaxf(v0.z * ir.z, floor));
          a0[4 * q + 3] = 0.5f * __logf(fmaxf(v0.w * ir.w, floor));
          if (has1) {
            bad |= !isfinite(v1.x) | !isfinite(v1.y) | !isfinite(v1.z) | !isfinite(v1.w);
            a1[4 * q] = 0.5f * __logf(fmaxf(v1.x * ir.x, floor));
            a1[4 * q + 1] = 0.5f * __logf(fmaxf(v1.y * ir.y, floor));
            a1[4 * q + 2] = 0.5f * __logf(fmaxf(v1.z * ir.z, floor));
            a1[4 * q + 3] = 0.5f * __logf(fmaxf(v1.w * ir.w, floor));
          } else {
            a1[4 * q] = a1[4 * q + 1] = a1[4 * q + 2] = a1[4 * q + 3] = 0.f;
          }
        }
      }
      prefetch(pr + gridDim.x);
    } else {
      for (int j = threadIdx.x; j < M; j += blockDim.x) {
        TIn v0 = i0[j];
        bad |= !finite_elem(v0);
        a0[j] = log_ratio_elem<TIn>(v0, inv_ref[j], ref64[j], floor);
        if (has1) {
          TIn v1 = i1[j];
          bad |= !finite_elem(v1);
          a1[j] = log_ratio_elem<TIn>(v1, inv_ref[j], ref64[j], floor);
        } else {
          a1[j] = 0.f;
        }
      }
    }
    __syncthreads();
    pad_pair<float, float>(x, a0, a1, M, L, pad_zero);
    hilbert_pair_stockham<float, MAXB>(x, tw, L, log2L);
    float* p0 = phi + r0 * (int64_t)M;
    float* p1 = phi + r1 * (int64_t)M;
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      cplx<float> v = x[pl + j];
      p0[j] = v.x * invL;
      if (has1) p1[j] = v.y * invL;
    }
    __syncthreads();
  }
  if (bad) atomicOr(flags, 2);
}

// ALS (Whittaker smoother with asymmetric weights) on 32 rows per warp (lane = row).  Each sweep
// back-substitutes the previous system (in the order its factorisation left) and, in the same pass,
// factorises the next system in that order (the penalty D^T D is persymmetric, so the reversed
// system has the same band values by position).  Factors (L1, L2, g/D) live in a [row][spectrum]
// fp64 state so that a warp's accesses are coalesced; y and z move through a 32x33 smem tile.
template <typename TY, typename TZ>
__global__ void __launch_bounds__(128, 4)
als_rows_kernel(const TY* __restrict__ y, int64_t n, int M, double lam, double p, int iters,
                double* __restrict__ st, int64_t nb, TZ* __restrict__ z) {
  __shared__ double tile[4][32][33];   // y tile in; in the last sweep overwritten by z (same slot)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = ((int64_t)blockIdx.x * 4 + warp) * 32;
  if (s0 >= n) return;
  const int64_t s = s0 + lane;
  const bool valid = s < n;
  double* L1 = st;
  double* L2 = st + (int64_t)M * nb;
  double* GD = st + 2 * (int64_t)M * nb;
  const int ntile = (M + 31) >> 5;
  const double q = 1.0 - p;
  for (int sw = 0; sw <= iters; ++sw) {
    const bool asc = (sw & 1) == 0;
    const bool do_bsub = sw > 0, do_fact = sw < iters;
    double zp1 = 0.0, zp2 = 0.0;
    double Dm1 = 0.0, Dm2 = 0.0, L1m1 = 0.0, L2m1 = 0.0, L2m2 = 0.0, gm1 = 0.0, gm2 = 0.0;
    // software pipeline: the (L1, L2, g/D) of the next PF rows are loaded PF rows ahead so the
    // dependent fp64 recurrence does not wait on L2/HBM latency every row
    constexpr int PF = 4;
    double nl1[PF], nl2[PF], ngd[PF];
    auto row_of = [&](int t) { return asc ? t : (M - 1 - t); };
    if (do_bsub) {
#pragma unroll
      for (int q2 = 0; q2 < PF; ++q2) {
        const int t = q2;
        if (t < M) {
          const int64_t ix = (int64_t)row_of(t) * nb + s;
          nl1[q2] = L1[ix]; nl2[q2] = L2[ix]; ngd[q2] = GD[ix];
        }
      }
    }
    for (int tt = 0; tt < ntile; ++tt) {
      const int tile_i = asc ? tt : (ntile - 1 - tt);
      const int r0 = tile_i * 32;
      // coalesced load of the 32 spectra x 32 channels tile (row jj = spectrum s0+jj)
      __syncwarp();
      for (int jj = 0; jj < 32; ++jj) {
        const int64_t ss = s0 + jj;
        const int col = r0 + lane;
        tile[warp][jj][lane] = (ss < n && col < M) ? (double)y[ss * (int64_t)M + col] : 0.0;
      }
      __syncwarp();
#pragma unroll 1
      for (int u0 = 0; u0 < 32; u0 += PF) {
#pragma unroll
        for (int q2 = 0; q2 < PF; ++q2) {
          const int u = u0 + q2;
          const int jloc = asc ? u : 31 - u;
          const int i = r0 + jloc;
          if (i >= M) continue;
          const int t = asc ? i : (M - 1 - i);  // position in the new system's elimination order
          const double yv = tile[warp][lane][jloc];
          const int64_t idx = (int64_t)i * nb + s;
          double w = 1.0;
          double zval = 0.0;
          if (do_bsub) {
            const double l1 = nl1[q2], l2 = nl2[q2], gd = ngd[q2];
            if (t + PF < M) {   // prefetch PF rows ahead (same ring slot)
              const int64_t ix = (int64_t)row_of(t + PF) * nb + s;
              nl1[q2] = L1[ix]; nl2[q2] = L2[ix]; ngd[q2] = GD[ix];
            }
            zval = gd - l1 * zp1 - l2 * zp2;
            zp2 = zp1;
            zp1 = zval;
            w = (yv > zval) ? p : q;
          }
          if (do_fact) {
            // band values of W + lam D^T D at position t (D^T D: diag 1,5,6..6,5,1; first
            // off-diagonal -2,-4..-4,-2; second off-diagonal 1)
            const double d0 = (t == 0 || t == M - 1) ? 1.0 : ((t == 1 || t == M - 2) ? 5.0 : 6.0);
            const double d1 = (t >= M - 1) ? 0.0 : ((t == 0 || t == M - 2) ? -2.0 : -4.0);
            const double a0 = w + lam * d0;
            const double a1 = lam * d1;
            const double a2 = (t <= M - 3) ? lam : 0.0;
            const double D = a0 - L1m1 * L1m1 * Dm1 - L2m2 * L2m2 * Dm2;
            const double rD = rcp64(D);
            const double l1n = (a1 - L2m1 * L1m1 * Dm1) * rD;
            const double l2n = a2 * rD;
            const double g = w * yv - L1m1 * gm1 - L2m2 * gm2;
            if (valid) { L1[idx] = l1n; L2[idx] = l2n; GD[idx] = g * rD; }
            Dm2 = Dm1; Dm1 = D;
            L2m2 = L2m1; L2m1 = l2n;
            L1m1 = l1n;
            gm2 = gm1; gm1 = g;
          } else {
            tile[warp][lane][jloc] = zval;
          }
        }
      }
      if (!do_fact) {
        __syncwarp();
        for (int jj = 0; jj < 32; ++jj) {
          const int64_t ss = s0 + jj;
          const int col = r0 + lane;
          if (ss < n && col < M) z[ss * (int64_t)M + col] = (TZ)tile[warp][jj][lane];
        }
      }
    }
  }
}

// Few-row variant (the |q| <= 2k rows of fPEC, Eq. 16): one warp per row, the factor state in shared
// memory (4M doubles) so the serial fp64 recurrence sees smem instead of L2 latency.  Same sweep
// order and arithmetic as als_rows_kernel.
template <typename TY, typename TZ>
__global__ void __launch_bounds__(32) als_rows_smem_kernel(const TY* __restrict__ y, int M, double lam, double p,
                                                           int iters, TZ* __restrict__ z) {
  extern __shared__ __align__(16) double sh[];
  double* yv = sh;
  double* L1 = yv + M;
  double* L2 = L1 + M;
  double* GD = L2 + M;
  const int row = blockIdx.x, lane = threadIdx.x;
  for (int i = lane; i < M; i += 32) yv[i] = (double)y[(int64_t)row * M + i];
  __syncwarp();
  if (lane == 0) {
    const double q = 1.0 - p;
    for (int sw = 0; sw <= iters; ++sw) {
      const bool asc = (sw & 1) == 0;
      const bool do_bsub = sw > 0, do_fact = sw < iters;
      double zp1 = 0.0, zp2 = 0.0;
      double Dm1 = 0.0, Dm2 = 0.0, L1m1 = 0.0, L2m1 = 0.0, L2m2 = 0.0, gm1 = 0.0, gm2 = 0.0;
      for (int t = 0; t < M; ++t) {
        const int i = asc ? t : (M - 1 - t);
        const double yy = yv[i];
        double w = 1.0, zval = 0.0;
        if (do_bsub) {
          zval = GD[i] - L1[i] * zp1 - L2[i] * zp2;
          zp2 = zp1;
          zp1 = zval;
          w = (yy > zval) ? p : q;
        }
        if (do_fact) {
          const double d0 = (t == 0 || t == M - 1) ? 1.0 : ((t == 1 || t == M - 2) ? 5.0 : 6.0);
          const double d1 = (t >= M - 1) ? 0.0 : ((t == 0 || t == M - 2) ? -2.0 : -4.0);
          const double a2 = (t <= M - 3) ? lam : 0.0;
          const double D = w + lam * d0 - L1m1 * L1m1 * Dm1 - L2m2 * L2m2 * Dm2;
          const double rD = rcp64(D);
          const double l1n = (lam * d1 - L2m1 * L1m1 * Dm1) * rD;
          const double l2n = a2 * rD;
          const double g = w * yy - L1m1 * gm1 - L2m2 * gm2;
          L1[i] = l1n; L2[i] = l2n; GD[i] = g * rD;
          Dm2 = Dm1; Dm1 = D;
          L2m2 = L2m1; L2m1 = l2n;
          L1m1 = l1n;
          gm2 = gm1; gm1 = g;
        } else {
          yv[i] = zval;    // y is dead after the last factorisation: reuse it for z
        }
      }
    }
  }
  __syncwarp();
  for (int i = lane; i < M; i += 32) z[(int64_t)row * M + i] = (TZ)yv[i];
}

template <typename TIn, int MAXB>
__global__ void __launch_bounds__(kDirectThreads, 2)
direct_finish_kernel(const TIn* __restrict__ I, int64_t n, int M, const float* __restrict__ inv_ref,
                     const double* __restrict__ ref64, float floor, int L, int log2L, int pad_zero,
                     const float2* __restrict__ tw_g, const float* __restrict__ phi,
                     const float* __restrict__ phierr, int h, void* __restrict__ out, int imag_only) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* P0 = reinterpret_cast<double*>(smem);
  double* P1 = P0 + (M + 1);
  double* P2 = P1 + (M + 1);
  double* ybuf = P2 + (M + 1);
  double* wsum = ybuf + M;                                   // 96 doubles
  double* red = wsum + 96;                                   // 64 doubles
  cplx<float>* tw = reinterpret_cast<cplx<float>*>(red + 64);
  cplx<float>* x = tw + (L >> 1);
  float* a0 = reinterpret_cast<float*>(x + L);
  float* a1 = a0 + M;
  float2* kb = reinterpret_cast<float2*>(a1 + M);
  float* pd0 = reinterpret_cast<float*>(kb + M);   // phi - phi_err of row r0 / r1 (read with the other rows)
  float* pd1 = pd0 + M;
  float* pe_s = reinterpret_cast<float*>(kb);
  for (int j = threadIdx.x; j < (L >> 1); j += blockDim.x) { float2 t = tw_g[j]; tw[j].x = t.x; tw[j].y = t.y; }
  const int64_t npairs = (n + 1) >> 1;
  const int pl = (L - M) >> 1;
  const float invL = 1.0f / (float)L;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const SgConst sgk = sg_const(h);
  for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int64_t r0 = 2 * pr, r1 = r0 + 1;
    const bool has1 = r1 < n;
    const float* e0 = phierr + r0 * (int64_t)M;
    const float* e1 = has1 ? phierr + r1 * (int64_t)M : e0;
    // every row this pair needs (I, phi, phi_err of both spectra) loaded in one batch per element
#pragma unroll 4
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      const TIn v0 = I[r0 * (int64_t)M + j];
      const TIn v1 = has1 ? I[r1 * (int64_t)M + j] : (TIn)0;
      const float f0 = phi[r0 * (int64_t)M + j], g0 = e0[j];
      const float f1 = has1 ? phi[r1 * (int64_t)M + j] : 0.f, g1 = has1 ? e1[j] : 0.f;
      a0[j] = log_ratio_elem<TIn>(v0, inv_ref[j], ref64[j], floor);
      a1[j] = has1 ? log_ratio_elem<TIn>(v1, inv_ref[j], ref64[j], floor) : 0.f;
      pd0[j] = f0 - g0;
      pd1[j] = f1 - g1;
      pe_s[j] = g0;          // phi_err rows for the padded transform (kb's space, dead until the r loop)
      pe_s[M + j] = g1;
    }
    __syncthreads();
    pad_pair<float, float>(x, pe_s, pe_s + M, M, L, pad_zero);   // (syncs)
    hilbert_pair_stockham<float, MAXB>(x, tw, L, log2L);
    for (int r = 0; r < 2; ++r) {
      if (r == 1 && !has1) break;
      const int64_t row = r0 + r;
      const float* pdr = r == 0 ? pd0 : pd1;
      const float* aa = r == 0 ? a0 : a1;
      for (int j = threadIdx.x; j < M; j += blockDim.x) {
        const float hpe = (r == 0 ? x[pl + j].x : x[pl + j].y) * invL;
        const float ap = aa[j] + hpe;              // a' = a + H{phi_err}
        const float pp = pdr[j];                   // phi' = phi - phi_err
        // hardware sin/cos after a two-term reduction to [-pi, pi] and the hardware exp: ~1e-6 absolute,
        // an order below the 1e-5 direct-KK tolerance (the accurate sincosf/expf were a long sequence)
        const float kq = __fsub_rn(__fadd_rn(pp * 0.15915494309189535f, 12582912.0f), 12582912.0f);
        const float rr = fmaf(kq, 1.7484556e-07f, fmaf(-kq, 6.2831854820251465f, pp));
        float sn, cs;
        __sincosf(rr, &sn, &cs);
        const float mag = __expf(ap);
        kb[j] = make_float2(mag * cs, mag * sn);
        ybuf[j] = (double)(mag * cs);
      }
      __syncthreads();
      block_prefix3(ybuf, M, P0, P1, P2, wsum);
      // min of the trend, mean of Re K'
      double tmin = 1e300;
      for (int j = threadIdx.x; j < M; j += blockDim.x) {
        const double T = sg_point(P0, P1, P2, M, h, j, sgk);
        ybuf[j] = T;
        tmin = fmin(tmin, T);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      if (lane == 0) red[wid] = tmin;
      __syncthreads();
      double gmin = red[0];
      for (int w2 = 1; w2 < nw; ++w2) gmin = fmin(gmin, red[w2]);
      const double mean = P0[M] / (double)M;
      for (int j = threadIdx.x; j < M; j += blockDim.x) {
        const double T = gmin <= 0.0 ? mean : ybuf[j];
        const float2 kv = kb[j];
        const float it = (float)rcp64(T);   // MUFU seed + two Newton steps (~1 ulp)
        if (imag_only) {
          reinterpret_cast<float*>(out)[row * (int64_t)M + j] = kv.y * it;
        } else {
          reinterpret_cast<float2*>(out)[row * (int64_t)M + j] = make_float2(kv.x * it, kv.y * it);
        }
      }
      __syncthreads();
    }
  }
}

inline int ilog2(int L) { int r = 0; while ((1 << r) < L) ++r; return r; }

int grid_for(int64_t work, int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = (int64_t)sms * per_sm;
  if (work < g) g = work;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_direct_phase(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                         float floor, int L, int pad_zero, const float2* tw, float* phi, int* flags, cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = (size_t)(L / 2 + L) * sizeof(float2) + 2 * (size_t)M * sizeof(float);
  const int grid = grid_for((n + 1) / 2, 6);
  const bool big = L > 8 * kDirectThreads;
  if (L > 16 * kDirectThreads) throw Status(11, "direct path: FFT length above 4096");
  auto launch = [&](auto kf, const auto* in) {
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kf<<<grid, kDirectThreads, smem, s>>>(in, n, M, inv_ref, ref64, floor, L, ilog2(L), pad_zero, tw, phi, flags);
  };
  if (in_f64) {
    if (big) launch(direct_phase_kernel<double, 2>, (const double*)I);
    else launch(direct_phase_kernel<double, 1>, (const double*)I);
  } else {
    if (big) launch(direct_phase_kernel<float, 2>, (const float*)I);
    else launch(direct_phase_kernel<float, 1>, (const float*)I);
  }
  check_launch("direct_phase");
}

void launch_als_rows(const void* y, int y_f64, int64_t n, int M, double lam, double p, int iters, double* state,
                     void* z, int z_f64, cudaStream_t s) {
  if (n <= 0) return;
  if (launch_als_part(y, y_f64, n, M, lam, p, iters, z, z_f64, s)) return;
  const size_t sm = (size_t)4 * M * sizeof(double);
  if (n <= 4096 && sm <= 200 * 1024) {
    // few rows: smem-resident state, one warp per row
#define FKK_ALS_SMEM(TY, TZ)                                                                          \
    {                                                                                                 \
      auto kf = als_rows_smem_kernel<TY, TZ>;                                                         \
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                 \
      kf<<<(unsigned)n, 32, sm, s>>>((const TY*)y, M, lam, p, iters, (TZ*)z);                         \
    }
    if (y_f64 && z_f64) FKK_ALS_SMEM(double, double)
    else if (!y_f64 && !z_f64) FKK_ALS_SMEM(float, float)
    else if (!y_f64 && z_f64) FKK_ALS_SMEM(float, double)
    else FKK_ALS_SMEM(double, float)
#undef FKK_ALS_SMEM
    check_launch("als_rows_smem");
    return;
  }
  const int64_t nb = ((n + 31) / 32) * 32;
  const int64_t warps = nb / 32;
  const int grid = (int)((warps + 3) / 4);
  if (y_f64 && z_f64)
    als_rows_kernel<double, double><<<grid, 128, 0, s>>>((const double*)y, n, M, lam, p, iters, state, nb, (double*)z);
  else if (!y_f64 && !z_f64)
    als_rows_kernel<float, float><<<grid, 128, 0, s>>>((const float*)y, n, M, lam, p, iters, state, nb, (float*)z);
  else if (!y_f64 && z_f64)
    als_rows_kernel<float, double><<<grid, 128, 0, s>>>((const float*)y, n, M, lam, p, iters, state, nb, (double*)z);
  else
    als_rows_kernel<double, float><<<grid, 128, 0, s>>>((const double*)y, n, M, lam, p, iters, state, nb, (float*)z);
  check_launch("als_rows");
}

size_t direct_finish_smem(int M, int L) {
  return (size_t)(4 * (M + 1) + 96 + 64) * sizeof(double) + (size_t)(L / 2 + L) * sizeof(float2) +
         4 * (size_t)M * sizeof(float) + (size_t)M * sizeof(float2) + 64;
}

void launch_direct_finish(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                          float floor, int L, int pad_zero, const float2* tw, const float* phi, const float* phierr,
                          int sg_half, void* out, int out_imag_only, cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = direct_finish_smem(M, L);
  const int grid = grid_for((n + 1) / 2, 2);
  const bool big = L > 8 * kDirectThreads;
  if (L > 16 * kDirectThreads) throw Status(11, "direct path: FFT length above 4096");
  auto launch = [&](auto kf, const auto* in) {
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kf<<<grid, kDirectThreads, smem, s>>>(in, n, M, inv_ref, ref64, floor, L, ilog2(L), pad_zero, tw, phi, phierr,
                                          sg_half, out, out_imag_only);
  };
  if (in_f64) {
    if (big) launch(direct_finish_kernel<double, 2>, (const double*)I);
    else launch(direct_finish_kernel<double, 1>, (const double*)I);
  } else {
    if (big) launch(direct_finish_kernel<float, 2>, (const float*)I);
    else launch(direct_finish_kernel<float, 1>, (const float*)I);
  }
  check_launch("direct_finish");
}

}  // namespace fkk
