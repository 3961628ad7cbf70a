// Reconstruction (F11, Eq. 23):
//   K[n, j] = exp(sum_i US[n,i] B_amp[i,j]) * (cos + i sin)(sum_i US[n,i] B_ph[i,j]),
// CUDA-core fp32 variant: 64 pixels x 128 channels per CTA; warp w owns 8 pixels, lane l owns
// channels l + 32m (m < 4) so the complex64 stores of a warp are 256 contiguous bytes.  B is stored
// column-interleaved (amp_j, ph_j) so one float2 smem load feeds both accumulators of a channel.
#include <cuda_runtime.h>
#include <math.h>

#include "fkk_internal.h"

namespace fkk {

namespace {

constexpr int RP = 64;    // pixels per CTA
constexpr int RC = 128;   // channels per CTA
constexpr int RK = 32;    // rank chunk

__device__ __forceinline__ float2 cis_exp(float amp, float ph) {
  // range-reduce the phase to [-pi, pi] before the fast sincos
  const float k = rintf(ph * 0.15915494309189535f);
  const float r = fmaf(-k, 6.2831854820251465f, ph);
  const float r2 = fmaf(k, 1.7484556e-07f, r);   // 2*pi = 6.2831854820251465 - 1.7484556e-07
  float sn, cs;
  __sincosf(r2, &sn, &cs);
  const float m = __expf(amp);
  return make_float2(m * cs, m * sn);
}

__global__ void __launch_bounds__(256) reconstruct_simt_kernel(const float* __restrict__ US, int64_t n, int k, int ldus,
                                                               const float* __restrict__ Bi, int M,
                                                               void* __restrict__ out, int imag_only) {
  __shared__ __align__(16) float Us[RK][RP];          // [rank][pixel]
  __shared__ __align__(16) float2 Bs[RK][RC];         // [rank][channel] (amp, ph)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t p0 = (int64_t)blockIdx.x * RP;
  const int c0 = blockIdx.y * RC;
  float am[8][4], ph[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) { am[a][b] = 0.f; ph[a][b] = 0.f; }
  for (int k0 = 0; k0 < k; k0 += RK) {
    for (int idx = tid; idx < RK * RP; idx += 256) {
      const int pr = idx / RK, kk = idx % RK;
      const int64_t p = p0 + pr;
      Us[kk][pr] = (p < n && k0 + kk < k) ? US[p * ldus + k0 + kk] : 0.f;
    }
    for (int idx = tid; idx < RK * RC; idx += 256) {
      const int kk = idx / RC, c = idx % RC;
      float2 v = make_float2(0.f, 0.f);
      if (k0 + kk < k && c0 + c < M) v = __ldg(reinterpret_cast<const float2*>(Bi) + (int64_t)(k0 + kk) * M + c0 + c);
      Bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < RK; ++kk) {
      float u[8];
      *reinterpret_cast<float4*>(&u[0]) = *reinterpret_cast<const float4*>(&Us[kk][w * 8]);
      *reinterpret_cast<float4*>(&u[4]) = *reinterpret_cast<const float4*>(&Us[kk][w * 8 + 4]);
      float2 b[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) b[m] = Bs[kk][lane + 32 * m];
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          am[x][m] = fmaf(u[x], b[m].x, am[x][m]);
          ph[x][m] = fmaf(u[x], b[m].y, ph[x][m]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    const int64_t p = p0 + w * 8 + x;
    if (p >= n) break;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int c = c0 + lane + 32 * m;
      if (c < M) {
        const float2 v = cis_exp(am[x][m], ph[x][m]);
        if (imag_only) __stcs(reinterpret_cast<float*>(out) + p * M + c, v.y);
        else __stcs(reinterpret_cast<float2*>(out) + p * M + c, v);
      }
    }
  }
}

}  // namespace

void launch_reconstruct_simt(const float* US, int64_t n, int k, int ldus, const float* Bi, int M, void* out,
                             int out_imag_only, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid((unsigned)((n + RP - 1) / RP), (unsigned)((M + RC - 1) / RC));
  reconstruct_simt_kernel<<<grid, 256, 0, s>>>(US, n, k, ldus, Bi, M, out, out_imag_only);
  check_launch("reconstruct_simt");
}

}  // namespace fkk
