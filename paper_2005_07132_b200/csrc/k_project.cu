// Projection US = A0 W (F5: US = A V_k = U_k S_k, with W = D_f V_k so that the
// f-scaling of Eq. 10 is folded in) and per-block column extremes for q (Eqs. 13-15,
// PAPER.md:117-121).  CUDA-core fp32 variant: 128 pixels x kp columns per CTA, 8 x CPT register
// blocks, channel chunks of 32 staged in smem.  Ties in the extremes -> lowest pixel index.
#include <cuda_runtime.h>
#include <math.h>

#include "fkk_internal.h"

namespace fkk {

namespace {

constexpr int PR = 128;   // pixels per CTA
constexpr int PK = 32;    // channels per chunk

template <int CPT>   // columns per thread; kp = 16 * CPT
__global__ void __launch_bounds__(256) project_simt_kernel(const float* __restrict__ A, int64_t n, int M,
                                                           const float* __restrict__ W, int k,
                                                           float* __restrict__ US, float* __restrict__ ext_val,
                                                           int64_t* __restrict__ ext_idx, int64_t row_offset) {
  constexpr int KP = 16 * CPT;
  constexpr int kMain = (PK * (PR + 4) + PK * KP) * 4;
  constexpr int kRed = 2 * 16 * KP * 8;
  __shared__ __align__(16) unsigned char smem_raw[kMain > kRed ? kMain : kRed];
  float(*As)[PR + 4] = reinterpret_cast<float(*)[PR + 4]>(smem_raw);
  float(*Ws)[KP] = reinterpret_cast<float(*)[KP]>(smem_raw + PK * (PR + 4) * 4);
  float(*rv)[16][KP] = reinterpret_cast<float(*)[16][KP]>(smem_raw);             // aliases As/Ws after the K loop
  int(*rix)[16][KP] = reinterpret_cast<int(*)[16][KP]>(smem_raw + 2 * 16 * KP * 4);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t p0 = (int64_t)blockIdx.x * PR;
  float acc[8][CPT];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < CPT; ++b) acc[a][b] = 0.f;
  for (int c0 = 0; c0 < M; c0 += PK) {
    // A chunk: 128 pixels x 32 channels = 1024 float4; transpose into As[channel][pixel]
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int idx = tid + h * 256;
      const int pr = idx >> 3, c4 = (idx & 7) * 4;
      const int64_t p = p0 + pr;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < n && c0 + c4 < M) v = __ldg(reinterpret_cast<const float4*>(A + p * (int64_t)M + c0 + c4));
      As[c4 + 0][pr] = v.x;
      As[c4 + 1][pr] = v.y;
      As[c4 + 2][pr] = v.z;
      As[c4 + 3][pr] = v.w;
    }
    for (int idx = tid; idx < PK * KP / 4; idx += 256) {
      const int r = idx / (KP / 4), c4 = (idx % (KP / 4)) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c0 + r < M) v = __ldg(reinterpret_cast<const float4*>(W + (int64_t)(c0 + r) * KP + c4));
      *reinterpret_cast<float4*>(&Ws[r][c4]) = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < PK; ++kk) {
      float a[8], b[CPT];
      *reinterpret_cast<float4*>(&a[0]) = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      *reinterpret_cast<float4*>(&a[4]) = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
#pragma unroll
      for (int b2 = 0; b2 < CPT; ++b2) b[b2] = Ws[kk][tx + 16 * b2];
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < CPT; ++y) acc[x][y] = fmaf(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
  // store US and per-thread column extremes over its 8 pixels
#pragma unroll
  for (int y = 0; y < CPT; ++y) {
    const int c = tx + 16 * y;
    float vmax = -INFINITY, vmin = INFINITY;
    int imax = 0x7fffffff, imin = 0x7fffffff;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int pl = ty * 8 + x;
      const int64_t p = p0 + pl;
      if (p < n) {
        const float v = acc[x][y];
        US[p * KP + c] = v;   // stride kp; columns >= k are exact zeros (W padded with zeros)
        if (v > vmax) { vmax = v; imax = pl; }   // ascending pl: strict > keeps the lowest index
        if (v < vmin) { vmin = v; imin = pl; }
      }
    }
    rv[0][ty][c] = vmax; rix[0][ty][c] = imax;
    rv[1][ty][c] = vmin; rix[1][ty][c] = imin;
  }
  __syncthreads();
  for (int c = tid; c < k; c += 256) {
    float vmax = -INFINITY, vmin = INFINITY;
    int imax = 0x7fffffff, imin = 0x7fffffff;
    for (int g = 0; g < 16; ++g) {   // ascending pixel groups
      if (rv[0][g][c] > vmax) { vmax = rv[0][g][c]; imax = rix[0][g][c]; }
      if (rv[1][g][c] < vmin) { vmin = rv[1][g][c]; imin = rix[1][g][c]; }
    }
    const int64_t o = ((int64_t)blockIdx.x * k + c) * 2;
    ext_val[o] = vmax;
    ext_idx[o] = imax == 0x7fffffff ? INT64_MAX : row_offset + p0 + imax;
    ext_val[o + 1] = vmin;
    ext_idx[o + 1] = imin == 0x7fffffff ? INT64_MAX : row_offset + p0 + imin;
  }
}

}  // namespace

int project_num_blocks(int64_t n) { return (int)((n + PR - 1) / PR); }

void launch_project_simt(const float* A, int64_t n, int M, const float* W, int k, int kp, float* US, float* ext_val,
                         int64_t* ext_idx, int64_t row_offset, cudaStream_t s) {
  if (n <= 0) return;
  const int grid = project_num_blocks(n);
  switch (kp) {
    case 16: project_simt_kernel<1><<<grid, 256, 0, s>>>(A, n, M, W, k, US, ext_val, ext_idx, row_offset); break;
    case 32: project_simt_kernel<2><<<grid, 256, 0, s>>>(A, n, M, W, k, US, ext_val, ext_idx, row_offset); break;
    case 64: project_simt_kernel<4><<<grid, 256, 0, s>>>(A, n, M, W, k, US, ext_val, ext_idx, row_offset); break;
    case 128: project_simt_kernel<8><<<grid, 256, 0, s>>>(A, n, M, W, k, US, ext_val, ext_idx, row_offset); break;
    default: throw Status(1, "project: unsupported padded rank " + std::to_string(kp));
  }
  check_launch("project_simt");
}

}  // namespace fkk
