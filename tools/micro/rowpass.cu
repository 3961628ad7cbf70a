// Micro-benchmark of the tridiagonalisation's per-row pass (copy of row_pass's loop shape): cycles per
// call for one warp, with and without the pending update, at several row lengths.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double row_pass(double* row, int m0, int M, bool pending, double vr, double wr,
                                           const double* vp, const double* wp, const double* v, double* pub) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if (pending) {
#pragma unroll 4
    for (int c = m0 + lane; c < M; c += 32) {
      const double a = row[c] - (vr * wp[c] + wr * vp[c]);
      row[c] = a;
      if (pub) pub[c] = a;
      acc = fma(a, v[c], acc);
    }
  } else {
#pragma unroll 4
    for (int c = m0 + lane; c < M; c += 32) {
      const double a = row[c];
      if (pub) pub[c] = a;
      acc = fma(a, v[c], acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}
// (c) __restrict__ + 4 independent accumulators, loads of 4 iterations issued together
__device__ __forceinline__ double row_pass_reg(double* __restrict__ row, int m0, int M, bool pending, double vr,
                                               double wr, const double* __restrict__ vp, const double* __restrict__ wp,
                                               const double* __restrict__ v) {
  const int lane = threadIdx.x & 31;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int c = m0 + lane;
  for (; c + 96 < M; c += 128) {
    double a[4], vv[4], ww[4], pp[4];
    // every load of the group first (explicit: the compiler keeps loads behind the row stores)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = row[c + 32 * u]; vv[u] = v[c + 32 * u];
      ww[u] = pending ? wp[c + 32 * u] : 0.0; pp[u] = pending ? vp[c + 32 * u] : 0.0;
    }
    if (pending) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] -= vr * ww[u] + wr * pp[u];
#pragma unroll
      for (int u = 0; u < 4; ++u) row[c + 32 * u] = a[u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = fma(a[u], vv[u], acc[u]);
  }
  for (; c < M; c += 32) {
    double a = row[c];
    if (pending) { a -= vr * wp[c] + wr * vp[c]; row[c] = a; }
    acc[0] = fma(a, v[c], acc[0]);
  }
  double r = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}
__global__ void k2(int M, int m0, int pending, int reps, long long* cyc, double* out) {
  extern __shared__ double sm[];
  double* rows = sm;
  double* vp = rows + 16 * M; double* wp = vp + M; double* v = wp + M;
  for (int i = threadIdx.x; i < 19 * M; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double s = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    s += row_pass_reg(rows + warp * M, m0, M, pending, vp[warp], wp[warp], vp, wp, v);
    __syncwarp();
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) { cyc[warp] = (t1 - t0) / reps; out[warp] = s; }
}
__global__ void k(int M, int m0, int pending, int reps, long long* cyc, double* out, double* gpub) {
  extern __shared__ double sm[];
  double* rows = sm;            // 16 rows
  double* vp = rows + 16 * M; double* wp = vp + M; double* v = wp + M;
  for (int i = threadIdx.x; i < 19 * M; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double s = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    s += row_pass(rows + warp * M, m0, M, pending, vp[warp], wp[warp], vp, wp, v, nullptr);
    __syncwarp();
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) { cyc[warp] = (t1 - t0) / reps; out[warp] = s; }
}
int main() {
  long long* cyc; double* out;
  cudaMalloc(&cyc, 64 * 8); cudaMalloc(&out, 64 * 8);
  const int M = 1000;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 19 * M * 8);
  for (int nw : {1, 7})
    for (int pending : {0, 1})
      for (int m : {100, 500, 999}) {
        k<<<1, 32 * nw, 19 * M * 8>>>(M, M - m, pending, 200, cyc, out, nullptr);
        long long h[64];
        cudaMemcpy(h, cyc, nw * 8, cudaMemcpyDeviceToHost);
        printf("warps %2d pending %d m %4d: %6lld cycles per row pass (warp 0)", nw, pending, m, h[0]);
        cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 19 * M * 8);
        k2<<<1, 32 * nw, 19 * M * 8>>>(M, M - m, pending, 200, cyc, out);
        cudaMemcpy(h, cyc, nw * 8, cudaMemcpyDeviceToHost);
        printf("   register variant %6lld\n", h[0]);
      }
  return 0;
}
