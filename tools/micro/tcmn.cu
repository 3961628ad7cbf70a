// Micro-test: tcgen05.mma kind::tf32 with MN-major SWIZZLE_128B operands (the layout a TMA SW128 box
// [K rows][32 fp32] produces), M = N = 128, K = 8.  X[mn][k] at box (mn / 32), row k, 16-B chunk
// ((mn % 32) / 4) ^ (k % 8), element mn % 4.  LBO = MN box stride, SBO = 8-row K atom stride.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_2005_07132_b200/csrc/tc_common.cuh"
using namespace fkk;

__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = tc::make_sdesc(saddr, lbo, sbo);
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(128) kmn(const float* A, const float* B, float* D, int lbo_mode) {
  __shared__ __align__(1024) unsigned char sa[4 * 1024];
  __shared__ __align__(1024) unsigned char sb[4 * 1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 8; e += 128) {
    const int mn = e >> 3, k = e & 7;
    const int off = (mn >> 5) * 1024 + k * 128 + ((((mn & 31) >> 2) ^ (k & 7)) << 4) + (mn & 3) * 4;
    *reinterpret_cast<float*>(sa + off) = A[mn * 8 + k];
    *reinterpret_cast<float*>(sb + off) = B[mn * 8 + k];
  }
  tc::fence_proxy_async_smem();
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&tslot, 128);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    // lbo_mode 0: LBO = MN box stride (1024), SBO = K atom stride (unused for K = 8 -> 8192)
    // lbo_mode 1: swapped
    const uint32_t lbo = lbo_mode ? 8192 : 1024, sbo = lbo_mode ? 1024 : 8192;
    const uint64_t da = make_sdesc_sw128(tc::smem_u32(sa), lbo, sbo);
    const uint64_t db = make_sdesc_sw128(tc::smem_u32(sb), lbo, sbo);
    const uint32_t idesc = tc::make_idesc_tf32(128, 128, true, true);
    tc::mma_tf32(tmem, da, db, idesc, 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int cb = 0; cb < 8; ++cb) {
    float v[16];
    tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + cb * 16, v);
    for (int q = 0; q < 16; ++q) D[(warp * 32 + lane) * 128 + cb * 16 + q] = v[q];
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

static float tf32t(float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  const int n = 128;
  float *hA = (float*)malloc(n * 8 * 4), *hB = (float*)malloc(n * 8 * 4), *hD = (float*)malloc(n * n * 4);
  srand(3);
  for (int i = 0; i < n * 8; ++i) { hA[i] = (rand() % 20001 - 10000) / 9973.0f; hB[i] = (rand() % 20001 - 10000) / 9967.0f; }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, n * 8 * 4); cudaMalloc(&dB, n * 8 * 4); cudaMalloc(&dD, n * n * 4);
  cudaMemcpy(dA, hA, n * 8 * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, n * 8 * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, n * n * 4);
    kmn<<<1, 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, n * n * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxv = 0;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
      double s = 0; for (int k = 0; k < 8; ++k) s += (double)tf32t(hA[i * 8 + k]) * tf32t(hB[j * 8 + k]);
      maxerr = fmax(maxerr, fabs(s - hD[i * n + j])); maxv = fmax(maxv, fabs(s));
    }
    printf("lbo_mode %d: %s  max err %.3e (max |D| %.3f)\n", mode, cudaGetErrorString(e), maxerr, maxv);
  }
}
