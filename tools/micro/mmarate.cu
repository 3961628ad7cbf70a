// tcgen05.mma kind::tf32 issue rate from shared memory, 128 x N x 8 per instruction, for the operand
// layouts the kernels use: (0) interleaved K-major with a 16-B pad per 8-row group (SBO 1040, the Gram
// image), (1) interleaved unpadded (SBO 1024), (2) SWIZZLE_128B K-major (SBO 1024, layout type 2).
// One CTA, one elected thread issues 12 MMAs per "stage" (4 k-steps x 3 products) for NIT stages.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2005_07132_b200/csrc/tc_common.cuh"
using namespace fkk;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N>
__global__ void __launch_bounds__(128) k(int mode, int nit, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  // A hi, A lo (128 rows), B hi, B lo (N rows), 32 K (128 B per row), 17 KB each incl. pad room
  constexpr int OPA = 128 * 128 + 16 * 16, OPB = N * 128 + (N / 8) * 16;
  unsigned char* ah = sm;
  unsigned char* al = ah + OPA;
  unsigned char* bh = al + OPA;
  unsigned char* bl = bh + ((OPB + 1023) & ~1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (int)(2 * OPA + 2 * ((OPB + 1023) & ~1023)) / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 1.0f;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&tslot, 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t idesc = tc::make_idesc_tf32(128, N, false, false);
    const uint32_t sbo = mode == 0 ? 1040 : 1024;
    uint64_t dah, dal, dbh, dbl;
    if (mode == 2) {
      dah = desc_sw128(tc::smem_u32(ah)); dal = desc_sw128(tc::smem_u32(al));
      dbh = desc_sw128(tc::smem_u32(bh)); dbl = desc_sw128(tc::smem_u32(bl));
    } else {
      dah = tc::make_sdesc(tc::smem_u32(ah), 128, sbo); dal = tc::make_sdesc(tc::smem_u32(al), 128, sbo);
      dbh = tc::make_sdesc(tc::smem_u32(bh), 128, sbo); dbl = tc::make_sdesc(tc::smem_u32(bl), 128, sbo);
    }
    const uint32_t kstep = mode == 2 ? 32 : 256;   // 8 tf32 along K: 32 B in a swizzle row, 2 core matrices otherwise
    long long t0 = clock64();
    if (tc::elect_one()) {
      for (int it = 0; it < nit; ++it) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t o = ks * kstep;
          tc::mma_tf32(tmem + N, tc::sdesc_add(dal, o), tc::sdesc_add(dbh, o), idesc, it > 0 || ks > 0);
          tc::mma_tf32(tmem + N, tc::sdesc_add(dah, o), tc::sdesc_add(dbl, o), idesc, 1u);
          tc::mma_tf32(tmem, tc::sdesc_add(dah, o), tc::sdesc_add(dbh, o), idesc, it > 0 || ks > 0);
        }
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  const int nit = 2000;
  for (int N : {128, 256})
    for (int mode = 0; mode < 3; ++mode) {
      const size_t smem = 160 * 1024;
      if (N == 128) { cudaFuncSetAttribute(k<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k<128><<<1, 128, smem>>>(mode, nit, d); }
      else { cudaFuncSetAttribute(k<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k<256><<<1, 128, smem>>>(mode, nit, d); }
      long long h = 0; cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double cyc = (double)h / (nit * 12.0);
      const double flop = 2.0 * 128 * N * 8;
      printf("N %3d layout %d: %6.1f cycles per MMA  (%5.0f flop/clk; %s)\n", N, mode, cyc, flop / cyc, cudaGetErrorString(e));
    }
  return 0;
}
