// Self-test of the tcgen05 plumbing (test hook fkk_debug_tc_mma): one CTA stages A (128 x 8) and
// B (N x 8) fp32 tiles into shared memory in a chosen UMMA layout, issues one tcgen05.mma
// kind::tf32 (K = 8), and copies the TMEM accumulator to global D (128 x N, row-major).
// mode bit 0: A MN-major (else K-major); bit 1: B MN-major; bit 2: pad the strips/groups by 16 B.
#include <cuda_runtime.h>

#include "fkk_internal.h"
#include "tc_common.cuh"

namespace fkk {

namespace {

__global__ void __launch_bounds__(128) tc_selftest_kernel(int mode, const float* __restrict__ A,
                                                          const float* __restrict__ B, float* __restrict__ D, int N) {
  __shared__ __align__(1024) unsigned char sm[2 * 128 * 48 + 2 * 256 * 48];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool a_mn = mode & 1, b_mn = mode & 2, pad = mode & 4;
  unsigned char* sa = sm;
  unsigned char* sb = sm + 128 * 48;
  // K-major: core matrix = 8 rows x 16 B (4 k); rows contiguous, K-chunks at LBO, 8-row groups at SBO
  //   LBO = 128 (+16 if pad), SBO = 2 * LBO
  // MN-major: core matrix = 8 k x 16 B (4 mn); k rows contiguous, 4-mn strips at SBO = 128 (+16)
  const uint32_t kl_lbo = pad ? 144 : 128, kl_sbo = 2 * kl_lbo;
  const uint32_t mn_sbo = pad ? 144 : 128;
  for (int e = tid; e < 128 * 8; e += 128) {
    const int r = e >> 3, k = e & 7;
    const float v = tc::tf32_rna(A[r * 8 + k]);
    uint32_t off;
    if (a_mn) off = (r >> 2) * mn_sbo + k * 16 + (r & 3) * 4;
    else off = (r >> 3) * kl_sbo + (k >> 2) * kl_lbo + (r & 7) * 16 + (k & 3) * 4;
    *reinterpret_cast<float*>(sa + off) = v;
  }
  for (int e = tid; e < N * 8; e += 128) {
    const int r = e >> 3, k = e & 7;
    const float v = tc::tf32_rna(B[r * 8 + k]);
    uint32_t off;
    if (b_mn) off = (r >> 2) * mn_sbo + k * 16 + (r & 3) * 4;
    else off = (r >> 3) * kl_sbo + (k >> 2) * kl_lbo + (r & 7) * 16 + (k & 3) * 4;
    *reinterpret_cast<float*>(sb + off) = v;
  }
  tc::fence_proxy_async_smem();
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(&tslot, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint64_t da = a_mn ? tc::make_sdesc(tc::smem_u32(sa), 128, mn_sbo) : tc::make_sdesc(tc::smem_u32(sa), kl_lbo, kl_sbo);
    const uint64_t db = b_mn ? tc::make_sdesc(tc::smem_u32(sb), 128, mn_sbo) : tc::make_sdesc(tc::smem_u32(sb), kl_lbo, kl_sbo);
    const uint32_t idesc = tc::make_idesc_tf32(128, N, a_mn, b_mn);
    tc::mma_tf32(tmem, da, db, idesc, 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int cb = 0; cb < N / 16; ++cb) {
    float v[16];
    tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + cb * 16, v);
    for (int q = 0; q < 16; ++q) D[(warp * 32 + lane) * N + cb * 16 + q] = v[q];
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

}  // namespace

void launch_tc_selftest(int mode, const float* A, const float* B, float* D, int N, cudaStream_t s) {
  tc_selftest_kernel<<<1, 128, 0, s>>>(mode, A, B, D, N);
  check_launch("tc_selftest");
}

}  // namespace fkk
