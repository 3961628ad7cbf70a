// Micro-test of the 2-CTA (cta_group::2) tcgen05.mma kind::tf32 plumbing: D(256x256) = A(256x8) B(256x8)^T
// with A rows 128r.. and B rows 128r.. staged in CTA r of a cluster pair (K-major, no swizzle).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_2005_07132_b200/csrc/tc_common.cuh"
using namespace fkk;

__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) k2(const float* A, const float* B, float* D, int bmode) {
  __shared__ __align__(1024) unsigned char sa[128 * 32];
  __shared__ __align__(1024) unsigned char sb[256 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t r = cluster_rank();
  // K-major core matrices: 8 rows x 16 B (4 k), rows contiguous; K-chunk at LBO = 128, 8-row group at SBO = 256
  for (int e = tid; e < 128 * 8; e += 128) {
    const int row = e >> 3, k = e & 7;
    const int off = (row >> 3) * 256 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
    *reinterpret_cast<float*>(sa + off) = tc::tf32_rna(A[(r * 128 + row) * 8 + k]);
  }
  // bmode 0: CTA r holds B rows 128r.. (N split); bmode 1: both CTAs hold all 256 rows
  const int nb = bmode ? 256 : 128;
  for (int e = tid; e < nb * 8; e += 128) {
    const int row = e >> 3, k = e & 7;
    const int grow = bmode ? row : (int)(r * 128 + row);
    const int off = (row >> 3) * 256 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
    *reinterpret_cast<float*>(sb + off) = tc::tf32_rna(B[grow * 8 + k]);
  }
  tc::fence_proxy_async_smem();
  if (tid == 0) { tc::mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tslot)), "r"(256u) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (r == 0 && tid == 0) {
    const uint64_t da = tc::make_sdesc(tc::smem_u32(sa), 128, 256);
    const uint64_t db = tc::make_sdesc(tc::smem_u32(sb), 128, 256);
    const uint32_t idesc = tc::make_idesc_tf32(256, 256, false, false);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0u) : "memory");
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(tc::smem_u32(&bar)), "h"((unsigned short)3) : "memory");
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int cb = 0; cb < 16; ++cb) {
    float v[16];
    tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + cb * 16, v);
    for (int q = 0; q < 16; ++q) D[(r * 128 + warp * 32 + lane) * 256 + cb * 16 + q] = v[q];
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u) : "memory");
}

static float tf32(float x) { unsigned u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  const int n = 256;
  float *hA = (float*)malloc(n * 8 * 4), *hB = (float*)malloc(n * 8 * 4), *hD = (float*)malloc(n * n * 4);
  srand(1);
  for (int i = 0; i < n * 8; ++i) { hA[i] = (rand() % 2001 - 1000) / 997.0f; hB[i] = (rand() % 2001 - 1000) / 991.0f; }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, n * 8 * 4); cudaMalloc(&dB, n * 8 * 4); cudaMalloc(&dD, n * n * 4);
  cudaMemcpy(dA, hA, n * 8 * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, n * 8 * 4, cudaMemcpyHostToDevice);
  for (int bmode = 0; bmode < 2; ++bmode) {
    cudaMemset(dD, 0, n * n * 4);
    k2<<<2, 128>>>(dA, dB, dD, bmode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, n * n * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxv = 0;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
      double s = 0; for (int k = 0; k < 8; ++k) s += (double)tf32(hA[i * 8 + k]) * tf32(hB[j * 8 + k]);
      maxerr = fmax(maxerr, fabs(s - hD[i * n + j])); maxv = fmax(maxv, fabs(s));
    }
    printf("bmode %d: %s  max err %.3e (max |D| %.3f)\n", bmode, cudaGetErrorString(e), maxerr, maxv);
  }
}
