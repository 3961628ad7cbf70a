// Grid-barrier latency probes on sm_100a (148 co-resident CTAs, 512 threads): cost per barrier of
// several designs, optionally with a burst of global stores before each barrier (release cost).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void flat(unsigned* ctr, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
  }
  __syncthreads();
}
__device__ __forceinline__ void flat_relaxed(unsigned* ctr, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
    unsigned v;
    do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ void hier(unsigned* ctr, unsigned& target, unsigned ncl, unsigned rank) {
  csync();   // includes the CTA-wide sync (aligned: all threads)
  target += gridDim.x / ncl;
  if (rank == 0 && threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
  }
  csync();
}
// flags: CTA b publishes epoch in flag[b*32]; CTA 0 gathers with 148 threads, then releases go
__device__ __forceinline__ void flags(unsigned* fl, unsigned* go, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(fl + blockIdx.x * 32), "r"(epoch) : "memory");
  if (blockIdx.x == 0) {
    if (threadIdx.x < gridDim.x) {
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl + threadIdx.x * 32) : "memory"); } while ((int)(v - epoch) < 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(go), "r"(epoch) : "memory");
  } else if (threadIdx.x == 0) {
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(go) : "memory"); } while ((int)(v - epoch) < 0);
  }
  __syncthreads();
}
// split: arrivals on the counter line (atom returns the old value); the last arriver publishes the
// epoch on a separate flag line that everyone polls
__device__ __forceinline__ void split(unsigned* ctr, unsigned* flag, unsigned epoch, bool relaxed_poll) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(ctr), "r"(1u) : "memory");
    if (old + 1 == epoch * gridDim.x) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    } else {
      unsigned v;
      if (relaxed_poll) {
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while ((int)(v - epoch) < 0);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while ((int)(v - epoch) < 0);
      }
    }
  }
  __syncthreads();
}
// all-poll: every CTA publishes its epoch in its own word; threads 0..P-1 of every CTA poll one
// word each (packed: 32 words per 128-B line) -- no atomics, one hop
__device__ __forceinline__ void allpoll(unsigned* fl, unsigned epoch, int stride) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(fl + blockIdx.x * stride), "r"(epoch) : "memory");
  if (threadIdx.x < gridDim.x) {
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl + threadIdx.x * stride) : "memory"); } while ((int)(v - epoch) < 0);
  }
  __syncthreads();
}
__device__ __forceinline__ void allpoll_relaxed(unsigned* fl, unsigned epoch, int stride) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(fl + blockIdx.x * stride), "r"(epoch) : "memory");
  if (threadIdx.x < gridDim.x) {
    unsigned v;
    do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl + threadIdx.x * stride) : "memory"); } while ((int)(v - epoch) < 0);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  __syncthreads();
}
__global__ void kbar(int mode, int iters, int nst, unsigned* ctr, unsigned* fl, double* scratch) {
  unsigned target = 0, ncl = 1, rank = 0;
  if (mode == 2) {
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  }
  for (int it = 0; it < iters; ++it) {
    for (int c = threadIdx.x; c < nst; c += blockDim.x) scratch[(size_t)blockIdx.x * 4096 + c] = it + c;
    if (mode == 0) flat(ctr, target);
    else if (mode == 1) flat_relaxed(ctr, target);
    else if (mode == 2) hier(ctr, target, ncl, rank);
    else if (mode == 3) flags(fl, fl + 148 * 32 + 64, it + 1);
    else if (mode == 4 || mode == 5) split(ctr, ctr + 64, it + 1, mode == 5);
    else if (mode == 6) allpoll(fl, it + 1, 1);
    else if (mode == 7) allpoll(fl, it + 1, 32);
    else allpoll_relaxed(fl, it + 1, 1);
  }
}
int main() {
  unsigned* ctr; unsigned* fl; double* scr;
  cudaMalloc(&ctr, 4096); cudaMalloc(&fl, 148 * 128 + 4096); cudaMalloc(&scr, 148 * 4096 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2000;
  for (int mode = 0; mode < 9; ++mode)
    for (int cl : {1, 2, 4, 8})
      for (int nst : {0, 512}) {
        if ((mode == 2) != (cl > 1)) continue;
        int grid = 148 / cl * cl;
        cudaMemset(ctr, 0, 4096); cudaMemset(fl, 0, 148 * 128 + 4096);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension; at[1].val.clusterDim.x = cl; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(512); cfg.attrs = at; cfg.numAttrs = cl > 1 ? 2 : 1;
        if (cl > 1) {
          int ncl = 0;
          cfg.numAttrs = 1; cfg.attrs = at + 1;
          cudaOccupancyMaxActiveClusters(&ncl, (void*)kbar, &cfg);
          cfg.attrs = at; cfg.numAttrs = 2;
          if (ncl * cl < grid) grid = ncl * cl;
          cfg.gridDim = dim3(grid);
        }
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, kbar, mode, iters, nst, ctr, fl, scr);
        cudaEventRecord(b);
        cudaError_t e2 = cudaEventSynchronize(b);
        float ms = 0; cudaEventElapsedTime(&ms, a, b);
        printf("mode %d cluster %d grid %d stores %4d: %7.3f us/barrier  (%s %s)\n", mode, cl, grid, nst, ms * 1e3 / iters,
               cudaGetErrorString(e), cudaGetErrorString(e2));
      }
  return 0;
}
