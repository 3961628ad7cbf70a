// Reconstruction (F11, Eq. 23) on the 5th-generation tensor cores:
//   K[p, c] = exp(sum_i US[p,i] B_amp[i,c]) * (cos + i sin)(sum_i US[p,i] B_ph[i,c])
// as one GEMM D = US . B^T per 128-pixel tile and NCH-channel chunk, B's rows interleaved
// (amp_c, ph_c) so TMEM columns (2j, 2j+1) are the exponent and phase of channel j; 3xTF32
// (hi*hi + hi*lo + lo*hi; K = kr = roundup8(k) is short, so one TMEM accumulator suffices).
//   warps 0-3  : producers - the US tile (128 x kr) -> tf32 hi/lo -> K-major smem (LBO 144 B pad)
//   warps 4-11 : epilogue  - tcgen05.ld, exp/sincos into a per-thread smem slot, then one bulk
//                copy (cp.async.bulk smem -> global) per thread: its pixel row's half of the chunk
//                (contiguous 128 B of complex64), double-buffered; 4 TMEM accumulators rotate.
//                (Measured: faster than staging a tile and storing coalesced rows after a named
//                barrier, 2.77 vs 3.35 ms at cfg3.)
//   warp 12    : TMEM alloc; B-chunk bulk copies (cp.async.bulk, mbarrier tx) and the MMA issue
// B is pre-staged once per basis in global memory in the exact K-major smem image (hi, lo).
// Persistent CTAs walk pixel tiles; the B chunk sequence repeats per tile (L2-resident, ~1 MB).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "fkk_internal.h"
#include "tc_common.cuh"

namespace fkk {

namespace {

constexpr int RTM = 128;          // pixels per tile (UMMA M)
constexpr int RT_THREADS = 416;
constexpr int A_LBO = 144;        // padded: conflict-free producer stores
constexpr int B_LBO = 128;
constexpr int SLOT = 144;         // epilogue staging slot per thread (128 B + pad)

struct RtGeom {
  int kr, nch, N, nchunks;
  int a_sbo, a_bytes;             // per hi / lo
  int b_sbo, b_part, b_stage;     // part = hi or lo block, stage = hi + lo
};

__host__ __device__ inline RtGeom rt_geom(int k, int M) {
  RtGeom g;
  g.kr = (k + 7) / 8 * 8;
  g.nch = g.kr <= 64 ? 32 : 16;
  g.N = 2 * g.nch;
  g.nchunks = (M + g.nch - 1) / g.nch;
  g.a_sbo = (g.kr / 4) * A_LBO;
  g.a_bytes = (RTM / 8) * g.a_sbo;
  g.b_sbo = (g.kr / 4) * B_LBO;
  g.b_part = (g.N / 8) * g.b_sbo;
  g.b_stage = 2 * g.b_part;
  return g;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float2 cis_exp(float amp, float ph) {
  const float kq = rintf(ph * 0.15915494309189535f);
  const float r = fmaf(-kq, 6.2831854820251465f, ph);
  const float r2 = fmaf(kq, 1.7484556e-07f, r);
  float sn, cs;
  __sincosf(r2, &sn, &cs);
  const float m = __expf(amp);
  return make_float2(m * cs, m * sn);
}

__global__ void __launch_bounds__(RT_THREADS, 1)
reconstruct_tc_kernel(const float* __restrict__ US, int64_t n, int k, int ldus, const float* __restrict__ bimg, int M,
                      void* __restrict__ out, int imag_only) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const RtGeom g = rt_geom(k, M);
  unsigned char* a_hi = smem;
  unsigned char* a_lo = smem + g.a_bytes;
  unsigned char* bst = smem + 2 * g.a_bytes;                 // 2 stages
  unsigned char* stg = bst + 2 * g.b_stage;                  // [2][256 threads][SLOT]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + 2 * 256 * SLOT);
  uint64_t* a_full = bars;          // producers -> MMA (count 128)
  uint64_t* a_empty = bars + 1;     // MMA commit -> producers
  uint64_t* b_full = bars + 2;      // [2] bulk copy tx
  uint64_t* b_empty = bars + 4;     // [2] MMA commit
  uint64_t* acc_full = bars + 6;    // [4] MMA commit -> epilogue
  uint64_t* acc_empty = bars + 10;  // [4] epilogue (256) -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (n + RTM - 1) / RTM;
  if (tid == 0) {
    tc::mbar_init(a_full, 128);
    tc::mbar_init(a_empty, 1);
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&b_full[s], 1); tc::mbar_init(&b_empty[s], 1); }
    for (int b = 0; b < 4; ++b) { tc::mbar_init(&acc_full[b], 1); tc::mbar_init(&acc_empty[b], 256); }
    tc::fence_mbar_init();
  }
  if (warp == 12) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producers: US tile
    uint32_t ph = 0;
    const int kq = g.kr / 4;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      tc::mbar_wait(a_empty, ph ^ 1);
      const int64_t p0 = t * RTM;
      for (int idx = tid; idx < RTM * kq; idx += 128) {
        const int p = idx / kq, c = idx - p * kq;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p0 + p < n) v = __ldg(reinterpret_cast<const float4*>(US + (p0 + p) * (int64_t)ldus + 4 * c));
        float4 hi, lo;
        tc::split4(v, hi, lo);
        const int off = (p >> 3) * g.a_sbo + c * A_LBO + (p & 7) * 16;
        *reinterpret_cast<float4*>(a_hi + off) = hi;
        *reinterpret_cast<float4*>(a_lo + off) = lo;
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(a_full);
      ph ^= 1;
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3, half = (warp - 4) >> 2;
    const int et = tid - 128;                    // 0..255
    const int nq = g.nch / 2;                    // channels handled by this thread per chunk
    uint32_t ph[4] = {0, 0, 0, 0};
    int64_t gq = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t p = t * RTM + lg * 32 + lane;
      for (int ch = 0; ch < g.nchunks; ++ch, ++gq) {
        const int b = (int)(gq & 3);
        tc::mbar_wait(&acc_full[b], ph[b]);
        ph[b] ^= 1;
        tc::tc_fence_after();
        const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(b * g.N + half * g.nch);
        // the slot written two chunks ago must have been read by its bulk copy
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        unsigned char* slot = stg + ((gq & 1) * 256 + et) * SLOT;
        for (int j0 = 0; j0 < nq; j0 += 8) {   // 8 channels = 16 TMEM columns per tcgen05.ld
          float v[16];
          tc::tmem_ld16(tb + 2 * j0, v);
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            const float2 z0 = cis_exp(v[2 * q], v[2 * q + 1]);
            const float2 z1 = cis_exp(v[2 * q + 2], v[2 * q + 3]);
            if (imag_only) *reinterpret_cast<float2*>(slot + (j0 + q) * 4) = make_float2(z0.y, z1.y);
            else *reinterpret_cast<float4*>(slot + (j0 + q) * 8) = make_float4(z0.x, z0.y, z1.x, z1.y);
          }
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&acc_empty[b]);
        const int c0 = ch * g.nch + half * nq;
        const int nvalid = min(nq, M - c0);
        if (p < n && nvalid > 0) {
          const uint32_t es = imag_only ? 4u : 8u;
          unsigned char* gdst = reinterpret_cast<unsigned char*>(out) + ((size_t)p * M + c0) * es;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                       "r"(tc::smem_u32(slot)), "r"((uint32_t)nvalid * es)
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp == 12 && lane == 0) {
    // ------------------------------------------------------------ B loader + MMA issue
    const uint32_t idesc = tc::make_idesc_tf32(RTM, g.N, false, false);
    const uint32_t sa_hi = tc::smem_u32(a_hi), sa_lo = tc::smem_u32(a_lo), sb = tc::smem_u32(bst);
    uint32_t a_ph = 0, bf_ph[2] = {0, 0}, be_ph[2] = {0, 0}, ae_ph[4] = {0, 0, 0, 0};
    int64_t gq = 0;
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total = my_tiles * g.nchunks;
    if (total > 0) bulk_g2s(sb, bimg, g.b_stage, &b_full[0]);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      tc::mbar_wait(a_full, a_ph);
      a_ph ^= 1;
      tc::tc_fence_after();
      for (int ch = 0; ch < g.nchunks; ++ch, ++gq) {
        // prefetch the next chunk's B into the other stage (its previous MMAs must be done)
        if (gq + 1 < total) {
          const int s1 = (int)((gq + 1) & 1);
          if (gq >= 1) { tc::mbar_wait(&b_empty[s1], be_ph[s1]); be_ph[s1] ^= 1; }
          const int ch1 = (int)((gq + 1) % g.nchunks);
          bulk_g2s(sb + s1 * g.b_stage, reinterpret_cast<const unsigned char*>(bimg) + (size_t)ch1 * g.b_stage,
                   g.b_stage, &b_full[s1]);
        }
        const int s = (int)(gq & 1);
        tc::mbar_wait(&b_full[s], bf_ph[s]);
        bf_ph[s] ^= 1;
        const int b = (int)(gq & 3);
        if (gq >= 4) { tc::mbar_wait(&acc_empty[b], ae_ph[b]); ae_ph[b] ^= 1; }
        tc::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * g.N);
        const uint32_t bh = sb + s * g.b_stage, bl = bh + g.b_part;
        for (int ks = 0; ks < g.kr / 8; ++ks) {
          const uint64_t dah = tc::make_sdesc(sa_hi + ks * 2 * A_LBO, A_LBO, g.a_sbo);
          const uint64_t dal = tc::make_sdesc(sa_lo + ks * 2 * A_LBO, A_LBO, g.a_sbo);
          const uint64_t dbh = tc::make_sdesc(bh + ks * 2 * B_LBO, B_LBO, g.b_sbo);
          const uint64_t dbl = tc::make_sdesc(bl + ks * 2 * B_LBO, B_LBO, g.b_sbo);
          tc::mma_tf32(d, dal, dbh, idesc, ks > 0 ? 1u : 0u);
          tc::mma_tf32(d, dah, dbl, idesc, 1u);
          tc::mma_tf32(d, dah, dbh, idesc, 1u);
        }
        tc::mma_commit(&b_empty[s]);
        tc::mma_commit(&acc_full[b]);
      }
      tc::mma_commit(a_empty);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 12) tc::tmem_dealloc(tmem, 512);
}

// B image: per chunk ch, part (hi, lo), row r (= 2*local channel + {amp, ph}), K index i.
__global__ void build_bimg_kernel(const float* __restrict__ Bi, int k, int M, float* __restrict__ bimg) {
  const RtGeom g = rt_geom(k, M);
  const int64_t total = (int64_t)g.nchunks * g.N * g.kr;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % g.kr);
    const int r = (int)((e / g.kr) % g.N);
    const int ch = (int)(e / ((int64_t)g.kr * g.N));
    const int c = ch * g.nch + (r >> 1);
    float v = 0.f;
    if (c < M && i < k) v = Bi[((int64_t)i * M + c) * 2 + (r & 1)];
    float hi, lo;
    tc::split_tf32(v, hi, lo);
    const int64_t base = (int64_t)ch * g.b_stage + (r >> 3) * g.b_sbo + (i >> 2) * B_LBO + (r & 7) * 16 + (i & 3) * 4;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bimg) + base) = hi;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bimg) + base + g.b_part) = lo;
  }
}

size_t rt_smem(int k, int M) {
  const RtGeom g = rt_geom(k, M);
  return (size_t)2 * g.a_bytes + 2 * (size_t)g.b_stage + 2 * 256 * SLOT + 16 * 8 + 64;
}

}  // namespace

size_t reconstruct_tc_bimg_floats(int k, int M) {
  const RtGeom g = rt_geom(k, M);
  return (size_t)g.nchunks * g.b_stage / 4;
}

void launch_build_bimg(const float* Bi, int k, int M, float* bimg, cudaStream_t s) {
  build_bimg_kernel<<<256, 256, 0, s>>>(Bi, k, M, bimg);
  check_launch("build_bimg");
}

void launch_reconstruct_tc(const float* US, int64_t n, int k, int ldus, const float* bimg, int M, void* out,
                           int out_imag_only, cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = rt_smem(k, M);
  if (smem > 227 * 1024) throw Status(10, "reconstruct_tc: k too large for the smem tile");
  FKK_CUDA_CHECK(cudaFuncSetAttribute(reconstruct_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (n + RTM - 1) / RTM;
  const int grid = (int)std::min<int64_t>(ntiles, sms);
  reconstruct_tc_kernel<<<grid, RT_THREADS, smem, s>>>(US, n, k, ldus, bimg, M, out, out_imag_only);
  check_launch("reconstruct_tc");
}

}  // namespace fkk
