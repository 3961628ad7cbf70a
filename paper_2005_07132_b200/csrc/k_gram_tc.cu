// Gram matrix G0 = A0^T A0 (F2, the normal matrix of the truncated SVD) on the
// 5th-generation tensor cores: tcgen05.mma kind::tf32 with the 3xTF32 split (reading A22):
//   G ~ hi_i hi_j + (hi_i lo_j + lo_i hi_j),  hi = rna_tf32(x), lo = rna_tf32(x - hi).
//
// Accuracy design (measured on B200): the tensor-core fp32 accumulator
// truncates on every add (~0.4 half-ulp bias per tcgen05.mma), so a long TMEM accumulation drifts
// (-3e-5 relative after 8192 pixels).  Hence
//   * hi*hi and the two cross terms accumulate in separate TMEM accumulators (the cross-term sum is
//     2^-11 smaller, its bias negligible);
//   * every GPERIOD = 128 pixels the accumulators are drained by 4 epilogue warps into an fp32
//     running sum held in registers (IEEE round-to-nearest adds), double-buffered so the MMAs on
//     the other accumulator pair continue; every 8192 pixels the running sum is added into this
//     CTA's fp64 partial tile (deterministic; summed over the row splits by gram_tc_reduce).
//
// Tiles: 128 x 128 blocks (ti <= tj) of G; CTA = (tile, row split).  Operands K-major in smem
// (K = pixel): core matrix = 8 channels x 16 B (4 pixels); the KC/4 core matrices of an
// 8-channel group are contiguous (LBO = 128 B), groups SBO = 32*KC + 16 B apart (pad: conflict-free
// 128-bit stores).  A0 is channel-contiguous, so a producer thread loads 4 pixels x 4 channels
// (four float4) and transposes them in registers into four 16-B core-matrix rows.
//   warps 0-7  : producers (fp32 loads one stage ahead in registers, tf32 hi/lo split, st.shared)
//   warps 8-15 : epilogue (tcgen05.ld of TMEM lanes 32*(w%4)..; two warps per lane group, 64 columns
//                each; fp32 running sum in registers, fp64 flush)
//   warp 16    : TMEM allocation and the single-thread tcgen05.mma issue
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "fkk_internal.h"
#include "tc_common.cuh"

namespace fkk {

namespace {

constexpr int GT = 128;                    // tile edge (i and j)
constexpr int GKC = 32;                    // pixels per stage
constexpr int GSTAGES = 3;
constexpr int GPERIOD = 128;               // pixels per TMEM accumulation period
constexpr int GFLUSH = 8192;               // pixels per fp64 flush of the register sum
constexpr int GLBO = 128;                  // K-adjacent core matrices
constexpr int GSBO = (GKC / 4) * GLBO + 16;   // 8-channel groups: 1040 B
constexpr int GOP_BYTES = (GT / 8) * GSBO;    // one 128-channel operand, hi or lo: 16640 B
constexpr int GSTAGE_BYTES = 4 * GOP_BYTES;   // A hi, A lo, B hi, B lo
constexpr int GSMEM = GSTAGES * GSTAGE_BYTES + 256;
constexpr int GPROD = 256;                 // producer threads
constexpr int GTHREADS = 544;
constexpr uint32_t GTMEM_COLS = 512;       // 2 buffers x (hi 128 + mid 128)

static_assert(GFLUSH % GPERIOD == 0 && GPERIOD % GKC == 0, "period layout");

// 4 pixels x 4 channels of A0 (four float4, channel-contiguous rows)
__device__ __forceinline__ void load_block(const float* __restrict__ A, int M, int64_t px0, int64_t pend, int col,
                                           float4 (&x)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    x[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (px0 + q < pend && col < M) x[q] = __ldg(reinterpret_cast<const float4*>(A + (px0 + q) * (int64_t)M + col));
  }
}
// -> tf32 hi/lo -> four 16-B K-major core-matrix rows (channel c4*4+e, pixels 4*p4..4*p4+3)
__device__ __forceinline__ void store_block(const float4 (&x)[4], unsigned char* hi_base, unsigned char* lo_base,
                                            int c4, int p4) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int r = c4 * 4 + e;
    const int off = (r >> 3) * GSBO + p4 * GLBO + (r & 7) * 16;
    const float v0 = e == 0 ? x[0].x : e == 1 ? x[0].y : e == 2 ? x[0].z : x[0].w;
    const float v1 = e == 0 ? x[1].x : e == 1 ? x[1].y : e == 2 ? x[1].z : x[1].w;
    const float v2 = e == 0 ? x[2].x : e == 1 ? x[2].y : e == 2 ? x[2].z : x[2].w;
    const float v3 = e == 0 ? x[3].x : e == 1 ? x[3].y : e == 2 ? x[3].z : x[3].w;
    float4 h, l;
    tc::split_fast(v0, h.x, l.x);
    tc::split_fast(v1, h.y, l.y);
    tc::split_fast(v2, h.z, l.z);
    tc::split_fast(v3, h.w, l.w);
    *reinterpret_cast<float4*>(hi_base + off) = h;
    *reinterpret_cast<float4*>(lo_base + off) = l;
  }
}

__global__ void __launch_bounds__(GTHREADS, 1)
gram_tc_kernel(const float* __restrict__ A, int64_t n, int M, const int2* __restrict__ tiles, int ntiles,
               double* __restrict__ partials) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GSTAGES * GSTAGE_BYTES);
  uint64_t* full = bars;                  // [GSTAGES]  producers -> MMA
  uint64_t* empty = bars + GSTAGES;       // [GSTAGES]  MMA commit -> producers
  uint64_t* acc_full = bars + 2 * GSTAGES;    // [2] MMA commit -> epilogue
  uint64_t* acc_empty = acc_full + 2;         // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = blockIdx.x % ntiles, split = blockIdx.x / ntiles, nsplit = gridDim.x / ntiles;
  const int ti = tiles[t].x, tj = tiles[t].y;
  const bool diag = ti == tj;
  const int64_t rb = n * split / nsplit, re = n * (split + 1) / nsplit;
  const int64_t nper = re > rb ? (re - rb + GPERIOD - 1) / GPERIOD : 0;

  if (tid == 0) {
    for (int s = 0; s < GSTAGES; ++s) { tc::mbar_init(&full[s], GPROD); tc::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&acc_full[b], 1); tc::mbar_init(&acc_empty[b], 256); }
    tc::fence_mbar_init();
  }
  if (warp == 16) tc::tmem_alloc(tmem_slot, GTMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ------------------------------------------------------------ producers (one item per operand)
    const int c4 = tid & 31, p4 = tid >> 5;     // channel quad, pixel quad
    float4 xa[4], xb[4];
    int64_t k0 = rb;
    if (k0 < re) {
      load_block(A, M, k0 + 4 * p4, re, ti * GT + 4 * c4, xa);
      if (!diag) load_block(A, M, k0 + 4 * p4, re, tj * GT + 4 * c4, xb);
    }
    int stage = 0;
    uint32_t phase = 0;
    for (; k0 < re; k0 += GKC) {
      tc::mbar_wait(&empty[stage], phase ^ 1);
      unsigned char* st = smem + stage * GSTAGE_BYTES;
      store_block(xa, st, st + GOP_BYTES, c4, p4);
      if (!diag) store_block(xb, st + 2 * GOP_BYTES, st + 3 * GOP_BYTES, c4, p4);
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&full[stage]);
      if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
      const int64_t kn = k0 + GKC;           // prefetch the next stage into registers
      if (kn < re) {
        load_block(A, M, kn + 4 * p4, re, ti * GT + 4 * c4, xa);
        if (!diag) load_block(A, M, kn + 4 * p4, re, tj * GT + 4 * c4, xb);
      }
    }
  } else if (warp < 16) {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3;                       // TMEM lane group (warp % 4)
    const int chalf = (warp - 8) >> 2;             // column half: 0 -> 0..63, 1 -> 64..127
    const int i = lg * 32 + lane;                  // tile row
    double* part = partials + (int64_t)blockIdx.x * (GT * GT);   // [j][i]
    float S[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) S[q] = 0.f;
    uint32_t ph = 0;   // bit b: phase of accumulator b (bit mask, not an indexed array)
    bool first = true;
    for (int64_t pidx = 0; pidx < nper; ++pidx) {
      const int b = (int)(pidx & 1);
      tc::mbar_wait(&acc_full[b], ((ph >> b) & 1u));
      ph ^= 1u << b;
      tc::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(256 * b + 64 * chalf);
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        float h[16], m[16];
        tc::tmem_ld16(tb + cb * 16, h);
        tc::tmem_ld16(tb + 128 + cb * 16, m);
#pragma unroll
        for (int q = 0; q < 16; ++q) S[cb * 16 + q] += h[q] + m[q];
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[b]);
      const bool last = pidx == nper - 1;
      if (last || ((pidx + 1) * GPERIOD) % GFLUSH == 0) {
        // fp64 flush in batches of 16: the batch's loads are issued together (one L2 round trip per
        // batch; load/store interleaving per entry serialised 64 round trips, which stalled the MMA
        // warp on acc_empty for ~18% of the kernel)
#pragma unroll
        for (int q0 = 0; q0 < 64; q0 += 16) {
          double old[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) old[u] = first ? 0.0 : part[(int64_t)(64 * chalf + q0 + u) * GT + i];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            part[(int64_t)(64 * chalf + q0 + u) * GT + i] = old[u] + (double)S[q0 + u];
            S[q0 + u] = 0.f;
          }
        }
        first = false;
      }
    }
    if (nper == 0)
      for (int q = 0; q < 64; ++q) part[(int64_t)(64 * chalf + q) * GT + i] = 0.0;
  } else {
    // ------------------------------------------------------------ MMA issue (warp 16 runs the loop; one
    // elected lane issues -- descriptors stay in uniform registers)
    constexpr uint32_t idesc = tc::make_idesc_tf32(GT, GT, false, false);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t eph = 0;   // bit b: phase of acc_empty[b]
    const uint32_t sbase = tc::smem_u32(smem);
    const uint64_t d00 = tc::make_sdesc(sbase, GLBO, GSBO);
    for (int64_t pidx = 0; pidx < nper; ++pidx) {
      const int b = (int)(pidx & 1);
      if (pidx >= 2) {
        tc::mbar_wait(&acc_empty[b], ((eph >> b) & 1u));
        eph ^= 1u << b;
        tc::tc_fence_after();
      }
      const uint32_t d_hi = tmem + 256 * b, d_mid = d_hi + 128;
      const int64_t p0 = rb + pidx * GPERIOD, p1 = (re < p0 + GPERIOD) ? re : (p0 + GPERIOD);
      uint32_t acc = 0;
      for (int64_t k0 = p0; k0 < p1; k0 += GKC) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint64_t dah = tc::sdesc_add(d00, (uint32_t)(stage * GSTAGE_BYTES)), dal = tc::sdesc_add(dah, GOP_BYTES);
        const uint64_t dbh = diag ? dah : tc::sdesc_add(dah, 2 * GOP_BYTES);
        const uint64_t dbl = diag ? dal : tc::sdesc_add(dah, 3 * GOP_BYTES);
        if (tc::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < GKC / 8; ++ks) {
            const uint32_t ko = ks * 2 * GLBO;   // 8 pixels = 2 K-core matrices
            tc::mma_tf32(d_mid, tc::sdesc_add(dal, ko), tc::sdesc_add(dbh, ko), idesc, acc);   // lo_i * hi_j
            tc::mma_tf32(d_mid, tc::sdesc_add(dah, ko), tc::sdesc_add(dbl, ko), idesc, 1);     // hi_i * lo_j
            tc::mma_tf32(d_hi, tc::sdesc_add(dah, ko), tc::sdesc_add(dbh, ko), idesc, acc);    // hi_i * hi_j
            acc = 1;
          }
          tc::mma_commit(&empty[stage]);
        }
        acc = 1;
        __syncwarp();
        if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::mma_commit(&acc_full[b]);
      __syncwarp();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 16) tc::tmem_dealloc(tmem, GTMEM_COLS);
}

// ---------------------------------------------------------------------------------------------
// Pre-split variant.  The log-ratio pass (F1) also writes A0 in the exact smem image the MMA reads:
// per 128-channel block cb and 32-pixel stage q, the tf32 hi and lo K-major core-matrix blocks
// (GOP_BYTES each, padding included) at Apre + ((cb nq + q) 2 + part) GOP_BYTES.  The Gram CTA then
// needs no producer threads: one loader lane bulk-copies (cp.async.bulk, mbarrier tx) 2 or 4 blocks
// per stage, so the A0 stream has no register lookahead limit and no transposes on the Gram's SMs.
// Pixels >= n and channels >= M are zero in the image; split boundaries are stage aligned.
__device__ __forceinline__ float half_ln(float x) {
  float l2;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(x));
  return 0.34657359027997264f * l2;   // ln 2 / 2
}

__global__ void __launch_bounds__(256, 4) logratio_pre_kernel(const float* __restrict__ I, int64_t n, int M,
                                                           const float* __restrict__ inv_ref, float floor,
                                                           float* __restrict__ A, unsigned char* __restrict__ Apre,
                                                           int64_t nq, int nT, int* __restrict__ flags, int raw) {
  // the image block (hi + lo, 2 GOP_BYTES) is assembled in shared memory and leaves with ONE bulk
  // copy (full-line writes); double-buffered; the next item's I loads are issued before this item's
  // arithmetic (register prefetch)
  extern __shared__ __align__(128) unsigned char simg[];   // [2][2 GOP_BYTES]
  const int c4 = threadIdx.x & 31, p4 = threadIdx.x >> 5;
  int bad = 0;
  const int64_t items = nq * nT;
  float4 xn[4];
  auto load = [&](int64_t it) {
    const int64_t q = it / nT;
    const int col = (int)(it - q * nT) * GT + 4 * c4;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t px = q * GKC + 4 * p4 + e;
      xn[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (it < items && px < n && col < M) xn[e] = __ldcs(reinterpret_cast<const float4*>(I + px * (int64_t)M + col));
    }
  };
  load(blockIdx.x);
  const int buf = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t q = it / nT;
    const int cb = (int)(it - q * nT);
    const int col = cb * GT + 4 * c4;
    float4 x[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = xn[e];
    load(it + gridDim.x);
    float4 ir = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!raw && col < M) ir = *reinterpret_cast<const float4*>(inv_ref + col);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t px = q * GKC + 4 * p4 + e;
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
      if (px < n && col < M) {
        const float4 v = x[e];
        bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
        if (raw) {   // image of the raw cube (the conventional workflow's SVD, reading A26)
          o = v;
        } else {
          // hardware log2 (<= 2 ulp, as the projection's raw-cube converters: reading A25); the
          // argument is >= floor > 0, so flush-to-zero never applies
          o.x = half_ln(fmaxf(v.x * ir.x, floor));
          o.y = half_ln(fmaxf(v.y * ir.y, floor));
          o.z = half_ln(fmaxf(v.z * ir.z, floor));
          o.w = half_ln(fmaxf(v.w * ir.w, floor));
        }
        if (A) *reinterpret_cast<float4*>(A + px * (int64_t)M + col) = o;   // A == nullptr: image only
      }
      x[e] = o;
    }
    // the single buffer was last read by the bulk store issued one item ago (its smem reads finish
    // while this item's loads and logs run); one buffer -> 33 KB per CTA, 4 CTAs per SM
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
    unsigned char* hi = simg + buf * 2 * GOP_BYTES;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = c4 * 4 + e;
      const int off = (r >> 3) * GSBO + p4 * GLBO + (r & 7) * 16;
      const float v0 = e == 0 ? x[0].x : e == 1 ? x[0].y : e == 2 ? x[0].z : x[0].w;
      const float v1 = e == 0 ? x[1].x : e == 1 ? x[1].y : e == 2 ? x[1].z : x[1].w;
      const float v2 = e == 0 ? x[2].x : e == 1 ? x[2].y : e == 2 ? x[2].z : x[2].w;
      const float v3 = e == 0 ? x[3].x : e == 1 ? x[3].y : e == 2 ? x[3].z : x[3].w;
      float4 h, l;
      tc::split_fast(v0, h.x, l.x);
      tc::split_fast(v1, h.y, l.y);
      tc::split_fast(v2, h.z, l.z);
      tc::split_fast(v3, h.w, l.w);
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(hi + GOP_BYTES + off) = l;
    }
    tc::fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned char* dst = Apre + ((size_t)(cb * nq + q) * 2) * GOP_BYTES;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(tc::smem_u32(hi)),
                   "r"((uint32_t)(2 * GOP_BYTES))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, 2);
}

__device__ __forceinline__ void bulk_g2s_g(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

constexpr int GPTHREADS = 320;   // warps 0-7 epilogue, 8 MMA issue, 9 bulk loader

__global__ void __launch_bounds__(GPTHREADS, 1)
gram_pre_kernel(const unsigned char* __restrict__ Apre, int64_t n, int64_t nq, const int2* __restrict__ tiles,
                int ntiles, double* __restrict__ partials, unsigned long long* __restrict__ dbg) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GSTAGES * GSTAGE_BYTES);
  uint64_t* full = bars;                  // [GSTAGES]  bulk copies (tx) -> MMA
  uint64_t* empty = bars + GSTAGES;       // [GSTAGES]  MMA commit -> loader
  uint64_t* acc_full = bars + 2 * GSTAGES;    // [2] MMA commit -> epilogue
  uint64_t* acc_empty = acc_full + 2;         // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = blockIdx.x % ntiles, split = blockIdx.x / ntiles, nsplit = gridDim.x / ntiles;
  const int ti = tiles[t].x, tj = tiles[t].y;
  const bool diag = ti == tj;
  const int64_t qb = nq * split / nsplit, qe = nq * (split + 1) / nsplit;     // stage range
  constexpr int SPP = GPERIOD / GKC;                                            // stages per period
  const int64_t nper = qe > qb ? (qe - qb + SPP - 1) / SPP : 0;

  if (tid == 0) {
    for (int s = 0; s < GSTAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&acc_full[b], 1); tc::mbar_init(&acc_empty[b], 256); }
    tc::fence_mbar_init();
  }
  if (warp == 8) tc::tmem_alloc(tmem_slot, GTMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ------------------------------------------------------------ epilogue (as gram_tc_kernel)
    const int lg = warp & 3;
    const int chalf = warp >> 2;
    const int i = lg * 32 + lane;
    double* part = partials + (int64_t)blockIdx.x * (GT * GT);   // [j][i]
    float S[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) S[q] = 0.f;
    uint32_t ph = 0;   // bit b: phase of accumulator b (bit mask, not an indexed array)
    bool first = true;
    for (int64_t pidx = 0; pidx < nper; ++pidx) {
      const int b = (int)(pidx & 1);
      tc::mbar_wait(&acc_full[b], ((ph >> b) & 1u));
      ph ^= 1u << b;
      tc::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(256 * b + 64 * chalf);
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        float h[16];
        tc::tmem_ld16(tb + cb * 16, h);
#pragma unroll
        for (int q = 0; q < 16; ++q) S[cb * 16 + q] += h[q];
        tc::tmem_ld16(tb + 128 + cb * 16, h);
#pragma unroll
        for (int q = 0; q < 16; ++q) S[cb * 16 + q] += h[q];
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[b]);
      const bool last = pidx == nper - 1;
      if (last || ((pidx + 1) * GPERIOD) % GFLUSH == 0) {
        // fp64 flush in batches of 16: the batch's loads are issued together (one L2 round trip per
        // batch; load/store interleaving per entry serialised 64 round trips, which stalled the MMA
        // warp on acc_empty for ~18% of the kernel)
#pragma unroll
        for (int q0 = 0; q0 < 64; q0 += 16) {
          double old[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) old[u] = first ? 0.0 : part[(int64_t)(64 * chalf + q0 + u) * GT + i];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            part[(int64_t)(64 * chalf + q0 + u) * GT + i] = old[u] + (double)S[q0 + u];
            S[q0 + u] = 0.f;
          }
        }
        first = false;
      }
    }
    if (nper == 0)
      for (int q = 0; q < 64; ++q) part[(int64_t)(64 * chalf + q) * GT + i] = 0.0;
  } else if (warp == 8) {
    // ------------------------------------------------------------ MMA issue
    constexpr uint32_t idesc = tc::make_idesc_tf32(GT, GT, false, false);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t eph = 0;   // bit b: phase of acc_empty[b]
    const uint64_t d00 = tc::make_sdesc(tc::smem_u32(smem), GLBO, GSBO);
    unsigned long long w_full = 0, w_acc = 0;   // dbg: cycles waiting for operands / for the epilogue
    const unsigned long long t_start = clock64();
    for (int64_t pidx = 0; pidx < nper; ++pidx) {
      const int b = (int)(pidx & 1);
      if (pidx >= 2) {
        const unsigned long long c0 = dbg ? clock64() : 0;
        tc::mbar_wait(&acc_empty[b], ((eph >> b) & 1u));
        if (dbg) w_acc += clock64() - c0;
        eph ^= 1u << b;
        tc::tc_fence_after();
      }
      const uint32_t d_hi = tmem + 256 * b, d_mid = d_hi + 128;
      const int64_t q0 = qb + pidx * SPP, q1 = (qe < q0 + SPP) ? qe : (q0 + SPP);
      uint32_t acc = 0;
      for (int64_t q = q0; q < q1; ++q) {
        const unsigned long long c0 = dbg ? clock64() : 0;
        tc::mbar_wait(&full[stage], phase);
        if (dbg) w_full += clock64() - c0;
        tc::tc_fence_after();
        const uint64_t dah = tc::sdesc_add(d00, (uint32_t)(stage * GSTAGE_BYTES)), dal = tc::sdesc_add(dah, GOP_BYTES);
        const uint64_t dbh = diag ? dah : tc::sdesc_add(dah, 2 * GOP_BYTES);
        const uint64_t dbl = diag ? dal : tc::sdesc_add(dah, 3 * GOP_BYTES);
        if (tc::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < GKC / 8; ++ks) {
            const uint32_t ko = ks * 2 * GLBO;
            tc::mma_tf32(d_mid, tc::sdesc_add(dal, ko), tc::sdesc_add(dbh, ko), idesc, acc);   // lo_i * hi_j
            tc::mma_tf32(d_mid, tc::sdesc_add(dah, ko), tc::sdesc_add(dbl, ko), idesc, 1);     // hi_i * lo_j
            tc::mma_tf32(d_hi, tc::sdesc_add(dah, ko), tc::sdesc_add(dbh, ko), idesc, acc);    // hi_i * hi_j
            acc = 1;
          }
          tc::mma_commit(&empty[stage]);
        }
        acc = 1;
        __syncwarp();
        if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::mma_commit(&acc_full[b]);
      __syncwarp();
    }
    if (dbg && lane == 0) {
      dbg[blockIdx.x * 4 + 0] = clock64() - t_start;
      dbg[blockIdx.x * 4 + 1] = w_full;
      dbg[blockIdx.x * 4 + 2] = w_acc;
      dbg[blockIdx.x * 4 + 3] = (unsigned long long)diag;
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------ bulk loader (warp 9, one lane)
    const uint32_t sbase = tc::smem_u32(smem);
    const uint32_t bytes = (diag ? 2u : 4u) * GOP_BYTES;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t q = qb; q < qe; ++q) {
      tc::mbar_wait(&empty[stage], phase ^ 1);
      const uint32_t st = sbase + stage * GSTAGE_BYTES;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&full[stage])),
                   "r"(bytes)
                   : "memory");
      const unsigned char* a = Apre + ((size_t)(ti * nq + q) * 2) * GOP_BYTES;
      bulk_g2s_g(st, a, 2 * GOP_BYTES, &full[stage]);                       // A hi, A lo (adjacent)
      if (!diag) {
        const unsigned char* bsrc = Apre + ((size_t)(tj * nq + q) * 2) * GOP_BYTES;
        bulk_g2s_g(st + 2 * GOP_BYTES, bsrc, 2 * GOP_BYTES, &full[stage]);  // B hi, B lo
      }
      if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 8) tc::tmem_dealloc(tmem, GTMEM_COLS);
}

__global__ void gram_tc_reduce_kernel(const double* __restrict__ partials, int ntiles, int nsplit, int M,
                                      const int* __restrict__ tile_of, int nT, double* __restrict__ G, int accumulate) {
  const int64_t total = (int64_t)M * M;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / M), c = (int)(e % M);
    const int i = min(r, c), j = max(r, c);
    const int ti = i / GT, tj = j / GT;
    const int t = tile_of[ti * nT + tj];
    const int64_t off = (int64_t)(j - tj * GT) * GT + (i - ti * GT);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += partials[((int64_t)sp * ntiles + t) * (GT * GT) + off];
    G[e] = accumulate ? G[e] + s : s;
  }
}

}  // namespace

// Tile list of the upper triangle of 128 x 128 blocks (ti <= tj).
void gram_tc_tiles(int M, std::vector<int2>& tiles, std::vector<int>& tile_of, int& nT) {
  nT = (M + GT - 1) / GT;
  tiles.clear();
  tile_of.assign((size_t)nT * nT, -1);
  for (int ti = 0; ti < nT; ++ti)
    for (int tj = ti; tj < nT; ++tj) {
      tile_of[ti * nT + tj] = (int)tiles.size();
      tiles.push_back(make_int2(ti, tj));
    }
}

int gram_tc_splits(int ntiles, int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int ns = std::max(1, sms / std::max(1, ntiles));
  // fewer than two tiles per SM (cfg4: 13 blocks, 91 tiles): equal pixel ranges for at least four waves
  // of CTAs -- one CTA per tile left 57 of 148 SMs idle (cfg4 at 1M rows: 18.6 ms with 1 range per
  // tile, 13.1 with 3, 12.8 with 8, 14.2 with 7; 8 to 24 ranges within 1% at 2M rows)
  if (2 * ntiles > sms) {   // and a last wave at least 95% full (91 tiles: 8 ranges = 4.92 waves, not 7 = 4.30)
    const int lo = (4 * sms + ntiles - 1) / ntiles, hi = 2 * lo;
    double best = 0.0;
    ns = lo;
    for (int c = lo; c <= hi; ++c) {
      const int64_t ctas = (int64_t)ntiles * c, waves = (ctas + sms - 1) / sms;
      const double eff = (double)ctas / (double)(waves * sms);
      if (eff > best + 1e-9) { best = eff; ns = c; }
      if (eff >= 0.95) break;
    }
  }
  if (const char* ev = getenv("FKK_GRAM_SPLITS")) ns = std::max(1, atoi(ev));   // A/B only
  const int64_t by_rows = std::max<int64_t>(1, n / 1024);
  return (int)std::min<int64_t>(ns, by_rows);
}

size_t gram_tc_partial_doubles(int ntiles, int nsplit) { return (size_t)ntiles * nsplit * GT * GT; }

void launch_gram_tc(const float* A, int64_t n, int M, const int2* d_tiles, int ntiles, int nsplit, double* partials,
                    cudaStream_t s) {
  FKK_CUDA_CHECK(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GSMEM));
  gram_tc_kernel<<<ntiles * nsplit, GTHREADS, GSMEM, s>>>(A, n, M, d_tiles, ntiles, partials);
  check_launch("gram_tc");
}

void launch_gram_tc_reduce(const double* partials, int ntiles, int nsplit, int M, const int* d_tile_of, int nT,
                           double* G, int accumulate, cudaStream_t s) {
  gram_tc_reduce_kernel<<<1024, 256, 0, s>>>(partials, ntiles, nsplit, M, d_tile_of, nT, G, accumulate);
  check_launch("gram_tc_reduce");
}

}  // namespace fkk

namespace fkk {

size_t gram_pre_bytes(int64_t n, int nT) {
  const int64_t nq = (n + GKC - 1) / GKC;
  return (size_t)nT * nq * 2 * GOP_BYTES;
}

void launch_logratio_pre(const float* I, int64_t n, int M, int nT, const float* inv_ref, float floor, float* A,
                         unsigned char* Apre, int* flags, cudaStream_t s, int raw) {
  if (n <= 0) return;
  const int64_t nq = (n + GKC - 1) / GKC;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = nq * nT;
  const int grid = (int)std::min<int64_t>(items, (int64_t)sms * 4);
  const int smem = 2 * GOP_BYTES;
  FKK_CUDA_CHECK(cudaFuncSetAttribute(logratio_pre_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  logratio_pre_kernel<<<grid, 256, smem, s>>>(I, n, M, inv_ref, floor, A, Apre, nq, nT, flags, raw);
  check_launch("logratio_pre");
}

void launch_gram_pre(const unsigned char* Apre, int64_t n, const int2* d_tiles, int ntiles, int nsplit,
                     double* partials, cudaStream_t s) {
  const int64_t nq = (n + GKC - 1) / GKC;
  FKK_CUDA_CHECK(cudaFuncSetAttribute(gram_pre_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GSMEM));
  // FKK_GRAM_DBG (debug only): per-CTA MMA-warp cycle split (total, waiting for operands, waiting
  // for the epilogue) of each launch, printed to stderr; synchronises the stream
  static const bool gdbg = getenv("FKK_GRAM_DBG") != nullptr;
  unsigned long long* dbg = nullptr;
  const int nblk = ntiles * nsplit;
  if (gdbg) FKK_CUDA_CHECK(cudaMalloc(&dbg, (size_t)nblk * 4 * sizeof(unsigned long long)));
  gram_pre_kernel<<<nblk, GPTHREADS, GSMEM, s>>>(Apre, n, nq, d_tiles, ntiles, partials, dbg);
  check_launch("gram_pre");
  if (gdbg) {
    std::vector<unsigned long long> h((size_t)nblk * 4);
    FKK_CUDA_CHECK(cudaMemcpyAsync(h.data(), dbg, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    FKK_CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFree(dbg);
    double tot[2][3] = {{0, 0, 0}, {0, 0, 0}};
    int cnt[2] = {0, 0};
    for (int b = 0; b < nblk; ++b) {
      const int dg = (int)h[b * 4 + 3];
      for (int q = 0; q < 3; ++q) tot[dg][q] += (double)h[b * 4 + q];
      cnt[dg]++;
    }
    for (int dg = 0; dg < 2; ++dg)
      if (cnt[dg])
        fprintf(stderr, "gram_pre dbg %s: %d CTAs, mean cycles total %.0f, wait operands %.0f, wait epilogue %.0f\n",
                dg ? "diag" : "offdiag", cnt[dg], tot[dg][0] / cnt[dg], tot[dg][1] / cnt[dg], tot[dg][2] / cnt[dg]);
  }
}

}  // namespace fkk
