// Projection US = A0 W (F5: US = A V_k = U_k S_k, with W = D_f V_k folding in the
// f-scaling of Eq. 10; also the first GEMM of ML apply, Eq. 25) on the tensor cores, with the
// per-tile column extremes that feed q (Eqs. 13-15; ties -> lowest pixel).
// tcgen05.mma kind::tf32, 3xTF32; M = 128 pixels per tile, N = kp, K = channels in stages of 32.
//   warps 0-7 : producers - A0 tile (128 px x 32 ch) fp32 loads FOUR stages ahead in registers (the
//               kernel streams A0 from HBM: >= 48 KB per SM must be in flight to cover the latency),
//               tf32 hi/lo split, K-major smem (LBO 144 B pad: conflict-free 16-B stores)
//   warps 8-11: epilogue  - tcgen05.ld of the 128 x kp accumulator (TMEM lane = pixel), US row
//               stores, per-column (max, argmax, min, argmin) by warp shuffles + smem
//   warp 12   : TMEM alloc, W-stage bulk copies (cp.async.bulk, mbarrier tx), MMA issue
// W^T is pre-staged (hi, lo) per K-stage in the exact K-major smem image by build_wimg.
// Persistent CTAs walk pixel tiles.  Accuracy: the tensor-core accumulator truncates on each add
// (DESIGN.md "Gram accuracy"), so hi*hi accumulates per 512-channel segment in its own TMEM
// accumulator and the two cross terms in another; the epilogue adds them in fp32 (round to nearest).
// Two accumulator sets alternate between tiles when they fit in the 512 TMEM columns.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "fkk_internal.h"
#include "tc_common.cuh"
#include "tma.h"

namespace fkk {

namespace {

constexpr int PTM = 128;           // pixels per tile
constexpr int PKC = 32;            // channels per stage
constexpr int PA_LBO = 144, PA_SBO = (PKC / 4) * PA_LBO;     // 1152
constexpr int PA_BYTES = (PTM / 8) * PA_SBO;                  // 18432 per hi / lo
constexpr int PB_LBO = 128, PB_SBO = (PKC / 4) * PB_LBO;     // 1024
constexpr int PTHREADS = 416;
constexpr int PPROD = 256;         // producer threads

__host__ __device__ inline int pb_part(int kp) { return (kp / 8) * PB_SBO; }       // hi or lo
__host__ __device__ inline int pb_stage(int kp) { return 2 * pb_part(kp); }
__host__ __device__ inline int p_stage_bytes(int kp) { return 2 * PA_BYTES + pb_stage(kp); }
__host__ __device__ inline int p_nstages(int kp) { return kp <= 64 ? 4 : 3; }
// channels per hi*hi accumulator segment: 512 (the truncating fp32 TMEM accumulation stays within
// the 1e-5 projection bar), longer when the (segments + cross) accumulator set would not leave two
// A slots (128 columns) of tensor memory: k = 100 (kp = 128) at M = 1600 takes 2 segments of 800
__host__ __device__ inline int p_seg_len(int M, int kp) {
  int nseg = (M + 511) / 512;
  while (nseg > 1 && (nseg + 1) * kp > 384) --nseg;
  return (((M + nseg - 1) / nseg) + 31) & ~31;
}
__host__ __device__ inline int p_nseg(int M, int kp) { return (M + p_seg_len(M, kp) - 1) / p_seg_len(M, kp); }
__host__ __device__ inline int p_set_cols(int M, int kp) { return (p_nseg(M, kp) + 1) * kp; }
__host__ __device__ inline int p_nbuf(int M, int kp) { return 2 * p_set_cols(M, kp) <= 512 ? 2 : 1; }

__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(PTHREADS, 1)
project_tc_kernel(const float* __restrict__ A, int64_t n, int M, const float* __restrict__ wimg, int kp,
                  float* __restrict__ US, float* __restrict__ ext_val, int64_t* __restrict__ ext_idx, int k,
                  int64_t row_offset, int want_ext) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int SB = p_stage_bytes(kp);
  const int PSTAGES = p_nstages(kp);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PSTAGES * SB);
  uint64_t* full = bars;                         // [PSTAGES] producers (128) + W tx
  uint64_t* empty = bars + PSTAGES;              // [PSTAGES] MMA commit
  uint64_t* acc_full = bars + 2 * PSTAGES;       // [2]
  uint64_t* acc_empty = acc_full + 2;            // [2] epilogue (128)
  float* red_v = reinterpret_cast<float*>(acc_empty + 2);      // [4 warps][2][128 cols]
  int* red_i = reinterpret_cast<int*>(red_v + 4 * 2 * 128);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_i + 4 * 2 * 128);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (n + PTM - 1) / PTM;
  const int nst = (M + PKC - 1) / PKC;           // K stages per tile
  if (tid == 0) {
    for (int s = 0; s < PSTAGES; ++s) { tc::mbar_init(&full[s], PPROD + 1); tc::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&acc_full[b], 1); tc::mbar_init(&acc_empty[b], 128); }
    tc::fence_mbar_init();
  }
  const int nseg = p_nseg(M, kp), setc = p_set_cols(M, kp), nbuf = p_nbuf(M, kp);
  const int pseg = p_seg_len(M, kp);
  if (warp == 12) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ------------------------------------------------------------ producers
    // item (pixel p, channel quad c4): p = idx >> 3, c4 = idx & 7; 4 items per thread per stage;
    // register slots X0..X3 rotate and hold the next four stages
    float4 X0[4], X1[4];
    int stage = 0;
    uint32_t phase = 0;
    auto load = [&](float4 (&x)[4], int64_t pos) {   // pos = linear (tile, stage) index of this CTA
      const int64_t t = blockIdx.x + (pos / nst) * gridDim.x;
      const int st = (int)(pos % nst);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int idx = tid + PPROD * h;
        const int p = idx >> 3, c4 = idx & 7;
        const int64_t pp = t * PTM + p;
        const int col = st * PKC + 4 * c4;
        x[h] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < ntiles && pp < n && col < M) x[h] = __ldg(reinterpret_cast<const float4*>(A + pp * (int64_t)M + col));
      }
    };
    auto store = [&](const float4 (&x)[4]) {
      tc::mbar_wait(&empty[stage], phase ^ 1);
      unsigned char* sa = smem + stage * SB;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int idx = tid + PPROD * h;
        const int p = idx >> 3, c4 = idx & 7;
        float4 hi, lo;
        tc::split4(x[h], hi, lo);
        const int off = (p >> 3) * PA_SBO + c4 * PA_LBO + (p & 7) * 16;
        *reinterpret_cast<float4*>(sa + off) = hi;
        *reinterpret_cast<float4*>(sa + PA_BYTES + off) = lo;
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&full[stage]);
      if (++stage == PSTAGES) { stage = 0; phase ^= 1; }
    };
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t npos = my_tiles * nst;
    float4 X2[4], X3[4];
    load(X0, 0);
    load(X1, 1);
    load(X2, 2);
    load(X3, 3);
    for (int64_t pos = 0; pos < npos; pos += 4) {   // four register slots: loads run 4 stages ahead
      store(X0);
      load(X0, pos + 4);
      if (pos + 1 >= npos) break;
      store(X1);
      load(X1, pos + 5);
      if (pos + 2 >= npos) break;
      store(X2);
      load(X2, pos + 6);
      if (pos + 3 >= npos) break;
      store(X3);
      load(X3, pos + 7);
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 8;
    uint32_t ph = 0;   // bit s: phase of slot s (bit mask: an indexed array lives in local memory)
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = (int)(it % nbuf);
      tc::mbar_wait(&acc_full[b], (ph >> b) & 1u);
      ph ^= 1u << b;
      tc::tc_fence_after();
      const int row = ew * 32 + lane;
      const int64_t p = t * PTM + row;
      const bool valid = p < n;
      const uint32_t tb = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(b * setc);
      for (int c0 = 0; c0 < kp; c0 += 16) {
        float v[16], w[16];
        tc::tmem_ld16(tb + nseg * kp + c0, v);                 // cross terms
        for (int sg = 0; sg < nseg; ++sg) {                     // + hi*hi segments (fp32 RN)
          tc::tmem_ld16(tb + sg * kp + c0, w);
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] += w[q];
        }
        if (valid) {
#pragma unroll
          for (int q = 0; q < 16; q += 4)
            *reinterpret_cast<float4*>(US + p * kp + c0 + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
        if (want_ext) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            // warp max/min with the smallest row among ties, by redux.sync on order-preserving
            // integer keys (+0 canonicalises -0, which compares equal to it)
            const uint32_t u = __float_as_uint(v[q] + 0.0f);
            const uint32_t key = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
            const uint32_t kM = __reduce_max_sync(0xffffffffu, valid ? key : 0u);
            const uint32_t km = __reduce_min_sync(0xffffffffu, valid ? key : 0xffffffffu);
            const int imax = (int)__reduce_min_sync(0xffffffffu, (valid && key == kM) ? (uint32_t)row : 0x7fffffffu);
            const int imin = (int)__reduce_min_sync(0xffffffffu, (valid && key == km) ? (uint32_t)row : 0x7fffffffu);
            const float vmax = imax == 0x7fffffff ? -INFINITY
                                                  : __uint_as_float((kM & 0x80000000u) ? (kM & 0x7fffffffu) : ~kM);
            const float vmin = imin == 0x7fffffff ? INFINITY
                                                  : __uint_as_float((km & 0x80000000u) ? (km & 0x7fffffffu) : ~km);
            if (lane == 0) {
              red_v[(ew * 2 + 0) * 128 + c0 + q] = vmax;
              red_i[(ew * 2 + 0) * 128 + c0 + q] = imax;
              red_v[(ew * 2 + 1) * 128 + c0 + q] = vmin;
              red_i[(ew * 2 + 1) * 128 + c0 + q] = imin;
            }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[b]);
      if (want_ext) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int c = ew * 32 + lane; c < k; c += 128) {
          float vM = -INFINITY, vm = INFINITY;
          int iM = 0x7fffffff, im = 0x7fffffff;
          for (int w2 = 0; w2 < 4; ++w2) {   // ascending pixel groups: strict compare keeps the lowest row
            const float a = red_v[(w2 * 2) * 128 + c], bmn = red_v[(w2 * 2 + 1) * 128 + c];
            const int ia = red_i[(w2 * 2) * 128 + c], ib = red_i[(w2 * 2 + 1) * 128 + c];
            if (a > vM || (a == vM && ia < iM)) { vM = a; iM = ia; }
            if (bmn < vm || (bmn == vm && ib < im)) { vm = bmn; im = ib; }
          }
          const int64_t o = (t * (int64_t)k + c) * 2;
          ext_val[o] = vM;
          ext_idx[o] = iM == 0x7fffffff ? INT64_MAX : row_offset + t * PTM + iM;
          ext_val[o + 1] = vm;
          ext_idx[o + 1] = im == 0x7fffffff ? INT64_MAX : row_offset + t * PTM + im;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  } else if (warp == 12) {
    // ------------------------------------------------------------ W stages + MMA issue (whole warp runs
    // the loop; one elected lane issues -- descriptors stay in uniform registers)
    const uint32_t idesc = tc::make_idesc_tf32(PTM, kp, false, false);
    const uint32_t sbase = tc::smem_u32(smem);
    const int WB = pb_stage(kp), WP = pb_part(kp);
    const uint64_t da0 = tc::make_sdesc(sbase, PA_LBO, PA_SBO);
    const uint64_t dw0 = tc::make_sdesc(sbase + 2 * PA_BYTES, PB_LBO, PB_SBO);
    // W stage copies run PSTAGES - 1 positions ahead of the MMAs (their L2 latency is not exposed):
    // position q (tile-major, stage-minor) uses slot q % PSTAGES; its W copy is issued once the slot's
    // previous MMAs (position q - PSTAGES) have completed.
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t npos = my_tiles * nst;
    uint32_t wph = 0;                                     // bit s: empty-phase of slot s for the W issuer
    auto issue_w = [&](int64_t q) {
      const int sl = (int)(q % PSTAGES);
      if (q >= PSTAGES) tc::mbar_wait(&empty[sl], ((wph >> sl) & 1) ^ 1);
      wph ^= 1u << sl;
      const int stq = (int)(q % nst);
      if (tc::elect_one())
        bulk_g2s(sbase + sl * SB + 2 * PA_BYTES, reinterpret_cast<const unsigned char*>(wimg) + (size_t)stq * WB, WB,
                 &full[sl]);
      __syncwarp();
    };
    for (int64_t q = 0; q < PSTAGES - 1 && q < npos; ++q) issue_w(q);
    int stage = 0;
    uint32_t phase = 0, ae = 0;   // ae bit b: phase of accumulator b
    int64_t it = 0, pos = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = (int)(it % nbuf);
      if (it >= nbuf) { tc::mbar_wait(&acc_empty[b], (ae >> b) & 1u); ae ^= 1u << b; tc::tc_fence_after(); }
      const uint32_t dset = tmem + (uint32_t)(b * setc);
      const uint32_t dx = dset + nseg * kp;
      for (int st = 0; st < nst; ++st, ++pos) {
        if (pos + PSTAGES - 1 < npos) issue_w(pos + PSTAGES - 1);
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint64_t dah = tc::sdesc_add(da0, (uint32_t)(stage * SB)), dal = tc::sdesc_add(dah, PA_BYTES);
        const uint64_t dbh = tc::sdesc_add(dw0, (uint32_t)(stage * SB)), dbl = tc::sdesc_add(dbh, (uint32_t)WP);
        const int sg = (st * PKC) / pseg;
        const uint32_t dh = dset + sg * kp;
        const bool seg_start = (st * PKC) % pseg == 0;
        if (tc::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < PKC / 8; ++ks) {
            const uint32_t oa = ks * 2 * PA_LBO, ob = ks * 2 * PB_LBO;
            const uint32_t accx = (st > 0 || ks > 0) ? 1u : 0u;
            const uint32_t acch = (!seg_start || ks > 0) ? 1u : 0u;
            tc::mma_tf32(dx, tc::sdesc_add(dal, oa), tc::sdesc_add(dbh, ob), idesc, accx);
            tc::mma_tf32(dx, tc::sdesc_add(dah, oa), tc::sdesc_add(dbl, ob), idesc, 1u);
            tc::mma_tf32(dh, tc::sdesc_add(dah, oa), tc::sdesc_add(dbh, ob), idesc, acch);
          }
          tc::mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == PSTAGES) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::mma_commit(&acc_full[b]);
      __syncwarp();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 12) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------------------------
// TMA + TMEM-A variant (default when the A0 row pitch is a multiple of 16 B).  The A0 tile (128 px x
// 32 ch fp32) arrives by TMA (SWIZZLE_128B, conflict-free row reads); four converter warps read one
// pixel row per thread, split it into tf32 hi/lo (round to nearest) and write both into TENSOR
// memory (tcgen05.st), where the MMAs read the A operand.  The only shared-memory operand stream is
// W (bulk copies from L2), so the kernel is bounded by HBM rather than by shared-memory bandwidth
// (the smem-A version moved ~136 KB of smem traffic per 16 KB of A0, this one ~72 KB).
//   warp 0   : A0 TMA producer (raw ring)        warp 2: W stage producer (W ring)
//   warp 1   : TMEM alloc, MMA issue            warps 4-7, 12-15: converters (warp % 4 = TMEM lane
//                                               quadrant; two warps split the 32 channels of a stage)
//   warps 8-11: epilogue (as above)
constexpr int QKC = 32;                       // channels per stage (one 128-B swizzle row)
constexpr int QA_BYTES = PTM * QKC * 4;       // 16 KB raw tile
constexpr int QTHREADS = 512;
__host__ __device__ inline int q_w_part(int kp) { return kp * QKC * 4; }     // hi or lo: kp rows x 128 B
__host__ __device__ inline int q_nw(int kp) { return kp <= 64 ? 6 : 3; }    // W ring slots
__host__ __device__ inline int q_nraw(int kp) { return (208 * 1024 - q_nw(kp) * 2 * q_w_part(kp)) / QA_BYTES; }
__host__ __device__ inline int q_ring_bytes(int kp) { return q_nraw(kp) * QA_BYTES + q_nw(kp) * 2 * q_w_part(kp); }
// TMEM: accumulator sets at columns [0, nbuf setc), then NA A slots of 2 x 32 columns (hi | lo)
__host__ __device__ inline int q_nbuf(int M, int kp) { return ((2 * p_set_cols(M, kp) + 127) & ~127) + 2 * 2 * QKC <= 512 ? 2 : 1; }
__host__ __device__ inline int q_abase(int M, int kp) { return (q_nbuf(M, kp) * p_set_cols(M, kp) + 127) & ~127; }
__host__ __device__ inline int q_na(int M, int kp) { return (512 - q_abase(M, kp)) / (2 * QKC); }

// SWIZZLE_128B K-major descriptor: 8-row x 128-B atoms stacked at SBO = 1024 B, LBO unused,
// layout type 2 (bits 61-63); the K offset inside the atom advances the start address.
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// ring cursor: slot and phase parity of consecutive positions in a ring of n slots
struct Ring {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) { slot = 0; phase ^= 1; }
  }
};

__global__ void __launch_bounds__(QTHREADS, 1)
project_tma_kernel(const __grid_constant__ CUtensorMap amap, int64_t n, int M, const float* __restrict__ wimg, int kp,
                   float* __restrict__ US, float* __restrict__ ext_val, int64_t* __restrict__ ext_idx, int k,
                   int64_t row_offset, int want_ext, int nbuf, int abase, int NA, const float* __restrict__ inv_ref,
                   float floor, int ir_smem, int pseg) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int NR = q_nraw(kp), NW = q_nw(kp);
  const int WP = q_w_part(kp);
  unsigned char* ring_a = smem;                              // [NR][16 KB]
  unsigned char* ring_w = ring_a + NR * QA_BYTES;            // [NW][2 WP]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + q_ring_bytes(kp));
  uint64_t* a_full = bars;               // [NR] TMA tx
  uint64_t* a_empty = a_full + NR;       // [NR] converters (4 warps)
  uint64_t* w_full = a_empty + NR;       // [NW] bulk tx
  uint64_t* w_empty = w_full + NW;       // [NW] MMA commit
  uint64_t* t_full = w_empty + NW;       // [NA] converters (4 warps): A hi/lo in TMEM
  uint64_t* t_empty = t_full + NA;       // [NA] MMA commit
  uint64_t* acc_full = t_empty + NA;     // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2] epilogue (128)
  float* red_v = reinterpret_cast<float*>(acc_empty + 2);      // [4 warps][2][128 cols]
  int* red_i = reinterpret_cast<int*>(red_v + 4 * 2 * 128);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_i + 4 * 2 * 128);
  // inv_ref staged in shared memory (raw-cube mode, when it fits): the converters' per-stage L1 loads
  // of it were their largest stall
  float* sir = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) & ~(uintptr_t)15);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (n + PTM - 1) / PTM;
  const int nst = (M + QKC - 1) / QKC;
  if (tid == 0) {
    for (int s2 = 0; s2 < NR; ++s2) { tc::mbar_init(&a_full[s2], 1); tc::mbar_init(&a_empty[s2], 8); }
    for (int s2 = 0; s2 < NW; ++s2) { tc::mbar_init(&w_full[s2], 1); tc::mbar_init(&w_empty[s2], 1); }
    for (int s2 = 0; s2 < NA; ++s2) { tc::mbar_init(&t_full[s2], 8); tc::mbar_init(&t_empty[s2], 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&acc_full[b], 1); tc::mbar_init(&acc_empty[b], 128); }
    tc::fence_mbar_init();
    tma::prefetch_map(&amap);
  }
  const int nseg = (M + pseg - 1) / pseg, setc = (nseg + 1) * kp;
  if (ir_smem)
    for (int c = tid; c < ((M + 31) & ~31); c += blockDim.x) sir[c] = inv_ref[c];
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_a = tmem + (uint32_t)abase;   // A slots
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t npos = my_tiles * nst;

  if (warp == 0) {
    // ------------------------------------------------------------ A0 TMA producer (raw ring)
    Ring ra;
    for (int64_t pos = 0; pos < npos; ++pos, ra.next(NR)) {
      const int64_t t = blockIdx.x + (pos / nst) * gridDim.x;
      const int st = (int)(pos % nst);
      tc::mbar_wait(&a_empty[ra.slot], ra.phase ^ 1);
      if (tc::elect_one()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&a_full[ra.slot])),
                     "r"((uint32_t)QA_BYTES)
                     : "memory");
        tma::load_2d(&amap, tc::smem_u32(ring_a + ra.slot * QA_BYTES), tc::smem_u32(&a_full[ra.slot]), st * QKC,
                     (int)(t * PTM));
      }
      __syncwarp();
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ W stage producer (W ring, from L2)
    Ring rw;
    for (int64_t pos = 0; pos < npos; ++pos, rw.next(NW)) {
      const int st = (int)(pos % nst);
      tc::mbar_wait(&w_empty[rw.slot], rw.phase ^ 1);
      if (tc::elect_one()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&w_full[rw.slot])),
                     "r"((uint32_t)(2 * WP))
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         tc::smem_u32(ring_w + rw.slot * 2 * WP)),
                     "l"(reinterpret_cast<const unsigned char*>(wimg) + (size_t)st * 2 * WP), "r"((uint32_t)(2 * WP)),
                     "r"(tc::smem_u32(&w_full[rw.slot]))
                     : "memory");
      }
      __syncwarp();
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 12) {
    // ------------------------------------------------------------ converters: smem row -> TMEM hi | lo
    // two warps per TMEM lane quadrant (warps 4-7: channels 0-15 of the stage, 12-15: channels 16-31)
    const int q = warp & 3, r = q * 32 + lane;            // pixel row = TMEM lane
    const int hc = warp >= 12 ? 16 : 0;                    // first channel of this warp's half
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    Ring ra, rt;
    // explicit shared-space loads (the swizzled row and inv_ref): the generic pointers above compile
    // to generic LD.E, whose latency was the converters' largest stall
    const uint32_t ring_a_s = tc::smem_u32(ring_a) + (uint32_t)(r * 128);
    const uint32_t sir_s = tc::smem_u32(sir);
    const float kHalfLn2 = 0.34657359027997264f;
    int st = 0;
    for (int64_t pos = 0; pos < npos; ++pos, ra.next(NR), rt.next(NA)) {
      tc::mbar_wait(&a_full[ra.slot], ra.phase);
      const uint32_t rows = ring_a_s + (uint32_t)(ra.slot * QA_BYTES);
      float x[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int cc = (hc >> 2) + c;   // logical 16-B chunk
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x[4 * c]), "=f"(x[4 * c + 1]), "=f"(x[4 * c + 2]), "=f"(x[4 * c + 3])
                     : "r"(rows + (uint32_t)((cc ^ (r & 7)) << 4)));
      }
      if (inv_ref) {
        // the tile is the raw cube: A0 = 1/2 ln(max(I / I_ref, floor)) here (hardware log2, flush to
        // zero: the argument is >= floor > 0; channels >= M zero like the A0 image), so the log-ratio
        // pass never writes A0 to HBM
        const int c0 = st * QKC + hc;
        // inv_ref is zero-padded to a multiple of 32: broadcast float4 loads, no predication
        float ir[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (ir_smem) {
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(ir[4 * u]), "=f"(ir[4 * u + 1]), "=f"(ir[4 * u + 2]), "=f"(ir[4 * u + 3])
                         : "r"(sir_s + (uint32_t)((c0 + 4 * u) * 4)));
          } else {
            const float4 v4 = __ldg(reinterpret_cast<const float4*>(inv_ref + c0) + u);
            ir[4 * u] = v4.x; ir[4 * u + 1] = v4.y; ir[4 * u + 2] = v4.z; ir[4 * u + 3] = v4.w;
          }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float l2;
          asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(fmaxf(x[i] * ir[i], floor)));
          x[i] = kHalfLn2 * l2;
        }
        const int nvalid = M - c0;   // channels c0 + i, i < nvalid, are real
        if (nvalid < 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = i < nvalid ? x[i] : 0.0f;
        }
      }
      if (++st == nst) st = 0;
      float hi[16], lo[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) tc::split_fast(x[i], hi[i], lo[i]);
      tc::mbar_wait(&t_empty[rt.slot], rt.phase ^ 1);
      tc::tc_fence_after();
      const uint32_t ta = tmem_a + lane_off + (uint32_t)(rt.slot * 2 * QKC) + (uint32_t)hc;
      tc::tmem_st16(ta, hi);
      tc::tmem_st16(ta + QKC, lo);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(&a_empty[ra.slot]);
        tc::mbar_arrive(&t_full[rt.slot]);
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ------------------------------------------------------------ epilogue (as project_tc_kernel)
    const int ew = warp - 8;
    uint32_t ph = 0;   // bit s: phase of slot s (bit mask: an indexed array lives in local memory)
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = (int)(it % nbuf);
      tc::mbar_wait(&acc_full[b], (ph >> b) & 1u);
      ph ^= 1u << b;
      tc::tc_fence_after();
      const int row = ew * 32 + lane;
      const int64_t p = t * PTM + row;
      const bool valid = p < n;
      const uint32_t tb = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(b * setc);
      for (int c0 = 0; c0 < kp; c0 += 16) {
        float v[16], w[16];
        tc::tmem_ld16(tb + nseg * kp + c0, v);
        for (int sg = 0; sg < nseg; ++sg) {
          tc::tmem_ld16(tb + sg * kp + c0, w);
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] += w[q];
        }
        if (valid) {
#pragma unroll
          for (int q = 0; q < 16; q += 4)
            *reinterpret_cast<float4*>(US + p * kp + c0 + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
        if (want_ext) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            // warp max/min with the smallest row among ties, by redux.sync on order-preserving
            // integer keys (+0 canonicalises -0, which compares equal to it)
            const uint32_t u = __float_as_uint(v[q] + 0.0f);
            const uint32_t key = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
            const uint32_t kM = __reduce_max_sync(0xffffffffu, valid ? key : 0u);
            const uint32_t km = __reduce_min_sync(0xffffffffu, valid ? key : 0xffffffffu);
            const int imax = (int)__reduce_min_sync(0xffffffffu, (valid && key == kM) ? (uint32_t)row : 0x7fffffffu);
            const int imin = (int)__reduce_min_sync(0xffffffffu, (valid && key == km) ? (uint32_t)row : 0x7fffffffu);
            const float vmax = imax == 0x7fffffff ? -INFINITY
                                                  : __uint_as_float((kM & 0x80000000u) ? (kM & 0x7fffffffu) : ~kM);
            const float vmin = imin == 0x7fffffff ? INFINITY
                                                  : __uint_as_float((km & 0x80000000u) ? (km & 0x7fffffffu) : ~km);
            if (lane == 0) {
              red_v[(ew * 2 + 0) * 128 + c0 + q] = vmax;
              red_i[(ew * 2 + 0) * 128 + c0 + q] = imax;
              red_v[(ew * 2 + 1) * 128 + c0 + q] = vmin;
              red_i[(ew * 2 + 1) * 128 + c0 + q] = imin;
            }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[b]);
      if (want_ext) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int c = ew * 32 + lane; c < k; c += 128) {
          float vM = -INFINITY, vm = INFINITY;
          int iM = 0x7fffffff, im = 0x7fffffff;
          for (int w2 = 0; w2 < 4; ++w2) {
            const float a = red_v[(w2 * 2) * 128 + c], bmn = red_v[(w2 * 2 + 1) * 128 + c];
            const int ia = red_i[(w2 * 2) * 128 + c], ib = red_i[(w2 * 2 + 1) * 128 + c];
            if (a > vM || (a == vM && ia < iM)) { vM = a; iM = ia; }
            if (bmn < vm || (bmn == vm && ib < im)) { vm = bmn; im = ib; }
          }
          const int64_t o = (t * (int64_t)k + c) * 2;
          ext_val[o] = vM;
          ext_idx[o] = iM == 0x7fffffff ? INT64_MAX : row_offset + t * PTM + iM;
          ext_val[o + 1] = vm;
          ext_idx[o + 1] = im == 0x7fffffff ? INT64_MAX : row_offset + t * PTM + im;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issue (A from TMEM, W from smem)
    const uint32_t idesc = tc::make_idesc_tf32(PTM, kp, false, false);
    Ring rw, rt;
    uint32_t ae = 0;   // bit b: phase of accumulator b
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = (int)(it % nbuf);
      if (it >= nbuf) { tc::mbar_wait(&acc_empty[b], (ae >> b) & 1u); ae ^= 1u << b; tc::tc_fence_after(); }
      const uint32_t dset = tmem + (uint32_t)(b * setc);
      const uint32_t dx = dset + nseg * kp;
      for (int st = 0; st < nst; ++st, rw.next(NW), rt.next(NA)) {
        tc::mbar_wait(&w_full[rw.slot], rw.phase);
        tc::mbar_wait(&t_full[rt.slot], rt.phase);
        tc::tc_fence_after();
        const uint32_t sw = tc::smem_u32(ring_w + rw.slot * 2 * WP);
        const uint64_t dbh = make_sdesc_sw128(sw), dbl = make_sdesc_sw128(sw + WP);
        const uint32_t tah = tmem_a + (uint32_t)(rt.slot * 2 * QKC), tal = tah + QKC;
        const int sg = (st * QKC) / pseg;
        const uint32_t dh = dset + sg * kp;
        const bool seg_start = (st * QKC) % pseg == 0;
        if (tc::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < QKC / 8; ++ks) {
            const uint32_t o = ks * 32;   // 8 tf32 = 32 B along K inside the 128-B swizzle row
            const uint32_t accx = (st > 0 || ks > 0) ? 1u : 0u;
            const uint32_t acch = (!seg_start || ks > 0) ? 1u : 0u;
            tc::mma_tf32_ts(dx, tal + ks * 8, tc::sdesc_add(dbh, o), idesc, accx);
            tc::mma_tf32_ts(dx, tah + ks * 8, tc::sdesc_add(dbl, o), idesc, 1u);
            tc::mma_tf32_ts(dh, tah + ks * 8, tc::sdesc_add(dbh, o), idesc, acch);
          }
          tc::mma_commit(&t_empty[rt.slot]);
          tc::mma_commit(&w_empty[rw.slot]);
          if (st == nst - 1) tc::mma_commit(&acc_full[b]);   // same issuing thread as the MMAs
        }
        __syncwarp();
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// W^T image for the TMA variant, per K-stage st: [hi | lo], each kp rows x 128 B in the SWIZZLE_128B
// K-major layout (16-B chunk index XOR row mod 8).
__global__ void build_wimg_sw_kernel(const double* __restrict__ V, const double* __restrict__ fscale,
                                     const double* __restrict__ cscale, int M, int k, int kp, float* __restrict__ wimg) {
  const int nst = (M + QKC - 1) / QKC;
  const int64_t total = (int64_t)nst * kp * QKC;
  const int WP = q_w_part(kp);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int jj = (int)(e % QKC);
    const int nrow = (int)((e / QKC) % kp);
    const int st = (int)(e / ((int64_t)QKC * kp));
    const int j = st * QKC + jj;
    double v = 0.0;
    if (j < M && nrow < k) {
      v = V[(int64_t)nrow * M + j];
      if (fscale) v *= fscale[j];
      if (cscale) v *= cscale[nrow];
    }
    float hi, lo;
    tc::split_tf32((float)v, hi, lo);
    const int64_t off = (int64_t)st * 2 * WP + nrow * 128 + (((jj >> 2) ^ (nrow & 7)) << 4) + (jj & 3) * 4;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(wimg) + off) = hi;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(wimg) + off + WP) = lo;
  }
}

size_t qt_smem(int kp) {
  return 1024 + (size_t)q_ring_bytes(kp) + 2 * (q_nraw(kp) + q_nw(kp) + 8) * 8 + 4 * 8 + 4 * 2 * 128 * 8 + 64;
}

// TMA variant unless FKK_PROJECT_MODE=0 or the A0 pitch is not a multiple of 16 B
bool project_use_tma(int M, int kp) {
  static int mode = -1;
  if (mode < 0) {
    const char* ev = getenv("FKK_PROJECT_MODE");
    mode = ev ? atoi(ev) : 1;
  }
  return mode != 0 && M % 4 == 0 && qt_smem(kp) <= 227 * 1024 && q_na(M, kp) >= 2;
}

// W^T image per K-stage st: rows n (rank, < kp), K = channel j in the stage, K-major hi/lo.
__global__ void build_wimg_kernel(const double* __restrict__ V, const double* __restrict__ fscale,
                                  const double* __restrict__ cscale, int M, int k, int kp, float* __restrict__ wimg) {
  const int nst = (M + PKC - 1) / PKC;
  const int64_t total = (int64_t)nst * kp * PKC;
  const int WB = pb_stage(kp), WP = pb_part(kp);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int jj = (int)(e % PKC);
    const int nrow = (int)((e / PKC) % kp);
    const int st = (int)(e / ((int64_t)PKC * kp));
    const int j = st * PKC + jj;
    double v = 0.0;
    if (j < M && nrow < k) {
      v = V[(int64_t)nrow * M + j];
      if (fscale) v *= fscale[j];
      if (cscale) v *= cscale[nrow];
    }
    float hi, lo;
    tc::split_tf32((float)v, hi, lo);
    const int64_t off = (int64_t)st * WB + (nrow >> 3) * PB_SBO + (jj >> 2) * PB_LBO + (nrow & 7) * 16 + (jj & 3) * 4;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(wimg) + off) = hi;
    *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(wimg) + off + WP) = lo;
  }
}

size_t pt_smem(int kp) { return (size_t)p_nstages(kp) * p_stage_bytes(kp) + 2 * 4 * 8 + 4 * 8 + 4 * 2 * 128 * 8 + 64; }

}  // namespace

bool project_raw_ok(int M, int kp) { return project_use_tma(M, kp); }

size_t project_tc_wimg_floats(int M, int kp) { return (size_t)((M + PKC - 1) / PKC) * pb_stage(kp) / 4; }

int project_tc_num_blocks(int64_t n) { return (int)((n + PTM - 1) / PTM); }

void launch_build_wimg(const double* V, const double* fscale, const double* cscale, int M, int k, int kp, float* wimg,
                       cudaStream_t s) {
  if (project_use_tma(M, kp))
    build_wimg_sw_kernel<<<256, 256, 0, s>>>(V, fscale, cscale, M, k, kp, wimg);
  else
    build_wimg_kernel<<<256, 256, 0, s>>>(V, fscale, cscale, M, k, kp, wimg);
  check_launch("build_wimg");
}

void launch_project_tc(const float* A, int64_t n, int M, const float* wimg, int k, int kp, float* US, float* ext_val,
                       int64_t* ext_idx, int64_t row_offset, int want_ext, cudaStream_t s, const float* inv_ref,
                       float floor) {
  if (inv_ref && !project_use_tma(M, kp)) throw Status(10, "project_tc: raw-cube input needs the TMA variant");
  if (n <= 0) return;
  if (project_use_tma(M, kp)) {
    if (kp > 128 || kp % 16 || p_set_cols(M, kp) > 512)
      throw Status(10, "project_tc: unsupported rank padding / channel count");
    size_t smem = qt_smem(kp);
    const size_t irbytes = (size_t)((M + 31) & ~31) * sizeof(float) + 32;
    const int ir_smem = (inv_ref && smem + irbytes <= 227 * 1024) ? 1 : 0;
    if (ir_smem) smem += irbytes;
    FKK_CUDA_CHECK(cudaFuncSetAttribute(project_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const CUtensorMap amap = tma::make_2d_f32(A, (uint64_t)n, (uint64_t)M, (uint64_t)M * 4, PTM, QKC, 128);
    const int64_t ntiles = (n + PTM - 1) / PTM;
    const int grid = (int)std::min<int64_t>(ntiles, sms);
    // hi*hi segment length (FKK_PROJECT_SEGLEN: A/B only, a multiple of 32) and the TMEM split it implies
    int pseg = p_seg_len(M, kp);
    if (const char* ev = getenv("FKK_PROJECT_SEGLEN")) pseg = std::max(32, atoi(ev) / 32 * 32);
    const int setc = ((M + pseg - 1) / pseg + 1) * kp;
    if (setc > 512 - 2 * QKC) throw Status(10, "project_tc: segment length leaves no A slot");
    int nbuf = ((2 * setc + 127) & ~127) + 2 * 2 * QKC <= 512 ? 2 : 1;
    int abase = (nbuf * setc + 127) & ~127;
    int na = std::min(8, (512 - abase) / (2 * QKC));
    if (const char* ev = getenv("FKK_PROJECT_NBUF")) {   // A/B only
      nbuf = 1;
      abase = (setc + 127) & ~127;
      na = std::min(8, (512 - abase) / (2 * QKC));
      if (atoi(ev) > 0) na = std::min(na, atoi(ev));
    }
    project_tma_kernel<<<grid, QTHREADS, smem, s>>>(amap, n, M, wimg, kp, US, ext_val, ext_idx, k, row_offset, want_ext,
                                                    nbuf, abase, na, inv_ref, floor, ir_smem, pseg);
    check_launch("project_tma");
    return;
  }
  const size_t smem = pt_smem(kp);
  if (smem > 227 * 1024 || kp > 128 || kp % 16 || p_set_cols(M, kp) > 512)
    throw Status(10, "project_tc: unsupported rank padding / channel count");
  FKK_CUDA_CHECK(cudaFuncSetAttribute(project_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (n + PTM - 1) / PTM;
  const int grid = (int)std::min<int64_t>(ntiles, sms);
  project_tc_kernel<<<grid, PTHREADS, smem, s>>>(A, n, M, wimg, kp, US, ext_val, ext_idx, k, row_offset, want_ext);
  check_launch("project_tc");
}

}  // namespace fkk
