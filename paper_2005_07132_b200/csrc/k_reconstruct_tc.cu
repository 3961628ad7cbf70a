// Reconstruction (F11, Eq. 23) on the 5th-generation tensor cores:
//   K[p, c] = exp(sum_i US[p,i] B_amp[i,c]) * (cos + i sin)(sum_i US[p,i] B_ph[i,c])
// as one GEMM D = US . B^T per 128-pixel tile and NCH-channel chunk, B's rows interleaved
// (amp_c, ph_c) so TMEM columns (2j, 2j+1) are the exponent and phase of channel j; 3xTF32
// (hi*hi + hi*lo + lo*hi; K = kr = roundup8(k) is short, so one TMEM accumulator suffices).
//   warps 0-3  : producers - the US tile (128 x kr), one pixel row per thread -> tf32 hi/lo ->
//                TENSOR memory (tcgen05.st; A slots double-buffered when they fit), where the MMAs
//                read the A operand: shared memory carries only the B chunks (the smem-A version
//                re-read the 128 x kr A tile for every 64-column chunk: ~4.6 MB of smem reads per tile)
//   warps 4-11 : epilogue  - tcgen05.ld, exp/sincos into a swizzled smem box [128 px][half chunk]
//                (one pixel row per thread, conflict-free through the TMA swizzle), then ONE 2-D
//                TMA tensor store per box (cp.async.bulk.tensor, out-of-range rows / channels
//                clipped by the TMA unit); boxes double-buffered per half; 4 TMEM accumulators
//                rotate.  (The previous per-thread 128-B bulk copies issued 44 M TMA operations at
//                cfg3 and ran at 2.7 ms.)
//   warp 12    : TMEM alloc; B-chunk bulk copies (cp.async.bulk, mbarrier tx) and the MMA issue
// B is pre-staged once per basis in global memory in the exact K-major smem image (hi, lo).
// Persistent CTAs walk pixel tiles; the B chunk sequence repeats per tile (L2-resident, ~1 MB).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "fkk_internal.h"
#include "tc_common.cuh"
#include "tma.h"

namespace fkk {

namespace {

constexpr int RTM = 128;          // pixels per tile (UMMA M)
constexpr int RT_PARTS = 4;       // epilogue: 4 warps per TMEM lane group, each a quarter of the chunk
constexpr int RT_EPI = 128 * RT_PARTS;
constexpr int RT_THREADS = 128 + RT_EPI + 64;   // + MMA warp + B loader warp
constexpr int A_LBO = 128;        // unpadded (the A tile is stored once per tile; conflicts there are cheap)
constexpr int B_LBO = 128;
static_assert(A_LBO == B_LBO, "the MMA loop advances both descriptors by the same K offset");
#ifndef FKK_RT_NBUF
#define FKK_RT_NBUF 3
#endif
constexpr int RT_NBUF = FKK_RT_NBUF;   // epilogue output boxes per part (a store may lag RT_NBUF - 1 chunks)
constexpr int RT_NBOX_PAIR = 4;        // pair mode: two pair slots of two boxes per part
__host__ __device__ constexpr int rt_nbox(bool pair) { return pair ? RT_NBOX_PAIR : RT_NBUF; }

struct RtGeom {
  int kr, nch, N, nchunks;
  int a_sbo, a_bytes;             // per hi / lo
  int b_sbo, b_part, b_stage;     // part = hi or lo block, stage = hi + lo
};

// Channels per chunk: 32 (N = 64 TMEM columns per accumulator) unless 16 is what buys a second A
// slot (64 < kr <= 96: 4 x 32 + 2 x 2 kr <= 512).  For 96 < kr <= 128 both leave one A slot, and
// 16-channel chunks only double the epilogue's per-chunk barriers / stores and halve the MMA N
// (cfg4, k = 100: 4 channels per thread between two barriers).  FKK_RT_NCH=16|32 forces (A/B only).
inline int rt_pick_nch(int k) {
  const int kr = (k + 7) / 8 * 8;
  static const int force = getenv("FKK_RT_NCH") ? atoi(getenv("FKK_RT_NCH")) : 0;
  if ((force == 16 || force == 32) && (force == 16 || kr <= 128)) return force;
  return (kr <= 64 || (kr > 96 && kr <= 128)) ? 32 : 16;
}

__host__ __device__ inline RtGeom rt_geom(int k, int M, int nch) {
  RtGeom g;
  g.kr = (k + 7) / 8 * 8;
  g.nch = nch;
  g.N = 2 * g.nch;
  g.nchunks = (M + g.nch - 1) / g.nch;
  g.a_sbo = (g.kr / 4) * A_LBO;
  g.a_bytes = (RTM / 8) * g.a_sbo;
  g.b_sbo = (g.kr / 4) * B_LBO;
  g.b_part = (g.N / 8) * g.b_sbo;
  g.b_stage = 2 * g.b_part;
  return g;
}

// TMEM: 4 rotating accumulators (columns [0, 4 N)), then the A slots (hi kr | lo kr), 128-aligned
__host__ __device__ inline int rt_a_base(const RtGeom& g) { return (4 * g.N + 127) & ~127; }
__host__ __device__ inline int rt_a_slots(const RtGeom& g) { return rt_a_base(g) + 4 * g.kr <= 512 ? 2 : 1; }

__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float2 cis_exp(float amp, float ph) {
  // nearest integer by the 1.5 x 2^23 trick (two FADDs on the FMA pipe instead of FRND on the
  // multi-function unit, which the sin / cos / ex2 already load; |ph| / 2 pi < 2^22)
  const float kq = __fsub_rn(__fadd_rn(ph * 0.15915494309189535f, 12582912.0f), 12582912.0f);
  const float r = fmaf(-kq, 6.2831854820251465f, ph);
  const float r2 = fmaf(kq, 1.7484556e-07f, r);
  float sn, cs;
  __sincosf(r2, &sn, &cs);
  const float m = __expf(amp);
  return make_float2(m * cs, m * sn);
}

// output box: 128 pixel rows x (nch/2 channels) of one chunk half; row bytes = 16 B granules
__host__ __device__ inline int rt_row_bytes(const RtGeom& g, int imag_only) {
  return (g.nch / RT_PARTS) * (imag_only ? 4 : 8);
}
__host__ __device__ inline int rt_box_region(const RtGeom& g) { return (RTM * (g.nch / RT_PARTS) * 8 + 1023) / 1024 * 1024; }

// RT_BST: B-chunk stages (bulk copies run RT_BST - 1 chunks ahead); 3 when the smem fits, else 2
// PAIR: the epilogue drains two consecutive chunks per step (one barrier pair, one bulk-store group
// for both; RT_NBOX_PAIR boxes per part = two pair slots) -- half the per-chunk synchronisation
template <int RT_BST, bool PAIR>
__global__ void __launch_bounds__(RT_THREADS, 1)
reconstruct_tc_kernel(const float* __restrict__ US, int64_t n, int k, int ldus, const float* __restrict__ bimg, int M,
                      const __grid_constant__ CUtensorMap tmap_out, int imag_only, int nch) {   // 0 complex, 1 Im, 2 linear real
  extern __shared__ __align__(1024) unsigned char smem[];
  const RtGeom g = rt_geom(k, M, nch);
  // [RT_NBUF][2 halves][box]; the TMA swizzle pattern is a function of the smem address -> 1024-align
  unsigned char* stg = smem + ((1024 - (tc::smem_u32(smem) & 1023)) & 1023);
  unsigned char* bst = stg + rt_nbox(PAIR) * RT_PARTS * rt_box_region(g);   // RT_BST stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(bst + RT_BST * g.b_stage);
  uint64_t* a_full = bars;                      // [2] producers -> MMA (count 128)
  uint64_t* a_empty = bars + 2;                 // [2] MMA commit -> producers
  uint64_t* b_full = bars + 4;                  // [RT_BST] bulk copy tx
  uint64_t* b_empty = b_full + RT_BST;          // [RT_BST] MMA commit
  uint64_t* acc_full = b_empty + RT_BST;        // [4] MMA commit -> epilogue
  uint64_t* acc_empty = acc_full + 4;           // [4] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (n + RTM - 1) / RTM;
  if (tid == 0) {
    for (int a = 0; a < 2; ++a) { tc::mbar_init(&a_full[a], 128); tc::mbar_init(&a_empty[a], 1); }
    for (int s = 0; s < RT_BST; ++s) { tc::mbar_init(&b_full[s], 1); tc::mbar_init(&b_empty[s], 1); }
    for (int b = 0; b < 4; ++b) { tc::mbar_init(&acc_full[b], 1); tc::mbar_init(&acc_empty[b], RT_EPI); }
    tc::fence_mbar_init();
  }
  if (warp == 4 + RT_EPI / 32) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nas = rt_a_slots(g);
  const uint32_t tmem_a = tmem + (uint32_t)rt_a_base(g);   // A slot a: [hi kr | lo kr] columns

  if (warp < 4) {
    // ------------------------------------------------------------ producers: US tile -> TMEM
    const int r = tid;                                        // pixel row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t ph = 0;   // bit s: phase of slot s (bit mask: an indexed array lives in local memory)
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int a = (int)(it % nas);
      tc::mbar_wait(&a_empty[a], ((ph >> a) & 1u) ^ 1u);
      ph ^= 1u << a;
      tc::tc_fence_after();
      const int64_t p = t * RTM + r;
      const float* src = US + p * (int64_t)ldus;
      const uint32_t ta = tmem_a + lane_off + (uint32_t)(a * 2 * g.kr);
      for (int c = 0; c < g.kr; c += 8) {
        float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
        if (p < n) {
          v0 = __ldg(reinterpret_cast<const float4*>(src + c));
          v1 = __ldg(reinterpret_cast<const float4*>(src + c + 4));
        }
        float hi[8], lo[8];
        const float x[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) tc::split_fast(x[i], hi[i], lo[i]);
        tc::tmem_st8(ta + c, hi);
        tc::tmem_st8(ta + g.kr + c, lo);
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&a_full[a]);
    }
  } else if (warp < 4 + RT_EPI / 32) {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3, half = (warp - 4) >> 2;   // half = part (quarter of the chunk)
    const int nq = g.nch / RT_PARTS;             // channels handled by this thread per chunk
    const int rb = rt_row_bytes(g, imag_only);   // 64, 32 or 16 B = TMA swizzle width (16: none)
    const int r = lg * 32 + lane;                // pixel row within the tile
    const int swz = rb >= 32 ? ((r * rb) >> 7) & (rb / 16 - 1) : 0;
    const bool issuer = lg == 0 && lane == 0;
    const uint32_t bar_id = 1 + half;            // named barrier of the 128 threads of this part
    if (issuer) tma::prefetch_map(&tmap_out);
    uint32_t ph = 0;   // bit b: phase of accumulator b (a bit mask: a dynamically indexed array lived in local memory)
    int64_t gq = 0;
    if constexpr (PAIR) {
      auto emitp = [&](unsigned char* rowp, const float* v, int j0, int cnt) {
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          if (q >= cnt) break;
          if (imag_only == 2) {
            const int byte = (j0 + q) * 4;
            const int gsn = (byte >> 4) ^ swz;
            *reinterpret_cast<float2*>(rowp + gsn * 16 + (byte & 15)) = make_float2(v[2 * q], v[2 * q + 2]);
            continue;
          }
          const float2 z0 = cis_exp(v[2 * q], v[2 * q + 1]);
          const float2 z1 = cis_exp(v[2 * q + 2], v[2 * q + 3]);
          if (imag_only) {
            const int byte = (j0 + q) * 4;
            const int gsn = (byte >> 4) ^ swz;
            *reinterpret_cast<float2*>(rowp + gsn * 16 + (byte & 15)) = make_float2(z0.y, z1.y);
          } else {
            const int gsn = ((j0 + q) >> 1) ^ swz;
            *reinterpret_cast<float4*>(rowp + gsn * 16) = make_float4(z0.x, z0.y, z1.x, z1.y);
          }
        }
      };
      const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      const int64_t total = my_tiles * g.nchunks;
      for (int64_t q = 0; q < total; q += 2) {
        const bool two = q + 1 < total;
        const int b0 = (int)(q & 3), b1 = (int)((q + 1) & 3);
        tc::mbar_wait(&acc_full[b0], (ph >> b0) & 1u);
        ph ^= 1u << b0;
        if (two) {
          tc::mbar_wait(&acc_full[b1], (ph >> b1) & 1u);
          ph ^= 1u << b1;
        }
        tc::tc_fence_after();
        // the pair slot's boxes must have been read by the stores of the pair before last
        if (issuer) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(RT_NBOX_PAIR / 2 - 1) : "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        const int slot = (int)((q >> 1) % (RT_NBOX_PAIR / 2));
        unsigned char* box0 = stg + ((slot * 2) * RT_PARTS + half) * rt_box_region(g);
        unsigned char* box1 = stg + ((slot * 2 + 1) * RT_PARTS + half) * rt_box_region(g);
        const uint32_t tb0 = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(b0 * g.N + half * 2 * nq);
        const uint32_t tb1 = two ? tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(b1 * g.N + half * 2 * nq) : tb0;
        if (nq >= 8) {
          for (int j0 = 0; j0 < nq; j0 += 8) {
            float v0[16], v1[16];
            tc::tmem_ld16_x2(tb0 + 2 * j0, tb1 + 2 * j0, v0, v1);   // (a lone last chunk loads its own twice)
            emitp(box0 + r * rb, v0, j0, 8);
            if (two) emitp(box1 + r * rb, v1, j0, 8);
          }
        } else {
          float v0[16], v1[16];
          tc::tmem_ld8(tb0, v0);
          tc::tmem_ld8(tb1, v1);
          emitp(box0 + r * rb, v0, 0, 4);
          if (two) emitp(box1 + r * rb, v1, 0, 4);
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&acc_empty[b0]);
        if (two) tc::mbar_arrive(&acc_empty[b1]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        if (issuer) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) break;
            const int64_t gqu = q + u;
            const int64_t t = blockIdx.x + (gqu / g.nchunks) * gridDim.x;
            const int ch = (int)(gqu % g.nchunks);
            const int c0 = ch * g.nch + half * nq;
            const int x = imag_only ? c0 : 2 * c0;
            tma::store_2d(&tmap_out, tc::smem_u32(u == 0 ? box0 : box1), x, (int)(t * RTM));
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    } else
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int ch = 0; ch < g.nchunks; ++ch, ++gq) {
        const int b = (int)(gq & 3);
        tc::mbar_wait(&acc_full[b], (ph >> b) & 1u);
        ph ^= 1u << b;
        tc::tc_fence_after();
        const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(b * g.N + half * 2 * nq);
        // box buffer of this chunk must have been read by its store from RT_NBUF chunks ago
        if (issuer) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(RT_NBUF - 1) : "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        unsigned char* box = stg + ((gq % RT_NBUF) * RT_PARTS + half) * rt_box_region(g);
        unsigned char* row = box + r * rb;
        auto emit = [&](const float* v, int j0, int cnt) {
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            if (q >= cnt) break;
            if (imag_only == 2) {   // linear real: the amp column itself, US . V^T (reading A26)
              const int byte = (j0 + q) * 4;
              const int gsn = (byte >> 4) ^ swz;
              *reinterpret_cast<float2*>(row + gsn * 16 + (byte & 15)) = make_float2(v[2 * q], v[2 * q + 2]);
              continue;
            }
            const float2 z0 = cis_exp(v[2 * q], v[2 * q + 1]);
            const float2 z1 = cis_exp(v[2 * q + 2], v[2 * q + 3]);
            if (imag_only) {
              const int byte = (j0 + q) * 4;     // two floats = 8 B: half a 16-B granule
              const int gsn = (byte >> 4) ^ swz;
              *reinterpret_cast<float2*>(row + gsn * 16 + (byte & 15)) = make_float2(z0.y, z1.y);
            } else {
              const int gsn = ((j0 + q) >> 1) ^ swz;
              *reinterpret_cast<float4*>(row + gsn * 16) = make_float4(z0.x, z0.y, z1.x, z1.y);
            }
          }
        };
        if (nq >= 8) {
          for (int j0 = 0; j0 < nq; j0 += 8) {   // 8 channels = 16 TMEM columns per tcgen05.ld
            float v[16];
            tc::tmem_ld16(tb + 2 * j0, v);
            emit(v, j0, 8);
          }
        } else {                                 // 4 channels = 8 TMEM columns
          float v[16];
          tc::tmem_ld8(tb, v);
          emit(v, 0, 4);
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&acc_empty[b]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        if (issuer) {
          const int c0 = ch * g.nch + half * nq;
          const int x = imag_only ? c0 : 2 * c0;
          tma::store_2d(&tmap_out, tc::smem_u32(box), x, (int)(t * RTM));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp == 4 + RT_EPI / 32) {
    // ------------------------------------------------------------ B loader + MMA issue (whole warp runs
    // the loop; one elected lane issues -- descriptors stay in uniform registers)
    const uint32_t idesc = tc::make_idesc_tf32(RTM, g.N, false, false);
    const uint32_t sb = tc::smem_u32(bst);
    const uint64_t db00 = tc::make_sdesc(sb, B_LBO, g.b_sbo);
    uint32_t a_ph = 0, bf_ph = 0, ae_ph = 0;   // bit s: phase of stage / slot / accumulator s
    int64_t it = 0;
    int64_t gq = 0;
    const int nks = g.kr / 8;
    // (the B chunks come from the loader warp: the MMA warp never waits on its own commits, so the
    //  tensor pipe gets chunk gq's MMAs while chunk gq-1's are still executing)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int a = (int)(it % nas);
      tc::mbar_wait(&a_full[a], (a_ph >> a) & 1u);
      a_ph ^= 1u << a;
      tc::tc_fence_after();
      const uint32_t tah = tmem_a + (uint32_t)(a * 2 * g.kr), tal = tah + (uint32_t)g.kr;
      for (int ch = 0; ch < g.nchunks; ++ch, ++gq) {
        const int s = (int)(gq % RT_BST);
        tc::mbar_wait(&b_full[s], (bf_ph >> s) & 1);
        bf_ph ^= 1u << s;
        const int b = (int)(gq & 3);
        if (gq >= 4) { tc::mbar_wait(&acc_empty[b], (ae_ph >> b) & 1u); ae_ph ^= 1u << b; }
        tc::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * g.N);
        const uint64_t dbh0 = tc::sdesc_add(db00, (uint32_t)(s * g.b_stage));
        const uint64_t dbl0 = tc::sdesc_add(dbh0, (uint32_t)g.b_part);
        if (tc::elect_one()) {
          for (int ks = 0; ks < nks; ++ks) {
            const uint32_t o = ks * 2 * B_LBO;
            tc::mma_tf32_ts(d, tal + ks * 8, tc::sdesc_add(dbh0, o), idesc, ks > 0 ? 1u : 0u);
            tc::mma_tf32_ts(d, tah + ks * 8, tc::sdesc_add(dbl0, o), idesc, 1u);
            tc::mma_tf32_ts(d, tah + ks * 8, tc::sdesc_add(dbh0, o), idesc, 1u);
          }
          tc::mma_commit(&b_empty[s]);
          tc::mma_commit(&acc_full[b]);
          if (ch == g.nchunks - 1) tc::mma_commit(&a_empty[a]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 5 + RT_EPI / 32) {
    // ------------------------------------------------------------ B-chunk loader (bulk copies, ring of RT_BST)
    const uint32_t sb = tc::smem_u32(bst);
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total = my_tiles * g.nchunks;
    uint32_t be_ph = 0;
    for (int64_t q = 0; q < total; ++q) {
      const int s1 = (int)(q % RT_BST);
      if (q >= RT_BST) { tc::mbar_wait(&b_empty[s1], (be_ph >> s1) & 1); be_ph ^= 1u << s1; }
      const int ch1 = (int)(q % g.nchunks);
      if (tc::elect_one())
        bulk_g2s(sb + s1 * g.b_stage, reinterpret_cast<const unsigned char*>(bimg) + (size_t)ch1 * g.b_stage, g.b_stage,
                 &b_full[s1]);
      __syncwarp();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 4 + RT_EPI / 32) tc::tmem_dealloc(tmem, 512);
}

// B image: per chunk ch, part (hi, lo), row r (= 2*local channel + {amp, ph}), K index i.
__global__ void build_bimg_kernel(const float* __restrict__ Bi, int k, int M, float* __restrict__ bimg, int nch) {
  const RtGeom g = rt_geom(k, M, nch);
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

size_t rt_smem(int k, int M, int RT_BST, bool pair) {
  const RtGeom g = rt_geom(k, M, rt_pick_nch(k));
  return (size_t)rt_nbox(pair) * RT_PARTS * rt_box_region(g) + RT_BST * (size_t)g.b_stage + 20 * 8 + 64 + 1024;
}

}  // namespace

size_t reconstruct_tc_bimg_floats(int k, int M) {
  const RtGeom g = rt_geom(k, M, rt_pick_nch(k));
  return (size_t)g.nchunks * g.b_stage / 4;
}

void launch_build_bimg(const float* Bi, int k, int M, float* bimg, cudaStream_t s) {
  build_bimg_kernel<<<256, 256, 0, s>>>(Bi, k, M, bimg, rt_pick_nch(k));
  check_launch("build_bimg");
}

void launch_reconstruct_tc(const float* US, int64_t n, int k, int ldus, const float* bimg, int M, void* out,
                           int out_imag_only, cudaStream_t s) {
  if (n <= 0) return;
  const int nch = rt_pick_nch(k);
  const RtGeom g0 = rt_geom(k, M, nch);
  if (rt_a_base(g0) + 2 * g0.kr > 512) throw Status(10, "reconstruct_tc: k too large for tensor memory");
  // pair mode when its four boxes per part still leave >= 3 B-chunk stages (cfg3); else one chunk per step
  static const int force_pair = getenv("FKK_RT_PAIR") ? atoi(getenv("FKK_RT_PAIR")) : -1;   // A/B only
  bool pair = force_pair != 0 && rt_smem(k, M, force_pair == 1 ? 2 : 3, true) <= 227 * 1024;
  int bst = 4;
  while (bst > 2 && rt_smem(k, M, bst, pair) > 227 * 1024) --bst;
  const size_t smem = rt_smem(k, M, bst, pair);
  if (smem > 227 * 1024) throw Status(10, "reconstruct_tc: k too large for the smem tile");
  auto kern = pair ? (bst == 4 ? reconstruct_tc_kernel<4, true> : bst == 3 ? reconstruct_tc_kernel<3, true>
                                                                          : reconstruct_tc_kernel<2, true>)
                   : (bst == 4 ? reconstruct_tc_kernel<4, false> : bst == 3 ? reconstruct_tc_kernel<3, false>
                                                                            : reconstruct_tc_kernel<2, false>);
  FKK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (n + RTM - 1) / RTM;
  const int grid = (int)std::min<int64_t>(ntiles, sms);
  const RtGeom g = rt_geom(k, M, nch);
  const int rb = rt_row_bytes(g, out_imag_only);
  const uint64_t cols = out_imag_only ? (uint64_t)M : 2 * (uint64_t)M;
  const CUtensorMap tm = tma::make_2d_f32(out, (uint64_t)n, cols, cols * 4, RTM, rb / 4, rb);
  kern<<<grid, RT_THREADS, smem, s>>>(US, n, k, ldus, bimg, M, tm, out_imag_only, nch);
  check_launch("reconstruct_tc");
}

}  // namespace fkk
