// Direct (conventional) per-spectrum KK + PEC + SEC (Eqs. 3-5), K7 in DESIGN.md.
//   direct_phase  : a = 1/2 ln(max(I/I_ref, floor)); phi = H{a}         (D1-D2, fp32 FFT)
//   als_seg       : phi_err = ALS baseline of phi (k_als.cu)             (D3, fp64, readings A6/A7)
//   direct_finish : a' = a + H{phi_err}; phi' = phi - phi_err; K' = e^{a'} e^{i phi'};
//                   T = SG trend(Re K') (fp64 moments; scalar mean if min T <= 0); K = K'/T  (D4-D5)
//
// One CTA of L/16 threads per PAIR of spectra: H is real-linear, so one complex transform of
// x_ext0 + i x_ext1 gives H{x0} + i H{x1} ("two for one").  The transforms are the radix-16 Stockham
// passes of fft_r16.cuh (compile-time pass plan per L): the forward transform's first pass gathers
// the padded rows through the padding map (reading A3; -1 = zero pad), its last pass applies the
// Hilbert multiplier (-i for 0 < f < L/2, +i above, 0 at DC and Nyquist; readings A2, A4), and the
// inverse transform's last pass hands over the centre M samples.
#include <cuda_runtime.h>
#include <math.h>

#include <cstdlib>
#include <type_traits>

#include "fft_r16.cuh"
#include "fkk_internal.h"

namespace fkk {

namespace {

template <typename TIn>
__device__ __forceinline__ float log_ratio_elem(const TIn v, const float inv_ref, const double ref64, float floor) {
  if constexpr (sizeof(TIn) == 8) {
    double r = (double)v / ref64;
    return (float)(0.5 * log(fmax(r, (double)floor)));
  } else {
    float r = (float)v * inv_ref;
    return 0.5f * __logf(fmaxf(r, floor));   // hardware log (<= 2 ulp; reading A27)
  }
}

// one-dimensional bulk copy global -> shared (TMA engine), completion counted on an mbarrier
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WB_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WB_%=;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// fp64 reciprocal: MUFU seed + two Newton steps (~1 ulp)
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// CTAs per SM the register budget is sized for (launch bounds: 128 registers at L = 2048; 4 measured
// 61.4 ms per cfg3 direct pass against 62.6 ms with 3 CTAs / 168 registers)
#ifndef FKK_DIRECT_MINB
#define FKK_DIRECT_MINB 4
#endif

template <int LOG2L>
__host__ __device__ constexpr int threads_of() { return (1 << LOG2L) / 16 < 32 ? 32 : (1 << LOG2L) / 16; }

// Hilbert transform of the two rows held (as floats) in rows0 / rows1 (inside buffer Y), result
// handed to `out(j, h0, h1)` for the centre samples j < M (scaled by 1/L).  X, Y: padded complex
// length-L buffers.  Every thread of the CTA calls this (the passes idle threads >= L/16).
template <int LOG2L, typename Out>
__device__ __forceinline__ void hilbert_pair(const float2* __restrict__ tw, const int* __restrict__ pmap, int M,
                                             float2* X, float2* Y, const float* rows0, const float* rows1, Out&& out) {
  using PL = fft16::Plan<LOG2L>;
  constexpr int L = PL::L;
  const int pl = (L - M) >> 1;
  const float invL = 1.0f / (float)L;
  auto gather = [&](int i) {
    const int src = __ldg(pmap + i);
    return src < 0 ? make_float2(0.f, 0.f) : make_float2(rows0[src], rows1[src]);
  };
  // forward: pass 0 gather -> X, pass 1 X -> Y, pass 2 Y -> target (NP = 3: X; NP = 2: Y; NP = 1: X)
  float2* tgt = PL::NP == 2 ? Y : X;
  auto mult = [&](int f, float2 v) {
    float2 o;
    if (f == 0 || f == (L >> 1)) o = make_float2(0.f, 0.f);
    else if (f < (L >> 1)) o = make_float2(v.y, -v.x);   // * (-i)
    else o = make_float2(-v.y, v.x);                      // * (+i)
    tgt[fft16::pad(f)] = o;
  };
  if constexpr (PL::NP == 1) fft16::pass<LOG2L, 0, false>(tw, gather, mult);
  else fft16::transform<LOG2L, false>(tw, X, Y, gather, mult);
  __syncthreads();
  // inverse: input tgt; pass 0 tgt -> oth, pass 1 oth -> tgt, pass 2 tgt -> out
  float2* oth = PL::NP == 2 ? X : Y;
  auto ld = [&](int i) { return tgt[fft16::pad(i)]; };
  auto st = [&](int i, float2 v) {
    const int j = i - pl;
    if (j >= 0 && j < M) out(j, v.x * invL, v.y * invL);
  };
  if constexpr (PL::NP == 1) fft16::pass<LOG2L, 0, true>(tw, ld, st);
  else fft16::transform<LOG2L, true>(tw, oth, tgt, ld, st);
}

template <typename TIn, int LOG2L>
__global__ void __launch_bounds__(threads_of<LOG2L>(), (2048 / threads_of<LOG2L>()) * FKK_DIRECT_MINB / 16)
direct_phase_kernel(const TIn* __restrict__ I, int64_t n, int M, const float* __restrict__ inv_ref,
                    const double* __restrict__ ref64, float floor, const float2* __restrict__ tw,
                    const int* __restrict__ pmap, float* __restrict__ phi, int* __restrict__ flags) {
  constexpr int L = 1 << LOG2L, NT = threads_of<LOG2L>();
  constexpr int PADL = fft16::padded_len(L);
  extern __shared__ __align__(16) unsigned char smem[];
  float2* X = reinterpret_cast<float2*>(smem);
  float2* Y = X + PADL;
  float* a0 = reinterpret_cast<float*>(Y);
  float* a1 = a0 + M;
  const int tid = threadIdx.x;
  const int64_t npairs = (n + 1) >> 1;
  int bad = 0;
  for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int64_t r0 = 2 * pr, r1 = r0 + 1;
    const bool has1 = r1 < n;
    const TIn* i0 = I + r0 * (int64_t)M;
    const TIn* i1 = I + r1 * (int64_t)M;
    if constexpr (sizeof(TIn) == 4) {
      for (int q = tid; 4 * q < M; q += NT) {   // M % 4 == 0: float4 rows
        const float4 ir = *reinterpret_cast<const float4*>(inv_ref + 4 * q);
        const float4 v0 = __ldcs(reinterpret_cast<const float4*>(i0) + q);
        const float4 v1 = has1 ? __ldcs(reinterpret_cast<const float4*>(i1) + q) : make_float4(1.f, 1.f, 1.f, 1.f);
        bad |= !isfinite(v0.x) | !isfinite(v0.y) | !isfinite(v0.z) | !isfinite(v0.w);
        bad |= !isfinite(v1.x) | !isfinite(v1.y) | !isfinite(v1.z) | !isfinite(v1.w);
        a0[4 * q] = 0.5f * __logf(fmaxf(v0.x * ir.x, floor));
        a0[4 * q + 1] = 0.5f * __logf(fmaxf(v0.y * ir.y, floor));
        a0[4 * q + 2] = 0.5f * __logf(fmaxf(v0.z * ir.z, floor));
        a0[4 * q + 3] = 0.5f * __logf(fmaxf(v0.w * ir.w, floor));
        a1[4 * q] = 0.5f * __logf(fmaxf(v1.x * ir.x, floor));
        a1[4 * q + 1] = 0.5f * __logf(fmaxf(v1.y * ir.y, floor));
        a1[4 * q + 2] = 0.5f * __logf(fmaxf(v1.z * ir.z, floor));
        a1[4 * q + 3] = 0.5f * __logf(fmaxf(v1.w * ir.w, floor));
      }
    } else {
      for (int j = tid; j < M; j += NT) {
        const TIn v0 = i0[j];
        const TIn v1 = has1 ? i1[j] : (TIn)1;
        bad |= !isfinite(v0) | !isfinite(v1);
        a0[j] = log_ratio_elem<TIn>(v0, inv_ref[j], ref64[j], floor);
        a1[j] = log_ratio_elem<TIn>(v1, inv_ref[j], ref64[j], floor);
      }
    }
    __syncthreads();
    float* p0 = phi + r0 * (int64_t)M;
    float* p1 = phi + r1 * (int64_t)M;
    hilbert_pair<LOG2L>(tw, pmap, M, X, Y, a0, a1, [&](int j, float h0, float h1) {
      p0[j] = h0;
      if (has1) p1[j] = h1;
    });
    __syncthreads();
  }
  if (bad) atomicOr(flags, 2);
}

// ---------------------------------------------------------------------------------------------
// direct_finish: thread t owns the C = ceil(M / NT) <= 8 consecutive channels [tC, tC + C) for the
// pointwise work and the SG trend (reading A8): the order-2 least-squares value in the (2h+1)-window
// centred at c = clamp(j, h, M-1-h), from the window moments Q_k = sum_{i in window} i^k y_i
// (k = 0..2), which come from fp64 prefix sums (chunk prefixes by a block scan plus at most C-1
// partial terms) and slide one channel at a time along a thread's chunk.
struct SgK {
  double n, K2, K4, idet, iK2;
};
__device__ __forceinline__ SgK sg_k(int h) {
  SgK k;
  k.n = 2.0 * h + 1.0;
  const double hd = (double)h;
  k.K2 = hd * (hd + 1.0) * (2.0 * hd + 1.0) / 3.0;
  k.K4 = hd * (hd + 1.0) * (2.0 * hd + 1.0) * (3.0 * hd * hd + 3.0 * hd - 1.0) / 15.0;
  k.idet = 1.0 / (k.n * k.K4 - k.K2 * k.K2);
  k.iK2 = 1.0 / k.K2;
  return k;
}
// branch-free form: at j = c the linear and quadratic terms are exact zeros
__device__ __forceinline__ double sg_eval_full(double Q0, double Q1, double Q2, int c, int j, const SgK& k) {
  const double cd = (double)c;
  const double S0 = Q0, S1 = Q1 - cd * Q0, S2 = Q2 - 2.0 * cd * Q1 + cd * cd * Q0;
  const double c0 = (k.K4 * S0 - k.K2 * S2) * k.idet;
  const double c2 = (k.n * S2 - k.K2 * S0) * k.idet;
  const double c1 = S1 * k.iK2;
  const double d = (double)(j - c);
  return fma(fma(c2, d, c1), d, c0);
}

// PF: the phi_err rows of the NEXT pair are bulk-copied into a staging buffer while this pair's SG
// trend runs, and this pair's I / phi rows are prefetched into L2 before its transforms (fp32 input,
// M % 4 == 0).
template <typename TIn, int LOG2L, bool PF>
__global__ void __launch_bounds__(threads_of<LOG2L>(), (2048 / threads_of<LOG2L>()) * FKK_DIRECT_MINB / 16)
direct_finish_kernel(const TIn* __restrict__ I, int64_t n, int M, const float* __restrict__ inv_ref,
                     const double* __restrict__ ref64, float floor, const float2* __restrict__ tw,
                     const int* __restrict__ pmap, const float* __restrict__ phi, const float* __restrict__ phierr,
                     int h, void* __restrict__ out, int imag_only) {
  constexpr int L = 1 << LOG2L, NT = threads_of<LOG2L>();
  constexpr int PADL = fft16::padded_len(L);
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  float2* X = reinterpret_cast<float2*>(smem);
  float2* Y = X + PADL;
  double* pre = reinterpret_cast<double*>(Y + PADL);   // [NT + 1][6]: chunk prefixes (3 moments x 2 rows)
  double* red = pre + 6 * (NT + 1);                    // [NW][8] scan / min scratch
  float* S = reinterpret_cast<float*>(red + NW * 8);   // PF: staged phi_err rows [2][M]
  uint64_t* bar = reinterpret_cast<uint64_t*>(S + 2 * M);
  float* e0 = PF ? S : reinterpret_cast<float*>(Y);    // phi_err rows (consumed by the forward pass)
  float* e1 = e0 + M;
  float* hb = reinterpret_cast<float*>(Y) + 2 * M;     // H{phi_err} rows (written by the inverse pass)
  float* y0 = reinterpret_cast<float*>(X);             // Re K' rows (after the transforms)
  float* y1 = y0 + M;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // L = 4096 (256 threads): 8 channels per thread when M is a multiple of 8 (the float4 path; cfg4's
  // M = 1600 takes 200 threads x 8 instead of 229 x 7 scalar: 144 -> 136 ms per 4M spectra); shorter
  // transforms keep ceil(M / NT) (the generalised rule cost cfg3 0.7 ms: other register allocation)
  const int C = (NT >= 256 && M % 8 == 0 && M <= 8 * NT) ? 8 : (M + NT - 1) / NT;   // (NT < 256: as before)
  const int j0 = tid * C;
  // the SG constants live in shared memory and are loaded for the trend section only (held in
  // registers across the whole pair loop they added to the finish kernel's spills)
  __shared__ SgK sgk_s;
  if (tid == 0) sgk_s = sg_k(h);
  __syncthreads();
  const int64_t npairs = (n + 1) >> 1;
  const uint32_t rowb = (uint32_t)M * 4u;
  auto issue = [&](int64_t pr) {   // thread 0: bulk copies of pair pr's phi_err rows into S
    const int64_t r0 = 2 * pr;
    const bool two = r0 + 1 < n;
    mbar_expect(bar, two ? 2 * rowb : rowb);
    bulk_row(S, phierr + r0 * (int64_t)M, rowb, bar);
    if (two) bulk_row(S + M, phierr + (r0 + 1) * (int64_t)M, rowb, bar);
  };
  if constexpr (PF) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0 && (int64_t)blockIdx.x < npairs) issue(blockIdx.x);
  }
  uint32_t ph = 0;
  for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int64_t r0 = 2 * pr, r1 = r0 + 1;
    const bool has1 = r1 < n;
    const int64_t o0 = r0 * (int64_t)M, o1 = has1 ? r1 * (int64_t)M : o0;
    if constexpr (PF) {
      if (tid == 0) {   // read after the transforms: in L2 by then
        prefetch_l2(I + o0, rowb);
        prefetch_l2(phi + o0, rowb);
        if (has1) {
          prefetch_l2(I + o1, rowb);
          prefetch_l2(phi + o1, rowb);
        }
      }
      mbar_wait_parity(bar, ph);
      ph ^= 1u;
    } else {
      for (int j = tid; j < M; j += NT) {
        e0[j] = phierr[o0 + j];
        e1[j] = phierr[o1 + j];
      }
      __syncthreads();
    }
    hilbert_pair<LOG2L>(tw, pmap, M, X, Y, e0, has1 || !PF ? e1 : e0, [&](int j, float a, float b) {
      hb[j] = a;
      hb[M + j] = b;
    });
    __syncthreads();
    // pointwise: a' = a + H{phi_err}, phi' = phi - phi_err, K' = exp(a') cis(phi'); chunk moments of Re K'
    // (a full 8-channel f32 chunk moves as float4 pairs: the scalar loads were the largest stall)
    float kre[2][8], kim[2][8];
    double s[6] = {0, 0, 0, 0, 0, 0};
    const bool vec = sizeof(TIn) == 4 && C == 8 && j0 + 8 <= M;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int64_t o = r ? o1 : o0;
      float va[8], vh[8], vp[8];
      if (vec) {
        const float4* ip = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(I) + o + j0);
        const float4* rp = reinterpret_cast<const float4*>(inv_ref + j0);
        const float4* pp4 = reinterpret_cast<const float4*>(phi + o + j0);
        const float4* ep4 = PF ? reinterpret_cast<const float4*>(S + ((r && has1) ? M : 0) + j0)
                               : reinterpret_cast<const float4*>(phierr + o + j0);
        const float4* hp4 = reinterpret_cast<const float4*>(hb + r * M + j0);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const float4 x = __ldcs(ip + h2), ir = rp[h2], f = __ldcs(pp4 + h2), e = PF ? ep4[h2] : __ldcs(ep4 + h2),
                       hh = hp4[h2];
          const float xs[4] = {x.x, x.y, x.z, x.w}, is[4] = {ir.x, ir.y, ir.z, ir.w};
          const float fs[4] = {f.x, f.y, f.z, f.w}, es[4] = {e.x, e.y, e.z, e.w}, hs[4] = {hh.x, hh.y, hh.z, hh.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            va[4 * h2 + u] = 0.5f * __logf(fmaxf(xs[u] * is[u], floor));
            vh[4 * h2 + u] = hs[u];
            vp[4 * h2 + u] = fs[u] - es[u];
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = j0 + c;
          va[c] = vh[c] = vp[c] = 0.f;
          if (c < C && j < M) {
            va[c] = log_ratio_elem<TIn>(I[o + j], inv_ref[j], ref64[j], floor);
            vh[c] = hb[r * M + j];
            vp[c] = phi[o + j] - (PF ? S[((r && has1) ? M : 0) + j] : phierr[o + j]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = j0 + c;
        kre[r][c] = kim[r][c] = 0.f;
        if (c < C && j < M) {
          const float ap = va[c] + vh[c];
          const float pp = vp[c];
          // hardware sin/cos after a two-term reduction to [-pi, pi] and the hardware exp (reading A27)
          const float kq = __fsub_rn(__fadd_rn(pp * 0.15915494309189535f, 12582912.0f), 12582912.0f);
          const float rr = fmaf(kq, 1.7484556e-07f, fmaf(-kq, 6.2831854820251465f, pp));
          float sn, cs;
          __sincosf(rr, &sn, &cs);
          const float mag = __expf(ap);
          kre[r][c] = mag * cs;
          kim[r][c] = mag * sn;
          const double yv = (double)kre[r][c], dj = (double)j;
          s[3 * r] += yv;
          s[3 * r + 1] = fma(dj, yv, s[3 * r + 1]);
          s[3 * r + 2] = fma(dj * dj, yv, s[3 * r + 2]);
        }
      }
    }
    // (X was last read by the inverse transform, before the barrier above)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = j0 + c;
      if (c < C && j < M) { y0[j] = kre[0][c]; y1[j] = kre[1][c]; }
    }
    // block exclusive scan of the chunk moments (6 doubles per thread)
    double inc[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) inc[q] = s[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const double t = __shfl_up_sync(0xffffffffu, inc[q], o);
        if (lane >= o) inc[q] += t;
      }
    }
    if (lane == 31) {
#pragma unroll
      for (int q = 0; q < 6; ++q) red[wid * 8 + q] = inc[q];
    }
    __syncthreads();
    if constexpr (PF) {   // every thread has read this pair's staged rows: stage the next pair
      if (tid == 0 && pr + gridDim.x < npairs) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(pr + gridDim.x);
      }
    }
    double off[6] = {0, 0, 0, 0, 0, 0};
    for (int w2 = 0; w2 < wid; ++w2) {
#pragma unroll
      for (int q = 0; q < 6; ++q) off[q] += red[w2 * 8 + q];
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) pre[tid * 6 + q] = off[q] + inc[q] - s[q];
    if (tid == NT - 1) {
#pragma unroll
      for (int q = 0; q < 6; ++q) pre[NT * 6 + q] = off[q] + inc[q];
    }
    __syncthreads();
    // prefix at idx in [0, M] from the nearest chunk boundary: forward terms from t C, or backward
    // terms from (t + 1) C, at most C / 2 <= 4 of them (a fixed, predicated loop: no divergence)
    auto prefix = [&](int r, int idx, double& P0, double& P1, double& P2) {
      const int t = idx / C, rem = idx - t * C;
      const bool back = 2 * rem > C && t < NT;
      const int tb = back ? t + 1 : t;
      P0 = pre[tb * 6 + 3 * r];
      P1 = pre[tb * 6 + 3 * r + 1];
      P2 = pre[tb * 6 + 3 * r + 2];
      const float* yy = r ? y1 : y0;
      const int i0 = back ? idx : t * C;
      const int nterm = back ? C - rem : rem;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        const float fv = (u < nterm && i < M) ? yy[i < M ? i : M - 1] : 0.f;
        const double v = back ? -(double)fv : (double)fv, di = (double)i;
        P0 += v;
        P1 = fma(di, v, P1);
        P2 = fma(di * di, v, P2);
      }
    };
    float tr[2][8];
    double tmin[2] = {1e300, 1e300};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float* yy = r ? y1 : y0;
      // window moments at the first channel's centre (the centres of a chunk's channels are
      // non-decreasing by 0 or 1 per channel, so the rest slide)
      double Q0 = 0, Q1 = 0, Q2 = 0;
      int cprev = j0 < h ? h : j0;
      if (cprev > M - 1 - h) cprev = M - 1 - h;
      {   // (threads past M compute a valid, unused window)
        double A0, A1, A2, B0, B1, B2;
        prefix(r, cprev + h + 1, A0, A1, A2);
        prefix(r, cprev - h, B0, B1, B2);
        Q0 = A0 - B0;
        Q1 = A1 - B1;
        Q2 = A2 - B2;
      }
      // every thread runs the same instructions for its 8 channel slots (predicated, no divergence:
      // the edge threads' centres stay, the interior threads' slide; a stay adds zero terms)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = j0 + c;
        int cc = j < h ? h : j;
        if (cc > M - 1 - h) cc = M - 1 - h;
        const bool sl = cc != cprev;
        const int ia = cc + h, ib = cprev - h;   // both inside [0, M) for any centre in [h, M-1-h]
        const float fa = yy[ia], fb = yy[ib];
        const double va = sl ? (double)fa : 0.0, vb = sl ? (double)fb : 0.0, da = (double)ia, db = (double)ib;
        Q0 += va - vb;
        Q1 += da * va - db * vb;
        Q2 += da * da * va - db * db * vb;
        cprev = cc;
        const double Tv = sg_eval_full(Q0, Q1, Q2, cc, j, sgk_s);
        const bool ok = c < C && j < M;
        tmin[r] = ok ? fmin(tmin[r], Tv) : tmin[r];
        tr[r][c] = ok ? (float)rcp64(Tv) : 0.f;   // 1/T, unless the spectrum falls back to the mean
      }
    }
    // min of the trend per spectrum (fallback to the scalar mean if <= 0, reading A9)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tmin[r] = fmin(tmin[r], __shfl_xor_sync(0xffffffffu, tmin[r], o));
    }
    if (lane == 0) { red[wid * 8 + 6] = tmin[0]; red[wid * 8 + 7] = tmin[1]; }
    __syncthreads();
    double gmin0 = 1e300, gmin1 = 1e300;
    for (int w2 = 0; w2 < NW; ++w2) { gmin0 = fmin(gmin0, red[w2 * 8 + 6]); gmin1 = fmin(gmin1, red[w2 * 8 + 7]); }
    const float im0 = (float)rcp64(pre[NT * 6 + 0] / (double)M), im1 = (float)rcp64(pre[NT * 6 + 3] / (double)M);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r == 1 && !has1) break;
      const int64_t o = r ? o1 : o0;
      const bool fb = (r ? gmin1 : gmin0) <= 0.0;
      const float imean = r ? im1 : im0;
      float it[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) it[c] = fb ? imean : tr[r][c];
      if (C == 8 && j0 + 8 <= M) {   // 16-B stores (o + j0 is a multiple of 8 elements: M % 4 == 0, j0 = 8t)
        if (imag_only) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + o + j0);
          __stcs(dst, make_float4(kim[r][0] * it[0], kim[r][1] * it[1], kim[r][2] * it[2], kim[r][3] * it[3]));
          __stcs(dst + 1, make_float4(kim[r][4] * it[4], kim[r][5] * it[5], kim[r][6] * it[6], kim[r][7] * it[7]));
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float2*>(out) + o + j0);
#pragma unroll
          for (int h2 = 0; h2 < 4; ++h2)
            __stcs(dst + h2, make_float4(kre[r][2 * h2] * it[2 * h2], kim[r][2 * h2] * it[2 * h2],
                                         kre[r][2 * h2 + 1] * it[2 * h2 + 1], kim[r][2 * h2 + 1] * it[2 * h2 + 1]));
        }
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = j0 + c;
          if (c < C && j < M) {
            if (imag_only) reinterpret_cast<float*>(out)[o + j] = kim[r][c] * it[c];
            else reinterpret_cast<float2*>(out)[o + j] = make_float2(kre[r][c] * it[c], kim[r][c] * it[c]);
          }
        }
      }
    }
    __syncthreads();
  }
}

inline int ilog2(int L) { int r = 0; while ((1 << r) < L) ++r; return r; }

int occupancy_grid(const void* kf, int threads, size_t smem, int64_t work) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kf, threads, smem);
  int64_t g = (int64_t)sms * (per < 1 ? 1 : per);
  if (work < g) g = work;
  return (int)(g < 1 ? 1 : g);
}

template <int LOG2L> struct LogTag { static constexpr int v = LOG2L; };

// dispatch on the compile-time FFT length
template <typename F>
void with_log2(int log2L, F&& f) {
  switch (log2L) {
    case 4: f(LogTag<4>{}); break;
    case 5: f(LogTag<5>{}); break;
    case 6: f(LogTag<6>{}); break;
    case 7: f(LogTag<7>{}); break;
    case 8: f(LogTag<8>{}); break;
    case 9: f(LogTag<9>{}); break;
    case 10: f(LogTag<10>{}); break;
    case 11: f(LogTag<11>{}); break;
    case 12: f(LogTag<12>{}); break;
    default: throw Status(10, "direct path: FFT length must be in [16, 4096]");
  }
}

}  // namespace

// direct_finish prefetch pipeline (PF) for fp32 rows of a multiple of 4 channels (measured: 13.5 against
// 14.0 ms per cfg3 pass; the same staging in direct_phase measured slower, 5.53 against 5.40 ms);
// FKK_DIRECT_PREFETCH=0 turns it off
inline bool direct_pf(int in_f64, int M) {
  static const int env = [] {
    const char* e = getenv("FKK_DIRECT_PREFETCH");
    return e ? atoi(e) : 1;
  }();
  return env != 0 && !in_f64 && M % 4 == 0;
}

size_t direct_phase_smem(int L) { return 2 * (size_t)fft16::padded_len(L) * sizeof(float2); }
size_t direct_finish_smem(int M, int L, bool pf) {
  const int T = L / 16;
  const int NT = T < 32 ? 32 : T;
  return 2 * (size_t)fft16::padded_len(L) * sizeof(float2) + (size_t)6 * (NT + 1) * sizeof(double) +
         (size_t)(NT / 32) * 8 * sizeof(double) + (pf ? 2 * (size_t)M * sizeof(float) + 16 : 0);
}

void launch_direct_phase(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                         float floor, int L, const float2* tw, const int* pmap, float* phi, int* flags, cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = direct_phase_smem(L);
  const int64_t npairs = (n + 1) / 2;
  auto launch = [&](auto lt, auto in_tag) {
    constexpr int LG = decltype(lt)::v;
    using TIn = decltype(in_tag);
    auto kf = direct_phase_kernel<TIn, LG>;
    constexpr int NT = threads_of<LG>();
    FKK_CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = occupancy_grid((const void*)kf, NT, smem, npairs);
    kf<<<grid, NT, smem, s>>>(reinterpret_cast<const TIn*>(I), n, M, inv_ref, ref64, floor, tw, pmap, phi, flags);
  };
  if (in_f64) with_log2(ilog2(L), [&](auto lt) { launch(lt, double{}); });
  else with_log2(ilog2(L), [&](auto lt) { launch(lt, float{}); });
  check_launch("direct_phase");
}

void launch_als_rows(const void* y, int y_f64, int64_t n, int M, double lam, double p, int iters, void* z, int z_f64,
                     cudaStream_t s, int* solves, unsigned* ctr) {
  if (n <= 0) return;
  if (!launch_als_part(y, y_f64, n, M, lam, p, iters, z, z_f64, s, solves, ctr))
    throw Status(10, "ALS: M must be in [8, 4096] and its segment state must fit in shared memory");
}

void launch_direct_finish(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                          float floor, int L, const float2* tw, const int* pmap, const float* phi, const float* phierr,
                          int sg_half, void* out, int out_imag_only, cudaStream_t s) {
  if (n <= 0) return;
  // one thread per 16 FFT points holds at most 8 channels of each row
  if (2 * M > L) throw Status(10, "direct path: the FFT length must be at least 2 M");
  const bool pf = direct_pf(in_f64, M);
  const size_t smem = direct_finish_smem(M, L, pf);
  const int64_t npairs = (n + 1) / 2;
  auto launch = [&](auto lt, auto in_tag, auto pf_tag) {
    constexpr int LG = decltype(lt)::v;
    using TIn = decltype(in_tag);
    auto kf = direct_finish_kernel<TIn, LG, decltype(pf_tag)::value>;
    constexpr int NT = threads_of<LG>();
    FKK_CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = occupancy_grid((const void*)kf, NT, smem, npairs);
    kf<<<grid, NT, smem, s>>>(reinterpret_cast<const TIn*>(I), n, M, inv_ref, ref64, floor, tw, pmap, phi, phierr,
                              sg_half, out, out_imag_only);
  };
  if (in_f64) with_log2(ilog2(L), [&](auto lt) { launch(lt, double{}, std::false_type{}); });
  else if (pf) with_log2(ilog2(L), [&](auto lt) { launch(lt, float{}, std::true_type{}); });
  else with_log2(ilog2(L), [&](auto lt) { launch(lt, float{}, std::false_type{}); });
  check_launch("direct_finish");
}

}  // namespace fkk
