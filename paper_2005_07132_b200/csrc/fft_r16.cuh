// Radix-16 Stockham FFT of one complex length-L sequence (L = 2^LOG2L, 32 <= L <= 4096) by a CTA of
// L/16 threads, for the direct path's Hilbert transforms ("direct path").
//
//   * every pass is compile-time (radix R, sub-transform size Ns): no integer division, twiddle
//     indices are shifts and masks;
//   * each thread holds 16 values per pass in registers (16 / R butterflies of radix R), so a pass
//     is one shared-memory read, register DFTs and one shared-memory write (ping-pong buffers: a
//     thread stores a butterfly's outputs right after computing it; one barrier per pass);
//   * the first pass reads its inputs through a caller functor (the padded log-ratio, straight from
//     global memory) and the last pass hands its outputs to a caller functor (the Hilbert multiplier,
//     or the result rows) -- the transform's own loads and stores are the only smem traffic;
//   * shared layout: element i at i + (i >> 4) (one pad per 16 elements), which makes the contiguous
//     16-element groups of the first pass and the strided groups of the others bank-conflict free.
//
// Stockham step (R, Ns): butterfly b < L/R, k = b mod Ns: v[r] = x[b + r L/R] * w^(r k L/(Ns R)),
// v = DFT_R(v), y[(b - k) R + k + r Ns] = v[r]  (natural order in and out).
// Twiddles tw[t] = exp(-2 pi i t / L), t < L (fp64-accurate table, computed on the host).
#pragma once
#include <cuda_runtime.h>

#ifndef FKK_FFT_TWIDDLE_POW2
#define FKK_FFT_TWIDDLE_POW2 1
#endif

namespace fkk {
namespace fft16 {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {   // * -i (forward) / * +i (inverse)
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
// * exp(-+ i pi / 4)
template <bool INV>
__device__ __forceinline__ float2 mul_w8(float2 a) {
  const float s = 0.70710678118654752440f;
  return INV ? make_float2(s * (a.x - a.y), s * (a.x + a.y)) : make_float2(s * (a.x + a.y), s * (a.y - a.x));
}
template <bool INV>
__device__ __forceinline__ float2 mul_w8_3(float2 a) {   // * exp(-+ 3 i pi / 4)
  const float s = 0.70710678118654752440f;
  return INV ? make_float2(-s * (a.x + a.y), s * (a.x - a.y)) : make_float2(s * (a.y - a.x), -s * (a.x + a.y));
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const float2 t2 = cadd(v[1], v[3]), t3 = mul_mi<INV>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else if constexpr (R == 8) {
    float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft<4, INV>(e);
    dft<4, INV>(o);
    o[1] = mul_w8<INV>(o[1]);
    o[2] = mul_mi<INV>(o[2]);
    o[3] = mul_w8_3<INV>(o[3]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q] = cadd(e[q], o[q]);
      v[q + 4] = csub(e[q], o[q]);
    }
  } else {   // 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
    float2 y[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      float2 t[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
      dft<4, INV>(t);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) y[k1][n2] = t[k1];
    }
    // twiddles w16^(n2 k1)
    const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;   // cos, sin (pi/8)
    const float2 w1 = make_float2(c1, INV ? s1 : -s1), w3 = make_float2(s1, INV ? c1 : -c1);
    y[1][1] = cmulf(y[1][1], w1);
    y[1][2] = mul_w8<INV>(y[1][2]);
    y[1][3] = cmulf(y[1][3], w3);
    y[2][1] = mul_w8<INV>(y[2][1]);
    y[2][2] = mul_mi<INV>(y[2][2]);
    y[2][3] = mul_w8_3<INV>(y[2][3]);
    y[3][1] = cmulf(y[3][1], w3);
    y[3][2] = mul_w8_3<INV>(y[3][2]);
    // w16^9 = -w16^1
    {
      const float2 t = cmulf(y[3][3], w1);
      y[3][3] = make_float2(-t.x, -t.y);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      dft<4, INV>(y[k1]);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = y[k1][k2];
    }
  }
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int L) { return L + L / 16; }

template <int LOG2L>
struct Plan {
  static constexpr int L = 1 << LOG2L;
  static constexpr int T = L / 16;                       // threads
  static constexpr int NP = (LOG2L + 3) / 4;             // passes
  static constexpr int LAST_R = 1 << (LOG2L - 4 * (NP - 1));
  template <int P> __host__ __device__ static constexpr int radix() { return P == NP - 1 ? LAST_R : 16; }
  template <int P> __host__ __device__ static constexpr int ns() { return 1 << (4 * P); }
};

// One Stockham pass P of the plan; `load(i)` gives input element i, `store(i, v)` takes output i.
template <int LOG2L, int P, bool INV, typename Load, typename Store>
__device__ __forceinline__ void pass(const float2* __restrict__ tw, Load&& load, Store&& store) {
  using PL = Plan<LOG2L>;
  constexpr int L = PL::L, T = PL::T;
  constexpr int R = PL::template radix<P>(), NS = PL::template ns<P>();
  constexpr int NB = 16 / R;            // butterflies per thread
  constexpr int STEP = L / (NS * R);    // twiddle index multiplier
  const int j = threadIdx.x;
  if (T < 32 && j >= T) return;         // short transforms: a warp wider than the plan
  // butterfly by butterfly: the load and store buffers of a pass are always different (ping-pong),
  // so a thread may store its outputs before the other threads have read their inputs
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int b = j + u * T;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = load(b + r * (L / R));
    const int k = b & (NS - 1);
    if constexpr (NS > 1) {
#if FKK_FFT_TWIDDLE_POW2
      // the power-of-two twiddles w^1, w^2, w^4, w^8 from the table, the rest as products of at most
      // three of them (fewer loads and live registers; <= 3 extra roundings per twiddle)
      float2 wp[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if ((1 << e) < R) {
          wp[e] = __ldg(tw + (1 << e) * k * STEP);
          if (INV) wp[e].y = -wp[e].y;
        }
      }
#pragma unroll
      for (int r = 1; r < R; ++r) {
        float2 w = make_float2(1.f, 0.f);
        bool first = true;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (r & (1 << e)) {
            w = first ? wp[e] : cmulf(w, wp[e]);
            first = false;
          }
        }
        v[r] = cmulf(v[r], w);
      }
#else
#pragma unroll
      for (int r = 1; r < R; ++r) {
        float2 w = __ldg(tw + r * k * STEP);
        if (INV) w.y = -w.y;
        v[r] = cmulf(v[r], w);
      }
#endif
    }
    dft<R, INV>(v);
    const int base = (b - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) store(base + r * NS, v[r]);
  }
}

// Whole transform: first pass from `load`, middle passes through the ping-pong buffers b0 / b1
// (padded layout), last pass into `store`.  The caller synchronises before reusing b0 / b1.
template <int LOG2L, bool INV, typename Load, typename Store>
__device__ __forceinline__ void transform(const float2* __restrict__ tw, float2* b0, float2* b1, Load&& load,
                                          Store&& store) {
  using PL = Plan<LOG2L>;
  constexpr int NP = PL::NP;
  auto sload0 = [&](int i) { return b0[pad(i)]; };
  auto sload1 = [&](int i) { return b1[pad(i)]; };
  auto sstore0 = [&](int i, float2 v) { b0[pad(i)] = v; };
  auto sstore1 = [&](int i, float2 v) { b1[pad(i)] = v; };
  if constexpr (NP == 1) {
    pass<LOG2L, 0, INV>(tw, load, store);
  } else {
    pass<LOG2L, 0, INV>(tw, load, sstore0);
    __syncthreads();
    if constexpr (NP == 2) {
      pass<LOG2L, 1, INV>(tw, sload0, store);
    } else {
      pass<LOG2L, 1, INV>(tw, sload0, sstore1);
      __syncthreads();
      // NP == 3 (L <= 4096)
      pass<LOG2L, 2, INV>(tw, sload1, store);
    }
  }
}

}  // namespace fft16
}  // namespace fkk
