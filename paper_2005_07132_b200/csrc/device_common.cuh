// Device helpers shared by the fKK-EC kernels (sm_100a).
//   * block-level radix-2 FFT Hilbert transform in shared memory (DIF forward -> multiplier in
//     bit-reversed order -> DIT inverse, no explicit permutation), two real rows per transform
//     ("two-for-one": H is real-linear, so IFFT(h FFT(x + i y)) = H{x} + i H{y});
//   * centred even-reflection / zero padding (reading A3);
//   * block scans and warp reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fkk {

template <typename T> struct cplx { T x, y; };

__device__ __forceinline__ int reflect_index(int j, int M) {
  // even reflection without repeating the edge sample, period 2(M-1) (numpy 'reflect')
  const int period = 2 * (M - 1);
  int r = j % period;
  if (r < 0) r += period;
  return r < M ? r : period - r;
}

// Twiddle table tw[j] = exp(-2 pi i j / L), j < L/2 (computed on the host in fp64).
// x: L complex values in shared memory, natural order in, bit-reversed order out (DIF).
template <typename T>
__device__ __forceinline__ void fft_dif_inplace(cplx<T>* x, const cplx<T>* tw, int L, int log2L) {
  for (int s = 0; s < log2L; ++s) {
    const int span = L >> (s + 1);
    const int tstride = 1 << s;  // twiddle index multiplier L/(2 span)
    const int ls = log2L - s - 1;
    for (int b = threadIdx.x; b < (L >> 1); b += blockDim.x) {
      const int grp = b >> ls, j = b & (span - 1);
      const int i0 = grp * 2 * span + j, i1 = i0 + span;
      cplx<T> a = x[i0], c = x[i1];
      cplx<T> w = tw[j * tstride];
      T dx = a.x - c.x, dy = a.y - c.y;
      x[i0].x = a.x + c.x;
      x[i0].y = a.y + c.y;
      x[i1].x = dx * w.x - dy * w.y;
      x[i1].y = dx * w.y + dy * w.x;
    }
    __syncthreads();
  }
}

// Inverse (unnormalised) DIT: bit-reversed order in, natural order out; uses conj twiddles.
template <typename T>
__device__ __forceinline__ void ifft_dit_inplace(cplx<T>* x, const cplx<T>* tw, int L, int log2L) {
  for (int s = 0; s < log2L; ++s) {
    const int span = 1 << s;
    const int tstride = L >> (s + 1);
    for (int b = threadIdx.x; b < (L >> 1); b += blockDim.x) {
      const int grp = b >> s, j = b - (grp << s);
      const int i0 = grp * 2 * span + j, i1 = i0 + span;
      cplx<T> a = x[i0], c = x[i1];
      cplx<T> w = tw[j * tstride];   // conj applied below
      T tx = c.x * w.x + c.y * w.y;  // c * conj(w)
      T ty = c.y * w.x - c.x * w.y;
      x[i0].x = a.x + tx;
      x[i0].y = a.y + ty;
      x[i1].x = a.x - tx;
      x[i1].y = a.y - ty;
    }
    __syncthreads();
  }
}

// Hilbert multiplier h(f) = -i sgn-like (f < L/2: -i; f > L/2: +i; f in {0, L/2}: 0), applied at
// bit-reversed position p: f == 0 <-> p == 0, f == L/2 <-> p == 1, f < L/2 <-> p even.
template <typename T>
__device__ __forceinline__ void hilbert_multiplier_bitrev(cplx<T>* x, int L) {
  for (int pidx = threadIdx.x; pidx < L; pidx += blockDim.x) {
    cplx<T> v = x[pidx];
    cplx<T> o;
    if (pidx < 2) { o.x = 0; o.y = 0; }
    else if ((pidx & 1) == 0) { o.x = v.y; o.y = -v.x; }   // * (-i)
    else { o.x = -v.y; o.y = v.x; }                        // * (+i)
    x[pidx] = o;
  }
  __syncthreads();
}

// Fill x (L complex) from two real rows r0, r1 (length M, shared or global) with centred padding.
template <typename T, typename S>
__device__ __forceinline__ void pad_pair(cplx<T>* x, const S* r0, const S* r1, int M, int L, int pad_zero) {
  const int pl = (L - M) >> 1;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    int j = i - pl;
    cplx<T> v;
    if (j >= 0 && j < M) { v.x = (T)r0[j]; v.y = (T)r1[j]; }
    else if (pad_zero) { v.x = 0; v.y = 0; }
    else { int r = reflect_index(j, M); v.x = (T)r0[r]; v.y = (T)r1[r]; }
    x[i] = v;
  }
  __syncthreads();
}

// H{r0} + i H{r1} left in x[pl .. pl+M) (scaled by 1/L by the caller when reading).
template <typename T>
__device__ __forceinline__ void hilbert_pair_inplace(cplx<T>* x, const cplx<T>* tw, int L, int log2L) {
  fft_dif_inplace<T>(x, tw, L, log2L);
  hilbert_multiplier_bitrev<T>(x, L);
  ifft_dit_inplace<T>(x, tw, L, log2L);
}

// ---------------------------------------------------------------------------------------------
// Stockham autosort FFT, radix 8 (last pass radix 4 or 2), one CTA, in place: each pass loads all of
// a butterfly's R inputs into registers, barriers, and writes the R outputs (natural order in and
// out).  Versus the radix-2 loop above: log8 instead of log2 passes over shared memory and two
// barriers per pass.  tw[t] = exp(-2 pi i t / L) for t < L/2 (tw[t + L/2] = -tw[t]).
template <typename T>
__device__ __forceinline__ cplx<T> cmul(cplx<T> a, cplx<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ cplx<T> tw_at(const cplx<T>* tw, int t, int L, bool inv) {
  const int h = L >> 1;
  cplx<T> w = tw[t < h ? t : t - h];
  if (t >= h) { w.x = -w.x; w.y = -w.y; }
  if (inv) w.y = -w.y;
  return w;
}
// in-register DFT of size R in {2, 4, 8}; forward uses exp(-2 pi i / R), inverse exp(+2 pi i / R)
template <typename T, int R, bool INV>
__device__ __forceinline__ void dft_small(cplx<T>* v) {
  auto mul_mi = [](cplx<T> a) -> cplx<T> { return INV ? cplx<T>{-a.y, a.x} : cplx<T>{a.y, -a.x}; };  // * -i (fwd)
  if constexpr (R == 2) {
    const cplx<T> a = v[0], b = v[1];
    v[0] = {a.x + b.x, a.y + b.y};
    v[1] = {a.x - b.x, a.y - b.y};
  } else if constexpr (R == 4) {
    const cplx<T> t0 = {v[0].x + v[2].x, v[0].y + v[2].y}, t1 = {v[0].x - v[2].x, v[0].y - v[2].y};
    const cplx<T> t2 = {v[1].x + v[3].x, v[1].y + v[3].y};
    const cplx<T> t3 = mul_mi(cplx<T>{v[1].x - v[3].x, v[1].y - v[3].y});
    v[0] = {t0.x + t2.x, t0.y + t2.y};
    v[2] = {t0.x - t2.x, t0.y - t2.y};
    v[1] = {t1.x + t3.x, t1.y + t3.y};
    v[3] = {t1.x - t3.x, t1.y - t3.y};
  } else {
    cplx<T> e[4], o[4];
    e[0] = v[0]; e[1] = v[2]; e[2] = v[4]; e[3] = v[6];
    o[0] = v[1]; o[1] = v[3]; o[2] = v[5]; o[3] = v[7];
    dft_small<T, 4, INV>(e);
    dft_small<T, 4, INV>(o);
    const T s = (T)0.70710678118654752440;
    // w8^k, k = 0..3 (forward: exp(-i pi k / 4))
    const cplx<T> o1 = INV ? cplx<T>{s * (o[1].x - o[1].y), s * (o[1].x + o[1].y)}
                           : cplx<T>{s * (o[1].x + o[1].y), s * (o[1].y - o[1].x)};
    const cplx<T> o2 = mul_mi(o[2]);
    const cplx<T> o3 = INV ? cplx<T>{-s * (o[3].x + o[3].y), s * (o[3].x - o[3].y)}
                           : cplx<T>{s * (o[3].y - o[3].x), -s * (o[3].x + o[3].y)};
    v[0] = {e[0].x + o[0].x, e[0].y + o[0].y};
    v[4] = {e[0].x - o[0].x, e[0].y - o[0].y};
    v[1] = {e[1].x + o1.x, e[1].y + o1.y};
    v[5] = {e[1].x - o1.x, e[1].y - o1.y};
    v[2] = {e[2].x + o2.x, e[2].y + o2.y};
    v[6] = {e[2].x - o2.x, e[2].y - o2.y};
    v[3] = {e[3].x + o3.x, e[3].y + o3.y};
    v[7] = {e[3].x - o3.x, e[3].y - o3.y};
  }
}
// one Stockham pass of radix R with current sub-transform size Ns (L / R butterflies)
template <typename T, int R, bool INV, int MAXB>
__device__ __forceinline__ void stockham_pass(cplx<T>* x, const cplx<T>* tw, int L, int Ns) {
  // MAXB radix-8 butterflies (8 MAXB values) per thread: L <= 8 MAXB blockDim; a radix-4 / radix-2
  // pass gives each thread 8 / R butterflies so it holds the same 8 MAXB values
  constexpr int NBT = MAXB * (8 / R);
  const int nb = L / R;
  cplx<T> v[NBT][R];
  int jj[NBT];
#pragma unroll
  for (int u = 0; u < NBT; ++u) {
    const int j = threadIdx.x + u * blockDim.x;
    jj[u] = j;
    if (j < nb) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[u][r] = x[j + r * nb];
      const int k = j % Ns;
      if (Ns > 1) {
        const int step = (L / (Ns * R)) * k;
        {
          // w^r from one table load and r-1 complex products (~r x 6e-8 relative): the other table
          // loads were half of the pass's shared-memory reads
          const cplx<T> w1 = tw_at(tw, step, L, INV);
          cplx<T> wr = w1;
#pragma unroll
          for (int r = 1; r < R; ++r) {
            v[u][r] = cmul(v[u][r], wr);
            wr = cmul(wr, w1);
          }
        }
      }
      dft_small<T, R, INV>(v[u]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < NBT; ++u) {
    const int j = jj[u];
    if (j < nb) {
      if (sizeof(T) == 4 && Ns == 1 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        // first pass: this thread's R outputs are contiguous (x[j R + r]) -> 16-B stores (the 8-B
        // stores at a 64-B lane stride were 16-way bank conflicted)
        float4* dst = reinterpret_cast<float4*>(x + j * R);
#pragma unroll
        for (int r = 0; r < R; r += 2)
          dst[r / 2] = make_float4((float)v[u][r].x, (float)v[u][r].y, (float)v[u][r + 1].x, (float)v[u][r + 1].y);
      } else {
        const int k = j % Ns;
        const int base = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) x[base + r * Ns] = v[u][r];
      }
    }
  }
  __syncthreads();
}
template <typename T, bool INV, int MAXB>
__device__ __forceinline__ void stockham_fft(cplx<T>* x, const cplx<T>* tw, int L, int log2L) {
  int Ns = 1, rem = log2L;
  while (rem >= 3) { stockham_pass<T, 8, INV, MAXB>(x, tw, L, Ns); Ns *= 8; rem -= 3; }
  if (rem == 2) stockham_pass<T, 4, INV, MAXB>(x, tw, L, Ns);
  else if (rem == 1) stockham_pass<T, 2, INV, MAXB>(x, tw, L, Ns);
}
// Hilbert multiplier in natural order: f in (0, L/2) -> -i, f in (L/2, L) -> +i, f in {0, L/2} -> 0
template <typename T>
__device__ __forceinline__ void hilbert_multiplier_natural(cplx<T>* x, int L) {
  for (int f = threadIdx.x; f < L; f += blockDim.x) {
    const cplx<T> v = x[f];
    cplx<T> o;
    if (f == 0 || f == (L >> 1)) { o.x = 0; o.y = 0; }
    else if (f < (L >> 1)) { o.x = v.y; o.y = -v.x; }   // * (-i)
    else { o.x = -v.y; o.y = v.x; }                      // * (+i)
    x[f] = o;
  }
  __syncthreads();
}
// H{r0} + i H{r1} in x[pl .. pl+M) (unnormalised: the caller scales by 1/L); requires L <= 8 MAXB blockDim
template <typename T, int MAXB>
__device__ __forceinline__ void hilbert_pair_stockham(cplx<T>* x, const cplx<T>* tw, int L, int log2L) {
  stockham_fft<T, false, MAXB>(x, tw, L, log2L);
  hilbert_multiplier_natural<T>(x, L);
  stockham_fft<T, true, MAXB>(x, tw, L, log2L);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive prefix sums of three fp64 sequences (y, j*y, j^2*y) over j = 0..M-1 into P0/P1/P2
// (length M+1, P[0] = 0).  `wsum` is scratch of 3 * 32 doubles.  Block-wide; ends synchronised.
__device__ __forceinline__ void block_prefix3(const double* y, int M, double* P0, double* P1, double* P2,
                                              double* wsum) {
  const int nt = blockDim.x;
  const int chunk = (M + nt - 1) / nt;
  const int beg = min(M, threadIdx.x * chunk), end = min(M, beg + chunk);
  double s0 = 0, s1 = 0, s2 = 0;
  for (int j = beg; j < end; ++j) { double v = y[j]; double dj = (double)j; s0 += v; s1 += dj * v; s2 += dj * dj * v; }
  // inclusive scan of per-thread totals
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double i0 = s0, i1 = s1, i2 = s2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o),
           t2 = __shfl_up_sync(0xffffffffu, i2, o);
    if (lane >= o) { i0 += t0; i1 += t1; i2 += t2; }
  }
  if (lane == 31) { wsum[wid] = i0; wsum[32 + wid] = i1; wsum[64 + wid] = i2; }
  __syncthreads();
  if (wid == 0) {
    const int nw = nt >> 5;
    double a0 = lane < nw ? wsum[lane] : 0, a1 = lane < nw ? wsum[32 + lane] : 0, a2 = lane < nw ? wsum[64 + lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double t0 = __shfl_up_sync(0xffffffffu, a0, o), t1 = __shfl_up_sync(0xffffffffu, a1, o),
             t2 = __shfl_up_sync(0xffffffffu, a2, o);
      if (lane >= o) { a0 += t0; a1 += t1; a2 += t2; }
    }
    if (lane < nw) { wsum[lane] = a0; wsum[32 + lane] = a1; wsum[64 + lane] = a2; }
  }
  __syncthreads();
  double o0 = i0 - s0 + (wid > 0 ? wsum[wid - 1] : 0.0);
  double o1 = i1 - s1 + (wid > 0 ? wsum[32 + wid - 1] : 0.0);
  double o2 = i2 - s2 + (wid > 0 ? wsum[64 + wid - 1] : 0.0);
  for (int j = beg; j < end; ++j) {
    P0[j] = o0; P1[j] = o1; P2[j] = o2;
    double v = y[j]; double dj = (double)j;
    o0 += v; o1 += dj * v; o2 += dj * dj * v;
  }
  if (end == M && beg < M) { P0[M] = o0; P1[M] = o1; P2[M] = o2; }
  __syncthreads();
}

// Savitzky-Golay order-2 trend at point i from window moment prefix sums (reading A8).
// Interior: centred quadratic least-squares value; edges: the quadratic fitted on the first/last
// w samples evaluated at i.  Exact rewriting of the per-window least-squares fit: with centred
// offsets k in [-h, h], c1 decouples and [n K2; K2 K4] [c0 c2]^T = [S0 S2]^T.
// the window constants of the local quadratic least-squares fit (computed once per kernel: the fp64
// divides are long instruction sequences and sg_point runs for every channel of every spectrum)
struct SgConst {
  double n, K2, K4, idet, iK2;
};
__device__ __forceinline__ SgConst sg_const(int h) {
  SgConst k;
  k.n = 2.0 * h + 1.0;
  const double hd = (double)h;
  k.K2 = hd * (hd + 1.0) * (2.0 * hd + 1.0) / 3.0;
  k.K4 = hd * (hd + 1.0) * (2.0 * hd + 1.0) * (3.0 * hd * hd + 3.0 * hd - 1.0) / 15.0;
  k.idet = 1.0 / (k.n * k.K4 - k.K2 * k.K2);
  k.iK2 = 1.0 / k.K2;
  return k;
}
__device__ __forceinline__ double sg_point(const double* P0, const double* P1, const double* P2, int M, int h, int i,
                                           const SgConst& kc) {
  int c = i;
  if (c < h) c = h;
  if (c > M - 1 - h) c = M - 1 - h;
  const int lo = c - h, hi = c + h + 1;
  const double Q0 = P0[hi] - P0[lo], Q1 = P1[hi] - P1[lo], Q2 = P2[hi] - P2[lo];
  const double cd = (double)c;
  const double S0 = Q0;
  const double S1 = Q1 - cd * Q0;
  const double S2 = Q2 - 2.0 * cd * Q1 + cd * cd * Q0;
  const double c0 = (kc.K4 * S0 - kc.K2 * S2) * kc.idet;
  if (c == i) return c0;
  const double c2 = (kc.n * S2 - kc.K2 * S0) * kc.idet;
  const double c1 = S1 * kc.iK2;
  const double k = (double)(i - c);
  return c0 + c1 * k + c2 * k * k;
}
__device__ __forceinline__ double sg_point(const double* P0, const double* P1, const double* P2, int M, int h, int i) {
  return sg_point(P0, P1, P2, M, h, i, sg_const(h));
}

}  // namespace fkk
