// Asymmetric-least-squares baseline D{.} (reading A6/A7): exactly `iters` solves of
// (W + lam D^T D) z = W y, w^0 = 1, then w_i = p if y_i > z_i else 1 - p -- all in fp64.
//
// Warp-partitioned solver: ONE warp per spectrum, the M rows split into P <= 32 contiguous
// segments (lane s owns rows [b_s, b_{s+1})).  The last two rows of every segment but the last are
// separators; each lane eliminates the interior of its segment (LDL^T of a pentadiagonal block),
// accumulating the Schur complement of its interior onto the two adjacent separators
// (C = Y^T D^-1 Y with Y = L^-1 [A_IS, f_I]: forward substitution only, no back-substitution
// needed).  The separators form a block-tridiagonal system with 2 x 2 blocks, solved by parallel
// cyclic reduction across the lanes (5 shuffle rounds).  Pass B forward-substitutes the corrected
// interior right-hand side; the next iteration's pass A back-substitutes it while it factorises the
// next system in the opposite direction (the elimination direction alternates).  Per-row state
// (l1, 1/D, g) lives in shared memory in a [row-in-segment][lane] layout (conflict-free), so the
// 10 solves never touch HBM: the spectrum is read once and the baseline written once.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "fkk_internal.h"

namespace fkk {

namespace {

__device__ __forceinline__ double rcp64a(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// one Newton step on the MUFU seed (~2^-44 relative): the LDL^T pivots of the ALS recurrence --
// a 1e-13 relative perturbation of the factorisation, far below the 1e-5 direct-KK tolerance
// (the second step was on the recurrence's critical path)
__device__ __forceinline__ double rcp64n1(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// band of lam D^T D (second differences): diagonal d0, first off-diagonal d1 (coupling i, i+1)
__device__ __forceinline__ double d0v(int i, int M) {
  return (i == 0 || i == M - 1) ? 1.0 : ((i == 1 || i == M - 2) ? 5.0 : 6.0);
}
__device__ __forceinline__ double d1v(int i, int M) { return (i == 0 || i == M - 2) ? -2.0 : -4.0; }
// A[i][j] for 1 <= |i - j| <= 2
__device__ __forceinline__ double cpl(int i, int j, int M, double lam) {
  return (abs(i - j) == 1) ? lam * d1v(min(i, j), M) : lam;
}

struct M2 {   // 2 x 2 matrix, row-major
  double a, b, c, d;
};
__device__ __forceinline__ M2 mul(const M2& x, const M2& y) {
  return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d};
}
__device__ __forceinline__ M2 inv(const M2& x) {
  const double r = rcp64a(x.a * x.d - x.b * x.c);
  return {x.d * r, -x.b * r, -x.c * r, x.a * r};
}
__device__ __forceinline__ double2 mulv(const M2& x, double2 v) {
  return make_double2(x.a * v.x + x.b * v.y, x.c * v.x + x.d * v.y);
}
__device__ __forceinline__ M2 shfl(const M2& x, int delta, bool up) {
  M2 r;
  if (up) {
    r.a = __shfl_up_sync(0xffffffffu, x.a, delta); r.b = __shfl_up_sync(0xffffffffu, x.b, delta);
    r.c = __shfl_up_sync(0xffffffffu, x.c, delta); r.d = __shfl_up_sync(0xffffffffu, x.d, delta);
  } else {
    r.a = __shfl_down_sync(0xffffffffu, x.a, delta); r.b = __shfl_down_sync(0xffffffffu, x.b, delta);
    r.c = __shfl_down_sync(0xffffffffu, x.c, delta); r.d = __shfl_down_sync(0xffffffffu, x.d, delta);
  }
  return r;
}
__device__ __forceinline__ double2 shflv(double2 v, int delta, bool up) {
  if (up) return make_double2(__shfl_up_sync(0xffffffffu, v.x, delta), __shfl_up_sync(0xffffffffu, v.y, delta));
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, delta), __shfl_down_sync(0xffffffffu, v.y, delta));
}

// segment of lane s: rows [seg_b(s), seg_b(s+1))
__device__ __forceinline__ int seg_b(int s, int M, int P) { return (s * M) / P; }   // s*M < 2^31 (M <= 4096)
__device__ __forceinline__ int seg_of(int col, int M, int P) {
  int s = (col * P) / M;
  if (s + 1 <= P && seg_b(s + 1, M, P) <= col) ++s;
  return s;
}

// lane exchange among the NL threads of one spectrum: out = mine of lane src (src clamped; callers
// ignore out-of-range sources).  NL = 32: shuffles; NL = 64 (two warps): through shared memory.
template <int NL, int W>
__device__ __forceinline__ void lane_get2(const double (&mine)[W], int src1, double (&out1)[W], int src2,
                                          double (&out2)[W], double* xs) {
  if constexpr (NL == 32) {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      out1[i] = __shfl_sync(0xffffffffu, mine[i], src1 & 31);
      out2[i] = __shfl_sync(0xffffffffu, mine[i], src2 & 31);
    }
  } else {
    __syncthreads();   // the previous exchange's reads are done
#pragma unroll
    for (int i = 0; i < W; ++i) xs[i * NL + threadIdx.x] = mine[i];
    __syncthreads();
    const int a = min(max(src1, 0), NL - 1), b = min(max(src2, 0), NL - 1);
#pragma unroll
    for (int i = 0; i < W; ++i) {
      out1[i] = xs[i * NL + a];
      out2[i] = xs[i * NL + b];
    }
  }
}
template <int NL>
__device__ __forceinline__ void spectrum_sync() {
  if constexpr (NL == 32) __syncwarp();
  else __syncthreads();
}

// NL threads (one or two warps) per spectrum, P <= NL segments: two warps halve the dependent chain
// of every lane (the solver is latency-bound at ~7 spectra per SM, the shared-memory limit)
template <typename TY, typename TZ, int NL>
__global__ void __launch_bounds__(NL) als_part_kernel(const TY* __restrict__ y, int64_t n, int M, int P, int T,
                                                      double lam, double p, int iters, TZ* __restrict__ z) {
  extern __shared__ __align__(16) double sh[];
  double* sl1 = sh;                  // [T][32] l1 of the current factorisation
  double* srd = sl1 + NL * T;        // [T][NL] 1/D
  double* sg = srd + NL * T;         // [T][NL] g = D^-1 L^-1 f~   (finally: z)
  double* xs = sg + NL * T;          // [10][NL] lane-exchange scratch (NL = 64)
  TY* sy = reinterpret_cast<TY*>(xs + (NL == 64 ? 10 * NL : 0));     // [T][NL] y (input precision)
  unsigned char* sw = reinterpret_cast<unsigned char*>(sy + NL * T);   // [T][NL] w: 1 -> p, 0 -> 1-p
  const int s = threadIdx.x;
  const bool act = s < P;
  const int b = act ? seg_b(s, M, P) : M, e = act ? seg_b(s + 1, M, P) : M;
  const bool hasL = act && s > 0, hasR = act && s < P - 1;
  const int nn = act ? (e - b) - (hasR ? 2 : 0) : 0;   // interior rows b .. b+nn-1
  // interiors touching rows 0, 1, M-2, M-1 (where D^T D's band differs) take the slow band lookup
  const bool edge = act && (b <= 1 || b + nn >= M - 1);
  const double q = 1.0 - p;
  const double lam2 = lam * lam, lam6 = 6.0 * lam, lamm4 = -4.0 * lam;

  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const TY* yr = y + row * (int64_t)M;
    spectrum_sync<NL>();
    for (int col = s; col < M; col += NL) {           // coalesced read, scatter to [t][lane]
      const int sc = seg_of(col, M, P);
      sy[(col - seg_b(sc, M, P)) * NL + sc] = yr[col];
    }
    spectrum_sync<NL>();
    double2 xL = make_double2(0.0, 0.0), xR = make_double2(0.0, 0.0);   // separator values (left: S_{s-1})
    for (int it = 0; it <= iters; ++it) {
      const bool dr = it & 1;                 // 0: ascending elimination, 1: descending
      const int ix0 = dr ? (nn - 1) * NL + s : s, dix = dr ? -NL : NL;
      const int i0 = dr ? b + nn - 1 : b, di = dr ? -1 : 1;
      const int na = dr ? e - 2 : b - 1;      // near-adjacent separator row
      const bool hasN = dr ? hasR : hasL, hasF = dr ? hasL : hasR;
      // ---------------- pass A: back-substitution of the previous system (it > 0) and factorisation
      //                  + forward substitution of the next (it < iters), in elimination order
      double z1 = 0.0, z2 = 0.0;
      double Dm1 = 0.0, rDm1 = 0.0, rDm2 = 0.0, L1m1 = 0.0, L1m2 = 0.0;
      double gf1 = 0.0, gf2 = 0.0, ga1 = 0.0, ga2 = 0.0, gb1 = 0.0, gb2 = 0.0;
      double Caa = 0.0, Cab = 0.0, Cbb = 0.0, Cfa = 0.0, Cfb = 0.0;
      const double ea0 = hasN ? cpl(i0, na, M, lam) : 0.0, eb0 = hasN ? lam : 0.0, ea1 = hasN ? lam : 0.0;
      using T_ = std::true_type;
      using F_ = std::false_type;
      auto passA = [&](auto bsub_c, auto fact_c) {
        constexpr bool BSUB = decltype(bsub_c)::value, FACT = decltype(fact_c)::value;
        int ix = ix0, i = i0;
        // the next row's shared-memory operands are loaded at the top of each step, before this row's
        // stores: the compiler otherwise orders every load behind the previous row's stores (the
        // arrays may alias) and the smem latency joins the dependent chain (tools/micro/rowpass.cu)
        const int ixmax = (T - 1) * NL + s;
        double cy = 0.0, cg = 0.0, cl1 = 0.0, crd = 0.0;
        if (nn > 0) {
          cy = (double)sy[ix];
          if constexpr (BSUB) { cg = sg[ix]; cl1 = sl1[ix]; crd = srd[ix]; }
        }
        // one row in elimination order; ea/eb = near-spike entries (t < 2), LASTROW: l1 = 0
        // EDGE: this position may hold one of the rows 0, 1, M-2, M-1 (where D^T D's band differs);
        // only the peeled positions t = 0, 1, nn-2, nn-1 can, so the main loop runs without the check
        auto step = [&](auto last_c, auto edge_c, double ea, double eb) {
          constexpr bool LASTROW = decltype(last_c)::value, EDGE = decltype(edge_c)::value;
          const double yv = cy;
          const double g_old = cg, l1_old = cl1, rd_old = crd;
          {
            const int ixn = min(max(ix + dix, s), ixmax);   // (clamped: past-the-segment rows are unused)
            cy = (double)sy[ixn];
            if constexpr (BSUB) { cg = sg[ixn]; cl1 = sl1[ixn]; crd = srd[ixn]; }
          }
          double wv = 1.0;
          if constexpr (BSUB) {
            // previous order: this row's l1 / l2 couple to the rows visited just before (z1, z2;
            // both zero at the first rows, where the stored l1 is zero too)
            const double zv = g_old - l1_old * z1 - lam * rd_old * z2;
            z2 = z1;
            z1 = zv;
            wv = yv > zv ? p : q;
            if constexpr (!FACT) sg[ix] = zv;
          }
          if constexpr (FACT) {
            double ld0 = lam6, ld1 = lamm4;
            if constexpr (EDGE) {
              if (edge) { ld0 = lam * d0v(i, M); ld1 = lam * d1v(dr ? i - 1 : i, M); }
            }
            const double D = (wv + ld0) - L1m1 * L1m1 * Dm1 - lam2 * rDm2;
            const double rd = rcp64n1(D);
            const double l1n = LASTROW ? 0.0 : (ld1 - lam * L1m1) * rd;
            const double L2m2 = lam * rDm2;
            const double gf = wv * yv - L1m1 * gf1 - L2m2 * gf2;
            const double ga = ea - L1m1 * ga1 - L2m2 * ga2, gb = eb - L1m1 * gb1 - L2m2 * gb2;
            const double ua = ga * rd, ub = gb * rd;
            Caa = fma(ga, ua, Caa);
            Cab = fma(ga, ub, Cab);
            Cbb = fma(gb, ub, Cbb);
            Cfa = fma(gf, ua, Cfa);
            Cfb = fma(gf, ub, Cfb);
            sl1[ix] = l1n;
            srd[ix] = rd;
            sw[ix] = wv == p ? 1 : 0;
            Dm1 = D;
            rDm2 = rDm1;
            rDm1 = rd;
            L1m2 = L1m1;
            L1m1 = l1n;
            gf2 = gf1; gf1 = gf;
            ga2 = ga1; ga1 = ga;
            gb2 = gb1; gb1 = gb;
          }
          ix += dix;
          i += di;
        };
        if (nn == 0) return;                      // lanes beyond the P segments
        step(F_{}, T_{}, ea0, eb0);               // t = 0   (nn >= 2 on active lanes)
        if (nn == 2) { step(T_{}, T_{}, ea1, 0.0); return; }
        step(F_{}, T_{}, ea1, 0.0);               // t = 1
#pragma unroll 2
        for (int t = 2; t < nn - 2; ++t) step(F_{}, F_{}, 0.0, 0.0);
        if (nn >= 4) step(F_{}, T_{}, 0.0, 0.0);  // t = nn - 2
        step(T_{}, T_{}, 0.0, 0.0);               // t = nn - 1
      };
      if (it == 0) passA(F_{}, T_{});
      else if (it < iters) passA(T_{}, T_{});
      else { passA(T_{}, F_{}); break; }
      // ---------------- far spike columns (nonzero only in the last two eliminated rows: after the
      //                  loop the shift registers hold t = nn-1 in *1 and t = nn-2 in *2)
      double Cff_aa = 0.0, Cff_ab = 0.0, Cff_bb = 0.0;                 // far x far (fa, ff)
      double Cnf_aa = 0.0, Cnf_ab = 0.0, Cnf_ba = 0.0, Cnf_bb = 0.0;   // near(na, nf) x far(fa, ff)
      double Cf_fa = 0.0, Cf_fb = 0.0;
      if (hasF) {
        const int r_last = dr ? b : b + nn - 1;                 // row eliminated last
        const int fa = dr ? b - 1 : e - 2;
        const double l1_nm2 = L1m2;                             // l1 of t = nn-2
        const double yfa0 = lam, yff0 = 0.0;                    // t = nn-2
        const double yfa1 = cpl(r_last, fa, M, lam) - l1_nm2 * lam, yff1 = lam;   // t = nn-1
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) {
          const double yfa = k2 ? yfa1 : yfa0, yff = k2 ? yff1 : yff0, rd = k2 ? rDm1 : rDm2;
          const double sga = k2 ? ga1 : ga2, sgb = k2 ? gb1 : gb2, sgf = k2 ? gf1 : gf2;
          Cff_aa = fma(yfa * rd, yfa, Cff_aa);
          Cff_ab = fma(yfa * rd, yff, Cff_ab);
          Cff_bb = fma(yff * rd, yff, Cff_bb);
          Cnf_aa = fma(sga * rd, yfa, Cnf_aa);
          Cnf_ab = fma(sga * rd, yff, Cnf_ab);
          Cnf_ba = fma(sgb * rd, yfa, Cnf_ba);
          Cnf_bb = fma(sgb * rd, yff, Cnf_bb);
          Cf_fa = fma(sgf * rd, yfa, Cf_fa);
          Cf_fb = fma(sgf * rd, yff, Cf_fb);
        }
      }
      // canonical blocks over the separator rows L = (b-2, b-1), R = (e-2, e-1)
      M2 CLL, CRR, CLR;
      double2 CfL, CfR;
      if (!dr) {   // near = L (na = L1, nf = L0), far = R (fa = R0, ff = R1)
        CLL = {Cbb, Cab, Cab, Caa};
        CRR = {Cff_aa, Cff_ab, Cff_ab, Cff_bb};
        CLR = {Cnf_ba, Cnf_bb, Cnf_aa, Cnf_ab};
        CfL = make_double2(Cfb, Cfa);
        CfR = make_double2(Cf_fa, Cf_fb);
      } else {     // near = R (na = R0, nf = R1), far = L (fa = L1, ff = L0)
        CRR = {Caa, Cab, Cab, Cbb};
        CLL = {Cff_bb, Cff_ab, Cff_ab, Cff_aa};
        CLR = {Cnf_ab, Cnf_bb, Cnf_aa, Cnf_ba};   // [L0 R0, L0 R1; L1 R0, L1 R1] = [ff.na, ff.nf; fa.na, fa.nf]
        CfR = make_double2(Cfa, Cfb);
        CfL = make_double2(Cf_fb, Cf_fa);
      }
      // ---------------- reduced block-tridiagonal system on the separators, lane s <-> S_s
      M2 nLL, nLR;
      double2 nCfL;
      {   // from lane s + 1
        const double mine[10] = {CLL.a, CLL.b, CLL.c, CLL.d, CLR.a, CLR.b, CLR.c, CLR.d, CfL.x, CfL.y};
        double o[10], o2[10];
        lane_get2<NL, 10>(mine, s + 1, o, s + 1, o2, xs);
        nLL = {o[0], o[1], o[2], o[3]};
        nLR = {o[4], o[5], o[6], o[7]};
        nCfL = make_double2(o[8], o[9]);
      }
      M2 Dk = {1.0, 0.0, 0.0, 1.0}, Uk = {0.0, 0.0, 0.0, 0.0};
      double2 rk = make_double2(0.0, 0.0);
      if (hasR) {
        const int i0s = e - 2, i1s = e - 1;
        const int l0 = (i0s - b) * NL + s, l1x = (i1s - b) * NL + s;
        const double w0 = it == 0 ? 1.0 : (sw[l0] ? p : q);
        const double w1 = it == 0 ? 1.0 : (sw[l1x] ? p : q);
        const double off = lam * d1v(i0s, M);
        Dk = {w0 + lam * d0v(i0s, M) - CRR.a - nLL.a, off - CRR.b - nLL.b, off - CRR.c - nLL.c,
              w1 + lam * d0v(i1s, M) - CRR.d - nLL.d};
        Uk = {-nLR.a, -nLR.b, -nLR.c, -nLR.d};
        rk = make_double2(w0 * (double)sy[l0] - CfR.x - nCfL.x, w1 * (double)sy[l1x] - CfR.y - nCfL.y);
      }
      M2 Lk;
      {   // from lane s - 1
        const double mine[4] = {Uk.a, Uk.b, Uk.c, Uk.d};
        double o[4], o2[4];
        lane_get2<NL, 4>(mine, s - 1, o, s - 1, o2, xs);
        Lk = {o[0], o[1], o[2], o[3]};
      }
      Lk = {Lk.a, Lk.c, Lk.b, Lk.d};   // transpose
      if (s == 0 || !hasR) Lk = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int h = 1; h < NL; h <<= 1) {
        const M2 Di = inv(Dk);
        const M2 Pm = mul(Di, Lk), Qm = mul(Di, Uk);
        const double2 sv = mulv(Di, rk);
        M2 Pdn, Qdn, Pup, Qup;
        double2 sdn, sup;
        {   // from lanes s - h and s + h
          const double mine[10] = {Pm.a, Pm.b, Pm.c, Pm.d, Qm.a, Qm.b, Qm.c, Qm.d, sv.x, sv.y};
          double dn[10], up[10];
          lane_get2<NL, 10>(mine, s - h, dn, s + h, up, xs);
          Pdn = {dn[0], dn[1], dn[2], dn[3]};
          Qdn = {dn[4], dn[5], dn[6], dn[7]};
          sdn = make_double2(dn[8], dn[9]);
          Pup = {up[0], up[1], up[2], up[3]};
          Qup = {up[4], up[5], up[6], up[7]};
          sup = make_double2(up[8], up[9]);
        }
        M2 nL = {0.0, 0.0, 0.0, 0.0}, nU = {0.0, 0.0, 0.0, 0.0};
        if (s - h >= 0) {
          const M2 a1 = mul(Lk, Pdn), a2 = mul(Lk, Qdn);
          const double2 a3 = mulv(Lk, sdn);
          nL = {-a1.a, -a1.b, -a1.c, -a1.d};
          Dk = {Dk.a - a2.a, Dk.b - a2.b, Dk.c - a2.c, Dk.d - a2.d};
          rk = make_double2(rk.x - a3.x, rk.y - a3.y);
        }
        if (s + h < NL) {
          const M2 b1 = mul(Uk, Qup), b2 = mul(Uk, Pup);
          const double2 b3 = mulv(Uk, sup);
          nU = {-b1.a, -b1.b, -b1.c, -b1.d};
          Dk = {Dk.a - b2.a, Dk.b - b2.b, Dk.c - b2.c, Dk.d - b2.d};
          rk = make_double2(rk.x - b3.x, rk.y - b3.y);
        }
        Lk = nL;
        Uk = nU;
      }
      xR = hasR ? mulv(inv(Dk), rk) : make_double2(0.0, 0.0);
      {   // from lane s - 1
        const double mine[2] = {xR.x, xR.y};
        double o[2], o2[2];
        lane_get2<NL, 2>(mine, s - 1, o, s - 1, o2, xs);
        xL = make_double2(o[0], o[1]);
      }
      if (!hasL) xL = make_double2(0.0, 0.0);
      if (hasR) {   // separator values of this solve; weights for the next
        const int l0 = (e - 2 - b) * NL + s, l1x = (e - 1 - b) * NL + s;
        sg[l0] = xR.x;
        sg[l1x] = xR.y;
        sw[l0] = (double)sy[l0] > xR.x ? 1 : 0;
        sw[l1x] = (double)sy[l1x] > xR.y ? 1 : 0;
      }
      // ---------------- pass B: forward substitution of the corrected interior right-hand side
      {
        const double x_na = dr ? xR.x : xL.y, x_nf = dr ? xR.y : xL.x;
        const double x_fa = dr ? xL.y : xR.x, x_ff = dr ? xL.x : xR.y;
        const int fa = dr ? b - 1 : e - 2;
        const int r_last = dr ? b : b + nn - 1;
        const double c0 = cpl(i0, na, M, lam) * x_na + lam * x_nf, c1 = lam * x_na;
        const double cL = cpl(r_last, fa, M, lam) * x_fa + lam * x_ff, cL2 = lam * x_fa;
        auto passB = [&](auto first_c) {
          constexpr bool FIRST = decltype(first_c)::value;
          double g1 = 0.0, g2 = 0.0, l1prev = 0.0, rdm1 = 0.0, rdm2 = 0.0;
          int ix = ix0;
          const int ixmaxB = (T - 1) * NL + s;
          // next row's operands loaded before this row's store (see pass A)
          unsigned char nw_ = 0;
          double ny = 0.0, nrd = 0.0, nl1 = 0.0;
          if (nn > 0) { nw_ = sw[ix]; ny = (double)sy[ix]; nrd = srd[ix]; nl1 = sl1[ix]; }
          auto stepB = [&](double corr) {
            const double wv = FIRST ? 1.0 : (nw_ ? p : q);
            const double f = wv * ny - corr;
            const double rd = nrd;
            const double l1c = nl1;
            {
              const int ixn = min(max(ix + dix, s), ixmaxB);
              nw_ = sw[ixn]; ny = (double)sy[ixn]; nrd = srd[ixn]; nl1 = sl1[ixn];
            }
            const double g = f - l1prev * g1 - lam * rdm2 * g2;
            sg[ix] = g * rd;
            g2 = g1;
            g1 = g;
            l1prev = l1c;
            rdm2 = rdm1;
            rdm1 = rd;
            ix += dix;
          };
          if (nn < 5) {
            for (int t = 0; t < nn; ++t)
              stepB((t == 0 ? c0 : 0.0) + (t == 1 ? c1 : 0.0) + (t == nn - 2 ? cL2 : 0.0) + (t == nn - 1 ? cL : 0.0));
          } else {
            stepB(c0);
            stepB(c1);
#pragma unroll 2
            for (int t = 2; t < nn - 2; ++t) stepB(0.0);
            stepB(cL2);
            stepB(cL);
          }
        };
        if (it == 0) passB(T_{});
        else passB(F_{});
      }
    }
    // ---------------- write z (interior from the last back-substitution, separators from the last solve)
    spectrum_sync<NL>();
    TZ* zr = z + row * (int64_t)M;
    for (int col = s; col < M; col += NL) {
      const int sc = seg_of(col, M, P);
      zr[col] = (TZ)sg[(col - seg_b(sc, M, P)) * NL + sc];
    }
  }
}

}  // namespace

// lanes per spectrum: 32 (one warp).  The two-warp variant (64 segments, FKK_ALS_LANES=64) halves every
// lane's dependent chain but adds a PCR level and shared-memory lane exchanges; measured on cfg3 rows it
// is no faster (13.06 vs 12.95 ms per 131,072 spectra: the extra exchange/separator work eats the gain)
static int als_lanes(int M) {
  const char* ev = getenv("FKK_ALS_LANES");
  const int want = ev ? atoi(ev) : 32;
  return (want == 64 && M / 4 >= 64) ? 64 : 32;
}

size_t als_part_smem(int M, int y_f64) {
  const int NL = als_lanes(M);
  const int P = M / 4 < NL ? M / 4 : NL;
  if (P < 2) return 0;
  const int T = (M + P - 1) / P;
  return (size_t)NL * T * (3 * sizeof(double) + (y_f64 ? 8 : 4) + 1) + (NL == 64 ? 10 * (size_t)NL * sizeof(double) : 0);
}

bool launch_als_part(const void* y, int y_f64, int64_t n, int M, double lam, double p, int iters, void* z, int z_f64,
                     cudaStream_t s) {
  const int NL = als_lanes(M);
  const int P = M / 4 < NL ? M / 4 : NL;
  if (P < 2 || n <= 0) return false;
  const int T = (M + P - 1) / P;
  const size_t sm = (size_t)NL * T * (3 * sizeof(double) + (y_f64 ? 8 : 4) + 1) +
                    (NL == 64 ? 10 * (size_t)NL * sizeof(double) : 0);
  int dev = 0, sms = 148, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (sm > (size_t)maxsm) return false;
#define FKK_ALS_PART(TY, TZ, L)                                                                       \
  {                                                                                                   \
    auto kf = als_part_kernel<TY, TZ, L>;                                                             \
    FKK_CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));   \
    int per = 1;                                                                                      \
    FKK_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kf, L, sm));                   \
    const int64_t g = std::min<int64_t>(n, (int64_t)sms * std::max(per, 1));                         \
    kf<<<(unsigned)g, L, sm, s>>>((const TY*)y, n, M, P, T, lam, p, iters, (TZ*)z);                   \
  }
#define FKK_ALS_TYPES(L)                                                                              \
  if (y_f64 && z_f64) FKK_ALS_PART(double, double, L)                                                 \
  else if (!y_f64 && !z_f64) FKK_ALS_PART(float, float, L)                                            \
  else if (!y_f64 && z_f64) FKK_ALS_PART(float, double, L)                                            \
  else FKK_ALS_PART(double, float, L)
  if (NL == 64) {
    FKK_ALS_TYPES(64)
  } else {
    FKK_ALS_TYPES(32)
  }
#undef FKK_ALS_TYPES
#undef FKK_ALS_PART
  check_launch("als_part");
  return true;
}

}  // namespace fkk
