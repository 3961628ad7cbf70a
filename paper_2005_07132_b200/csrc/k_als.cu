// Asymmetric-least-squares baseline D{.} (readings A6/A7): `iters` solves of
// (W + lam D^T D) z = W y, w^0 = 1, then w_i = p if y_i > z_i else 1 - p -- all in fp64.  The loop
// stops early once a solve leaves every weight unchanged: the next system would be identical, so its
// solution is the current one (the fp64 oracle always runs all `iters` solves).
//
// Warp-partitioned solver: ONE warp per spectrum, the M rows (extended to Mp = 32 T with zero-weight
// rows, see als_geo) split into 32 segments of T rows (lane s owns rows [sT, sT+T)).  The last two rows
// of every segment are separators; each lane eliminates the interior of its segment (LDL^T of a
// pentadiagonal block) while forward-substituting the right-hand side and the two near spike columns,
// accumulating the Schur complement C = Y^T D^-1 Y of its interior onto the adjacent separators.  The
// separators form a block-tridiagonal system with 2 x 2 blocks, solved by parallel cyclic reduction
// across the lanes (5 shuffle rounds).  Pass B forward-substitutes the corrected interior right-hand
// side; the next solve's pass A back-substitutes it while it factorises the next system in the
// opposite direction.  Equal segments make every row step warp-uniform, which the tensor-memory
// accesses below require.
//
// On-chip layout (one warp = one spectrum; one CTA per SM of up to 16 warps, up to four per TMEM lane
// quadrant):
//   tensor memory: the factor {l1, 1/D} (fp64) of interior row t of segment s at lane s of the warp's
//   quadrant, columns 4t .. 4t+3 after the warp's column offset (T = 32: 120 columns per spectrum,
//   four spectra per quadrant);
//   shared memory: row block t = { g[32] (fp64), y[32] (input precision) }, lane s at column s;
//   weights: one bit per row in a per-lane register mask (bit t = 1 <-> w = p).
// Moving the factor to tensor memory halves the shared memory per spectrum (28 -> 12 KB at M = 1000),
// so 16 instead of 7 spectra (warps) are resident per SM to hide the recurrences' latency.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "fkk_internal.h"
#include "tc_common.cuh"

namespace fkk {

namespace {

constexpr int NL = 32;   // lanes (segments) per spectrum
constexpr int WPC_MAX = 16;   // warps (spectra) per CTA: up to four per TMEM lane quadrant

__device__ __forceinline__ double rcp64a(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// one Newton step on the MUFU seed (~2^-44 relative): the LDL^T pivots of the ALS recurrence -- a
// 1e-13 relative perturbation of the factorisation, far below the 1e-5 direct-KK tolerance
__device__ __forceinline__ double rcp64n1(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// band of D^T D (second differences): diagonal d0, first off-diagonal d1 (coupling i, i+1)
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
// interior weights of a segment: one bit per interior row (bit r <-> segment row r; 1 <-> w = p) in
// a 64-bit (T <= 64) or 128-bit register.  A pass visits the rows in elimination order (ascending or
// descending); it reads and rebuilds the mask through "position order" words (bit t <-> t-th row
// visited), one shift per row, and converts with a bit reversal once per pass.
template <typename MT> struct MaskBits { static constexpr int N = 8 * (int)sizeof(MT); };
__device__ __forceinline__ unsigned long long mask_rev(unsigned long long m) { return __brevll(m); }
__device__ __forceinline__ unsigned __int128 mask_rev(unsigned __int128 m) {
  return ((unsigned __int128)__brevll((unsigned long long)m) << 64) | __brevll((unsigned long long)(m >> 64));
}
template <typename MT>   // row-order mask -> position-order cursor (bit 0 = first row visited)
__device__ __forceinline__ MT mask_cursor(MT m, int nn, bool desc) {
  return desc ? (MT)(mask_rev(m) >> (MaskBits<MT>::N - nn)) : m;
}
template <typename MT>
__device__ __forceinline__ bool mask_take(MT& c) {
  const bool v = (bool)(c & (MT)1);
  c >>= 1;
  return v;
}
template <typename MT>   // append the visited row's bit at the top (position t ends at bit N - nn + t)
__device__ __forceinline__ void mask_push(MT& m, bool v) {
  m = (MT)(m >> 1) | ((MT)v << (MaskBits<MT>::N - 1));
}
template <typename MT>   // pushed word -> row-order mask
__device__ __forceinline__ MT mask_final(MT m, int nn, bool desc) {
  return desc ? mask_rev(m) : (MT)(m >> (MaskBits<MT>::N - nn));
}

// TMEM: the factor of interior row t (l1, 1/D as two fp64 = four 32-bit columns 4t .. 4t+3) in the
// lane of its segment; one 32x32b access moves one row of all 32 segments.  The wait is tied to the
// destination registers so that no use of them can be scheduled before it.
__device__ __forceinline__ void tm_ld2(uint32_t ta, double& a, double& b) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3));
  a = __hiloint2double((int)r1, (int)r0);
  b = __hiloint2double((int)r3, (int)r2);
}
__device__ __forceinline__ void tm_st2(uint32_t ta, double a, double b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta),
               "r"(__double2loint(a)), "r"(__double2hiint(a)), "r"(__double2loint(b)), "r"(__double2hiint(b)));
}
__device__ __forceinline__ void tm_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// shared-memory row block (one per segment row t, all 32 lanes): g (fp64) | y (input precision)
template <typename TY>
struct RowLayout {
  static constexpr int OFF_G = 0;
  static constexpr int OFF_Y = 8 * NL;
  static constexpr int BYTES = 8 * NL + (int)sizeof(TY) * NL;
};

template <typename TY>
__device__ __forceinline__ double ld_y(const unsigned char* rowp, int s) {
  return (double)*reinterpret_cast<const TY*>(rowp + RowLayout<TY>::OFF_Y + s * (int)sizeof(TY));
}
__device__ __forceinline__ double& fld(unsigned char* rowp, int off, int s) {
  return *reinterpret_cast<double*>(rowp + off + 8 * s);
}

template <typename TY, typename TZ, typename MT>
__global__ void __launch_bounds__(NL * WPC_MAX, 1)
    als_seg_kernel(const TY* __restrict__ y, int64_t n, int M, int T, int P, uint32_t tcols, double lam, double p,
                   int iters, TZ* __restrict__ z, int* __restrict__ solves, unsigned* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char shm_all[];
  __shared__ uint32_t tmem_base_s;
  using RL = RowLayout<TY>;
  constexpr int RS = RL::BYTES;
  const int warp = threadIdx.x >> 5, s = threadIdx.x & (NL - 1), wpc = blockDim.x >> 5;
  if (warp == 0) tc::tmem_alloc(&tmem_base_s, tcols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // lane quadrant warp % 4 (the warps a quadrant can address), columns 4 (T-2) (warp / 4) onwards
  const uint32_t tbase = tmem_base_s + ((uint32_t)((warp & 3) * NL) << 16) + 4u * (uint32_t)(T - 2) * (uint32_t)(warp >> 2);
  unsigned char* const shm = shm_all + (size_t)warp * T * RS;
  const int Mp = P * T, nn = T - 2;         // every segment: interior rows 0 .. nn-1, separators nn, nn+1
  const bool act = s < P;
  const int b = s * T, e = b + T;
  const bool hasL = act && s > 0, hasR = act;
  const bool edge = s == 0;                 // rows 0 and 1 (D^T D's first band rows) are lane 0's t = 0, 1
  // rows M .. Mp-1 (padding of the last segment; all rows of inactive lanes) carry weight 0
  MT realm = 0;
  for (int t = 0; t < nn; ++t)
    if (b + t < M) realm |= (MT)1 << t;
  const bool real0 = e - 2 < M, real1 = e - 1 < M;
  const double q = 1.0 - p;
  const double lam2 = lam * lam, lam6 = 6.0 * lam, lamm4 = -4.0 * lam;
  int solves_local = 0;

  // spectra: from the launch's counter when given (the solve count varies 2..10 per spectrum, so a static
  // stride left the slowest warps ~10% behind the mean), else a static stride
  auto next_row = [&](int64_t cur) -> int64_t {
    if (!ctr) return cur < 0 ? (int64_t)blockIdx.x * wpc + warp : cur + (int64_t)gridDim.x * wpc;
    unsigned v = 0;
    if (s == 0) v = atomicAdd(ctr, 1u);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  for (int64_t row = next_row(-1); row < n; row = next_row(row)) {
    const TY* yr = y + row * (int64_t)M;
    __syncwarp();
    // lane s reads its own segment (L1 serves the strided lanes from the row's cached lines); the
    // [row][lane] shared stores are conflict-free
    for (int t = 0; t < T; ++t)
      *reinterpret_cast<TY*>(shm + t * RS + RL::OFF_Y + s * (int)sizeof(TY)) = (b + t < M) ? yr[b + t] : (TY)0;
    __syncwarp();
    MT im = 0;                 // interior weights (bit 1 <-> p); w^0 = 1 is handled by it == 0
    bool ws0 = false, ws1 = false;   // separator weights (rows e-2, e-1)
    bool sep_flip = true;      // a separator weight changed in the previous solve
    double2 xL = make_double2(0.0, 0.0), xR = make_double2(0.0, 0.0);
    int it = 0;
    for (;; ++it) {
      const bool dr = it & 1;                 // 0: ascending elimination, 1: descending
      const int i0 = dr ? b + nn - 1 : b, di = dr ? -1 : 1;
      const int r0 = dr ? nn - 1 : 0;         // segment row of the first eliminated row
      const int dstep = dr ? -RS : RS;
      const uint32_t tstep = dr ? (uint32_t)-4 : 4u;
      const int na = dr ? e - 2 : b - 1;      // near-adjacent separator row
      const bool hasN = dr ? hasR : hasL, hasF = dr ? hasL : hasR;
      const bool fact = it < iters;
      // ---------------- pass A: back-substitution of the previous system (it > 0) and factorisation
      //                  + forward substitution of the next (it < iters), in elimination order
      double z1 = 0.0, z2 = 0.0;
      double Dm1 = 0.0, rDm1 = 0.0, rDm2 = 0.0, L1m1 = 0.0, L1m2 = 0.0;
      double gf1 = 0.0, gf2 = 0.0, ga1 = 0.0, ga2 = 0.0, gb1 = 0.0, gb2 = 0.0;
      double Caa = 0.0, Cab = 0.0, Cbb = 0.0, Cfa = 0.0, Cfb = 0.0;
      bool iflip = false;
      const double ea0 = hasN ? cpl(i0, na, Mp, lam) : 0.0, eb0 = hasN ? lam : 0.0, ea1 = hasN ? lam : 0.0;
      using T_ = std::true_type;
      using F_ = std::false_type;
      auto passA = [&](auto bsub_c, auto fact_c) {
        constexpr bool BSUB = decltype(bsub_c)::value, FACT = decltype(fact_c)::value;
        unsigned char* rp = shm + r0 * RS;
        uint32_t tc_ = tbase + 4u * (uint32_t)r0;
        int i = i0;
        // the next row's operands are loaded at the top of each step, before this row's stores
        double cy = ld_y<TY>(rp, s), cg = 0.0, cl1 = 0.0, crd = 0.0;
        if constexpr (BSUB) {
          cg = fld(rp, RL::OFF_G, s);
          tm_ld2(tc_, cl1, crd);
        }
        MT new_m = 0;
        // one row in elimination order; ea/eb = near-spike entries (t < 2); LASTROW: l1 = 0 and no
        // prefetch; EDGE: this position may hold row 0 or 1
        auto step = [&](auto last_c, auto edge_c, double ea, double eb) {
          constexpr bool LASTROW = decltype(last_c)::value, EDGE = decltype(edge_c)::value;
          const double yv = cy;
          const double g_old = cg, l1_old = cl1, rd_old = crd;
          unsigned char* const cur = rp;
          const uint32_t ct = tc_;
          if constexpr (!LASTROW) {
            rp += dstep;
            tc_ += tstep;
            cy = ld_y<TY>(rp, s);
            if constexpr (BSUB) {
              cg = fld(rp, RL::OFF_G, s);
              tm_ld2(tc_, cl1, crd);
            }
          }
          double wv = 1.0;
          if constexpr (BSUB) {
            // previous order: this row's l1 / l2 couple to the rows visited just before (z1, z2;
            // both zero at the first rows, where the stored l1 is zero too)
            const double zv = g_old - l1_old * z1 - lam * rd_old * z2;
            z2 = z1;
            z1 = zv;
            const bool wp = yv > zv;
            mask_push<MT>(new_m, wp);
            wv = wp ? p : q;
            fld(cur, RL::OFF_G, s) = zv;          // kept: the output if this solve is the last
          }
          if constexpr (FACT) {
            wv = i < M ? wv : 0.0;
            double ld0 = lam6, ld1 = lamm4;
            if constexpr (EDGE) {
              const double e0 = lam * d0v(i, Mp), e1 = lam * d1v(dr ? i - 1 : i, Mp);
              ld0 = edge ? e0 : ld0;
              ld1 = edge ? e1 : ld1;
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
            tm_st2(ct, l1n, rd);
            Dm1 = D;
            rDm2 = rDm1;
            rDm1 = rd;
            L1m2 = L1m1;
            L1m1 = l1n;
            gf2 = gf1; gf1 = gf;
            ga2 = ga1; ga1 = ga;
            gb2 = gb1; gb1 = gb;
          }
          i += di;
        };
        step(F_{}, T_{}, ea0, eb0);               // t = 0   (nn >= 2)
        if (nn == 2) {
          step(T_{}, T_{}, ea1, 0.0);
        } else {
          step(F_{}, T_{}, ea1, 0.0);               // t = 1
#pragma unroll 2
          for (int t = 2; t < nn - 2; ++t) step(F_{}, F_{}, 0.0, 0.0);
          if (nn >= 4) step(F_{}, T_{}, 0.0, 0.0);  // t = nn - 2
          step(T_{}, T_{}, 0.0, 0.0);               // t = nn - 1
        }
        if constexpr (BSUB) {
          const MT nm = mask_final<MT>(new_m, nn, dr);
          iflip = ((nm ^ im) & realm) != 0;
          im = nm;
        }
      };
      if (it == 0) passA(F_{}, T_{});
      else if (fact) passA(T_{}, T_{});
      else passA(T_{}, F_{});
      // the previous solve changed no weight: this system equals it, so its solution is final
      // (interior z in the g slots from this pass A, separators from the previous reduction)
      if (it >= 2 && !__any_sync(0xffffffffu, iflip || sep_flip)) break;
      if (!fact) break;
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
        const double yfa1 = cpl(r_last, fa, Mp, lam) - l1_nm2 * lam, yff1 = lam;   // t = nn-1
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
      {   // from lane s + 1 (CLL is symmetric: 3 values); lanes beyond the P segments contribute zero
        const double mine[9] = {CLL.a, CLL.b, CLL.d, CLR.a, CLR.b, CLR.c, CLR.d, CfL.x, CfL.y};
        double o[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) o[i] = __shfl_down_sync(0xffffffffu, act ? mine[i] : 0.0, 1);
        if (s + 1 >= P) {   // the last segment's separator couples to nothing on its right
#pragma unroll
          for (int i = 0; i < 9; ++i) o[i] = 0.0;
        }
        nLL = {o[0], o[1], o[1], o[2]};
        nLR = {o[3], o[4], o[5], o[6]};
        nCfL = make_double2(o[7], o[8]);
      }
      unsigned char* const sep0 = shm + nn * RS;        // rows e-2, e-1 (segment rows nn, nn+1)
      unsigned char* const sep1 = sep0 + RS;
      M2 Dk = {1.0, 0.0, 0.0, 1.0}, Uk = {0.0, 0.0, 0.0, 0.0};
      double2 rk = make_double2(0.0, 0.0);
      double ys0 = 0.0, ys1 = 0.0;
      if (hasR) {
        const int i0s = e - 2, i1s = e - 1;
        ys0 = ld_y<TY>(sep0, s);
        ys1 = ld_y<TY>(sep1, s);
        const double w0 = real0 ? (it == 0 ? 1.0 : (ws0 ? p : q)) : 0.0;
        const double w1 = real1 ? (it == 0 ? 1.0 : (ws1 ? p : q)) : 0.0;
        const double off = lam * d1v(i0s, Mp);
        Dk = {w0 + lam * d0v(i0s, Mp) - CRR.a - nLL.a, off - CRR.b - nLL.b, off - CRR.c - nLL.c,
              w1 + lam * d0v(i1s, Mp) - CRR.d - nLL.d};
        Uk = {-nLR.a, -nLR.b, -nLR.c, -nLR.d};
        rk = make_double2(w0 * ys0 - CfR.x - nCfL.x, w1 * ys1 - CfR.y - nCfL.y);
      }
      // symmetric PCR (the separator system is SPD block tridiagonal, so L_s = U_{s-h}^T at every level):
      // with Dinv = D^-1, A = Dinv U, b = Dinv r, a level of stride h is
      //   D_s -= U_{s-h}^T A_{s-h} + U_s Dinv_{s+h} U_s^T,  r_s -= U_{s-h}^T b_{s-h} + U_s b_{s+h},
      //   U_s <- -U_s A_{s+h}
      // (14 doubles exchanged per level instead of 20 for the general form; D kept as (a, b, d))
      double Da = Dk.a, Db = Dk.b, Dd = Dk.d;
#pragma unroll
      for (int h = 1; h < NL; h <<= 1) {
        const double idet = rcp64a(Da * Dd - Db * Db);
        const double ia = Dd * idet, ib = -Db * idet, id = Da * idet;
        const M2 A = {ia * Uk.a + ib * Uk.c, ia * Uk.b + ib * Uk.d, ib * Uk.a + id * Uk.c, ib * Uk.b + id * Uk.d};
        const double2 bv = make_double2(ia * rk.x + ib * rk.y, ib * rk.x + id * rk.y);
        const double caa = Uk.a * A.a + Uk.c * A.c, cab = Uk.a * A.b + Uk.c * A.d, cbb = Uk.b * A.b + Uk.d * A.d;
        const double2 ev = make_double2(Uk.a * bv.x + Uk.c * bv.y, Uk.b * bv.x + Uk.d * bv.y);
        double up[9], dn[5];
        {
          const double mu[9] = {ia, ib, id, bv.x, bv.y, A.a, A.b, A.c, A.d};
          const double md[5] = {caa, cab, cbb, ev.x, ev.y};
#pragma unroll
          for (int i = 0; i < 9; ++i) up[i] = __shfl_down_sync(0xffffffffu, mu[i], h);
#pragma unroll
          for (int i = 0; i < 5; ++i) dn[i] = __shfl_up_sync(0xffffffffu, md[i], h);
        }
        if (s - h >= 0) {
          Da -= dn[0]; Db -= dn[1]; Dd -= dn[2];
          rk = make_double2(rk.x - dn[3], rk.y - dn[4]);
        }
        M2 nU = {0.0, 0.0, 0.0, 0.0};
        if (s + h < NL) {
          const double ja = up[0], jb = up[1], jd = up[2];
          const M2 Tm = {Uk.a * ja + Uk.b * jb, Uk.a * jb + Uk.b * jd, Uk.c * ja + Uk.d * jb, Uk.c * jb + Uk.d * jd};
          Da -= Tm.a * Uk.a + Tm.b * Uk.b;
          Db -= Tm.a * Uk.c + Tm.b * Uk.d;
          Dd -= Tm.c * Uk.c + Tm.d * Uk.d;
          rk = make_double2(rk.x - (Uk.a * up[3] + Uk.b * up[4]), rk.y - (Uk.c * up[3] + Uk.d * up[4]));
          nU = {-(Uk.a * up[5] + Uk.b * up[7]), -(Uk.a * up[6] + Uk.b * up[8]), -(Uk.c * up[5] + Uk.d * up[7]),
                -(Uk.c * up[6] + Uk.d * up[8])};
        }
        Uk = nU;
      }
      if (hasR) {
        const double idet = rcp64a(Da * Dd - Db * Db);
        xR = make_double2((Dd * rk.x - Db * rk.y) * idet, (Da * rk.y - Db * rk.x) * idet);
      } else {
        xR = make_double2(0.0, 0.0);
      }
      xL = make_double2(__shfl_up_sync(0xffffffffu, xR.x, 1), __shfl_up_sync(0xffffffffu, xR.y, 1));   // from lane s - 1
      if (!hasL) xL = make_double2(0.0, 0.0);
      sep_flip = false;
      if (hasR) {   // separator values of this solve (the output if it is the last); weights for the next
        fld(sep0, RL::OFF_G, s) = xR.x;
        fld(sep1, RL::OFF_G, s) = xR.y;
        const bool w0n = ys0 > xR.x, w1n = ys1 > xR.y;
        sep_flip = it == 0 || (real0 && w0n != ws0) || (real1 && w1n != ws1);
        ws0 = w0n;
        ws1 = w1n;
      }
      tm_st_wait();   // this pass A's factor rows are in TMEM before pass B reads them
      // ---------------- pass B: forward substitution of the corrected interior right-hand side
      {
        const double x_na = dr ? xR.x : xL.y, x_nf = dr ? xR.y : xL.x;
        const double x_fa = dr ? xL.y : xR.x, x_ff = dr ? xL.x : xR.y;
        const int fa = dr ? b - 1 : e - 2;
        const int r_last = dr ? b : b + nn - 1;
        const double c0 = cpl(i0, na, Mp, lam) * x_na + lam * x_nf, c1 = lam * x_na;
        const double cL = cpl(r_last, fa, Mp, lam) * x_fa + lam * x_ff, cL2 = lam * x_fa;
        auto passB = [&](auto first_c) {
          constexpr bool FIRST = decltype(first_c)::value;
          MT cur_m = mask_cursor<MT>(im, nn, dr);
          double g1 = 0.0, g2 = 0.0, l1prev = 0.0, rdm1 = 0.0, rdm2 = 0.0;
          unsigned char* rp = shm + r0 * RS;
          uint32_t tc_ = tbase + 4u * (uint32_t)r0;
          double ny = ld_y<TY>(rp, s), nrd, nl1;
          tm_ld2(tc_, nl1, nrd);
          auto stepB = [&](auto last_c, double corr) {
            constexpr bool LASTROW = decltype(last_c)::value;
            const double wv = FIRST ? 1.0 : (mask_take<MT>(cur_m) ? p : q);
            const double f = wv * ny - corr;      // padding rows: y = 0
            const double rd = nrd;
            const double l1c = nl1;
            unsigned char* const cur = rp;
            if constexpr (!LASTROW) {
              rp += dstep;
              tc_ += tstep;
              ny = ld_y<TY>(rp, s);
              tm_ld2(tc_, nl1, nrd);
            }
            const double g = f - l1prev * g1 - lam * rdm2 * g2;
            fld(cur, RL::OFF_G, s) = g * rd;
            g2 = g1;
            g1 = g;
            l1prev = l1c;
            rdm2 = rdm1;
            rdm1 = rd;
          };
          if (nn < 5) {
            for (int t = 0; t < nn; ++t) {
              const double corr = (t == 0 ? c0 : 0.0) + (t == 1 ? c1 : 0.0) + (t == nn - 2 ? cL2 : 0.0) + (t == nn - 1 ? cL : 0.0);
              if (t == nn - 1) stepB(T_{}, corr);
              else stepB(F_{}, corr);
            }
          } else {
            stepB(F_{}, c0);
            stepB(F_{}, c1);
#pragma unroll 2
            for (int t = 2; t < nn - 2; ++t) stepB(F_{}, 0.0);
            stepB(F_{}, cL2);
            stepB(T_{}, cL);
          }
        };
        if (it == 0) passB(T_{});
        else passB(F_{});
      }
    }
    tm_st_wait();
    solves_local += it;   // solves 0 .. it-1 were completed
    // ---------------- write z (interior from the last back-substitution, separators from the last solve)
    __syncwarp();
    TZ* zr = z + row * (int64_t)M;
    for (int t = 0; t < T; ++t)
      if (b + t < M) zr[b + t] = (TZ)*reinterpret_cast<const double*>(shm + t * RS + RL::OFF_G + 8 * s);
  }
  if (solves && s == 0) atomicAdd(solves, solves_local);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem_base_s, tcols);
}

// segment geometry: T rows per segment (>= 4: two interior rows and the two separator rows), P =
// ceil(M / T) <= 32 segments, system size Mp = P T >= M.  The rows M .. Mp-1 extend the last segment
// with weight 0: with zero weight they are free, the second differences they enter vanish on the linear
// extrapolation of z, so the first M rows of the extended minimiser are exactly the original one (DESIGN
// reading A31); every segment then has the same shape and the warp runs one row schedule.
// One CTA per SM (kernels that allocate tensor memory are not co-resident on B200: measured) holding
// wpc = 4 x (spectra per quadrant) warps, bounded by 16 (128 registers per thread) and shared memory.
struct Geo {
  int T, P, wpc;
  uint32_t cols;   // TMEM columns allocated: (wpc / 4) x 4 (T - 2), rounded up to a power of two
};
template <typename TY>
Geo als_geo(int M, size_t smem_max) {
  Geo g;
  g.T = std::max(4, (M + NL - 1) / NL);
  g.P = (M + g.T - 1) / g.T;
  const int per_q = std::max(0, std::min(WPC_MAX / 4, 512 / (4 * (g.T - 2))));
  int wpc = 4 * per_q;
  while (wpc > 4 && (size_t)wpc * g.T * RowLayout<TY>::BYTES > smem_max) wpc -= 4;
  g.wpc = wpc;
  g.cols = 32;
  while (g.cols < 4u * (uint32_t)(g.T - 2) * (uint32_t)(wpc / 4)) g.cols <<= 1;
  return g;
}

}  // namespace

size_t als_part_smem(int M, int y_f64) {
  if (M < 8) return 0;
  const size_t cap = 227 * 1024;
  if (y_f64) { const Geo g = als_geo<double>(M, cap); return (size_t)g.wpc * g.T * RowLayout<double>::BYTES; }
  const Geo g = als_geo<float>(M, cap);
  return (size_t)g.wpc * g.T * RowLayout<float>::BYTES;
}

bool launch_als_part(const void* y, int y_f64, int64_t n, int M, double lam, double p, int iters, void* z, int z_f64,
                     cudaStream_t s, int* solves, unsigned* ctr) {
  if (M < 8 || n <= 0) return false;
  int dev = 0, sms = 148, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t cap = (size_t)maxsm - 64;
  const Geo g = y_f64 ? als_geo<double>(M, cap) : als_geo<float>(M, cap);
  if (g.wpc < 4 || g.cols > 512) return false;
  const size_t sm = (size_t)g.wpc * g.T * (y_f64 ? RowLayout<double>::BYTES : RowLayout<float>::BYTES);
  if (sm > cap) return false;
  const int64_t gr = std::min<int64_t>((n + g.wpc - 1) / g.wpc, sms);
#define FKK_ALS_SEG(TY, TZ)                                                                           \
  {                                                                                                   \
    auto kf = g.T - 2 <= 64 ? als_seg_kernel<TY, TZ, unsigned long long> : als_seg_kernel<TY, TZ, unsigned __int128>; \
    FKK_CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));   \
    if (ctr) FKK_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));                              \
    kf<<<(unsigned)gr, NL * g.wpc, sm, s>>>((const TY*)y, n, M, g.T, g.P, g.cols, lam, p, iters, (TZ*)z, solves, ctr); \
  }
  if (y_f64 && z_f64) FKK_ALS_SEG(double, double)
  else if (!y_f64 && !z_f64) FKK_ALS_SEG(float, float)
  else if (!y_f64 && z_f64) FKK_ALS_SEG(float, double)
  else FKK_ALS_SEG(double, float)
#undef FKK_ALS_SEG
  check_launch("als_seg");
  return true;
}

}  // namespace fkk
