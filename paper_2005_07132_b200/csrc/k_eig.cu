// GPU fp64 top-k symmetric eigensolver for the Gram matrix (F4: the truncated SVD of A through
// G = A^T A; s_i = sqrt(lambda_i), V_k = top-k eigenvectors).  Same algorithm as the
// host reference solver (host_eig.cpp), laid out for the GPU:
//   tridiag   : Householder tridiagonalisation Q^T G Q = T in ONE cooperative kernel (grid barriers;
//               a 16-CTA cluster variant measured slower and is disabled).  Per
//               column every CTA forms the reflector redundantly in smem; one pass over the trailing
//               rows applies the previous column's rank-2 update lazily and forms p = tau A v; one
//               barrier; every CTA forms w = p - (tau/2)(p.v) v.  G stays L2-resident.
//   bisect    : warp per eigenvalue, 32-point Sturm multisection (33x narrowing per round)
//   inviter   : thread per eigenvector, partial-pivoting tridiagonal LU of T - lambda I, 3 solves
//   reorth    : classical Gram-Schmidt, twice, in descending-eigenvalue order (one CTA)
//   backxform : CTA per eigenvector, u = H_0 ... H_{M-3} z, then the sign rule (largest |.| > 0)
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "device_common.cuh"
#include "fkk_internal.h"
#include "tc_common.cuh"

namespace cg = cooperative_groups;

namespace fkk {

namespace {

constexpr int kEigThreads = 256;
constexpr int kTriThreads = 512;
constexpr int kSeg = 256;

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  // every warp reduces the nw partials with shuffles (fixed order: deterministic, same in all warps)
  double s = lane < nw ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// One pass over the trailing matrix and one barrier per column j: the rank-2 update of column j-1 is applied
// lazily while p_j = tau_j A^(j) v_j is formed, row by row (each row read and written once):
//   row_r(A^(j)) = row_r(A^(j-1)) - v_{j-1}[r] w_{j-1} - w_{j-1}[r] v_{j-1}
// Every CTA builds v_j from row j of A^(j-1) plus the pending update (symmetry: row j = column j).
template <bool kCluster>
__global__ void __launch_bounds__(kTriThreads) tridiag_kernel(double* __restrict__ A, int M, double* __restrict__ d,
                                                              double* __restrict__ e, double* __restrict__ tau,
                                                              double* __restrict__ pg) {
  auto barrier = [&]() {
    if constexpr (kCluster) cg::this_cluster().sync();
    else cg::this_grid().sync();
  };
  extern __shared__ __align__(16) double sm[];
  double* v = sm;            // v_j   (index i <-> row j+1+i)
  double* vp = sm + M;       // v_{j-1} (index i <-> row j+i)
  double* wp = sm + 2 * M;   // w_{j-1} (index i <-> row j+i)
  double* red = sm + 3 * M;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31;
  const int gwarp = (blockIdx.x * nt + tid) >> 5;
  const int nwarps = (gridDim.x * nt) >> 5;
  bool pending = false;      // (vp, wp) hold the update of column j-1
  double tprev = 0.0;
  for (int j = 0; j + 2 < M; ++j) {
    const int m = M - j - 1, base = j + 1;
    // reflector of the previous column goes to its (dead) row j-1, after everybody read that row
    if (j > 0 && blockIdx.x == 0) {
      double* rj = A + (int64_t)(j - 1) * M + j;
      for (int i = tid; i < m + 1; i += nt) rj[i] = tprev != 0.0 ? vp[i] : 0.0;
    }
    // x = column j of A^(j) below the diagonal (row j of A^(j-1) + pending update)
    const double* rowj = A + (int64_t)j * M;
    double s = 0.0;
    const double vpj = pending ? vp[0] : 0.0, wpj = pending ? wp[0] : 0.0;
    for (int i = tid; i < m; i += nt) {
      double x = rowj[base + i];
      if (pending) x -= vpj * wp[1 + i] + wpj * vp[1 + i];
      v[i] = x;
      s += x * x;
    }
    double djj = 0.0;
    if (tid == 0) { djj = rowj[j]; if (pending) djj -= 2.0 * vpj * wpj; }
    const double nrm2 = block_sum_d(s, red);
    const double x0 = v[0];
    const double nrm = sqrt(nrm2);
    const double alpha = x0 >= 0.0 ? -nrm : nrm;
    const double v0 = x0 - alpha;
    const double vtv = nrm2 - x0 * x0 + v0 * v0;
    const double t = (nrm == 0.0 || vtv == 0.0) ? 0.0 : 2.0 / vtv;
    __syncthreads();
    if (tid == 0) v[0] = v0;
    if (blockIdx.x == 0 && tid == 0) {
      d[j] = djj;
      e[j] = t == 0.0 ? x0 : alpha;
      tau[j] = t;
    }
    __syncthreads();
    // pass over the trailing rows: apply the pending update, write back, p = t A^(j) v.  A warp
    // task is (row, 256-column segment): 8 independent loads per lane in flight; the per-segment
    // partial dots are summed in a fixed order after the grid barrier (deterministic).
    const int nseg = (m + kSeg - 1) / kSeg;
    for (int task = gwarp; task < m * nseg; task += nwarps) {
      const int r = task / nseg, sg = task - r * nseg;
      double* row = A + (int64_t)(base + r) * M + base;
      const int c0 = sg * kSeg, c1 = min(m, c0 + kSeg);
      double acc = 0.0;
      if (pending) {
        const double vr = vp[1 + r], wr = wp[1 + r];
#pragma unroll 8
        for (int c = c0 + lane; c < c1; c += 32) {
          const double a = row[c] - (vr * wp[1 + c] + wr * vp[1 + c]);
          row[c] = a;
          acc = fma(a, v[c], acc);
        }
      } else {
#pragma unroll 8
        for (int c = c0 + lane; c < c1; c += 32) acc = fma(row[c], v[c], acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) pg[(int64_t)sg * M + r] = t * acc;
    }
    barrier();
    // w_j = p - (t/2)(p.v) v  -> becomes the pending update (index shift: row j+1+i -> i)
    double ps = 0.0;
    for (int i = tid; i < m; i += nt) {
      double pv = 0.0;
      for (int sg = 0; sg < nseg; ++sg) pv += pg[(int64_t)sg * M + i];
      wp[i] = pv;
      ps += pv * v[i];
    }
    const double K = 0.5 * t * block_sum_d(ps, red);
    for (int i = tid; i < m; i += nt) { wp[i] -= K * v[i]; vp[i] = v[i]; }
    if (t == 0.0) for (int i = tid; i < m; i += nt) { wp[i] = 0.0; vp[i] = 0.0; }
    __syncthreads();
    pending = true;
    tprev = t;
  }
  // flush: reflector of the last column and the trailing 2 x 2 block with the pending update
  if (blockIdx.x == 0) {
    const int j = M - 2;
    if (j > 0) {
      double* rj = A + (int64_t)(j - 1) * M + j;
      for (int i = tid; i < 2; i += nt) rj[i] = tprev != 0.0 ? vp[i] : 0.0;
    }
    if (tid == 0) {
      double a00 = A[(int64_t)(M - 2) * M + (M - 2)], a10 = A[(int64_t)(M - 1) * M + (M - 2)];
      double a11 = A[(int64_t)(M - 1) * M + (M - 1)];
      if (pending && M >= 3) {
        a00 -= 2.0 * vp[0] * wp[0];
        a10 -= vp[1] * wp[0] + wp[1] * vp[0];
        a11 -= 2.0 * vp[1] * wp[1];
      }
      d[M - 2] = a00;
      e[M - 2] = a10;
      d[M - 1] = a11;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Row-resident variant (default when the owned rows fit in shared memory): CTA c of the cooperative
// grid keeps rows r = c, c + P, c + 2P, ... of the working matrix in its shared memory for the whole
// tridiagonalisation, so the per-column pass touches no L2.  Per column j, with (v_{j-1}, w_{j-1})
// the pending rank-2 update:
//   after the barrier of column j-1: read p_{j-1} and column j of A^(j-1) (= row j, symmetry) in ONE
//     batch of L2 loads; form w_{j-1} = p - (t/2)(p.v) v; x = row j of A^(j); reflector v_j, t_j
//     (every CTA redundantly, on 4 warps: the "column chain");
//   pass: every owned row r > j gets the pending update (eagerly, in smem) and p_r = t_j A^(j)[r,:] v_j;
//     each row also emits its entry A^(j)[r][j+1] (column j+1 = row j+1 for the next chain);
//   one grid barrier.
// The last columns (trailing block small enough for the shared memory of ONE thread-block cluster)
// continue in tridiag_tail_kernel with cluster barriers (~0.2 us) instead of grid barriers (~1.5-2 us).
constexpr int kTsThreads = 512;
constexpr int kTsChain = 128;   // threads of the per-column chain (warps 0-3)
constexpr int kTsMaxM = 16 * kTsChain;   // chain registers: 16 entries per chain thread

__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// sum over the 128 chain threads: warp sums, then every chain thread adds the 4 partials in a fixed order
__device__ __forceinline__ double chain_sum(double v, double* buf) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
  asm volatile("bar.sync 1, 128;" ::: "memory");
  return (buf[0] + buf[1]) + (buf[2] + buf[3]);
}

// The column chain of column j, run by the 128 chain threads; chain thread ct owns the entries
// c = j + ct + 128 i (i < NPL) in registers: Pv = p_{j-1}[c], X = A^(j-1)[j][c] on entry (zero past M).
//   K = (t_{j-1}/2) p.v_{j-1};  w_{j-1} = p - K v_{j-1} -> wp;  x = X - v_{j-1}[j] w - w[j] v_{j-1}
//   (= row j of A^(j));  reflector v_j (x below the diagonal with v[j+1] = x[j+1] - alpha) -> v,
//   t_j = 2 / v.v -> red[8];  d[j], e[j], tau[j] by the writer.
// Only the two 128-thread sums synchronise.  pj = p_{j-1}[j], vj = v_{j-1}[j] are read by every thread
// before any wp write.
// sqrt and 1/x for the column chain's critical path: MUFU seeds + Newton steps (~1 ulp; the IEEE
// sequences were ~150 cycles of the per-column latency)
__device__ __forceinline__ double chain_sqrt(double x) {
  if (!(x > 0.0)) return 0.0;
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x * r, r, 1.5);
  r = r * fma(-0.5 * x * r, r, 1.5);
  const double s0 = x * r;
  return fma(0.5 * r, fma(-s0, s0, x), s0);
}
__device__ __forceinline__ double chain_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int NPL, bool SIGNAL_W = false>
__device__ __forceinline__ void column_chain(int j, int M, double (&Pv)[NPL], double (&X)[NPL], double pj,
                                             const double* vp, double* wp, double* v, double* red, double tprev,
                                             bool writer, double* d, double* e, double* tau) {
  const int ct = threadIdx.x;
  if (j > 0) {
    double V[NPL];
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int c = j + ct + kTsChain * i;
      V[i] = c < M ? vp[c] : 0.0;
      s = fma(Pv[i], V[i], s);
    }
    const double vj = vp[j];
    const double K = 0.5 * tprev * chain_sum(s, red);
    const double wj = tprev != 0.0 ? pj - K * vj : 0.0;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int c = j + ct + kTsChain * i;
      const double w = tprev != 0.0 ? Pv[i] - K * V[i] : 0.0;
      X[i] -= vj * w + wj * V[i];
      if (c < M) wp[c] = w;
    }
    // w is complete: the pass warps may apply the pending update to their rows while this chain
    // finishes the reflector (named barrier 2: 128 arrivals here + the 384 pass threads' bar.sync)
    if constexpr (SIGNAL_W) asm volatile("bar.arrive 2, %0;" ::"r"(kTsThreads) : "memory");
  }
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int c = j + ct + kTsChain * i;
    if (c > j && c < M) {
      s2 = fma(X[i], X[i], s2);
      v[c] = X[i];
    }
  }
  if (ct == 1) red[12] = X[0];   // x[j+1]
  if (ct == 0) red[13] = X[0];   // x[j]
  const double nrm2 = chain_sum(s2, red + 4);
  const double x0 = red[12];
  const double nrm = chain_sqrt(nrm2);
  const double alpha = x0 >= 0.0 ? -nrm : nrm;
  const double v0 = x0 - alpha;
  const double vtv = nrm2 - x0 * x0 + v0 * v0;
  const double t = (nrm == 0.0 || vtv == 0.0) ? 0.0 : 2.0 * chain_rcp(vtv);
  if (ct == 1) v[j + 1] = v0;
  if (ct == 0) {
    red[8] = t;
    if (writer) {
      d[j] = red[13];
      e[j] = t == 0.0 ? x0 : alpha;
      tau[j] = t;
    }
  }
}

// row[c] -= vr w[c] + wr v_{j-1}[c] for c >= m0 (one warp): the loads of four iterations are issued
// before their stores -- the compiler otherwise keeps every load behind the previous row store (the
// arrays may alias), a ~100-cycle dependent chain per iteration (tools/micro/rowpass.cu)
__device__ __forceinline__ void row_update(double* row, int m0, int M, double vr, double wr, const double* vp,
                                           const double* wp) {
  const int lane = threadIdx.x & 31;
  int c = m0 + lane;
  for (; c + 96 < M; c += 128) {
    double a[4], ww[4], pp[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = row[c + 32 * u];
      ww[u] = wp[c + 32 * u];
      pp[u] = vp[c + 32 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) row[c + 32 * u] = a[u] - (vr * ww[u] + wr * pp[u]);
  }
  for (; c < M; c += 32) row[c] -= vr * wp[c] + wr * vp[c];
}

// The pass over one owned row r > j (one warp): pending update row -= v_{j-1}[r] w + w[r] v_{j-1} (if
// pending) and the dot A^(j)[r,:] v_j over c > j.  Lane 0 handles c = j + 1 first, so row[j+1]
// (= A^(j)[r][j+1]) is its own write.
__device__ __forceinline__ double row_pass(double* row, int roff, int m0, int M, bool pending, double vr, double wr,
                                           const double* vp, const double* wp, const double* v, double* pub) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if (pending) {
    // groups of four iterations with every load before the group's stores (see row_update)
    int c = m0 + lane;
    for (; c + 96 < M; c += 128) {
      double a[4], ww[4], pp[4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = row[c + 32 * u - roff];
        ww[u] = wp[c + 32 * u];
        pp[u] = vp[c + 32 * u];
        vv[u] = v[c + 32 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] -= vr * ww[u] + wr * pp[u];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        row[c + 32 * u - roff] = a[u];
        if (pub) pub[c + 32 * u] = a[u];
        acc = fma(a[u], vv[u], acc);
      }
    }
    for (; c < M; c += 32) {
      const double a = row[c - roff] - (vr * wp[c] + wr * vp[c]);
      row[c - roff] = a;
      if (pub) pub[c] = a;
      acc = fma(a, v[c], acc);
    }
  } else {
#pragma unroll 4
    for (int c = m0 + lane; c < M; c += 32) {
      const double a = row[c - roff];
      if (pub) pub[c] = a;
      acc = fma(a, v[c], acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Trailing 2 x 2 block after the last column (j = M-3): w_{M-3} from p_{M-3} (pcur), the reflector
// v_{M-3} -> row M-3 of Wk, and d[M-2], e[M-2], d[M-1] from rows M-2, M-1 of A^(M-3) (published to Wk).
// One CTA; p read with loader(c).
template <typename PL>
__device__ __forceinline__ void tail_flush(int M, PL pload, const double* vp, double* wp, double tprev, double* red,
                                           double* Wk, double* d, double* e) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int j = M - 2;
  double s = 0.0;
  for (int c = j + tid; c < M; c += nt) {
    const double pv = pload(c);
    wp[c] = pv;
    s += pv * vp[c];
  }
  const double K = 0.5 * tprev * block_sum_d(s, red);
  for (int c = j + tid; c < M; c += nt) wp[c] = tprev != 0.0 ? wp[c] - K * vp[c] : 0.0;
  __syncthreads();
  double* rj = Wk + (int64_t)(j - 1) * M;
  for (int c = j + tid; c < M; c += nt) rj[c] = tprev != 0.0 ? vp[c] : 0.0;
  if (tid == 0) {
    const double* r0 = Wk + (int64_t)(M - 2) * M;
    const double* r1 = Wk + (int64_t)(M - 1) * M;
    d[M - 2] = __ldcg(r0 + M - 2) - 2.0 * vp[M - 2] * wp[M - 2];
    e[M - 2] = __ldcg(r1 + M - 2) - (vp[M - 1] * wp[M - 2] + wp[M - 1] * vp[M - 2]);
    d[M - 1] = __ldcg(r1 + M - 1) - 2.0 * vp[M - 1] * wp[M - 1];
  }
}

// Grid phase: columns j < jend (jend = M - 2: all).  With jend < M - 2 every CTA leaves its owned rows
// r >= jend (state A^(jend-1), columns >= jend) in Wk and CTA 0 the reflector v_{jend-1} in row jend-1,
// for tridiag_tail_kernel.
template <int NPL>
__global__ void __launch_bounds__(kTsThreads, 1) tridiag_rows_kernel(const double* __restrict__ G, double* __restrict__ Wk,
                                                                   int M, int jend, double* __restrict__ d,
                                                                   double* __restrict__ e, double* __restrict__ tau,
                                                                   double* __restrict__ Pg, unsigned int* __restrict__ ctr,
                                                                   int dbg) {
  extern __shared__ __align__(16) double sm[];
  const int P = gridDim.x, cta = blockIdx.x;
  const int R = (M - cta + P - 1) / P;            // owned rows: r = cta + i P, i < R
  double* rows = sm;                               // R x M
  double* vbuf0 = rows + (size_t)R * M;            // v_j / v_{j-1} ping-pong (absolute index)
  double* vbuf1 = vbuf0 + M;
  double* wp = vbuf1 + M;                          // w_{j-1}
  double* red = wp + M;                            // 32
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int i = 0; i < R; ++i) {
    const double* g = G + (int64_t)(cta + i * P) * M;
    for (int c = tid; c < M; c += nt) rows[(size_t)i * M + c] = g[c];
  }
  for (int c = tid; c < 3 * M; c += nt) vbuf0[c] = 0.0;   // no uninitialised value ever meets a zero weight
  __syncthreads();
  unsigned int target = 0;
  double tprev = 0.0;
  double* v = vbuf0;
  double* vp = vbuf1;
  long long tsr[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // dbg 3: phase clocks of CTA 0 at column 500
  auto stamp = [&](int j, int ph) {
    if (dbg == 3 && cta == 0 && tid == 0 && j == 500) tsr[ph] = clock64();
  };
  const int jstop = min(jend, M - 2);
  for (int j = 0; j < jstop; ++j) {
    stamp(j, 0);
    if (tid < kTsChain) {
      double X[NPL], Pv[NPL];
      double pj = 0.0;
      if (j == 0) {
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
          const int c = tid + kTsChain * i;
          X[i] = c < M ? G[c] : 0.0;
          Pv[i] = 0.0;
        }
      } else {
        const double* pprev = Pg + ((j - 1) & 1) * M;         // p_{j-1}
        const double* cprev = Pg + (2 + ((j - 1) & 1)) * M;   // column j of A^(j-1) = row j
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
          const int c = j + tid + kTsChain * i;
          Pv[i] = c < M ? __ldcg(pprev + c) : 0.0;
          X[i] = c < M ? __ldcg(cprev + c) : 0.0;
        }
        pj = __ldcg(pprev + j);
      }
      stamp(j, 1);
      column_chain<NPL, true>(j, M, Pv, X, pj, vp, wp, v, red, tprev, cta == 0, d, e, tau);
      stamp(j, 2);
    } else if (j > 0) {
      if (dbg != 5) {   // dbg 5: timing without the reflector stores (wrong results)
        // reflector v_{j-1} -> dead row j-1, a 1/P slice per CTA
        double* rj = Wk + (int64_t)(j - 1) * M;
        const int len = (M - j + P - 1) / P, c0 = j + cta * len, c1 = min(M, c0 + len);
        for (int c = c0 + tid - kTsChain; c < c1; c += nt - kTsChain) rj[c] = tprev != 0.0 ? vp[c] : 0.0;
      }
      // pending rank-2 update of the owned rows r > j as soon as w is known (overlaps the chain's
      // second half): row -= v_{j-1}[r] w + w[r] v_{j-1} over c > j; the pass then only reads
      asm volatile("bar.sync 2, %0;" ::"r"(kTsThreads) : "memory");
      const int m0u = j + 1;
      for (int i = warp - kTsChain / 32; i < R; i += nw - kTsChain / 32) {
        const int r = cta + i * P;
        if (r <= j || tprev == 0.0) continue;
        double* row = rows + (size_t)i * M;
        const double vr = vp[r], wr = wp[r];
        row_update(row, m0u, M, vr, wr, vp, wp);
      }
    }
    __syncthreads();
    const double t = red[8];
    stamp(j, 3);
    // ---- pass over the owned rows r > j: pending update (eager, smem), p_r = t A^(j)[r,:] v_j
    const int m0 = j + 1;
    const bool last = j + 3 == M;
    // one non-chain warp per owned row (the same warp that applied its pending update above); dbg 1:
    // timing without the pass
    for (int i = warp - kTsChain / 32; i < (dbg == 1 || warp < kTsChain / 32 ? 0 : R); i += nw - kTsChain / 32) {
      const int r = cta + i * P;
      if (r <= j) continue;
      double* row = rows + (size_t)i * M;
      const bool publish = last && (r == j + 1 || r == M - 1);   // rows for the trailing 2 x 2 flush
      const double acc = row_pass(row, 0, m0, M, false, 0.0, 0.0, vp, wp, v, publish ? Wk + (int64_t)r * M : nullptr);
      // p_r and A^(j)[r][j+1] into the column-parity buffers: a fast CTA's next pass never overwrites
      // what a slow CTA still reads
      if (lane == 0) {
        Pg[(j & 1) * M + r] = t * acc;
        Pg[(2 + (j & 1)) * M + r] = row[m0];
      }
    }
    stamp(j, 4);
    if (dbg != 2) {   // dbg 2: timing without the barrier (wrong results); = grid_barrier with stamps
      __syncthreads();
      stamp(j, 5);
      target += gridDim.x;
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
        unsigned int cv;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cv) : "l"(ctr) : "memory");
        } while ((int)(cv - target) < 0);
      }
      stamp(j, 6);
      __syncthreads();
    }
    stamp(j, 7);
    tprev = t;
    double* tmp = vp; vp = v; v = tmp;
  }
  if (jstop < M - 2) {
    // hand-over to the cluster tail: owned rows r >= jend (columns >= jend), reflector v_{jend-1}
    for (int i = 0; i < R; ++i) {
      const int r = cta + i * P;
      if (r < jend) continue;
      for (int c = jend + tid; c < M; c += nt) Wk[(int64_t)r * M + c] = rows[(size_t)i * M + c];
    }
    if (cta == 0 && jend > 0)
      for (int c = jend + tid; c < M; c += nt) Wk[(int64_t)(jend - 1) * M + c] = tprev != 0.0 ? vp[c] : 0.0;
  } else if (cta == 0 && M >= 3) {
    const double* pcur = Pg + ((M - 3) & 1) * M;
    tail_flush(M, [&](int c) { return __ldcg(pcur + c); }, vp, wp, tprev, red, Wk, d, e);
  }
  if (dbg == 3 && cta == 0 && tid == 0)
    for (int q = 0; q < 8; ++q) e[q] = (double)tsr[q];
}

// Cluster tail: columns j >= jend of the same algorithm on ONE cluster of CL CTAs, the trailing
// (M - jend)^2 block resident in their shared memory (rows r = jend + rank + i CL).  p_r and
// A^(j)[r][j+1] are pushed into every CTA's shared memory with st.shared::cluster during the pass
// (parity-buffered), so a column costs the chain, the pass and one cluster barrier -- no L2 round trip.
// Entry state (jend > 0): rows r >= jend of A^(jend-1) in Wk, v_{jend-1} in Wk row jend-1, p_{jend-1}
// and column jend of A^(jend-1) in the Pg parity buffers, t_{jend-1} = tau[jend-1].  jend = 0: G.
template <int NPL>
__global__ void __launch_bounds__(kTsThreads, 1) tridiag_tail_kernel(const double* __restrict__ G, double* __restrict__ Wk,
                                                                   int M, int jend, double* __restrict__ d,
                                                                   double* __restrict__ e, double* __restrict__ tau,
                                                                   const double* __restrict__ Pg, int dbg) {
  extern __shared__ __align__(16) double sm[];
  long long tsr[6] = {0, 0, 0, 0, 0, 0};   // dbg >= 3: phase clocks of rank 0 at column M - dcol
  const int dcol = (dbg >> 8) ? (dbg >> 8) : 100;
  dbg &= 0xff;
  uint32_t rank, CL;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(CL));
  const int mt = M - jend;
  const int R = (mt - (int)rank + (int)CL - 1) / (int)CL;   // owned rows r = jend + rank + i CL
  double* rows = sm;                                        // row i: rows + i mt, local column c - jend
  // vectors indexed by the absolute column c (size M each, so no pointer leaves the shared window);
  // same layout in every CTA of the cluster
  double* base = sm + (size_t)((mt + CL - 1) / CL) * mt;
  double* vbuf0 = base;
  double* vbuf1 = vbuf0 + M;
  double* wp = vbuf1 + M;
  double* pb = wp + M;      // pb + parity * M: p of the column with that parity
  double* cb = pb + 2 * M;  // cb + parity * M: column j+1 of A^(j)
  double* red = base + 7 * (size_t)M;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int pprev0 = (jend - 1) & 1;
  for (int i = 0; i < R; ++i) {
    const int r = jend + (int)rank + i * (int)CL;
    const double* src = jend > 0 ? Wk + (int64_t)r * M : G + (int64_t)r * M;
    for (int c = jend + tid; c < M; c += nt) rows[(size_t)i * mt + (c - jend)] = src[c];
  }
  for (int c = jend + tid; c < M; c += nt) {
    vbuf0[c] = 0.0;
    wp[c] = 0.0;
    vbuf1[c] = jend > 0 ? __ldcg(Wk + (int64_t)(jend - 1) * M + c) : 0.0;
    pb[pprev0 * M + c] = jend > 0 ? __ldcg(Pg + pprev0 * M + c) : 0.0;
    cb[pprev0 * M + c] = jend > 0 ? __ldcg(Pg + (2 + pprev0) * M + c) : G[c];
  }
  double tprev = jend > 0 ? tau[jend - 1] : 0.0;
  // remote addresses of the p / column buffers in every CTA of the cluster (lane q < CL: CTA q)
  uint32_t rpb = 0, rcb = 0;
  if (lane < (int)CL) {
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rpb) : "r"(tc::smem_u32(pb)), "r"(lane));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rcb) : "r"(tc::smem_u32(cb)), "r"(lane));
  }
  cluster_sync_all();
  double* v = vbuf0;
  double* vp = vbuf1;
  for (int j = jend; j + 2 < M; ++j) {
    const int pp = (j - 1) & 1, pc = j & 1;
    if (tid < kTsChain) {
      double X[NPL], Pv[NPL];
      const double* pprev = pb + pp * M;
      const double* cprev = cb + pp * M;
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        const int c = j + tid + kTsChain * i;
        Pv[i] = c < M ? pprev[c] : 0.0;
        X[i] = c < M ? cprev[c] : 0.0;
      }
      if (dbg >= 3 && rank == 0 && tid == 0 && j == M - dcol) tsr[0] = clock64();
      column_chain<NPL>(j, M, Pv, X, pprev[j], vp, wp, v, red, tprev, rank == 0, d, e, tau);
      if (dbg >= 3 && rank == 0 && tid == 0 && j == M - dcol) tsr[1] = clock64();
    } else if (j > 0) {
      double* rj = Wk + (int64_t)(j - 1) * M;
      const int len = (M - j + CL - 1) / CL, c0 = j + rank * len, c1 = min(M, c0 + len);
      for (int c = c0 + tid - kTsChain; c < c1; c += nt - kTsChain) rj[c] = tprev != 0.0 ? vp[c] : 0.0;
    }
    __syncthreads();
    if (dbg >= 3 && rank == 0 && tid == 0 && j == M - dcol) tsr[2] = clock64();
    const double t = red[8];
    const int m0 = j + 1;
    const bool last = j + 3 == M;
    for (int i = warp; i < R; i += nw) {
      const int r = jend + (int)rank + i * (int)CL;
      if (r <= j) continue;
      double* row = rows + (size_t)i * mt;
      const bool publish = last && (r == j + 1 || r == M - 1);
      const double acc = row_pass(row, jend, m0, M, j > 0, vp[r], wp[r], vp, wp, v, publish ? Wk + (int64_t)r * M : nullptr);
      const double cval = __shfl_sync(0xffffffffu, lane == 0 ? row[m0 - jend] : 0.0, 0);
      if (lane < (int)CL && dbg != 4) {   // dbg 4: timing without the pushes (wrong results)
        const uint32_t off = (uint32_t)((pc * M + r) * 8);
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rpb + off), "d"(t * acc) : "memory");
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rcb + off), "d"(cval) : "memory");
      }
    }
    if (dbg >= 3 && rank == 0 && tid == 0 && j == M - dcol) tsr[3] = clock64();
    cluster_sync_all();
    if (dbg >= 3 && rank == 0 && tid == 0 && j == M - dcol) tsr[4] = clock64();
    tprev = t;
    double* tmp = vp; vp = v; v = tmp;
  }
  if (rank == 0 && M >= 3) {
    const double* pcur = pb + ((M - 3) & 1) * M;
    tail_flush(M, [&](int c) { return pcur[c]; }, vp, wp, tprev, red, Wk, d, e);
  }
  if (dbg >= 3 && rank == 0 && tid == 0)
    for (int q = 0; q < 5; ++q) d[q] = (double)tsr[q];
}

size_t tridiag_rows_smem(int M, int P) {
  const int R = (M + P - 1) / P;
  return ((size_t)R * M + 3 * (size_t)M + 32) * sizeof(double);
}

size_t tridiag_tail_smem(int mt, int CL, int Mfull) {
  return ((size_t)((mt + CL - 1) / CL) * mt + 7 * (size_t)Mfull + 32) * sizeof(double);
}

// 1/q via the MUFU seed + two Newton steps (full fp64 accuracy for normal q; a Sturm count only
// needs the sign of each q to be right away from the eigenvalues)
__device__ __forceinline__ double fast_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double err = fma(-q, r, 1.0);
  r = fma(r, err, r);
  err = fma(-q, r, 1.0);
  return fma(r, err, r);
}

__device__ __forceinline__ int sturm_count_dev(const double* d, const double* e, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0) cnt++;
  for (int i = 1; i < n; ++i) {
    const double ee = e[i - 1];
    q = d[i] - x - ee * ee * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) cnt++;
  }
  return cnt;
}

// warp per eigenvalue index jj (jj-th largest); also computes ||T|| bounds
__global__ void bisect_kernel(const double* __restrict__ d, const double* __restrict__ e, int M, int k,
                              double* __restrict__ lam, double* __restrict__ tnorm_out) {
  extern __shared__ double bsm[];
  double* sd = bsm;          // d
  double* se2 = bsm + M;     // se2[i] = e[i-1]^2
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    sd[i] = d[i];
    se2[i] = i > 0 ? e[i - 1] * e[i - 1] : 0.0;
  }
  __shared__ int gred[2][32];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int jj = blockIdx.x;   // one CTA per eigenvalue
  if (jj >= k) return;
  double gl = 1e300, gu = -1e300, tn = 0.0;
  for (int i = lane; i < M; i += 32) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < M - 1 ? fabs(e[i]) : 0.0);
    gl = fmin(gl, d[i] - r);
    gu = fmax(gu, d[i] + r);
    tn = fmax(tn, fabs(d[i]) + r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
    tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
  }
  const double eps = 2.220446049250313e-16;
  const double pivmin = fmax(1e-300, tn * 1e-300);
  double lo = gl - 2.0 * eps * tn * M - 1e-300, hi = gu + 2.0 * eps * tn * M + 1e-300;
  const int idx = M - 1 - jj;   // ascending index
  // 256-point multisection per round (one CTA of 128 threads per eigenvalue, 2 interleaved Sturm
  // chains per thread).  The count uses the
  // division-free three-term form p_{i+1} = (d_i - x) p_i - e_{i-1}^2 p_{i-1} (q_i = p_{i+1} / p_i,
  // the LDL^T pivots of T - x I; #{q_i < 0} = #sign changes): one DFMA on the dependent chain per
  // step instead of a reciprocal; rescaled by a power of two every 8 steps (the ratios, hence the
  // signs, are unchanged).  Rounding: fl((d-x)p - e^2 p') = (...)(1 + delta) gives q_i with the same
  // relative error per step as the ratio form.
  constexpr int NCH = 2;
  const int NPT = blockDim.x * NCH;   // points per round over the whole CTA
  for (int round = 0; round < 64; ++round) {
    // absolute tolerance 2 eps ||T|| (LAPACK dstebz's default abstol scale): inverse iteration needs
    // lambda to O(eps ||T||), and every consumer compares eigenvalues normwise (sigma_i against
    // sigma_1); a relative-to-lambda stop spent ~3 extra rounds on the plateau eigenvalues
    if (hi - lo <= 2.0 * eps * tn + pivmin) break;
    const double w = (hi - lo) / (double)(NPT + 1);
    double x[NCH], p1[NCH], p2[NCH];
    int cnt[NCH];
#pragma unroll
    for (int u = 0; u < NCH; ++u) {
      x[u] = lo + w * (double)(threadIdx.x * NCH + u + 1);   // point g = tid * NCH + u at lo + w (g + 1)
      p2[u] = 1.0;
      p1[u] = d[0] - x[u];
      if (p1[u] == 0.0) p1[u] = -pivmin;
      cnt[u] = p1[u] < 0.0 ? 1 : 0;
    }
    auto step = [&](double dvh, double evh) {
#pragma unroll
      for (int u = 0; u < NCH; ++u) {
        // an exact zero needs no pivmin patch here: with p_{i+1} = +-0, q_i and q_{i+1} = -e^2 p_i / 0
        // have opposite signs, so the pair contributes exactly one negative pivot, as in the ratio
        // form with q_i -> -pivmin
        const double pn = fma(dvh - x[u], p1[u], -evh * p2[u]);
        cnt[u] += (int)(((unsigned)__double2hiint(pn) ^ (unsigned)__double2hiint(p1[u])) >> 31);
        p2[u] = p1[u];
        p1[u] = pn;
      }
    };
    auto rescale = [&]() {
#pragma unroll
      for (int u = 0; u < NCH; ++u) {
        const int ex = ((__double2hiint(p1[u]) >> 20) & 0x7ff) - 1023;
        if (ex > 256 || ex < -256) {
          const double sc = __hiloint2double((1023 - ex) << 20, 0);   // 2^-ex
          p1[u] *= sc;
          p2[u] *= sc;
        }
      }
    };
    int i = 1;
    if (i + 8 <= M) {
      // full blocks of 8 steps; the next block's (d, e^2) are loaded while this block computes
      double dv[8], ev[8], dn[8], en[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) { dv[h] = sd[i + h]; ev[h] = se2[i + h]; }
      for (; i + 8 <= M; i += 8) {
        const bool more = i + 16 <= M;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          dn[h] = more ? sd[i + 8 + h] : 0.0;
          en[h] = more ? se2[i + 8 + h] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) step(dv[h], ev[h]);
        rescale();
#pragma unroll
        for (int h = 0; h < 8; ++h) { dv[h] = dn[h]; ev[h] = en[h]; }
      }
    }
    for (; i < M; ++i) step(sd[i], se2[i]);
    // first point (in ascending order) with more than idx eigenvalues below it
    int g = NPT;
#pragma unroll
    for (int u = NCH - 1; u >= 0; --u)
      if (cnt[u] > idx) g = threadIdx.x * NCH + u;
    g = (int)__reduce_min_sync(0xffffffffu, (unsigned)g);
    if (lane == 0) gred[round & 1][wid] = g;   // parity slots: one barrier per round
    __syncthreads();
    g = gred[round & 1][0];
    for (int w2 = 1; w2 < nwarp; ++w2) g = min(g, gred[round & 1][w2]);
    const double nlo = lo + w * (double)g;            // point g-1 (or lo)
    const double nhi = g == NPT ? hi : lo + w * (double)(g + 1);
    lo = nlo;
    hi = nhi;
  }
  if (threadIdx.x == 0) {
    lam[jj] = 0.5 * (lo + hi);
    if (jj == 0) tnorm_out[0] = tn;
  }
}

// CTA (one warp) per eigenvector: inverse iteration on T - lambda I (LAPACK dgttrf/dgttrs logic),
// the LU factors in shared memory (lane 0 runs the recurrences; the warp fills and normalises).
__global__ void __launch_bounds__(32) inviter_kernel(const double* __restrict__ d, const double* __restrict__ e, int M,
                                                     int k, const double* __restrict__ lam,
                                                     const double* __restrict__ tnorm, double* __restrict__ Z) {
  extern __shared__ __align__(16) double sh[];
  const int jj = blockIdx.x;
  const int lane = threadIdx.x;
  double* dl = sh;
  double* dd = dl + M;
  double* du = dd + M;
  double* du2 = du + M;
  double* z = du2 + M;
  unsigned char* piv = reinterpret_cast<unsigned char*>(z + M);
  const double eps = 2.220446049250313e-16;
  const double tn = tnorm[0];
  const double tiny = eps * tn + 1e-300;
  double l = lam[jj];
  if (jj > 0 && fabs(lam[jj - 1] - l) < 10.0 * eps * tn) l -= 10.0 * eps * tn * jj;   // split exact ties
  for (int i = lane; i < M; i += 32) {
    dd[i] = d[i] - l;
    piv[i] = 0;
    if (i < M - 1) { dl[i] = e[i]; du[i] = e[i]; }
    if (i < M - 2) du2[i] = 0.0;
    uint64_t s = 0x9E3779B97F4A7C15ull * (uint64_t)(jj + 1) + 0xD1B54A32D192ED03ull * (uint64_t)(i + 1);
    s ^= s >> 31; s *= 0x7FB5D329728EA185ull; s ^= s >> 27; s *= 0x81DADEF4BC2DD44Dull; s ^= s >> 33;
    z[i] = ((double)(s >> 11) / 9007199254740992.0) - 0.5;
  }
  __syncwarp();
  if (lane == 0) {
    // LU with partial pivoting of the tridiagonal T - l I (LAPACK dgttrf order); the modified
    // diagonal and super-diagonal entries of the next row travel in registers (no smem round trip
    // on the dependent chain), reciprocals by MUFU seed + two Newton steps
    double di = dd[0], ui = M > 1 ? du[0] : 0.0;
#pragma unroll 2
    for (int i = 0; i < M - 1; ++i) {
      const double li = dl[i], dnext = dd[i + 1];
      const double unext = i < M - 2 ? du[i + 1] : 0.0;
      double dn, un;
      if (fabs(di) >= fabs(li)) {
        if (di == 0.0) di = tiny;
        const double f = li * fast_rcp(di);
        dl[i] = f;
        dd[i] = di;
        du[i] = ui;
        dn = dnext - f * ui;
        un = unext;
      } else {
        const double f = di * fast_rcp(li);
        dd[i] = li;
        dl[i] = f;
        du[i] = dnext;
        dn = ui - f * dnext;
        if (i < M - 2) du2[i] = unext;
        un = -f * unext;
        piv[i] = 1;
      }
      di = dn;
      ui = un;
    }
    dd[M - 1] = di;
  }
  __syncwarp();
  for (int i = lane; i < M; i += 32) {
    double v = dd[i];
    if (fabs(v) < tiny) v = v < 0 ? -tiny : tiny;
    dd[i] = 1.0 / v;     // keep reciprocals: the solves multiply
  }
  __syncwarp();
  // two solves: lambda is within 2 eps ||T|| of the eigenvalue, so each solve grows the wanted
  // component by ~gap / (eps ||T||) against the others; the CholQR2 that follows restores
  // orthogonality inside clusters.  A near-tie (relative gap to a computed neighbour below 1e-8)
  // gets a third solve: there the vector's mix inside the cluster converges more slowly, and the
  // per-column argmax of U S (q, Eqs. 13-15) depends on that mix.
  double gap = 1e300;
  if (jj > 0) gap = fmin(gap, fabs(lam[jj - 1] - lam[jj]));
  if (jj + 1 < k) gap = fmin(gap, fabs(lam[jj + 1] - lam[jj]));
  const int nsolve = gap < 1e-8 * tn ? 3 : 2;
  for (int it = 0; it < nsolve; ++it) {
    if (lane == 0) {
      // forward: apply P and L^-1 (the running entry in a register)
      double zi = z[0];
#pragma unroll 4
      for (int i = 0; i < M - 1; ++i) {   // branch-free: a = stored entry, b - f a = next running entry
        const double bi1 = z[i + 1], f = dl[i];
        const bool pv = piv[i] != 0;
        const double a = pv ? bi1 : zi, b = pv ? zi : bi1;
        z[i] = a;
        zi = fma(-f, a, b);
      }
      // backward: U^-1 (three-band), the two following entries in registers
      double z1 = zi * dd[M - 1], z2 = 0.0;
      z[M - 1] = z1;
      if (M > 1) {
        const double zz = (z[M - 2] - du[M - 2] * z1) * dd[M - 2];
        z[M - 2] = zz;
        z2 = z1;
        z1 = zz;
      }
#pragma unroll 4
      for (int i = M - 3; i >= 0; --i) {   // one DFMA on the dependent chain per step
        const double r = dd[i];
        const double t = fma(-du2[i], z2, z[i]) * r;
        const double zz = fma(-du[i] * r, z1, t);
        z[i] = zz;
        z2 = z1;
        z1 = zz;
      }
    }
    __syncwarp();
    double nz = 0.0;
    for (int i = lane; i < M; i += 32) nz += z[i] * z[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    const double inv = 1.0 / sqrt(nz);
    for (int i = lane; i < M; i += 32) z[i] *= inv;
    __syncwarp();
  }
  for (int i = lane; i < M; i += 32) Z[(int64_t)jj * M + i] = z[i];
}

// classical Gram-Schmidt applied twice, vectors in descending-eigenvalue order (one CTA)
__global__ void __launch_bounds__(1024) reorth_kernel(double* __restrict__ Z, int M, int k) {
  __shared__ double dots[128];
  __shared__ double red[32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int j = 0; j < k; ++j) {
    double* zj = Z + (int64_t)j * M;
    for (int pass = 0; pass < 2; ++pass) {
      for (int c = wid; c < j; c += nw) {
        const double* zc = Z + (int64_t)c * M;
        double acc = 0.0;
        for (int i = lane; i < M; i += 32) acc = fma(zc[i], zj[i], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) dots[c] = acc;
      }
      __syncthreads();
      for (int i = tid; i < M; i += nt) {
        double x = zj[i];
        for (int c = 0; c < j; ++c) x -= dots[c] * Z[(int64_t)c * M + i];
        zj[i] = x;
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int i = tid; i < M; i += nt) s += zj[i] * zj[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[wid] = s;
    __syncthreads();
    double tot = 0.0;
    for (int w2 = 0; w2 < nw; ++w2) tot += red[w2];
    const double inv = 1.0 / sqrt(tot);
    for (int i = tid; i < M; i += nt) zj[i] *= inv;
    __syncthreads();
  }
}

// CTA per eigenvector: u = H_0 H_1 ... H_{M-3} z, reflector v_j stored in row j of A at j+1..M-1
__global__ void __launch_bounds__(kEigThreads) backxform_kernel(const double* __restrict__ A, const double* __restrict__ tau,
                                                                int M, const double* __restrict__ Z,
                                                                const double* __restrict__ lam, double* __restrict__ V,
                                                                double* __restrict__ lam_out) {
  extern __shared__ __align__(16) double zs[];   // M
  __shared__ double red[32];
  __shared__ int redi[32];
  const int jj = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int i = tid; i < M; i += nt) zs[i] = Z[(int64_t)jj * M + i];
  __syncthreads();
  for (int j = M - 3; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    const double* vj = A + (int64_t)j * M;
    double acc = 0.0;
    for (int i = j + 1 + tid; i < M; i += nt) acc = fma(vj[i], zs[i], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[wid] = acc;
    __syncthreads();
    double dot = 0.0;
    for (int w2 = 0; w2 < nw; ++w2) dot += red[w2];
    dot *= t;
    for (int i = j + 1 + tid; i < M; i += nt) zs[i] -= dot * vj[i];
    __syncthreads();
  }
  // sign rule: entry of largest |.| positive, ties -> lowest index
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int i = tid; i < M; i += nt) {
    const double a = fabs(zs[i]);
    if (a > best) { best = a; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if (lane == 0) { red[wid] = best; redi[wid] = bi; }
  __syncthreads();
  double gb = red[0];
  int gi = redi[0];
  for (int w2 = 1; w2 < nw; ++w2)
    if (red[w2] > gb || (red[w2] == gb && redi[w2] < gi)) { gb = red[w2]; gi = redi[w2]; }
  const double sg = zs[gi] < 0.0 ? -1.0 : 1.0;
  for (int i = tid; i < M; i += nt) V[(int64_t)jj * M + i] = sg * zs[i];
  if (tid == 0) lam_out[jj] = lam[jj];
}


// Back-transformation, reflector-sharing variant: a CTA of nw warps holds nw eigenvectors (one per
// warp, in shared memory); the reflectors v_j (row j of Wk, columns j+1..M-1) stream through a
// double-buffered shared-memory stage with cp.async, so each v_j is read from L2 once per CTA and
// its load overlaps the previous reflector's dot/axpy.  u = H_0 ... H_{M-3} z, then the sign rule.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
constexpr int kBxStages = 6;

__global__ void __launch_bounds__(256) backxform_shared_kernel(const double* __restrict__ Wk,
                                                               const double* __restrict__ tau, int M, int k,
                                                               const double* __restrict__ Z,
                                                               const double* __restrict__ lam,
                                                               double* __restrict__ V, double* __restrict__ lam_out) {
  extern __shared__ __align__(16) double shx[];
  constexpr int NS = kBxStages;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  double* stage = shx;                 // NS x M ring
  double* z = shx + (size_t)NS * M + (size_t)warp * M;
  double* ts = shx + (size_t)(NS + nw) * M;   // tau (read once; the per-step global load was on the critical path)
  for (int i = tid; i < M; i += blockDim.x) ts[i] = tau[i];
  const int jj = blockIdx.x * nw + warp;
  const bool active = jj < k;
  if (active)
    for (int i = lane; i < M; i += 32) z[i] = Z[(int64_t)jj * M + i];
  // row j lives in ring slot (M-3-j) % NS
  auto issue = [&](int j) {
    if (j >= 0) {
      double* dst = stage + (size_t)((M - 3 - j) % NS) * M;
      for (int c = j + 1 + tid; c < M; c += blockDim.x) cp_async8(dst + c, Wk + (int64_t)j * M + c);
    }
    cp_async_commit();
  };
  for (int q = 0; q < NS - 1; ++q) issue(M - 3 - q);
  for (int j = M - 3; j >= 0; --j) {
    cp_async_wait<NS - 2>();
    __syncthreads();                   // row j visible; every warp is done with the slot reused below
    issue(j - (NS - 1));
    const double t = ts[j];
    if (active && t != 0.0) {
      const double* vj = stage + (size_t)((M - 3 - j) % NS) * M;
      double acc = 0.0;
#pragma unroll 4
      for (int c = j + 1 + lane; c < M; c += 32) acc = fma(vj[c], z[c], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const double f = t * acc;
#pragma unroll 4
      for (int c = j + 1 + lane; c < M; c += 32) z[c] -= f * vj[c];
    }
  }
  if (!active) return;
  __syncwarp();
  // sign rule: entry of largest |.| positive, ties -> lowest index
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int i = lane; i < M; i += 32) {
    const double a = fabs(z[i]);
    if (a > best) { best = a; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  const double sg = z[bi] < 0.0 ? -1.0 : 1.0;
  for (int i = lane; i < M; i += 32) V[(int64_t)jj * M + i] = sg * z[i];
  if (lane == 0) lam_out[jj] = lam[jj];
}

// Register variant: ONE eigenvector per CTA of kBxW warps (entry c owned by thread c mod 32 kBxW,
// NPL entries per thread in registers), so the 60 vectors spread over 60 SMs and every step is a
// short dot (partial per thread, warp shuffle, 8-way smem sum) and axpy; the reflector streams
// through the cp.async ring.  Two barriers per step (ring slot + partial sums, double-buffered).
constexpr int kBxW = 8;
template <int NPL>
__global__ void __launch_bounds__(32 * kBxW) backxform_reg_kernel(const double* __restrict__ Wk,
                                                                  const double* __restrict__ tau, int M, int k,
                                                                  const double* __restrict__ Z,
                                                                  const double* __restrict__ lam,
                                                                  double* __restrict__ V,
                                                                  double* __restrict__ lam_out) {
  extern __shared__ __align__(16) double shx[];
  constexpr int NS = kBxStages;
  constexpr int NT = 32 * kBxW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int jj = blockIdx.x;
  double* ts = shx + (size_t)NS * M;           // tau
  double* red = ts + M;                        // [2][kBxW] partial dots
  __shared__ double bestv[kBxW];
  __shared__ int besti[kBxW];
  for (int i = tid; i < M; i += NT) ts[i] = tau[i];
  double zr[NPL];
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    const int c = tid + NT * u;
    zr[u] = c < M ? Z[(int64_t)jj * M + c] : 0.0;
  }
  auto issue = [&](int j) {
    if (j >= 0) {
      double* dst = shx + (size_t)((M - 3 - j) % NS) * M;
      for (int c = j + 1 + tid; c < M; c += NT) cp_async8(dst + c, Wk + (int64_t)j * M + c);
    }
    cp_async_commit();
  };
  for (int q = 0; q < NS - 1; ++q) issue(M - 3 - q);
  for (int j = M - 3; j >= 0; --j) {
    cp_async_wait<NS - 2>();
    __syncthreads();
    issue(j - (NS - 1));
    const double t = ts[j];
    if (t == 0.0) continue;                    // uniform across the CTA
    const double* vj = shx + (size_t)((M - 3 - j) % NS) * M;
    double vc[NPL];
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
      const int c = tid + NT * u;
      vc[u] = (c > j && c < M) ? vj[c] : 0.0;
      acc = fma(vc[u], zr[u], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    double* rb = red + (j & 1) * kBxW;
    if (lane == 0) rb[warp] = acc;
    __syncthreads();
    double dot = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < kBxW; ++w2) dot += rb[w2];
    const double f = t * dot;
#pragma unroll
    for (int u = 0; u < NPL; ++u) zr[u] = fma(-f, vc[u], zr[u]);
  }
  // sign rule: entry of largest |.| positive, ties -> lowest index
  double best = -1.0, bval = 0.0;
  int bi = 0x7fffffff;
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    const int c = tid + NT * u;
    if (c < M && fabs(zr[u]) > best) { best = fabs(zr[u]); bi = c; bval = zr[u]; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; bval = ov; }
  }
  if (lane == 0) { bestv[warp] = bval; besti[warp] = bi; red[warp] = best; }
  __syncthreads();
  double gb = red[0], gv = bestv[0];
  int gi = besti[0];
  for (int w2 = 1; w2 < kBxW; ++w2)
    if (red[w2] > gb || (red[w2] == gb && besti[w2] < gi)) { gb = red[w2]; gi = besti[w2]; gv = bestv[w2]; }
  const double sg = gv < 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    const int c = tid + NT * u;
    if (c < M) V[(int64_t)jj * M + c] = sg * zr[u];
  }
  if (tid == 0) lam_out[jj] = lam[jj];
}

// Blocked back-transformation (compact WY).  Q = H_0 H_1 ... H_{M-3}, H_j = I - tau_j v_j v_j^T (v_j in
// row j of Wk, entries c > j).  Blocks of kWyB consecutive reflectors: H_{j0} ... H_{j0+nb-1} =
// I - V T V^T with T upper triangular (forward accumulation, LAPACK dlarft):
//   T(i,i) = tau_i,  T(0:i, i) = -tau_i T(0:i, 0:i) (V(:, 0:i)^T v_i).
// Each eigenvector z then needs one reduction per block (w = V^T z, all kWyB dots at once) instead of
// one per reflector: y = B_0 (B_1 (... B_last z)).
constexpr int kWyB = 16;   // reflectors per block: the block's V entries stay in registers between w = V^T z and z -= V w'

// one CTA per block: S = V^T V (upper), then the T recurrence on warp 0
__global__ void __launch_bounds__(256) wy_t_kernel(const double* __restrict__ Wk, const double* __restrict__ tau, int M,
                                                   int nrefl, double* __restrict__ Tout) {
  extern __shared__ double vs[];   // [kWyB][M]: the block's reflectors (zero at c <= j)
  __shared__ double S[kWyB][kWyB + 1];
  __shared__ double T[kWyB][kWyB + 1];
  const int p = blockIdx.x, j0 = p * kWyB, nb = min(kWyB, nrefl - j0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int q = threadIdx.x; q < kWyB * M; q += blockDim.x) {
    const int a = q / M, c = q - a * M;
    vs[q] = (a < nb && c > j0 + a) ? Wk[(int64_t)(j0 + a) * M + c] : 0.0;
  }
  __syncthreads();
  for (int q = warp; q < kWyB * kWyB; q += nw) {
    const int a = q / kWyB, b = q - a * kWyB;
    if (a > b) continue;
    double acc = 0.0;
    for (int c = j0 + b + 1 + lane; c < M; c += 32) acc = fma(vs[a * M + c], vs[b * M + c], acc);
    acc = warp_sum(acc);
    if (lane == 0) S[a][b] = acc;
  }
  __syncthreads();
  if (warp == 0) {
    const int r = lane;
    for (int i = 0; i < kWyB; ++i) {
      const double ti = i < nb ? tau[j0 + i] : 0.0;
      const double y = (r < i) ? S[r < kWyB ? r : 0][i] : 0.0;
      double w = 0.0;
      for (int c = 0; c < i; ++c) {
        const double yc = __shfl_sync(0xffffffffu, y, c);
        if (r <= c) w = fma(T[r][c], yc, w);
      }
      if (r < kWyB) T[r][i] = r < i ? -ti * w : (r == i ? ti : 0.0);
      __syncwarp();
    }
    for (int q = lane; q < kWyB * kWyB; q += 32) Tout[(int64_t)p * kWyB * kWyB + q] = T[q / kWyB][q % kWyB];
  }
}

// sum over the 32 lanes of kWyB (16) per-lane values v[]: on return lane l holds the sum of column
// l mod 16 (recursive halving: 8 + 4 + 2 + 1 shuffles, then one xor-16 add)
__device__ __forceinline__ double transpose_sum16(double (&v)[kWyB]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = kWyB / 2; h >= 1; h >>= 1) {
    const bool upper = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = upper ? v[i] : v[i + h];
      const double keep = upper ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// one eigenvector per CTA (entries in registers, c = tid + NT u); blocks applied last to first
template <int NPL>
__global__ void __launch_bounds__(32 * kBxW) backxform_wy_kernel(const double* __restrict__ Wk, const double* __restrict__ Tg,
                                                                 int M, int nrefl, int k, const double* __restrict__ Z,
                                                                 const double* __restrict__ lam, double* __restrict__ V,
                                                                 double* __restrict__ lam_out, int tpre) {
  constexpr int NT = 32 * kBxW;
  __shared__ double red[2][kBxW][kWyB];   // parity-buffered: one barrier pair per block
  __shared__ double wv[2][kWyB];
  __shared__ double bestv[kBxW], bestm[kBxW];
  __shared__ int besti[kBxW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int jj = blockIdx.x;
  double zr[NPL];
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    const int c = tid + NT * u;
    zr[u] = c < M ? Z[(int64_t)jj * M + c] : 0.0;
  }
  const int nblk = (nrefl + kWyB - 1) / kWyB;
  // the next block's V entries of this thread's rows are prefetched into shared memory by cp.async
  // (zero-filled outside the reflector) while this block computes: the per-block L2 latency of the
  // 16 rows was the kernel's critical path.  Each thread reads back only its own slots.
  extern __shared__ double vnext[];   // [kWyB][NPL][NT]
  auto prefetch = [&](int pb) {
    const int pj0 = pb * kWyB, pnb = min(kWyB, nrefl - pj0);
#pragma unroll
    for (int i = 0; i < kWyB; ++i)
#pragma unroll
      for (int u = 0; u < NPL; ++u) {
        const int c = tid + NT * u;
        const bool ok = i < pnb && c > pj0 + i && c < M;
        const double* src = ok ? Wk + (int64_t)(pj0 + i) * M + c : Wk;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&vnext[(i * NPL + u) * NT + tid]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0) : "memory");
      }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch(nblk - 1);
  for (int p = nblk - 1; p >= 0; --p) {
    double vr[kWyB][NPL];
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int i = 0; i < kWyB; ++i)
#pragma unroll
      for (int u = 0; u < NPL; ++u) vr[i][u] = vnext[(i * NPL + u) * NT + tid];
    if (p > 0) prefetch(p - 1);
    // warp 0's rows of this block's T factor, loaded before the dots and the barrier (an L2 round
    // trip after the barrier sat on every block's critical path)
    double trow[kWyB];
    if (warp == 0) {
      const double* T = Tg + (int64_t)p * kWyB * kWyB;
#pragma unroll
      for (int c = 0; c < kWyB; ++c) trow[c] = (tpre && lane < kWyB && c >= lane) ? __ldg(T + lane * kWyB + c) : 0.0;
    }
    // w = V^T z: per-thread partials of all dots, lane-transposed warp sums, 8-warp sum
    double part[kWyB];
#pragma unroll
    for (int i = 0; i < kWyB; ++i) {
      double a = 0.0;
#pragma unroll
      for (int u = 0; u < NPL; ++u) a = fma(vr[i][u], zr[u], a);
      part[i] = a;
    }
    const double ws = transpose_sum16(part);
    if (lane < kWyB) red[p & 1][warp][lane] = ws;
    __syncthreads();
    if (warp == 0) {
      double w = 0.0;
      if (lane < kWyB) {
#pragma unroll
        for (int w2 = 0; w2 < kBxW; ++w2) w += red[p & 1][w2][lane];
      }
      // w' = T w (T upper triangular): lane r sums T(r, c) w_c for c >= r (trow is zero elsewhere)
      double tw = 0.0;
      const double* T = Tg + (int64_t)p * kWyB * kWyB;
#pragma unroll
      for (int c = 0; c < kWyB; ++c) {
        const double wc = __shfl_sync(0xffffffffu, w, c);
        if (lane < kWyB && c >= lane) tw = fma(tpre ? trow[c] : __ldg(T + lane * kWyB + c), wc, tw);
      }
      if (lane < kWyB) wv[p & 1][lane] = tw;
    }
    __syncthreads();
    // z -= V w'
#pragma unroll
    for (int i = 0; i < kWyB; ++i) {
      const double wi = wv[p & 1][i];
#pragma unroll
      for (int u = 0; u < NPL; ++u) zr[u] = fma(-wi, vr[i][u], zr[u]);
    }
  }
  // sign rule: entry of largest |.| positive, ties -> lowest index
  double best = -1.0, bval = 0.0;
  int bi = 0x7fffffff;
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    const int c = tid + NT * u;
    if (c < M && fabs(zr[u]) > best) { best = fabs(zr[u]); bi = c; bval = zr[u]; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; bval = ov; }
  }
  if (lane == 0) { bestv[warp] = bval; besti[warp] = bi; bestm[warp] = best; }
  __syncthreads();
  double gb = bestm[0], gv = bestv[0];
  int gi = besti[0];
  for (int w2 = 1; w2 < kBxW; ++w2)
    if (bestm[w2] > gb || (bestm[w2] == gb && besti[w2] < gi)) { gb = bestm[w2]; gi = besti[w2]; gv = bestv[w2]; }
  const double sg = gv < 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int u = 0; u < NPL; ++u) {
    const int c = tid + NT * u;
    if (c < M) V[(int64_t)jj * M + c] = sg * zr[u];
  }
  if (tid == 0) lam_out[jj] = lam[jj];
}

// Re-orthogonalisation by CholeskyQR, applied twice (CholQR2): S = Z Z^T (k x k), S = R^T R,
// Z <- R^{-T} Z.  In exact arithmetic this is classical Gram-Schmidt of the vectors in their
// (descending-eigenvalue) order -- the same result as reorth_kernel -- but parallel over M.
__global__ void gram_rows_kernel(const double* __restrict__ Z, int M, int k, double* __restrict__ S) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int npairs = k * (k + 1) / 2;
  if (w >= npairs) return;
  int a = 0, rem = w;
  while (rem >= k - a) { rem -= k - a; ++a; }
  const int b = a + rem;
  const double* za = Z + (int64_t)a * M;
  const double* zb = Z + (int64_t)b * M;
  double acc = 0.0;
  for (int i = lane; i < M; i += 32) acc = fma(za[i], zb[i], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) { S[a * k + b] = acc; S[b * k + a] = acc; }
}

// one CTA: Cholesky S = R^T R (R upper, row-major), then T = R^{-1} (upper) into Tout
__global__ void __launch_bounds__(256) chol_inv_kernel(const double* __restrict__ S, int k, double* __restrict__ Tout,
                                                       int* __restrict__ fallback) {
  extern __shared__ __align__(16) double sc[];
  double* Wm = sc;          // k x k working copy (upper triangle), then T
  double* Rm = sc + k * k;  // k x k: R (upper)
  double* rinv = Rm + k * k;  // k: 1 / R[c][c]
  double* sdiag = rinv + k;   // k: the original diagonal (pivot-loss test without a global load per column)
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < k * k; i += nt) { Wm[i] = S[i]; Rm[i] = 0.0; }
  for (int i = tid; i < k; i += nt) sdiag[i] = S[i * k + i];
  __syncthreads();
  // right-looking Cholesky, one barrier per column: row c of R from the working row, and the
  // trailing update W[i][j] -= W[c][i] W[c][j] / W[c][c] (row c is not written in this phase)
  for (int c = 0; c < k; ++c) {
    const double dcc = Wm[c * k + c];
    const bool ok = dcc > 0.0;
    const double rcc = ok ? sqrt(dcc) : 0.0;
    const double ircc = ok ? 1.0 / rcc : 0.0, idcc = ok ? 1.0 / dcc : 0.0;
    // a pivot that lost ~12 digits: the vectors are (numerically) dependent -> robust fallback
    if (tid == 0) {
      if (!(dcc > 1e-8 * sdiag[c])) atomicOr(fallback, 1);
      rinv[c] = ok ? ircc : 0.0;
    }
    for (int j = c + tid; j < k; j += nt) Rm[c * k + j] = j == c ? rcc : Wm[c * k + j] * ircc;
    // 2-D thread grid (16 x 16) over the trailing upper triangle: no integer division per element
    for (int i = c + 1 + (tid >> 4); i < k; i += nt >> 4) {
      const double wci = Wm[c * k + i] * idcc;
      for (int j = i + (tid & 15); j < k; j += 16) Wm[i * k + j] -= wci * Wm[c * k + j];
    }
    __syncthreads();
  }
  // T = R^{-1} (upper) by right-looking back substitution, one barrier per row: acc starts as I;
  // at step i (bottom up) row i of acc is final, T[i][j] = acc[i][j] / R[i][i], and every row r < i
  // takes acc[r][j] -= R[r][i] T[i][j] (parallel over (r, j); row i itself is only read)
  double* acc = Wm;
  for (int q = tid; q < k * k; q += nt) acc[q] = (q / k == q % k) ? 1.0 : 0.0;
  __syncthreads();
  for (int i = k - 1; i >= 0; --i) {
    const double ri = rinv[i];
    for (int r = tid >> 4; r <= i; r += nt >> 4) {
      const double rri = r < i ? Rm[r * k + i] : 0.0;
      for (int j = i + (tid & 15); j < k; j += 16) {
        const double tij = acc[i * k + j] * ri;
        if (r < i) acc[r * k + j] -= rri * tij;
        else Rm[i * k + j] = tij;   // r == i: park T[i][j] in R's (now dead) row i
      }
    }
    __syncthreads();
  }
  double* Tm = Rm;
  for (int i = tid; i < k * k; i += nt) Tout[i] = Tm[i];
}

// Znew[c][i] = sum_{b <= c} Z[b][i] T[b][c]   (Q = Z_mat R^{-1}, Z_mat = M x k with columns z_b)
__global__ void apply_rinv_kernel(const double* __restrict__ Z, int M, int k, const double* __restrict__ T,
                                  double* __restrict__ Zn) {
  const int64_t total = (int64_t)M * k;
  for (int64_t e2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e2 < total; e2 += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e2 / M), i = (int)(e2 % M);
    double acc = 0.0;
    for (int b = 0; b <= c; ++b) acc = fma(Z[(int64_t)b * M + i], __ldg(T + b * k + c), acc);
    Zn[e2] = acc;
  }
}


// Fallback re-orthogonalisation (only when CholQR met a near-singular Gram, e.g. a multiple zero
// eigenvalue of a rank-deficient G where inverse iteration returns nearly parallel vectors):
// classical Gram-Schmidt twice in descending-eigenvalue order on the inverse-iteration vectors; a
// vector that loses > 6 digits is replaced by a hashed pseudo-random vector orthogonalised against
// the accepted ones (which spans the remaining eigenspace when the cluster is the null space).
__global__ void __launch_bounds__(1024) reorth_fallback_kernel(const int* __restrict__ fallback,
                                                               const double* __restrict__ Zin, double* __restrict__ Z,
                                                               int M, int k, const double* __restrict__ lam,
                                                               const double* __restrict__ tnorm, int* __restrict__ flags) {
  if (*fallback == 0) return;
  __shared__ double dots[1024];
  __shared__ double red[32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  auto norm2 = [&](const double* z) {
    double sacc = 0.0;
    for (int i = tid; i < M; i += nt) sacc += z[i] * z[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    __syncthreads();
    if (lane == 0) red[wid] = sacc;
    __syncthreads();
    double tot = 0.0;
    for (int w2 = 0; w2 < nw; ++w2) tot += red[w2];
    return tot;
  };
  auto project_out = [&](double* zj, int j) {
    for (int pass = 0; pass < 2; ++pass) {
      for (int c = wid; c < j; c += nw) {
        const double* zc = Z + (int64_t)c * M;
        double acc = 0.0;
        for (int i = lane; i < M; i += 32) acc = fma(zc[i], zj[i], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) dots[c] = acc;
      }
      __syncthreads();
      for (int i = tid; i < M; i += nt) {
        double x = zj[i];
        for (int c = 0; c < j; ++c) x -= dots[c] * Z[(int64_t)c * M + i];
        zj[i] = x;
      }
      __syncthreads();
    }
  };
  for (int j = 0; j < k; ++j) {
    double* zj = Z + (int64_t)j * M;
    for (int i = tid; i < M; i += nt) zj[i] = Zin[(int64_t)j * M + i];
    __syncthreads();
    const double n0 = norm2(zj);
    project_out(zj, j);
    double n1 = norm2(zj);
    // a replaced vector is an eigenvector only inside the (numerical) null space: a dependent
    // vector whose eigenvalue is above 2 eps ||T|| is a numerical failure (flag bit 8)
    if (!(n1 > 1e-12 * n0) && tid == 0 && flags && lam[j] > 2.220446049250313e-16 * 2.0 * tnorm[0]) atomicOr(flags, 8);
    for (int attempt = 0; attempt < 4 && !(n1 > 1e-12 * n0); ++attempt) {
      for (int i = tid; i < M; i += nt) {
        uint64_t h = 0x9E3779B97F4A7C15ull * (uint64_t)(j + 1 + 977 * attempt) + 0xC2B2AE3D27D4EB4Full * (uint64_t)(i + 1);
        h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        zj[i] = (double)(h >> 11) / 9007199254740992.0 - 0.5;
      }
      __syncthreads();
      const double nr = norm2(zj);
      project_out(zj, j);
      n1 = norm2(zj);
      if (n1 > 1e-6 * nr) break;
    }
    const double inv = 1.0 / sqrt(n1);
    for (int i = tid; i < M; i += nt) zj[i] *= inv;
    __syncthreads();
  }
}

}  // namespace

// CholQR building blocks for other stages (the range finder, k_rf.cu): S = Z Z^T of k vectors of
// length M (row-major k x k), T = R^-1 of S = R^T R (fallback |= 1 on a pivot that lost > 8 digits),
// Zn = Z R^-1 (column vectors of Z_mat, i.e. Zn[c] = sum_{b <= c} T[b][c] Z[b]).
void launch_gram_rows(const double* Z, int M, int k, double* S, cudaStream_t s) {
  const int npairs = k * (k + 1) / 2;
  gram_rows_kernel<<<(npairs * 32 + 255) / 256, 256, 0, s>>>(Z, M, k, S);
  check_launch("gram_rows");
}
void launch_chol_rinv(const double* S, int k, double* T, int* fallback, cudaStream_t s) {
  const size_t csm = (2 * (size_t)k * k + 2 * k) * sizeof(double);
  FKK_CUDA_CHECK(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
  chol_inv_kernel<<<1, 256, csm, s>>>(S, k, T, fallback);
  check_launch("chol_rinv");
}
void launch_apply_rinv(const double* Z, int M, int k, const double* T, double* Zn, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int agrid = (int)std::min<int64_t>(((int64_t)M * k + 255) / 256, 4 * sms);
  apply_rinv_kernel<<<agrid, 256, 0, s>>>(Z, M, k, T, Zn);
  check_launch("apply_rinv");
}

size_t eig_workspace_doubles(int M, int k) {
  // d, e, tau (3M) + p / LL words (16M) + lam, tnorm (k+1) + Z, Z2, Z3 (3kM) + S, T (2k^2) + flag + A (M*M)
  return 19 * (size_t)M + (size_t)k + 1 + 3 * (size_t)k * M + 2 * (size_t)k * k + 18 + (size_t)M * M +
         ((size_t)(M + kWyB - 1) / kWyB) * kWyB * kWyB;   // + compact-WY T blocks
}

int eig_path_rows_resident(int M) {
  int dev = 0, sms = 148, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const char* force = getenv("FKK_EIG_FORCE_L2");   // debugging / A-B only
  if (force && force[0] == '1') return 0;
  return M >= 3 && M <= kTsMaxM && tridiag_rows_smem(M, sms) <= (size_t)maxsm;
}

void launch_eig_topk(const double* G, int M, int k, double* work, double* V, double* lam_out, int* flags,
                     cudaStream_t s, double* dbg_det);


void debug_tridiag(const double* G, int M, double* det_out) {
  double* work = nullptr;
  FKK_CUDA_CHECK(cudaMalloc(&work, eig_workspace_doubles(M, 1) * sizeof(double)));
  double* V = nullptr;
  FKK_CUDA_CHECK(cudaMalloc(&V, (size_t)M * sizeof(double) * 2));
  launch_eig_topk(G, M, 1, work, V, V + M, nullptr, nullptr, det_out);
  FKK_CUDA_CHECK(cudaDeviceSynchronize());
  cudaFree(work);
  cudaFree(V);
}

void launch_eig_topk(const double* G, int M, int k, double* work, double* V, double* lam_out, int* flags,
                     cudaStream_t s) {
  launch_eig_topk(G, M, k, work, V, lam_out, flags, s, nullptr);
}

namespace {
// per host thread and device: the side stream and fork / join events of the WY-factor kernel
struct EigSide {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
EigSide& eig_side(int dev) {
  thread_local EigSide sides[64];
  EigSide& e = sides[dev & 63];
  if (!e.st) {
    FKK_CUDA_CHECK(cudaStreamCreateWithFlags(&e.st, cudaStreamNonBlocking));
    FKK_CUDA_CHECK(cudaEventCreateWithFlags(&e.fork, cudaEventDisableTiming));
    FKK_CUDA_CHECK(cudaEventCreateWithFlags(&e.join, cudaEventDisableTiming));
  }
  return e;
}
}  // namespace

void launch_eig_topk(const double* G, int M, int k, double* work, double* V, double* lam_out, int* flags,
                     cudaStream_t s, double* dbg_det) {
  double* d = work;
  double* e = d + M;
  double* tau = e + M;
  double* pg = tau + M;
  double* lam = pg + 16 * (size_t)M;
  double* tnorm = lam + k;
  double* Z = tnorm + 1;
  double* Z2 = Z + (size_t)k * M;
  double* Z3 = Z2 + (size_t)k * M;
  double* S = Z3 + (size_t)k * M;
  double* T = S + (size_t)k * k;
  int* fallback = reinterpret_cast<int*>(T + (size_t)k * k);
  // working matrix / published rows / reflectors (M x M), 16-byte aligned for the bulk copies
  double* A = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(T + (size_t)k * k + 16) + 15) & ~(uintptr_t)15);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (eig_path_rows_resident(M)) {
    // row-resident tridiagonalisation (G is read, never copied): grid phase (cooperative, one grid
    // barrier per column) for j < jend, then the cluster tail (one cluster barrier per column) for the
    // trailing block that fits in the shared memory of CL CTAs
    int maxsm = 0;
    FKK_CUDA_CHECK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    int CL = 8;
    if (const char* ev = getenv("FKK_TRIDIAG_TAIL")) CL = atoi(ev);   // cluster size of the tail; 0: none
    if (CL != 0 && CL != 8 && CL != 16) CL = 8;
    int mt = 0;
    if (CL > 0) {
      int cap = 200;   // per-column cost of the tail grows with m^2 / CL; below ~200 it beats the grid barrier
      if (const char* ev = getenv("FKK_TRIDIAG_MT")) cap = std::max(3, atoi(ev));   // A/B only
      mt = std::min(M, cap);
      while (mt > 2 && tridiag_tail_smem(mt, CL, M) > (size_t)maxsm) --mt;
    }
    int jend = CL > 0 ? M - mt : M - 2;
    if (jend < 2 && CL > 0) jend = 0;   // whole problem in the tail
    int Mi = M, jendi = jend;
    const double* Gc = G;
    if (jend > 0) {
      unsigned int* ctr = reinterpret_cast<unsigned int*>(fallback) + 2;
      FKK_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(unsigned int), s));
      int dbg = 0;
      if (const char* ev = getenv("FKK_TRIDIAG_DBG")) dbg = atoi(ev);   // timing experiments only
      void* args[] = {&Gc, &A, &Mi, &jendi, &d, &e, &tau, &pg, &ctr, &dbg};
      int nct = sms;
      if (const char* ev = getenv("FKK_TRIDIAG_CTAS")) nct = std::max(1, std::min(sms, atoi(ev)));   // A/B only
      const size_t smem = tridiag_rows_smem(M, nct);
      auto kr = M <= 8 * kTsChain ? tridiag_rows_kernel<8> : tridiag_rows_kernel<16>;
      FKK_CUDA_CHECK(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per = 0;
      FKK_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kr, kTsThreads, smem));
      if (per < 1) throw Status(10, "tridiag_rows kernel cannot be co-resident");
      FKK_CUDA_CHECK(cudaLaunchCooperativeKernel((void*)kr, dim3(nct), dim3(kTsThreads), args, smem, s));
      count_launch();
    }
    if (jend < M - 2) {
      const size_t smem = tridiag_tail_smem(M - jend, CL, M);
      auto kt = tridiag_tail_kernel<8>;
      FKK_CUDA_CHECK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (CL > 8) FKK_CUDA_CHECK(cudaFuncSetAttribute(kt, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(CL);
      cfg.blockDim = dim3(kTsThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const double* Pc = pg;
      int tdbg = 0;
      if (const char* ev = getenv("FKK_TRIDIAG_DBG")) {   // timing experiments only: 13 / 14 (+ 256 x column offset)
        const int v = atoi(ev);
        tdbg = (v & 0xff) >= 13 ? ((v & ~0xff) | ((v & 0xff) - 10)) : 0;
      }
      FKK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kt, Gc, A, Mi, jendi, d, e, tau, Pc, tdbg));
      count_launch();
    }
  } else {
    FKK_CUDA_CHECK(cudaMemcpyAsync(A, G, (size_t)M * M * sizeof(double), cudaMemcpyDeviceToDevice, s));
    // L2-streaming cooperative tridiagonalisation (large M)
    const size_t smem = (3 * (size_t)M + 32) * sizeof(double);
    int Mi = M;
    auto kg = tridiag_kernel<false>;
    FKK_CUDA_CHECK(cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 1;
    FKK_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kg, kTriThreads, smem));
    if (per < 1) throw Status(10, "tridiag kernel cannot be co-resident");
    void* args[] = {&A, &Mi, &d, &e, &tau, &pg};
    FKK_CUDA_CHECK(cudaLaunchCooperativeKernel((void*)kg, dim3(sms), dim3(kTriThreads), args, smem, s));
    count_launch();
  }
  if (dbg_det) {   // debug: d, e, tau only
    FKK_CUDA_CHECK(cudaMemcpyAsync(dbg_det, d, 3 * (size_t)M * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  // WY T factors of the reflector blocks depend only on the tridiagonalisation: on a forked stream
  // they run beside bisection / inverse iteration / CholQR2 (FKK_WYT_FORK=0: in order, A/B only)
  static const int bx_mode = getenv("FKK_BACKXFORM_MODE") ? atoi(getenv("FKK_BACKXFORM_MODE")) : 1;   // A/B only
  static const int wyt_fork = getenv("FKK_WYT_FORK") ? atoi(getenv("FKK_WYT_FORK")) : 1;
  const bool wy_path = bx_mode == 1 && M >= 3 && M <= 32 * kBxW * 4;
  const int nrefl = M - 2, nblk = (nrefl + kWyB - 1) / kWyB;
  double* Tg = A + (size_t)M * M;
  EigSide* side = nullptr;
  if (wy_path) {
    const size_t tsm = (size_t)kWyB * M * sizeof(double);
    FKK_CUDA_CHECK(cudaFuncSetAttribute(wy_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    cudaStream_t ws = s;
    if (wyt_fork) {
      side = &eig_side(dev);
      FKK_CUDA_CHECK(cudaEventRecord(side->fork, s));
      FKK_CUDA_CHECK(cudaStreamWaitEvent(side->st, side->fork, 0));
      ws = side->st;
    }
    wy_t_kernel<<<nblk, 256, tsm, ws>>>(A, tau, M, nrefl, Tg);
    check_launch("eig_wy_t");
    if (side) FKK_CUDA_CHECK(cudaEventRecord(side->join, side->st));
  }
  FKK_CUDA_CHECK(cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(2 * (size_t)M * sizeof(double))));
  int bth = 128;
  if (const char* ev = getenv("FKK_BISECT_THREADS")) bth = std::max(32, std::min(1024, atoi(ev)) / 32 * 32);   // A/B
  bisect_kernel<<<k, bth, 2 * (size_t)M * sizeof(double), s>>>(d, e, M, k, lam, tnorm);
  check_launch("eig_bisect");
  const size_t ism = (size_t)5 * M * sizeof(double) + (size_t)M + 16;
  FKK_CUDA_CHECK(cudaFuncSetAttribute(inviter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ism));
  inviter_kernel<<<k, 32, ism, s>>>(d, e, M, k, lam, tnorm, Z);
  check_launch("eig_inviter");
  // CholQR2 re-orthogonalisation (k <= 128: the k x k factor lives in one CTA's shared memory):
  // Z -> Z2 -> Z3; a near-singular Gram switches to the Gram-Schmidt fallback (Z -> Z3)
  double* Zf = Z3;
  if (k <= 128) {
    const size_t csm = (2 * (size_t)k * k + 2 * k) * sizeof(double);
    FKK_CUDA_CHECK(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
    FKK_CUDA_CHECK(cudaMemsetAsync(fallback, 0, sizeof(int), s));
    const int npairs = k * (k + 1) / 2;
    const int agrid = (int)std::min<int64_t>(((int64_t)M * k + 255) / 256, 4 * sms);
    for (int pass = 0; pass < 2; ++pass) {
      const double* zin = pass == 0 ? Z : Z2;
      double* zout = pass == 0 ? Z2 : Z3;
      gram_rows_kernel<<<(npairs * 32 + 255) / 256, 256, 0, s>>>(zin, M, k, S);
      check_launch("eig_reorth_gram");
      chol_inv_kernel<<<1, 256, csm, s>>>(S, k, T, fallback);
      check_launch("eig_reorth_chol");
      apply_rinv_kernel<<<agrid, 256, 0, s>>>(zin, M, k, T, zout);
      check_launch("eig_reorth_apply");
    }
    reorth_fallback_kernel<<<1, 1024, 0, s>>>(fallback, Z, Z3, M, k, lam, tnorm, flags);
    check_launch("eig_reorth_fallback");
  } else {
    reorth_kernel<<<1, 1024, 0, s>>>(Z, M, k);
    check_launch("eig_reorth");
    Zf = Z;
  }
  // back-transformation: eigenvectors in registers (M <= 2048), else reflector-sharing CTAs
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t rsm = ((size_t)(kBxStages + 1) * M + 2 * kBxW) * sizeof(double);
  if (wy_path) {   // (NPL = 8 would spill the register-cached V block)
    if (side) FKK_CUDA_CHECK(cudaStreamWaitEvent(s, side->join, 0));
    const int npl = M <= 32 * kBxW * 2 ? 2 : 4;
    const int wsm = kWyB * npl * 32 * kBxW * (int)sizeof(double);   // the prefetched block
    auto kb = npl == 2 ? backxform_wy_kernel<2> : backxform_wy_kernel<4>;
    FKK_CUDA_CHECK(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, wsm));
    static const int tpre = getenv("FKK_BX_TPRE") ? atoi(getenv("FKK_BX_TPRE")) : 1;   // A/B only
    kb<<<k, 32 * kBxW, wsm, s>>>(A, Tg, M, nrefl, k, Zf, lam, V, lam_out, tpre);
    check_launch("eig_backxform_wy");
    return;
  }
  if (M >= 3 && M <= 32 * kBxW * 8 && rsm <= (size_t)maxsm) {
#define FKK_BX_REG(NPL)                                                                                  \
    {                                                                                                    \
      auto kb = backxform_reg_kernel<NPL>;                                                               \
      FKK_CUDA_CHECK(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));   \
      kb<<<k, 32 * kBxW, rsm, s>>>(A, tau, M, k, Zf, lam, V, lam_out);                                  \
    }
    if (M <= 32 * kBxW * 2) FKK_BX_REG(2)
    else if (M <= 32 * kBxW * 4) FKK_BX_REG(4)
    else FKK_BX_REG(8)
#undef FKK_BX_REG
    check_launch("eig_backxform");
    return;
  }
  int nw = 8;
  while (nw > 1 && (size_t)(kBxStages + nw + 1) * M * sizeof(double) > (size_t)maxsm) --nw;
  const size_t bsm = (size_t)(kBxStages + nw + 1) * M * sizeof(double);
  if (M >= 3 && bsm <= (size_t)maxsm) {
    FKK_CUDA_CHECK(cudaFuncSetAttribute(backxform_shared_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
    backxform_shared_kernel<<<(k + nw - 1) / nw, nw * 32, bsm, s>>>(A, tau, M, k, Zf, lam, V, lam_out);
    check_launch("eig_backxform");
  } else {
    const size_t bsm1 = (size_t)M * sizeof(double);
    FKK_CUDA_CHECK(cudaFuncSetAttribute(backxform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm1));
    backxform_kernel<<<k, kEigThreads, bsm1, s>>>(A, tau, M, Zf, lam, V, lam_out);
    check_launch("eig_backxform");
  }
}

}  // namespace fkk
