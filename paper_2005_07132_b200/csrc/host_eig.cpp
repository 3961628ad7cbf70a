// Host fp64 top-k symmetric eigensolver for the Gram matrix G = A^T A (F4; PAPER.md:64-70,
// "truncated SVD": s_i = sqrt(lambda_i), V_k = top-k eigenvectors).  Self-contained (no LAPACK in
// the image):  Householder tridiagonalisation (OpenMP over rows)  ->  Sturm-count bisection for
// the k largest eigenvalues  ->  inverse iteration with partial-pivoting tridiagonal LU and
// modified Gram-Schmidt inside eigenvalue clusters  ->  back-transformation by the reflectors.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "fkk_internal.h"

namespace fkk {

namespace {

// Number of eigenvalues of the tridiagonal (d, e) strictly less than x (Sturm sequence).
int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (std::fabs(q) < pivmin) q = -pivmin;
  if (q < 0) cnt++;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (std::fabs(q) < pivmin) q = -pivmin;
    if (q < 0) cnt++;
  }
  return cnt;
}

// Solve (T - lam I) x = b in place with LU + partial pivoting (LAPACK dgttrf/dgttrs logic).
void tridiag_shift_solve(const double* d, const double* e, int n, double lam, double tiny,
                         std::vector<double>& dl, std::vector<double>& dd, std::vector<double>& du,
                         std::vector<double>& du2, std::vector<int>& ipiv, double* b) {
  for (int i = 0; i < n; ++i) { dd[i] = d[i] - lam; ipiv[i] = i; }
  for (int i = 0; i < n - 1; ++i) { dl[i] = e[i]; du[i] = e[i]; }
  for (int i = 0; i < n - 2; ++i) du2[i] = 0.0;
  for (int i = 0; i < n - 1; ++i) {
    if (std::fabs(dd[i]) >= std::fabs(dl[i])) {
      if (dd[i] == 0.0) dd[i] = tiny;
      double fact = dl[i] / dd[i];
      dl[i] = fact;
      dd[i + 1] -= fact * du[i];
    } else {
      double fact = dd[i] / dl[i];
      dd[i] = dl[i];
      dl[i] = fact;
      double temp = du[i];
      du[i] = dd[i + 1];
      dd[i + 1] = temp - fact * dd[i + 1];
      if (i < n - 2) {
        du2[i] = du[i + 1];
        du[i + 1] = -fact * du[i + 1];
      }
      ipiv[i] = i + 1;
    }
  }
  if (dd[n - 1] == 0.0) dd[n - 1] = tiny;
  for (int i = 0; i < n; ++i) if (std::fabs(dd[i]) < tiny) dd[i] = dd[i] < 0 ? -tiny : tiny;
  // forward: L y = P b
  for (int i = 0; i < n - 1; ++i) {
    int ip = ipiv[i];
    double temp = (ip == i ? b[i + 1] : b[i]) - dl[i] * b[ip];
    b[i] = b[ip];
    b[i + 1] = temp;
  }
  // backward: U x = y
  b[n - 1] /= dd[n - 1];
  if (n > 1) b[n - 2] = (b[n - 2] - du[n - 2] * b[n - 1]) / dd[n - 2];
  for (int i = n - 3; i >= 0; --i) b[i] = (b[i] - du[i] * b[i + 1] - du2[i] * b[i + 2]) / dd[i];
}

}  // namespace

int host_eig_topk(const double* G, int M, int k, double* V, double* lam) {
  if (M < 1 || k < 1 || k > M) return -1;
  std::vector<double> A((size_t)M * M);
  // symmetrise from the lower triangle
  for (int r = 0; r < M; ++r)
    for (int c = 0; c <= r; ++c) A[(size_t)r * M + c] = A[(size_t)c * M + r] = G[(size_t)r * M + c];
  std::vector<double> d(M), e(std::max(M - 1, 1)), tau(std::max(M - 2, 1), 0.0);
  std::vector<double> p(M), w(M);
  // --- 1. Householder tridiagonalisation: Q^T A Q = T, Q = H_0 ... H_{M-3}.
  for (int j = 0; j + 2 < M; ++j) {
    double* col = &w[0];
    int m = M - j - 1;   // length of the vector below the diagonal
    double nrm2 = 0.0;
    for (int i = 0; i < m; ++i) { col[i] = A[(size_t)(j + 1 + i) * M + j]; nrm2 += col[i] * col[i]; }
    double nrm = std::sqrt(nrm2);
    d[j] = A[(size_t)j * M + j];
    if (nrm == 0.0) { e[j] = 0.0; tau[j] = 0.0; for (int i = 0; i < m; ++i) A[(size_t)(j + 1 + i) * M + j] = 0.0; continue; }
    double alpha = col[0] >= 0 ? -nrm : nrm;
    double v0 = col[0] - alpha;
    double vtv = nrm2 - col[0] * col[0] + v0 * v0;
    if (vtv == 0.0) { e[j] = col[0]; tau[j] = 0.0; continue; }
    col[0] = v0;
    double t = 2.0 / vtv;
    tau[j] = t;
    e[j] = alpha;
    // store v in column j below the diagonal (and keep a dense copy in col)
    for (int i = 0; i < m; ++i) A[(size_t)(j + 1 + i) * M + j] = col[i];
    const int base = j + 1;
    // p = t * A22 v
#pragma omp parallel for schedule(static) if (m > 128)
    for (int r = 0; r < m; ++r) {
      const double* row = &A[(size_t)(base + r) * M + base];
      double s = 0.0;
      for (int c = 0; c < m; ++c) s += row[c] * col[c];
      p[r] = t * s;
    }
    double ptv = 0.0;
    for (int r = 0; r < m; ++r) ptv += p[r] * col[r];
    const double K = 0.5 * t * ptv;
    for (int r = 0; r < m; ++r) p[r] -= K * col[r];     // p <- w = p - K v
    // A22 -= v w^T + w v^T
#pragma omp parallel for schedule(static) if (m > 128)
    for (int r = 0; r < m; ++r) {
      double* row = &A[(size_t)(base + r) * M + base];
      const double vr = col[r], wr = p[r];
      for (int c = 0; c < m; ++c) row[c] -= vr * p[c] + wr * col[c];
    }
  }
  if (M >= 2) {
    d[M - 2] = A[(size_t)(M - 2) * M + (M - 2)];
    e[M - 2] = A[(size_t)(M - 1) * M + (M - 2)];
  }
  d[M - 1] = A[(size_t)(M - 1) * M + (M - 1)];

  // --- 2. bisection for the k largest eigenvalues of T
  std::vector<double> e2(std::max(M - 1, 1));
  double gl = d[0], gu = d[0], tnorm = 0.0;
  for (int i = 0; i < M; ++i) {
    double r = (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i < M - 1 ? std::fabs(e[i]) : 0.0);
    gl = std::min(gl, d[i] - r);
    gu = std::max(gu, d[i] + r);
    tnorm = std::max(tnorm, std::fabs(d[i]) + r);
  }
  for (int i = 0; i < M - 1; ++i) e2[i] = e[i] * e[i];
  const double eps = 2.220446049250313e-16;
  const double pivmin = std::max(1e-300, tnorm * 1e-300);
  const double width = gu - gl;
  gl -= 2.0 * eps * tnorm * M + 1e-300;
  gu += 2.0 * eps * tnorm * M + 1e-300;
  std::vector<double> ev(k);
#pragma omp parallel for schedule(dynamic)
  for (int jj = 0; jj < k; ++jj) {
    int idx = M - 1 - jj;   // ascending index of the jj-th largest eigenvalue
    double lo = gl, hi = gu;
    for (int it = 0; it < 200; ++it) {
      double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      if (hi - lo <= 2.0 * eps * std::max(std::fabs(lo), std::fabs(hi)) + pivmin) break;
      if (sturm_count(d.data(), e2.data(), M, mid, pivmin) > idx) hi = mid; else lo = mid;
    }
    ev[jj] = 0.5 * (lo + hi);
  }
  (void)width;

  // --- 3. inverse iteration (descending order), MGS inside clusters
  std::vector<double> Z((size_t)M * k);
  std::vector<double> dl(M), dd(M), du(M), du2(M);
  std::vector<int> ipiv(M);
  const double ortol = 1e-3 * tnorm;
  const double tiny = eps * tnorm + 1e-300;
  int cluster_start = 0;
  double prev_lam = 0.0;
  for (int jj = 0; jj < k; ++jj) {
    double l = ev[jj];
    if (jj > 0 && std::fabs(prev_lam - l) > ortol) cluster_start = jj;
    if (jj > cluster_start && std::fabs(l - prev_lam) < 10.0 * eps * tnorm) l = prev_lam - 10.0 * eps * tnorm;  // split exact ties
    prev_lam = l;
    double* z = &Z[(size_t)jj * M];
    uint64_t s = 0x9E3779B97F4A7C15ull * (uint64_t)(jj + 1);
    for (int i = 0; i < M; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      z[i] = ((double)(s >> 11) / 9007199254740992.0) - 0.5;
    }
    for (int it = 0; it < 4; ++it) {
      tridiag_shift_solve(d.data(), e.data(), M, l, tiny, dl, dd, du, du2, ipiv, z);
      for (int c = cluster_start; c < jj; ++c) {
        const double* zc = &Z[(size_t)c * M];
        double dot = 0.0;
        for (int i = 0; i < M; ++i) dot += zc[i] * z[i];
        for (int i = 0; i < M; ++i) z[i] -= dot * zc[i];
      }
      double nz = 0.0;
      for (int i = 0; i < M; ++i) nz += z[i] * z[i];
      nz = std::sqrt(nz);
      if (nz == 0.0 || !std::isfinite(nz)) return -2;
      for (int i = 0; i < M; ++i) z[i] /= nz;
    }
  }

  // --- 4. back-transformation u = H_0 H_1 ... H_{M-3} z
#pragma omp parallel for schedule(static)
  for (int jj = 0; jj < k; ++jj) {
    double* z = &Z[(size_t)jj * M];
    for (int j = M - 3; j >= 0; --j) {
      if (tau[j] == 0.0) continue;
      double dot = 0.0;
      for (int i = j + 1; i < M; ++i) dot += A[(size_t)i * M + j] * z[i];
      dot *= tau[j];
      for (int i = j + 1; i < M; ++i) z[i] -= dot * A[(size_t)i * M + j];
    }
    // sign rule: largest |entry| positive (ties -> lowest index)
    int am = 0;
    double best = -1.0;
    for (int i = 0; i < M; ++i) if (std::fabs(z[i]) > best) { best = std::fabs(z[i]); am = i; }
    double sg = z[am] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < M; ++i) V[(size_t)jj * M + i] = sg * z[i];
    lam[jj] = ev[jj];
  }
  return 0;
}

}  // namespace fkk
