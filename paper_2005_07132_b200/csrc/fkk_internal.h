// Internal declarations of the fKK-EC runtime: kernel launchers (one per .cu file) and the host
// eigensolver.  Everything here is C++; the public surface is include/fkk.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

namespace fkk {

struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FKK_CUDA_CHECK(expr)                                                                     \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess)                                                                       \
      throw ::fkk::Status(7, std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " +     \
                                 __FILE__ + ":" + std::to_string(__LINE__) + " (" #expr ")");    \
  } while (0)

// Launch counter (the bench reports kernel launches per call).
extern thread_local int64_t g_launches;
inline void count_launch(int n = 1) { g_launches += n; }
inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Status(7, std::string("kernel launch failed (") + what + "): " + cudaGetErrorString(e));
  count_launch();
}

// ---- reference / log-ratio prerequisites (k_misc.cu)
// inv_ref[j] = 1/I_ref[j] (fp32), ref64[j] = I_ref[j] (fp64); flags |= 1 if any I_ref <= 0 or non-finite.
void launch_prep_ref(const void* d_iref, int in_f64, int M, float* inv_ref, double* ref64, int* flags, cudaStream_t s);
// A0 = 1/2 ln(max(I/I_ref, floor)) (fp32, n x M); flags |= 2 on non-finite input.
void launch_logratio(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                     float floor, float* A, int* flags, cudaStream_t s);
void launch_colsum(const void* I, int in_f64, int64_t n, int M, double* colsum, cudaStream_t s);
void launch_noise_scale_from_sums(const double* colsum, int M, double inv_n, double alpha, double sg, double* f64,
                                  float* f32, cudaStream_t s);
void launch_fill(double* p, double v, int64_t n, cudaStream_t s);
void launch_bi_linear(const double* V, int k, int M, float* Bi, cudaStream_t s);
void launch_fill_f(float* p, float v, int64_t n, cudaStream_t s);
void launch_scale_gram(double* G, const double* f, int M, cudaStream_t s);
void launch_cast_w(const double* V, const double* fscale, const double* cscale, int M, int k, int kp, float* W,
                   cudaStream_t s);
void launch_gather_rows(const float* US, int k, int ldus, const int64_t* q_local, int nq, double* X, cudaStream_t s);
void launch_extremes_reduce(const float* ext_val, const int64_t* ext_idx, int nblk, int k, float* out_val,
                            int64_t* out_idx, cudaStream_t s);
void launch_add_f64(const double* a, const double* b, double* out, int64_t n, cudaStream_t s);

// ---- direct path (k_direct.cu)
// tw: exp(-2 pi i t / L) for t < L (fp32 from fp64); pmap: L padding-map entries (source channel
// of padded sample i, -1 for a zero pad; reading A3)
void launch_direct_phase(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                         float floor, int L, const float2* tw, const int* pmap, float* phi, int* flags, cudaStream_t s);
// ALS on rows of y (fp32 or fp64, row-major n x M) -> z (fp32 or fp64); state: 3*M*nb doubles, nb = 32*ceil(n/32)
// ctr (nullable, one unsigned of device memory): warps take spectra from it dynamically (reset here)
void launch_als_rows(const void* y, int y_f64, int64_t n, int M, double lam, double p, int iters, void* z, int z_f64,
                     cudaStream_t s, int* solves = nullptr, unsigned* ctr = nullptr);
void launch_direct_finish(const void* I, int in_f64, int64_t n, int M, const float* inv_ref, const double* ref64,
                          float floor, int L, const float2* tw, const int* pmap, const float* phi, const float* phierr,
                          int sg_half, void* out, int out_imag_only, cudaStream_t s);
size_t direct_finish_smem(int M, int L, bool pf);
// warp-partitioned fp64 ALS (k_als.cu), state in shared memory; false if M is out of its range
size_t als_part_smem(int M, int y_f64);
bool launch_als_part(const void* y, int y_f64, int64_t n, int M, double lam, double p, int iters, void* z, int z_f64,
                     cudaStream_t s, int* solves = nullptr, unsigned* ctr = nullptr);

// ---- factorized path
// Gram partials (k_gram.cu): 128 x 128 tiles of the upper triangle, nsplit row segments each.
int gram_num_tiles(int M);
int gram_num_splits(int64_t n, int M);
void launch_gram_simt(const float* A, int64_t n, int M, double* partials, int nsplit, cudaStream_t s);
void launch_gram_reduce(const double* partials, int nsplit, int M, double* G, int accumulate, cudaStream_t s);
// tcgen05 3xTF32 Gram (k_gram_tc.cu): 128 x 256 tiles of the upper triangle x row splits.
void gram_tc_tiles(int M, std::vector<int2>& tiles, std::vector<int>& tile_of, int& nTj);
int gram_tc_splits(int ntiles, int64_t n);
size_t gram_tc_partial_doubles(int ntiles, int nsplit);
void launch_gram_tc(const float* A, int64_t n, int M, const int2* d_tiles, int ntiles, int nsplit, double* partials,
                    cudaStream_t s);
void launch_gram_tc_reduce(const double* partials, int ntiles, int nsplit, int M, const int* d_tile_of, int nTj,
                           double* G, int accumulate, cudaStream_t s);
// Pre-split Gram (k_gram_tc.cu): the log-ratio pass also writes the MMA smem image of A0 (tf32 hi/lo
// K-major blocks per 128-channel block and 32-pixel stage); the Gram bulk-copies it (no producers).
// nT = number of 128-channel image blocks (>= ceil(M / 128); blocks past M are zero)
size_t gram_pre_bytes(int64_t n, int nT);
void launch_logratio_pre(const float* I, int64_t n, int M, int nT, const float* inv_ref, float floor, float* A,
                         unsigned char* Apre, int* flags, cudaStream_t s, int raw = 0);
// CTA-pair Gram fed by the image (k_gram_pre2.cu): 256 x 256 tiles (gram_tc2_tiles / _splits / _reduce)
int gram_pre2_image_blocks(int M);
void launch_gram_pre2(const unsigned char* Apre, int64_t n, const int2* d_tiles, int ntiles, int nsplit,
                      double* partials, cudaStream_t s);
void launch_gram_pre(const unsigned char* Apre, int64_t n, const int2* d_tiles, int ntiles, int nsplit,
                     double* partials, cudaStream_t s);
// CTA-pair tile list, split count and split reduction (k_gram_tc2.cu) used by the image-fed pair Gram above
void gram_tc2_tiles(int M, std::vector<int2>& tiles, std::vector<int>& tile_of, int& nT);
int gram_tc2_splits(int ntiles, int64_t n);
size_t gram_tc2_partial_doubles(int ntiles, int nsplit);
void launch_gram_tc2_reduce(const double* partials, int ntiles, int nsplit, int M, const int* d_tile_of, int nT,
                            double* G, int accumulate, cudaStream_t s);
// Projection US = A0 W (k_project.cu) with per-block column extremes [blk][c][2].
int project_num_blocks(int64_t n);
void launch_project_simt(const float* A, int64_t n, int M, const float* W, int k, int kp, float* US, float* ext_val,
                         int64_t* ext_idx, int64_t row_offset, cudaStream_t s);
// tcgen05 3xTF32 projection (k_project_tc.cu): W^T image per 32-channel K stage (hi, lo).
size_t project_tc_wimg_floats(int M, int kp);
int project_tc_num_blocks(int64_t n);
void launch_build_wimg(const double* V, const double* fscale, const double* cscale, int M, int k, int kp, float* wimg,
                       cudaStream_t s);
// the TMA projection can read the raw f32 cube and form A0 itself (log-ratio pass writes no A0)
bool project_raw_ok(int M, int kp);
void launch_project_tc(const float* A, int64_t n, int M, const float* wimg, int k, int kp, float* US, float* ext_val,
                       int64_t* ext_idx, int64_t row_offset, int want_ext, cudaStream_t s, const float* inv_ref = nullptr,
                       float floor = 0.f);
// Reconstruction K = exp(US B_amp) e^{i US B_ph} (k_reconstruct.cu); Bi: k x M x 2 (amp, ph);
// US: n x ldus fp32 (ldus >= k, columns >= k zero).
void launch_reconstruct_simt(const float* US, int64_t n, int k, int ldus, const float* Bi, int M, void* out,
                             int out_imag_only, cudaStream_t s);
// tcgen05 3xTF32 reconstruction (k_reconstruct_tc.cu): B image (K-major core matrices, hi/lo) built
// once per basis; bimg_floats() gives its size.
size_t reconstruct_tc_bimg_floats(int k, int M);
void launch_build_bimg(const float* Bi, int k, int M, float* bimg, cudaStream_t s);
void launch_reconstruct_tc(const float* US, int64_t n, int k, int ldus, const float* bimg, int M, void* out,
                           int out_imag_only, cudaStream_t s);
// Basis (k_basis.cu): all fp64, tiny.
void launch_hilbert_rows_f64(const double* X, int rows, int M, int ldx, double* out, int L, int pad_zero,
                             const double2* tw, cudaStream_t s);
void launch_sg_rows_f64(const double* X, int rows, int M, int h, double* out, cudaStream_t s);
// C[m x n] = alpha * op(A) op(B) (+ beta C); row-major; op = transpose if flag.
void launch_dgemm_small(int m, int n, int kk, const double* A, int lda, int ta, const double* B, int ldb, int tb,
                        double* C, int ldc, double beta, cudaStream_t s);
void launch_vt_over_f(const double* V /* M x k col-major */, const double* f, int M, int k, double* Vt_f,
                      cudaStream_t s);
// ridge: solve (C + lam I) Phi = R with lam = ridge_rel * lambda_max(C); writes lam to lam_out.
void launch_ridge(const double* C, int k, const double* R, int ncol, double ridge_rel, double* Phi, double* lam_out,
                  double* work, int* flags, cudaStream_t s);
void launch_assemble_B(const double* Vt_f, const double* HPhi, const double* Vsec, const double* Hv,
                       const double* Phi_pec, int k, int M, float* Bi, cudaStream_t s);

// ---- GPU eigensolver (k_eig.cu): top-k eigenpairs of the symmetric M x M fp64 G (device);
// V: k vectors of length M (= M x k column-major), lam_out: k descending.
void launch_gram_rows(const double* Z, int M, int k, double* S, cudaStream_t s);
void launch_chol_rinv(const double* S, int k, double* T, int* fallback, cudaStream_t s);
void launch_apply_rinv(const double* Z, int M, int k, const double* T, double* Zn, cudaStream_t s);
// ---- randomized range finder (k_rf.cu)
void rf_omega_host(uint64_t seed, int M, int l, double* omega_lxM);
void launch_rf_reduce(const double* partials, int nT, int nsplit, int M, int l, const double* f, double* Zraw,
                      double* SY, cudaStream_t s);
void launch_rf_combine(const double* Zq, int M, int l, const double* U, const double* lam, int k, double* V,
                       cudaStream_t s);
size_t eig_workspace_doubles(int M, int k);
// M >= 3; flags |= 8 if the re-orthogonalisation finds dependent vectors.  G is not modified.
void launch_eig_topk(const double* G, int M, int k, double* work, double* V, double* lam_out, int* flags,
                     cudaStream_t s);
int eig_path_rows_resident(int M);
void debug_tridiag(const double* G, int M, double* det_out);   // d, e, tau (3M doubles, device)   // 1: the row-resident (shared-memory) tridiagonalisation is used

void launch_tc_selftest(int mode, const float* A, const float* B, float* D, int N, cudaStream_t s);

// ---- host eigensolver (host_eig.cpp): returns 0 on success
int host_eig_topk(const double* G, int M, int k, double* V /* k vectors of length M */, double* lam);

}  // namespace fkk
