/*
 * fkk.h -- C-ABI of the B200-native fKK-EC hot path (arxiv 2005.07132).
 *
 * The method (PAPER.md = /root/reference/PAPER.md, cited as PAPER.md:<line> (section, Eq.)):
 *   inputs  : a CARS cube I (N spectra x M channels, "M spectra ... N frequency
 *             increments" -- letters swapped here to BASELINE.json's N pixels x M channels) and one
 *             surrogate reference spectrum I_ref;
 *   output  : K_CARS = chi^(3)/chi_nr per pixel (Eq. 2), complex; its imaginary part
 *             is the Raman-to-NRB ratio.
 *   paths   : fkk_transform      -- factorized fKK + fPEC + fSEC + reconstruction (Eqs. 6-23,
 *                                   PAPER.md:61-164), a collective over the pixel shards;
 *             fkk_apply_trained_basis -- ML:fKK-EC (Eqs. 24-25), local;
 *             kk_direct_batch    -- conventional per-spectrum KK + PEC + SEC (Eqs. 3-5,
 *                                   PAPER.md:36-55), local;
 *             fkk_svd            -- the truncated SVD alone;
 *             fkk_conventional   -- SVD-denoise of the raw cube + kk_direct (Fig. 1(a), NEXT 2).
 *
 * Conventions:
 *   - cube layout: row-major N x M, each spectrum contiguous; the frequency axis is uniform and
 *     ascending (a descending axis flips the Hilbert sign, reading A2);
 *   - log-ratio a = f * 1/2 ln(max(I/I_ref, ratio_floor)) (Eq. 6/10, readings A15/A16);
 *   - Hilbert: centred pad to L (REFLECT default, ZERO optional), multiplier -i sgn, DC and Nyquist
 *     zeroed, H{cos} = sin (readings A2-A4);
 *   - ALS: lambda = 1e4, p = 1e-3, 10 fp64 solves, w^0 = 1 (readings A6/A7);
 *   - SG trend: order 2, window 2 floor(0.375 M) + 1, polynomial edges (reading A8);
 *   - fPEC ridge lambda = ridge_rel * lambda_max(X^T X) (reading A11); q = sorted unique union of
 *     per-column argmax/argmin, ties to the lowest global pixel index (reading A12).
 *
 * Memory: every pointer named d_* is DEVICE memory (cudaMalloc / torch CUDA tensor) owned by the
 * caller; h_* is host memory owned by the caller.  Inputs are read-only.  All work is enqueued on
 * the plan's stream (fkk_plan_set_stream); calls that return host data synchronise that stream.
 * Errors: every function returns fkk_status and never throws; fkk_last_error(plan) gives a
 * message.  Device-detected errors (non-positive reference, non-finite input) of an asynchronous
 * call are returned by the next fkk_plan_sync() or synchronous call on the same plan.  On error
 * the contents of output buffers are unspecified.  A plan is not thread-safe.
 */
#ifndef FKK_H
#define FKK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FKK_OK = 0,
  FKK_ERR_INVALID_ARG = 1,        /* null pointer, bad shape/size/alignment, k out of range */
  FKK_ERR_NONFINITE_INPUT = 2,    /* NaN/Inf in the cube */
  FKK_ERR_BAD_REFERENCE = 3,      /* I_ref <= 0 or non-finite (Eq. 3 needs ln(I/I_ref)) */
  FKK_ERR_NUMERICAL = 4,          /* eigensolver / Cholesky failure ("increase ridge_rel") */
  FKK_ERR_INCOMPATIBLE_BASIS = 5, /* trained basis M or L differs from the plan */
  FKK_ERR_STATE = 6,              /* call order / plan state error */
  FKK_ERR_CUDA = 7,               /* CUDA runtime error */
  FKK_ERR_NCCL = 8,               /* NCCL error */
  FKK_ERR_OOM = 9,                /* workspace allocation failed */
  FKK_ERR_NOT_IMPLEMENTED = 10
} fkk_status;

typedef enum { FKK_PAD_REFLECT = 0, FKK_PAD_ZERO = 1 } fkk_pad_mode;
typedef enum { FKK_OUT_COMPLEX64 = 0, FKK_OUT_IMAG_F32 = 1 } fkk_out_layout;
typedef enum { FKK_IN_F32 = 0, FKK_IN_F64 = 1 } fkk_in_dtype;
/* Dense contractions (Gram, projection, reconstruction): tcgen05 3xTF32 (default) or an
 * exact-fp32 CUDA-core variant kept as a measured comparison. */
typedef enum { FKK_GEMM_3XTF32 = 0, FKK_GEMM_FP32_SIMT = 1 } fkk_gemm_impl;
typedef enum { FKK_F_ONE = 0, FKK_F_EQ9 = 1 } fkk_f_mode;

typedef enum { FKK_SVD_GRAM = 0, FKK_SVD_RANGE_FINDER = 1 } fkk_svd_mode;
typedef struct fkk_plan* fkk_plan_t;
typedef struct fkk_basis* fkk_basis_t;

typedef struct {
  int32_t n_freq;            /* M: 8 <= M <= 4096, M % 4 == 0 (16-B rows for vector loads) */
  int64_t max_rows;          /* max spectra per call on this rank (workspace sizing), >= 1 */
  int32_t rank_k;            /* k: 1 <= k <= min(M, 128, N_global) retained singular triplets */
  int32_t fft_len;           /* L: 0 -> 2*nextpow2(M); else a power of two >= M, <= 8192 */
  int32_t pad_mode;          /* fkk_pad_mode, default FKK_PAD_REFLECT (reading A3) */
  double ratio_floor;        /* clamp of I/I_ref before ln, default 1e-6 (reading A16); must be >= FLT_MIN */
  int32_t f_mode;            /* fkk_f_mode: f(omega) of Eq. 9 or f == 1 (default) */
  double f_alpha, f_sigma_g; /* Eq. 9 Poisson multiplier and Gaussian sigma */
  double als_lambda;         /* ALS smoothness, default 1e4 */
  double als_p;              /* ALS asymmetry, default 1e-3 */
  int32_t als_iters;         /* ALS solves, default 10 */
  int32_t sg_window;         /* 0 -> 2*floor(0.375*M)+1 (odd, <= M) */
  int32_t sg_order;          /* must be 2 */
  double ridge_rel;          /* fPEC ridge: lambda = ridge_rel * lambda_max(X^T X), default 1e-3 */
  double ml_ridge_rel;       /* ML ridge: lambda_ml = ml_ridge_rel * s_1^2, default 0 */
  int32_t gemm_impl;         /* fkk_gemm_impl */
  int32_t out_layout;        /* fkk_out_layout */
  int32_t in_dtype;          /* fkk_in_dtype of the cube and of I_ref */
  int32_t device;            /* CUDA device ordinal */
  int32_t world_size, rank;  /* pixel shards: this rank owns a contiguous block of rows */
  const uint8_t* nccl_id;    /* 128-byte ncclUniqueId from fkk_get_nccl_unique_id: required when world_size > 1;
                                with world_size == 1 it selects the NCCL backend over a 1-rank communicator
                                (exercises the collective path on one GPU); NULL: no communicator */
  int32_t loopback_shards;   /* >1: run the Gram/projection per virtual shard on one GPU and combine
                                in the multi-rank order (partition-invariance test mode) */
  /* F2-F4 method ("random sampling ('randomized') SVD", Halko 2011):
   * FKK_SVD_GRAM (default) = Gram A^T A + fp64 eigensolver; FKK_SVD_RANGE_FINDER = randomized subspace
   * iteration: Y = A Omega (Omega: M x (k + rf_oversample) Gaussian from SplitMix64 counters keyed by
   * rf_seed, oracle/range_finder_omega), rf_power_iters times {Y = A orth(A^T orth(Y))}, then the SVD
   * of B = orth(Y)^T A.  Needs k + rf_oversample <= min(M, 128), f32 input, world_size/loopback as
   * the Gram path (the l x M and l x l products are all-reduced). */
  int32_t svd_mode;          /* fkk_svd_mode, default FKK_SVD_GRAM */
  int32_t rf_oversample;     /* p >= 0, default 10 */
  int32_t rf_power_iters;    /* q >= 0, default 1 */
  uint64_t rf_seed;          /* test-matrix seed, default 0 */
} fkk_plan_desc;

/* Fill *d with the defaults above for the given M, k and max_rows. */
void fkk_plan_desc_init(fkk_plan_desc* d, int32_t n_freq, int32_t rank_k, int64_t max_rows);

fkk_status fkk_get_nccl_unique_id(uint8_t out[128]);
fkk_status fkk_plan_create(const fkk_plan_desc* d, fkk_plan_t* out);  /* allocates all workspace */
fkk_status fkk_plan_destroy(fkk_plan_t p);
const char* fkk_last_error(fkk_plan_t p);          /* valid until the next call on p; p may be NULL */
/* Enqueue subsequent work on cuda_stream (a cudaStream_t; NULL = the legacy default stream).  A new
 * plan starts on its own non-blocking stream. */
fkk_status fkk_plan_set_stream(fkk_plan_t p, void* cuda_stream);
fkk_status fkk_plan_sync(fkk_plan_t p);            /* synchronise; report deferred device errors */

/* fkk_svd -- truncated SVD A ~ U S V^T of the log-ratio matrix through the Gram
 * matrix G = A^T A (all-reduced over ranks).  Collective.  d_icars: n_rows x M (this rank's rows);
 * d_iref: M.  d_V_out: M x k fp32, column-major (each right singular vector contiguous), sign rule:
 * the entry of largest |.| is positive.  h_s_out: k singular values (host, descending).  Syncs. */
fkk_status fkk_svd(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref,
                   float* d_V_out, double* h_s_out);

/* fkk_transform -- full fKK-EC (F0..F11): Eq. 23
 *   K = exp[US (V^T/f + H{Phi_PEC} - V_SEC^T)] exp[i US (H{V^T/f} - Phi_PEC)].
 * Collective.  d_out: n_rows x M complex64 (re, im interleaved) or fp32 Im only (out_layout).
 * basis_out (nullable): receives a trained basis (caller frees with fkk_basis_destroy). */
fkk_status fkk_transform(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref,
                         void* d_out, fkk_basis_t* basis_out);

/* fkk_apply_trained_basis -- ML:fKK-EC (Eqs. 24-25): US_new = A_new W with
 * W = V diag(s^2/(s^2 + lambda_ml)), then Eq. 23 with the trained B.  Local (no collective).
 * Uses the trained reference and f stored in the basis. */
fkk_status fkk_apply_trained_basis(fkk_plan_t p, fkk_basis_t b, const void* d_icars,
                                   int64_t n_rows, void* d_out);

/* kk_direct_batch -- conventional per-spectrum KK + PEC + SEC (Eq. 5 in the log domain,
 * PAPER.md:53): a = 1/2 ln(I/I_ref); phi = H{a}; phi_err = ALS(phi); a' = a + H{phi_err};
 * phi' = phi - phi_err; K' = e^{a'} e^{i phi'}; K_CARS = K' / SGtrend(Re K').  Local. */
fkk_status kk_direct_batch(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref,
                           void* d_out);

/* fkk_conventional -- the paper's comparison baseline, Fig. 1(a) (
 * SURVEY 8(f) NEXT 2; reading A26): rank-k_keep SVD denoise of the RAW cube,
 * I_k = (I V_k) V_k^T with V_k the top eigenvectors of I^T I (same tensor-core Gram, GPU eigensolver
 * and projection as fkk_svd), then kk_direct_batch of every denoised spectrum.
 * k_keep in [1, rank_k].  d_icars: n_rows x M f32 (device), d_out: as kk_direct_batch.  The plan's
 * N x M workspace holds I_k.  Requires an f32 plan on the 3xTF32 path with world_size 1
 * (FKK_ERR_NOT_IMPLEMENTED otherwise).  Local, enqueued on the plan stream (one host sync after the
 * eigensolver). */
fkk_status fkk_conventional(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref, int32_t k_keep,
                            void* d_out);

/* Host-buffer variants (end-to-end: host->device copies, compute, device->host copies, all on the
 * plan's stream; they synchronise before returning).  h_* may be pageable or pinned. */
fkk_status fkk_transform_host(fkk_plan_t p, const void* h_icars, int64_t n_rows, const void* h_iref,
                              void* h_out, fkk_basis_t* basis_out);
/* fKK-EC (as fkk_transform) of n_cubes host-resident cubes of n_rows spectra each, streamed: cube
 * i+1's host->device copy and cube i-1's device->host copy overlap cube i's transform, over two copy
 * streams and two device cube-buffer pairs (allocated on first use, kept by the plan; 2 (in + out)
 * cube bytes).  h_icars[i] / h_out[i]: host cubes (pinned for the copies to overlap; an output
 * buffer may repeat with a stride of 2 or more).  h_cube_ms (nullable, n_cubes floats): per-cube
 * latency, H2D start to D2H end (CUDA events).  Each cube's result equals fkk_transform_host's.
 * Synchronises before returning; errors as fkk_transform. */
fkk_status fkk_transform_host_stream(fkk_plan_t p, const void* const* h_icars, int32_t n_cubes, int64_t n_rows,
                                     const void* h_iref, void* const* h_out, float* h_cube_ms);
fkk_status fkk_apply_trained_basis_host(fkk_plan_t p, fkk_basis_t b, const void* h_icars,
                                        int64_t n_rows, void* h_out);
fkk_status kk_direct_batch_host(fkk_plan_t p, const void* h_icars, int64_t n_rows,
                                const void* h_iref, void* h_out);
/* ML:fKK-EC apply of a host-resident cube streamed in batches
 * of `batch` spectra (<= max_rows): per batch a host->device copy, the apply (as
 * fkk_apply_trained_basis) and a device->host copy, pipelined over three streams with two device
 * buffer pairs (allocated on the first call and kept by the plan).  h_icars / h_out should be pinned
 * (cudaHostAlloc) for the copies to overlap.  h_batch_ms (nullable, ceil(n_rows / batch) floats):
 * each batch's end-to-end latency (H2D start to D2H end, CUDA events).  Synchronises before returning. */
fkk_status fkk_apply_trained_basis_stream(fkk_plan_t p, fkk_basis_t b, const void* h_icars, int64_t n_rows,
                                          int64_t batch, void* h_out, float* h_batch_ms);

fkk_status fkk_basis_destroy(fkk_basis_t b);
/* Basis metadata: M, k, L.  Any pointer may be NULL. */
fkk_status fkk_basis_info(fkk_basis_t b, int32_t* n_freq, int32_t* rank_k, int32_t* fft_len);

/* Stage tensors of the last fkk_transform / fkk_svd on p (stage-wise parity):
 *   G: M x M fp64 | S: k fp64 | V: M x k fp64 column-major | US: n_rows x k fp32 row-major |
 *   Q: nq int64 (global pixel indices, ascending) | HV: k x M fp64 | PHI_ERR: nq x M fp64 |
 *   PHI_PEC: k x M fp64 | V_SEC: k x M fp64 | B: k x M x 2 fp32 (amp, ph interleaved) |
 *   LAMBDA: 1 fp64 (fPEC ridge) | F: M fp64.
 * fkk_stage_size returns the byte size; fkk_get_stage copies min(bytes, size) bytes. */
typedef enum {
  FKK_STAGE_G = 0, FKK_STAGE_S, FKK_STAGE_V, FKK_STAGE_US, FKK_STAGE_Q, FKK_STAGE_HV,
  FKK_STAGE_PHI_ERR, FKK_STAGE_PHI_PEC, FKK_STAGE_V_SEC, FKK_STAGE_B, FKK_STAGE_LAMBDA, FKK_STAGE_F
} fkk_stage;
size_t fkk_stage_size(fkk_plan_t p, int32_t stage);
fkk_status fkk_get_stage(fkk_plan_t p, int32_t stage, void* dst, size_t bytes, int32_t dst_is_device);

/* Test hook: F5..F11 with caller-supplied V (d_V: M x k fp32 column-major), s (host) and q (host,
 * global pixel indices, ascending, nq <= 2k), skipping the SVD and the q selection. */
fkk_status fkk_transform_from(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref,
                              const float* d_V, const double* h_s, const int64_t* h_q, int32_t nq,
                              void* d_out);

/* Per-stage device times (ms) of the last call, measured with CUDA events on the plan stream when
 * timing is enabled.  names/ms arrays of length cap; returns the number of stages written. */
fkk_status fkk_enable_timing(fkk_plan_t p, int32_t on);
int32_t fkk_stage_times(fkk_plan_t p, const char** names, float* ms, int32_t cap);
/* Number of kernel launches issued by the last call (the bench reports it). */
int64_t fkk_last_launch_count(fkk_plan_t p);
/* Diagnostic: ALS solves summed over the spectra of the direct-path calls since the last query
 * (the ALS stops once a solve changes no weight, PAPER.md:45 / reading A6; iters per spectrum =
 * this / spectra).  Synchronises the plan stream and resets the counter; -1 on a CUDA error. */
int64_t fkk_debug_als_solves(fkk_plan_t p);
/* Host helper (no GPU): the range finder's test matrix Omega for seed, M x l row-major
 * into out_Mxl: entry (j, i) = sqrt(-2 ln u1) cos(2 pi u2), u1 = ((h(2c) >> 11) + 1) / 2^53,
 * u2 = (h(2c+1) >> 11) / 2^53, h = SplitMix64, counter c = seed 2^40 + j l + i.  Returns 0, or 1 on bad
 * arguments. */
int32_t fkk_range_finder_omega(uint64_t seed, int32_t M, int32_t l, double* out_Mxl);

/* Collectives supplied by the caller (host buffers; each returns 0 on success), for running the sharded
 * transform's exchange sequence without GPUs. */
typedef struct {
  void* ctx;
  int32_t world_size, rank;
  int32_t (*allgather)(void* ctx, const void* send, void* recv, size_t bytes);   /* recv: world x bytes */
  int32_t (*allreduce_sum_f64)(void* ctx, double* data, size_t n);
  int32_t (*allreduce_max_i32)(void* ctx, int32_t* data, size_t n);
} fkk_host_collectives;
/* The collective sequence of a pixel-sharded fkk_transform on host data, through
 * the same C++ sequence functions the NCCL path calls: row-count allgather (-> *row0_out, *n_global_out),
 * Gram all-reduce (G: M x M local partial in, global sum out), extremes allgather + merge (ext_val /
 * ext_idx: shards x k x 2 local column max / min and their GLOBAL pixel indices; -> q_out (<= 2k,
 * ascending), *nq_out), X = US[q] all-reduce (US_local: n_rows x k row-major; X_out: nq x k), error-flag
 * max-reduce (*flags in/out).  Collective over the caller's ranks; no GPU needed. */
fkk_status fkk_exchange_selftest(const fkk_host_collectives* comm, int64_t n_rows, int32_t M, int32_t k, int32_t shards,
                                 double* G, const float* ext_val, const int64_t* ext_idx, const float* US_local,
                                 int32_t* flags, int64_t* row0_out, int64_t* n_global_out, int64_t* q_out,
                                 int32_t* nq_out, double* X_out);

/* Test hook (tensor-core plumbing self-test): one tcgen05.mma kind::tf32 of A (128 x 8, row-major
 * fp32, device) times B^T (B: N x 8, N in {16, 32, ..., 256}) into D (128 x N fp32, device) with the
 * UMMA smem layout selected by mode (bit 0: A MN-major, bit 1: B MN-major, bit 2: 16-B padding).
 * Synchronises the device. */
fkk_status fkk_debug_tc_mma(int32_t mode, const float* d_A, const float* d_B, float* d_D, int32_t N);

/* Test hook (F4, PAPER.md:64, :70 -- the truncated SVD through the Gram eigenproblem): the GPU
 * eigensolver that fkk_svd/fkk_transform run, on a caller-supplied symmetric M x M fp64 matrix d_G
 * (device, row-major, both triangles; not modified).  d_V: k x M (vector j contiguous, device),
 * d_lam: k descending (device).  Sign rule as fkk_svd.  M >= 3, 1 <= k <= M, else INVALID_ARG;
 * dependent inverse-iteration vectors -> NUMERICAL.  Allocates its own workspace; synchronises. */
fkk_status fkk_debug_eig_topk(const double* d_G, int32_t M, int32_t k, double* d_V, double* d_lam);
/* 1 if the eigensolver keeps the working matrix resident in shared memory for this M (the
 * row-resident tridiagonalisation), 0 if it streams it through L2. */
int32_t fkk_debug_eig_path(int32_t M);
/* Test hook: the tridiagonalisation step of the eigensolver alone.  d_det (device, 3M doubles)
 * receives d (diagonal), e (off-diagonal, M-1 used) and tau (reflector factors). */
fkk_status fkk_debug_tridiag(const double* d_G, int32_t M, double* d_det);

/* ---------------- host-only helpers (no GPU needed; exercised by the CPU tests) ---------------- */
/* Top-k eigenpairs of a symmetric M x M fp64 matrix (row-major; only the lower triangle is read):
 * Householder tridiagonalisation, Sturm bisection, inverse iteration, back-transformation.
 * V: M x k column-major, lam: k descending.  Sign rule as fkk_svd. */
fkk_status fkk_host_eig_topk(const double* G, int32_t M, int32_t k, double* V, double* lam);
/* Rows [*row0, *row1) owned by `rank` of `world` for n_global rows (contiguous, ragged last). */
void fkk_shard_range(int64_t n_global, int32_t world, int32_t rank, int64_t* row0, int64_t* row1);
/* Merge per-rank column extremes into q (reading A12).  vals/idx: world x k x 2 arrays, [..][..][0]
 * = max, [1] = min, idx = global pixel index.  Writes the sorted unique union to q_out (capacity
 * 2k) and returns its length. */
int32_t fkk_merge_extremes(const float* vals, const int64_t* idx, int32_t world, int32_t k,
                           int64_t* q_out);

#ifdef __cplusplus
}
#endif
#endif /* FKK_H */
