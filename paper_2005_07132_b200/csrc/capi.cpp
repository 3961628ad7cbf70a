// C-ABI of the fKK-EC hot path (include/fkk.h): plan / workspace / stream management, the stage
// orchestration of the factorized path (F0..F11), ML reuse (F12)
// and the direct path (D1..D5), NCCL for the pixel-sharded collectives.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <cstdlib>

#include "../../include/fkk.h"
#include "fkk_internal.h"
#include "exchange.h"
#include <nvtx3/nvToolsExt.h>
#include <thread>

using fkk::Status;

// ------------------------------------------------------------------------------------------------
// NCCL, resolved at run time (only when the plan is given an nccl_id), so the library loads without it.
// ------------------------------------------------------------------------------------------------
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) { h = dlopen(n, RTLD_NOW | RTLD_GLOBAL); if (h) break; }
    if (!h) { err = "cannot dlopen libnccl.so.2"; return false; }
#define FKK_SYM(field, name) field = reinterpret_cast<decltype(field)>(dlsym(h, name)); if (!field) { err = "missing NCCL symbol " name; return false; }
    FKK_SYM(GetUniqueId, "ncclGetUniqueId");
    FKK_SYM(CommInitRank, "ncclCommInitRank");
    FKK_SYM(CommDestroy, "ncclCommDestroy");
    FKK_SYM(CommAbort, "ncclCommAbort");
    FKK_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    FKK_SYM(AllReduce, "ncclAllReduce");
    FKK_SYM(AllGather, "ncclAllGather");
    FKK_SYM(GetErrorString, "ncclGetErrorString");
#undef FKK_SYM
    return true;
  }
};
NcclApi g_nccl;

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Status(FKK_ERR_NCCL, std::string("NCCL ") + what + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
}

template <typename T>
T* dalloc(size_t count) {
  if (count == 0) count = 1;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Status(FKK_ERR_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed: " + cudaGetErrorString(e));
  }
  return static_cast<T*>(p);
}

int ilog2i(int L) { int r = 0; while ((1 << r) < L) ++r; return r; }
int next_pow2(int v) { int p = 1; while (p < v) p <<= 1; return p; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

// ------------------------------------------------------------------------------------------------
// Trained basis (ML:fKK-EC model: f, S, V, Phi_PEC, V_SEC -> W and B)
// ------------------------------------------------------------------------------------------------
struct fkk_basis {
  int M = 0, k = 0, kp = 0, L = 0, pad = 0, device = 0;
  double ratio_floor = 1e-6;
  float* inv_ref = nullptr;
  double* ref64 = nullptr;
  double* f64 = nullptr;
  float* W = nullptr;    // M x kp, D_f V diag(s^2/(s^2+lam_ml))
  float* Bi = nullptr;   // k x M x 2
  float* bimg = nullptr; // tensor-core B image (reconstruct_tc)
  bool bimg_valid = false;
  float* wimg = nullptr; // tensor-core W^T image (project_tc)
  double* V64 = nullptr;
  std::vector<double> s;
  ~fkk_basis() {
    cudaFree(inv_ref); cudaFree(ref64); cudaFree(f64); cudaFree(W); cudaFree(Bi); cudaFree(V64); cudaFree(bimg); cudaFree(wimg);
  }
};

// ------------------------------------------------------------------------------------------------
// Plan
// ------------------------------------------------------------------------------------------------
struct fkk_plan {
  bool a0_raw = false;   // A0 not materialised by the last svd_stage (projection reads the cube)
  fkk_plan_desc d{};
  int M = 0, k = 0, kp = 0, L = 0, log2L = 0, sg_half = 0, in_f64 = 0, pad_zero = 0;
  size_t in_elem = 4;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  // NCCL
  ncclComm_t comm = nullptr;
  bool use_nccl = false;   // nccl_id given: the NCCL backend (world_size > 1, or a 1-rank communicator)
  std::unique_ptr<fkk::Collectives> coll;   // the sharded exchange's collectives (local copy or NCCL)
  unsigned char* xscratch = nullptr;        // device staging of the control collectives (NCCL)
  size_t xscratch_bytes = 0;
  // device workspace (factorized)
  int* flags = nullptr;
  int* h_flags = nullptr;   // pinned
  float* inv_ref = nullptr;
  double* ref64 = nullptr;
  float2* tw32 = nullptr;
  int* pmap = nullptr;
  double2* tw64 = nullptr;
  float* A = nullptr;
  double* gram_part = nullptr;
  int gram_nsplit_cap = 0;
  double* G = nullptr;
  double* colsum = nullptr;
  double* f64 = nullptr;
  float* f32 = nullptr;
  double* V64 = nullptr;
  float* W = nullptr;
  float* US = nullptr;
  float* ext_val = nullptr;
  int64_t* ext_idx = nullptr;
  float* ext_out_val = nullptr;
  int64_t* ext_out_idx = nullptr;
  int64_t* q_dev = nullptr;
  double *X = nullptr, *Vt_f = nullptr, *Hv = nullptr, *P = nullptr, *Phi_err = nullptr, *XtX = nullptr,
         *XtPhi = nullptr, *Phi_pec = nullptr, *HPhi = nullptr, *tmp = nullptr, *Vsec = nullptr, *ridge_work = nullptr,
         *lam = nullptr;
  float* Bi = nullptr;
  float* bimg = nullptr;
  float* wimg = nullptr;
  double* eig_work = nullptr;
  double* lam_d = nullptr;
  // tcgen05 Gram
  int2* gtc_tiles = nullptr;
  int* gtc_tile_of = nullptr;
  int gtc_ntiles = 0, gtc_nTj = 0, gtc_nsplit = 0;
  // Gram variants (3xTF32): 0 = 1-CTA 128x128 fed by the pre-split A0 image, 1 = CTA pairs 256x256
  // fed by the image (default when ceil(M/128) is even), 2 = 1-CTA with in-kernel producers (fp64 input /
  // loopback shards), 3 = CTA pairs with in-kernel producers (measurement only).  FKK_GRAM_MODE overrides.
  int gram_mode = 0;
  bool gtc_pair = false;
  unsigned char* apre = nullptr;   // pre-split MMA image of A0
  int apre_blocks = 0;
  double* gtc_part = nullptr;
  // randomized range finder (svd_mode = FKK_SVD_RANGE_FINDER): l = k + oversample columns
  int rf_l = 0, rf_nsplit = 0;
  double *rf_omega = nullptr, *rf_part = nullptr, *rf_Z = nullptr, *rf_Zq = nullptr, *rf_Z2 = nullptr,
         *rf_SY = nullptr, *rf_S = nullptr, *rf_T = nullptr, *rf_U = nullptr, *rf_lam = nullptr;
  float *rf_wimg = nullptr, *rf_Y = nullptr;
  int2* rf_tiles = nullptr;
  int* rf_fallback = nullptr;
  // direct path (lazy)
  int64_t direct_batch = 0;
  float *phi = nullptr, *phierr = nullptr;
  int* als_solves = nullptr;   // ALS solves summed over the spectra of the direct calls (diagnostic)
  unsigned* als_ctr = nullptr;  // the direct ALS launches' dynamic spectrum counter
  // host-buffer variants (lazy)
  void* d_in_cube = nullptr;
  size_t d_in_cube_bytes = 0;
  void* d_out_cube = nullptr;
  size_t d_out_cube_bytes = 0;
  void* d_ref_buf = nullptr;
  // streamed ML apply (lazy): two input and two output batch buffers, copy-in / copy-out streams
  void* stream_bufs[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t stream_in_bytes = 0, stream_out_bytes = 0;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  // streamed host transform (lazy): two input and two output cube buffers
  void* cube_bufs[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t cube_in_bytes = 0, cube_out_bytes = 0;
  // last-call host state
  std::vector<double> h_s;
  std::vector<int64_t> h_q;
  int64_t last_rows = 0, last_row0 = 0, last_global_rows = 0;
  bool have_transform = false;
  // timing
  bool timing = false;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  std::vector<std::string> t_names;
  std::vector<float> t_ms;
  int64_t launches = 0;

  ~fkk_plan() {
    if (stream) cudaStreamSynchronize(stream);
    void* ptrs[] = {flags, inv_ref, ref64, tw32, pmap, tw64, A, gram_part, G, colsum, f64, f32, V64, W, US, ext_val,
                    ext_idx, ext_out_val, ext_out_idx, q_dev, X, Vt_f, Hv, P, Phi_err, XtX, XtPhi, Phi_pec, HPhi,
                    tmp, Vsec, ridge_work, lam, Bi, bimg, wimg, eig_work, lam_d, gtc_tiles, gtc_tile_of, gtc_part, apre, phi, phierr, als_solves, als_ctr, rf_omega, rf_part, rf_Z, rf_Zq, rf_Z2, rf_SY, rf_S, rf_T, rf_U, rf_lam,
                    rf_wimg, rf_Y, rf_tiles, rf_fallback, d_in_cube,
                    d_out_cube, d_ref_buf};
    for (void* p : ptrs) if (p) cudaFree(p);
    if (h_flags) cudaFreeHost(h_flags);
    for (void* b : stream_bufs) if (b) cudaFree(b);
    for (void* b : cube_bufs) if (b) cudaFree(b);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    for (auto& m : marks) cudaEventDestroy(m.second);
    coll.reset();
    if (xscratch) cudaFree(xscratch);
    if (comm && g_nccl.CommDestroy) g_nccl.CommDestroy(comm);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  int nq_cap() const { return 2 * k; }

  // NVTX: one range per C-ABI call (its name) and one per stage, closed at the stage's mark, so an
  // nsys/ncu timeline shows the paper's steps
  int nvtx_depth = 0;
  void nvtx_push(const char* name) { nvtxRangePushA(name); ++nvtx_depth; }
  void nvtx_pop_all() { while (nvtx_depth > 0) { nvtxRangePop(); --nvtx_depth; } }
  void mark(const char* name) {
    if (nvtx_depth > 1) { nvtxRangePop(); --nvtx_depth; }
    nvtxMarkA(name);
    if (nvtx_depth == 1) nvtx_push("stage");
    if (!timing) return;
    cudaEvent_t e;
    FKK_CUDA_CHECK(cudaEventCreate(&e));
    FKK_CUDA_CHECK(cudaEventRecord(e, stream));
    marks.emplace_back(name, e);
  }
  void begin_call(const char* name = "fkk_call") {
    nvtx_pop_all();
    nvtx_push(name);
    nvtx_push("stage");
    for (auto& m : marks) cudaEventDestroy(m.second);
    marks.clear();
    fkk::g_launches = 0;
    FKK_CUDA_CHECK(cudaSetDevice(d.device));
    mark("start");
  }
  void end_call() {
    nvtx_pop_all();
    launches = fkk::g_launches;
    t_names.clear();
    t_ms.clear();
    if (!timing || marks.size() < 2) return;
    FKK_CUDA_CHECK(cudaEventSynchronize(marks.back().second));
    for (size_t i = 1; i < marks.size(); ++i) {
      float ms = 0.f;
      FKK_CUDA_CHECK(cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second));
      t_names.push_back(marks[i].first);
      t_ms.push_back(ms);
    }
  }

  // deferred device errors: reads the pinned flag word after the stream drained.  In the collective
  // calls (`collective`, every rank at the same point) the word is first max-reduced over the ranks, so
  // a non-finite value in one rank's shard makes EVERY rank throw the same error instead of leaving
  // the others blocked in the next collective.
  void check_flags_sync(bool collective = false);
  void check_flags_sync_impl(bool collective) {
    if (collective && use_nccl) {
      if (!comm) throw Status(FKK_ERR_STATE, "the communicator was aborted by an earlier failure; recreate the plan");
      nccl_allreduce_flags();
    }
    FKK_CUDA_CHECK(cudaMemcpyAsync(h_flags, flags, sizeof(int), cudaMemcpyDeviceToHost, stream));
    if (collective) coll->sync();
    else FKK_CUDA_CHECK(cudaStreamSynchronize(stream));
    const int f = *h_flags;
    if (f) {
      FKK_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(int), stream));
      if (f & 1) throw Status(FKK_ERR_BAD_REFERENCE, "reference spectrum has a non-positive or non-finite value");
      if (f & 2) throw Status(FKK_ERR_NONFINITE_INPUT, "non-finite value in the input cube");
      if (f & 4) throw Status(FKK_ERR_NUMERICAL, "ridge system not positive definite (increase ridge_rel)");
      if (f & 8) throw Status(FKK_ERR_NUMERICAL, "eigensolver: inverse-iteration vectors are linearly dependent");
    }
  }

  void nccl_allreduce_flags();

  void ensure_direct() {
    if (phi) return;
    // phi / phi_err scratch of up to 8 GB (one batch for cfg3: 47.5 ms per pass against 48.3 ms in
    // 131,072-spectrum batches, fewer kernel tails)
    int64_t cap = std::max<int64_t>(4096, (int64_t)(8e9 / (8.0 * (double)M)));
    if (const char* ev = getenv("FKK_DIRECT_BATCH")) cap = std::max<int64_t>(64, atoll(ev));   // A/B only
    direct_batch = std::min<int64_t>(std::max<int64_t>(d.max_rows, 2), cap);
    direct_batch = ((direct_batch + 31) / 32) * 32;
    phi = dalloc<float>((size_t)direct_batch * M);
    phierr = dalloc<float>((size_t)direct_batch * M);
    als_solves = dalloc<int>(1);
    FKK_CUDA_CHECK(cudaMemset(als_solves, 0, sizeof(int)));
    als_ctr = dalloc<unsigned>(1);
  }
};

// one rank: the collectives are identities (the sequence code is shared with the NCCL path)
struct LocalCollectives : fkk::Collectives {
  fkk_plan* p;
  explicit LocalCollectives(fkk_plan* pl) : p(pl) {}
  void allgather_host(const void* send, void* recv, size_t bytes) override { std::memcpy(recv, send, bytes); }
  void allreduce_sum_f64(double*, size_t) override {}
  void allreduce_max_i32(int*, size_t) override {}
  void sync() override { FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream)); }
};

// NCCL over the plan's communicator, enqueued on the plan stream.  Control data is staged through a
// device scratch buffer sized at plan creation (no per-call allocation).  sync() polls the stream and
// ncclCommGetAsyncError against a deadline (FKK_NCCL_TIMEOUT_S, default 600 s): a peer that failed
// before a collective leaves this rank waiting, and the deadline turns that into ncclCommAbort and
// FKK_ERR_NCCL instead of a hang.
struct NcclCollectives : fkk::Collectives {
  fkk_plan* p;
  explicit NcclCollectives(fkk_plan* pl) : p(pl) {
    world = pl->d.world_size;
    rank = pl->d.rank;
  }
  void allgather_host(const void* send, void* recv, size_t bytes) override {
    if ((size_t)(world + 1) * bytes > p->xscratch_bytes) throw Status(FKK_ERR_STATE, "collective scratch too small");
    unsigned char* mine = p->xscratch + (size_t)world * bytes;
    FKK_CUDA_CHECK(cudaMemcpyAsync(mine, send, bytes, cudaMemcpyHostToDevice, p->stream));
    nccl_check(g_nccl.AllGather(mine, p->xscratch, bytes, ncclInt8, p->comm, p->stream), "AllGather");
    FKK_CUDA_CHECK(cudaMemcpyAsync(recv, p->xscratch, (size_t)world * bytes, cudaMemcpyDeviceToHost, p->stream));
    sync();
  }
  void allreduce_sum_f64(double* d, size_t n) override {
    nccl_check(g_nccl.AllReduce(d, d, n, ncclFloat64, ncclSum, p->comm, p->stream), "AllReduce(sum)");
  }
  void allreduce_max_i32(int* d, size_t n) override {
    nccl_check(g_nccl.AllReduce(d, d, n, ncclInt32, ncclMax, p->comm, p->stream), "AllReduce(max)");
  }
  void sync() override {
    static const double limit = getenv("FKK_NCCL_TIMEOUT_S") ? atof(getenv("FKK_NCCL_TIMEOUT_S")) : 600.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      const cudaError_t e = cudaStreamQuery(p->stream);
      if (e == cudaSuccess) return;
      if (e != cudaErrorNotReady) FKK_CUDA_CHECK(e);
      ncclResult_t ar = ncclSuccess;
      if (p->comm && g_nccl.CommGetAsyncError(p->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
        abort_comm();
        throw Status(FKK_ERR_NCCL, std::string("NCCL asynchronous error: ") + g_nccl.GetErrorString(ar));
      }
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > limit) {
        abort_comm();
        throw Status(FKK_ERR_NCCL, "collective not complete after " + std::to_string((int)limit) +
                                       " s (a peer rank failed or diverged): communicator aborted");
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  void abort_comm() {
    if (p->comm && g_nccl.CommAbort) g_nccl.CommAbort(p->comm);
    p->comm = nullptr;
  }
};

void fkk_plan::nccl_allreduce_flags() { coll->allreduce_max_i32(flags, 1); }
void fkk_plan::check_flags_sync(bool collective) { check_flags_sync_impl(collective); }

namespace {

void validate_desc(const fkk_plan_desc* d) {
  if (!d) throw Status(FKK_ERR_INVALID_ARG, "desc is NULL");
  if (d->n_freq < 8 || d->n_freq > 4096 || d->n_freq % 4) throw Status(FKK_ERR_INVALID_ARG, "n_freq must be in [8, 4096] and a multiple of 4");
  if (d->max_rows < 1) throw Status(FKK_ERR_INVALID_ARG, "max_rows must be >= 1");
  if (d->rank_k < 1 || d->rank_k > std::min(d->n_freq, 128)) throw Status(FKK_ERR_INVALID_ARG, "rank_k must be in [1, min(M, 128)]");
  if (d->fft_len) {
    if (d->fft_len < d->n_freq || (d->fft_len & (d->fft_len - 1)) || d->fft_len > 8192)
      throw Status(FKK_ERR_INVALID_ARG, "fft_len must be a power of two in [M, 8192]");
  }
  if (d->pad_mode != FKK_PAD_REFLECT && d->pad_mode != FKK_PAD_ZERO) throw Status(FKK_ERR_INVALID_ARG, "bad pad_mode");
  // >= FLT_MIN: the kernels take the log of max(I / I_ref, floor) in fp32 with flush-to-zero hardware lg2
  if (!(d->ratio_floor >= 1.1754943508222875e-38))
    throw Status(FKK_ERR_INVALID_ARG, "ratio_floor must be >= FLT_MIN (1.18e-38)");
  if (d->f_mode != FKK_F_ONE && d->f_mode != FKK_F_EQ9) throw Status(FKK_ERR_INVALID_ARG, "bad f_mode");
  if (!(d->als_lambda > 0) || !(d->als_p > 0 && d->als_p < 0.5) || d->als_iters < 1)
    throw Status(FKK_ERR_INVALID_ARG, "ALS needs lambda > 0, 0 < p < 0.5, iters >= 1");
  if (d->sg_order != 2) throw Status(FKK_ERR_INVALID_ARG, "sg_order must be 2");
  if (d->sg_window && (d->sg_window % 2 == 0 || d->sg_window < 5 || d->sg_window > d->n_freq))
    throw Status(FKK_ERR_INVALID_ARG, "sg_window must be odd, >= 5 and <= M");
  if (!(d->ridge_rel >= 0) || !(d->ml_ridge_rel >= 0)) throw Status(FKK_ERR_INVALID_ARG, "ridge weights must be >= 0");
  if (d->gemm_impl != FKK_GEMM_3XTF32 && d->gemm_impl != FKK_GEMM_FP32_SIMT) throw Status(FKK_ERR_INVALID_ARG, "bad gemm_impl");
  if (d->out_layout != FKK_OUT_COMPLEX64 && d->out_layout != FKK_OUT_IMAG_F32) throw Status(FKK_ERR_INVALID_ARG, "bad out_layout");
  if (d->in_dtype != FKK_IN_F32 && d->in_dtype != FKK_IN_F64) throw Status(FKK_ERR_INVALID_ARG, "bad in_dtype");
  if (d->world_size < 1 || d->rank < 0 || d->rank >= d->world_size) throw Status(FKK_ERR_INVALID_ARG, "bad world_size/rank");
  if (d->world_size > 1 && !d->nccl_id) throw Status(FKK_ERR_INVALID_ARG, "nccl_id must be given when world_size > 1");
  if (d->loopback_shards < 0 || d->loopback_shards > 64) throw Status(FKK_ERR_INVALID_ARG, "loopback_shards must be in [0, 64]");
  if (d->svd_mode != FKK_SVD_GRAM && d->svd_mode != FKK_SVD_RANGE_FINDER) throw Status(FKK_ERR_INVALID_ARG, "bad svd_mode");
  if (d->svd_mode == FKK_SVD_RANGE_FINDER) {
    if (d->rf_oversample < 0 || d->rf_power_iters < 0 || d->rf_power_iters > 16)
      throw Status(FKK_ERR_INVALID_ARG, "range finder: oversample >= 0, 0 <= power_iters <= 16");
    if (d->rank_k + d->rf_oversample > std::min(d->n_freq, 128))
      throw Status(FKK_ERR_INVALID_ARG, "range finder: k + oversample must be <= min(M, 128)");
    if (d->in_dtype != FKK_IN_F32 || d->gemm_impl != FKK_GEMM_3XTF32)
      throw Status(FKK_ERR_NOT_IMPLEMENTED, "range finder: f32 cube on the tensor-core path");
  }
}

void create_plan(const fkk_plan_desc* d, fkk_plan* p) {
  validate_desc(d);
  p->d = *d;
  p->M = d->n_freq;
  p->k = d->rank_k;
  p->kp = p->k <= 16 ? 16 : (p->k <= 32 ? 32 : (p->k <= 64 ? 64 : 128));
  p->L = d->fft_len ? d->fft_len : 2 * next_pow2(p->M);
  p->log2L = ilog2i(p->L);
  const int win = d->sg_window ? d->sg_window : 2 * (int)std::floor(0.375 * p->M) + 1;
  p->sg_half = (std::min(win, p->M % 2 ? p->M : p->M - 1) - 1) / 2;
  p->in_f64 = d->in_dtype == FKK_IN_F64;
  p->in_elem = p->in_f64 ? 8 : 4;
  p->pad_zero = d->pad_mode == FKK_PAD_ZERO;
  FKK_CUDA_CHECK(cudaSetDevice(d->device));
  FKK_CUDA_CHECK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  p->own_stream = true;
  const int M = p->M, k = p->k, kp = p->kp;
  const int64_t n = d->max_rows;
  p->flags = dalloc<int>(4);
  FKK_CUDA_CHECK(cudaMemset(p->flags, 0, 4 * sizeof(int)));
  FKK_CUDA_CHECK(cudaMallocHost(&p->h_flags, 4 * sizeof(int)));
  p->inv_ref = dalloc<float>((size_t)(M + 31) / 32 * 32);   // zero tail: the raw-cube projection reads 32-channel stages
  FKK_CUDA_CHECK(cudaMemset(p->inv_ref, 0, (size_t)(M + 31) / 32 * 32 * sizeof(float)));
  p->ref64 = dalloc<double>(M);
  // twiddles exp(-2 pi i j / L), fp64 on the host (fp32 copy: full period for the direct path's
  // radix-16 passes; fp64: half period for the basis transforms) and the padding map of the direct
  // path (source channel of each padded sample; reading A3)
  {
    std::vector<float2> t32(p->L);
    std::vector<double2> t64(p->L / 2);
    for (int j = 0; j < p->L; ++j) {
      const double a = -2.0 * M_PI * (double)j / (double)p->L;
      t32[j] = make_float2((float)std::cos(a), (float)std::sin(a));
      if (j < p->L / 2) t64[j] = make_double2(std::cos(a), std::sin(a));
    }
    p->tw32 = dalloc<float2>(p->L);
    p->tw64 = dalloc<double2>(p->L / 2);
    FKK_CUDA_CHECK(cudaMemcpy(p->tw32, t32.data(), t32.size() * sizeof(float2), cudaMemcpyHostToDevice));
    FKK_CUDA_CHECK(cudaMemcpy(p->tw64, t64.data(), t64.size() * sizeof(double2), cudaMemcpyHostToDevice));
    std::vector<int> pm(p->L);
    const int pl = (p->L - M) / 2, period = 2 * (M - 1);
    for (int i = 0; i < p->L; ++i) {
      const int t = i - pl;
      if (t >= 0 && t < M) pm[i] = t;
      else if (p->pad_zero) pm[i] = -1;
      else {   // even reflection without repeating the edge sample, period 2(M-1) (numpy 'reflect')
        int r = t % period;
        if (r < 0) r += period;
        pm[i] = r < M ? r : period - r;
      }
    }
    p->pmap = dalloc<int>(p->L);
    FKK_CUDA_CHECK(cudaMemcpy(p->pmap, pm.data(), pm.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  p->A = dalloc<float>((size_t)n * M);
  if (d->gemm_impl == FKK_GEMM_3XTF32) {
    std::vector<int2> tl;
    std::vector<int> tof;
    // CTA pairs (256 x 256 tiles) when they add no channel padding over 128 x 128 tiles: after the
    // batched fp64 flush they are faster (3.50 vs 3.61 ms at cfg3)
    int mode = ((M + 127) / 128) % 2 == 0 ? 1 : 0;
    // modes: 0 1-CTA image Gram, 1 CTA-pair image Gram, 2 fp32-A 1-CTA Gram (f64 input, loopback shards)
    if (const char* ev = getenv("FKK_GRAM_MODE")) mode = std::min(2, std::max(0, atoi(ev)));   // A/B and tests
    if ((mode == 0 || mode == 1) && (d->in_dtype || d->loopback_shards > 1)) mode = 2;   // image needs fp32, 1 shard
    p->gram_mode = mode;
    p->gtc_pair = mode == 1;
    if (p->gtc_pair) fkk::gram_tc2_tiles(M, tl, tof, p->gtc_nTj);
    else fkk::gram_tc_tiles(M, tl, tof, p->gtc_nTj);
    p->gtc_ntiles = (int)tl.size();
    p->gtc_nsplit = p->gtc_pair ? fkk::gram_tc2_splits(p->gtc_ntiles, n) : fkk::gram_tc_splits(p->gtc_ntiles, n);
    p->gtc_tiles = dalloc<int2>(tl.size());
    p->gtc_tile_of = dalloc<int>(tof.size());
    FKK_CUDA_CHECK(cudaMemcpy(p->gtc_tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice));
    FKK_CUDA_CHECK(cudaMemcpy(p->gtc_tile_of, tof.data(), tof.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (mode <= 1) {
      p->apre_blocks = mode == 1 ? fkk::gram_pre2_image_blocks(M) : (M + 127) / 128;
      // the range finder appends Y (N x 128) as one more image block
      const int extra = d->svd_mode == FKK_SVD_RANGE_FINDER ? 1 : 0;
      p->apre = dalloc<unsigned char>(fkk::gram_pre_bytes(n, p->apre_blocks + extra));
    }
    p->gtc_part = dalloc<double>(p->gtc_pair ? fkk::gram_tc2_partial_doubles(p->gtc_ntiles, p->gtc_nsplit)
                                             : fkk::gram_tc_partial_doubles(p->gtc_ntiles, p->gtc_nsplit));
  } else {
    p->gram_nsplit_cap = fkk::gram_num_splits(n, M);
    p->gram_part = dalloc<double>((size_t)p->gram_nsplit_cap * fkk::gram_num_tiles(M) * 128 * 128);
  }
  p->G = dalloc<double>((size_t)M * M);
  p->colsum = dalloc<double>(M);
  p->f64 = dalloc<double>(M);
  p->f32 = dalloc<float>(M);
  p->V64 = dalloc<double>((size_t)M * k);
  p->W = dalloc<float>((size_t)M * kp);
  p->US = dalloc<float>((size_t)n * kp);   // row stride kp, zero-padded columns
  const int nblk = fkk::project_num_blocks(n);
  p->ext_val = dalloc<float>((size_t)nblk * k * 2);
  p->ext_idx = dalloc<int64_t>((size_t)nblk * k * 2);
  p->ext_out_val = dalloc<float>((size_t)64 * k * 2);
  p->ext_out_idx = dalloc<int64_t>((size_t)64 * k * 2);
  const int nqc = p->nq_cap();
  p->q_dev = dalloc<int64_t>(nqc);
  p->X = dalloc<double>((size_t)nqc * k);
  p->Vt_f = dalloc<double>((size_t)k * M);
  p->Hv = dalloc<double>((size_t)k * M);
  p->P = dalloc<double>((size_t)nqc * M);
  p->Phi_err = dalloc<double>((size_t)nqc * M);
  p->XtX = dalloc<double>((size_t)k * k);
  p->XtPhi = dalloc<double>((size_t)k * M);
  p->Phi_pec = dalloc<double>((size_t)k * M);
  p->HPhi = dalloc<double>((size_t)k * M);
  p->tmp = dalloc<double>((size_t)k * M);
  p->Vsec = dalloc<double>((size_t)k * M);
  p->ridge_work = dalloc<double>((size_t)3 * k * k);
  p->lam = dalloc<double>(1);
  p->Bi = dalloc<float>((size_t)k * M * 2);
  p->bimg = dalloc<float>(fkk::reconstruct_tc_bimg_floats(k, M));
  p->wimg = dalloc<float>(fkk::project_tc_wimg_floats(M, kp));
  p->eig_work = dalloc<double>(fkk::eig_workspace_doubles(M, k));
  p->lam_d = dalloc<double>(k);
  if (d->svd_mode == FKK_SVD_RANGE_FINDER) {
    if (!p->apre) throw Status(FKK_ERR_NOT_IMPLEMENTED, "range finder: needs the pre-split image Gram path");
    const int l = k + d->rf_oversample;
    p->rf_l = l;
    const int nT = (M + 127) / 128;
    std::vector<int2> tl;
    for (int cb = 0; cb < nT; ++cb) tl.push_back(make_int2(cb, p->apre_blocks));
    tl.push_back(make_int2(p->apre_blocks, p->apre_blocks));
    p->rf_tiles = dalloc<int2>(tl.size());
    FKK_CUDA_CHECK(cudaMemcpy(p->rf_tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice));
    p->rf_nsplit = fkk::gram_tc_splits(nT + 1, n);
    p->rf_part = dalloc<double>((size_t)(nT + 1) * p->rf_nsplit * 128 * 128);
    p->rf_omega = dalloc<double>((size_t)l * M);
    std::vector<double> om((size_t)l * M);
    fkk::rf_omega_host(d->rf_seed, M, l, om.data());
    FKK_CUDA_CHECK(cudaMemcpy(p->rf_omega, om.data(), om.size() * sizeof(double), cudaMemcpyHostToDevice));
    p->rf_wimg = dalloc<float>(fkk::project_tc_wimg_floats(M, 128));
    p->rf_Y = dalloc<float>((size_t)n * 128);
    p->rf_Z = dalloc<double>((size_t)l * M);
    p->rf_Zq = dalloc<double>((size_t)l * M);
    p->rf_Z2 = dalloc<double>((size_t)l * M);
    p->rf_SY = dalloc<double>((size_t)l * l);
    p->rf_S = dalloc<double>((size_t)l * l);
    p->rf_T = dalloc<double>((size_t)l * l);
    p->rf_U = dalloc<double>((size_t)l * k);
    p->rf_lam = dalloc<double>(k);
    p->rf_fallback = dalloc<int>(1);
  }
  if (d->nccl_id) {   // (world_size 1 with an id: the NCCL backend over a 1-rank communicator)
    p->use_nccl = true;
    std::string e;
    if (!g_nccl.load(e)) throw Status(FKK_ERR_NCCL, e);
    ncclUniqueId id;
    std::memcpy(&id, d->nccl_id, sizeof(id));
    nccl_check(g_nccl.CommInitRank(&p->comm, d->world_size, id, d->rank), "CommInitRank");
    // control collectives: row counts (8 B) and the per-shard column extremes (shards x k x 2 x 8 B)
    const int shards = std::max(1, d->loopback_shards);
    p->xscratch_bytes = (size_t)(d->world_size + 1) * std::max<size_t>(64, (size_t)shards * k * 2 * sizeof(int64_t));
    p->xscratch = dalloc<unsigned char>(p->xscratch_bytes);
    p->coll.reset(new NcclCollectives(p));
  } else {
    p->coll.reset(new LocalCollectives(p));
  }
}

struct Shard { int64_t row0, rows; };

// Rows of all ranks (global row offset of this rank, global N): step 1 of exchange.h.
void exchange_rows(fkk_plan* p, int64_t n_rows, int64_t& row0, int64_t& n_global) {
  if (p->use_nccl && !p->comm)
    throw Status(FKK_ERR_STATE, "the communicator was aborted by an earlier failure; recreate the plan");
  fkk::exchange_rows(*p->coll, n_rows, &row0, &n_global);
}

void check_cube_args(fkk_plan* p, const void* cube, int64_t n_rows, const void* ref, const void* out) {
  if (!cube && n_rows > 0) throw Status(FKK_ERR_INVALID_ARG, "cube pointer is NULL");
  if (!out && n_rows > 0) throw Status(FKK_ERR_INVALID_ARG, "output pointer is NULL");
  if (!ref) throw Status(FKK_ERR_INVALID_ARG, "reference pointer is NULL");
  if (n_rows < 0 || n_rows > p->d.max_rows) throw Status(FKK_ERR_INVALID_ARG, "n_rows must be in [0, max_rows]");
  if (!aligned16(cube) || !aligned16(out)) throw Status(FKK_ERR_INVALID_ARG, "cube and output must be 16-byte aligned");
}

// F0..F4: log-ratio, Gram (all-reduced), eig -> V64 (device), s (host).
// Gram from the pre-split image (modes 0 / 1): fp64 partials per (tile, split), reduced into G
// (accumulated onto G when `accumulate`)
static void gram_from_image(fkk_plan* p, int64_t n_rows, int64_t nr, bool accumulate, cudaStream_t s) {
  const int M = p->M;
  if (p->gtc_pair) {
    const int ns = std::min(p->gtc_nsplit, fkk::gram_tc2_splits(p->gtc_ntiles, nr));
    fkk::launch_gram_pre2(p->apre, n_rows, p->gtc_tiles, p->gtc_ntiles, ns, p->gtc_part, s);
    fkk::launch_gram_tc2_reduce(p->gtc_part, p->gtc_ntiles, ns, M, p->gtc_tile_of, p->gtc_nTj, p->G, accumulate, s);
  } else {
    const int ns = std::min(p->gtc_nsplit, fkk::gram_tc_splits(p->gtc_ntiles, nr));
    fkk::launch_gram_pre(p->apre, n_rows, p->gtc_tiles, p->gtc_ntiles, ns, p->gtc_part, s);
    fkk::launch_gram_tc_reduce(p->gtc_part, p->gtc_ntiles, ns, M, p->gtc_tile_of, p->gtc_nTj, p->G, accumulate, s);
  }
}

// F2-F4 by the randomized range finder (Halko 2011 Alg. 4.4 + 5.1, as the oracle's
// randomized_svd): Y = A Omega; q times {Z = A^T orth(Y); Y = A orth(Z)}; then with Q = orth(Y):
// B = Q^T A = (A^T Q)^T, B B^T = U~ S^2 U~^T, V = B^T U~ S^-1.  orth(Y) is implicit: A^T Y and Y^T Y
// come out of one image-Gram launch (Y as an extra image block), Y^T Y = R^T R, A^T Q = (A^T Y) R^-1.
void rf_svd(fkk_plan* p, const float* cube, int64_t n_rows) {
  cudaStream_t s = p->stream;
  const int M = p->M, k = p->k, l = p->rf_l, nT = (M + 127) / 128;
  const int64_t nq = (n_rows + 31) / 32;
  unsigned char* yimg = p->apre + (size_t)p->apre_blocks * nq * 2 * 16640;
  FKK_CUDA_CHECK(cudaMemsetAsync(p->rf_fallback, 0, sizeof(int), s));
  // Y = A (D_f Omega)
  fkk::launch_build_wimg(p->rf_omega, p->f64, nullptr, M, l, 128, p->rf_wimg, s);
  fkk::launch_project_tc(cube, n_rows, M, p->rf_wimg, l, 128, p->rf_Y, p->ext_val, p->ext_idx, 0, 0, s, p->inv_ref,
                         (float)p->d.ratio_floor);
  const int q = p->d.rf_power_iters;
  const int ns = std::min(p->rf_nsplit, fkk::gram_tc_splits(nT + 1, std::max<int64_t>(n_rows, 1)));
  for (int it = 0; it <= q; ++it) {
    // A^T Y (nT tiles) and Y^T Y (one tile) from the image, all-reduced over ranks
    fkk::launch_logratio_pre(p->rf_Y, n_rows, 128, 1, p->inv_ref, 0.f, nullptr, yimg, p->flags, s, 1);
    fkk::launch_gram_pre(p->apre, n_rows, p->rf_tiles, nT + 1, ns, p->rf_part, s);
    fkk::launch_rf_reduce(p->rf_part, nT, ns, M, l, p->f64, p->rf_Z, p->rf_SY, s);
    p->coll->allreduce_sum_f64(p->rf_Z, (size_t)l * M);
    p->coll->allreduce_sum_f64(p->rf_SY, (size_t)l * l);
    // Zq = A^T Q = (A^T Y) R^-1 with Y^T Y = R^T R
    fkk::launch_chol_rinv(p->rf_SY, l, p->rf_T, p->rf_fallback, s);
    fkk::launch_apply_rinv(p->rf_Z, M, l, p->rf_T, p->rf_Zq, s);
    if (it == q) break;
    // power iteration: Y = A (D_f orth(Zq)), orth by CholQR2
    fkk::launch_gram_rows(p->rf_Zq, M, l, p->rf_S, s);
    fkk::launch_chol_rinv(p->rf_S, l, p->rf_T, p->rf_fallback, s);
    fkk::launch_apply_rinv(p->rf_Zq, M, l, p->rf_T, p->rf_Z2, s);
    fkk::launch_gram_rows(p->rf_Z2, M, l, p->rf_S, s);
    fkk::launch_chol_rinv(p->rf_S, l, p->rf_T, p->rf_fallback, s);
    fkk::launch_apply_rinv(p->rf_Z2, M, l, p->rf_T, p->rf_Zq, s);
    fkk::launch_build_wimg(p->rf_Zq, p->f64, nullptr, M, l, 128, p->rf_wimg, s);
    fkk::launch_project_tc(cube, n_rows, M, p->rf_wimg, l, 128, p->rf_Y, p->ext_val, p->ext_idx, 0, 0, s, p->inv_ref,
                           (float)p->d.ratio_floor);
  }
  p->mark("range_finder");
  // B B^T = Zq^T Zq (l x l); its top-k eigenpairs; V = Zq U diag(1/sigma), sign rule
  fkk::launch_gram_rows(p->rf_Zq, M, l, p->rf_S, s);
  fkk::launch_eig_topk(p->rf_S, l, k, p->eig_work, p->rf_U, p->rf_lam, p->flags, s);
  fkk::launch_rf_combine(p->rf_Zq, M, l, p->rf_U, p->rf_lam, k, p->V64, s);
  FKK_CUDA_CHECK(cudaMemcpyAsync(p->lam_d, p->rf_lam, k * sizeof(double), cudaMemcpyDeviceToDevice, s));
  std::vector<double> hl(k);
  int hfb = 0;
  FKK_CUDA_CHECK(cudaMemcpyAsync(hl.data(), p->rf_lam, k * sizeof(double), cudaMemcpyDeviceToHost, s));
  FKK_CUDA_CHECK(cudaMemcpyAsync(&hfb, p->rf_fallback, sizeof(int), cudaMemcpyDeviceToHost, s));
  p->check_flags_sync(true);
  if (hfb) throw Status(FKK_ERR_NUMERICAL, "range finder: CholQR met a numerically rank-deficient block (lower k + oversample)");
  p->h_s.assign(k, 0.0);
  for (int i = 0; i < k; ++i) {
    if (!std::isfinite(hl[i])) throw Status(FKK_ERR_NUMERICAL, "range finder produced a non-finite singular value");
    p->h_s[i] = std::sqrt(std::max(hl[i], 0.0));
  }
  p->mark("eig");
}

void svd_stage(fkk_plan* p, const void* d_icars, int64_t n_rows, const void* d_iref, int64_t n_global) {
  cudaStream_t s = p->stream;
  const int M = p->M, k = p->k;
  fkk::launch_prep_ref(d_iref, p->in_f64, M, p->inv_ref, p->ref64, p->flags, s);
  const bool pre = p->apre != nullptr;
  // with the pre-split Gram and the TMA projection, A0 is never materialised: the projection forms it
  // from the cube in its converter warps (saves writing and re-reading N x M fp32)
  p->a0_raw = pre && !p->in_f64 && p->d.gemm_impl == FKK_GEMM_3XTF32 && fkk::project_raw_ok(M, p->kp) && !getenv("FKK_A0_STORE");
  if (pre)
    fkk::launch_logratio_pre(static_cast<const float*>(d_icars), n_rows, M, p->apre_blocks, p->inv_ref,
                             (float)p->d.ratio_floor, p->a0_raw ? nullptr : p->A, p->apre, p->flags, s);
  else
    fkk::launch_logratio(d_icars, p->in_f64, n_rows, M, p->inv_ref, p->ref64, (float)p->d.ratio_floor, p->A, p->flags, s);
  if (p->d.f_mode == FKK_F_EQ9) {
    FKK_CUDA_CHECK(cudaMemsetAsync(p->colsum, 0, M * sizeof(double), s));
    fkk::launch_colsum(d_icars, p->in_f64, n_rows, M, p->colsum, s);
    p->coll->allreduce_sum_f64(p->colsum, M);
    fkk::launch_noise_scale_from_sums(p->colsum, M, 1.0 / (double)std::max<int64_t>(n_global, 1), p->d.f_alpha, p->d.f_sigma_g, p->f64, p->f32, s);
  } else {
    fkk::launch_fill(p->f64, 1.0, M, s);
    fkk::launch_fill_f(p->f32, 1.0f, M, s);
  }
  p->mark("logratio");
  if (p->d.svd_mode == FKK_SVD_RANGE_FINDER) {
    rf_svd(p, static_cast<const float*>(d_icars), n_rows);
    return;
  }
  // Gram: per (virtual) shard in rank order, fp64 partial sums
  const int shards = std::max(1, p->d.loopback_shards);
  for (int sh = 0; sh < shards; ++sh) {
    int64_t r0, r1;
    fkk_shard_range(n_rows, shards, sh, &r0, &r1);
    if (p->d.gemm_impl == FKK_GEMM_3XTF32) {
      const int64_t nr = std::max<int64_t>(r1 - r0, 1);
      if (pre) {
        gram_from_image(p, n_rows, nr, sh > 0, s);
      } else {
        const int ns = std::min(p->gtc_nsplit, fkk::gram_tc_splits(p->gtc_ntiles, nr));
        fkk::launch_gram_tc(p->A + r0 * (int64_t)M, r1 - r0, M, p->gtc_tiles, p->gtc_ntiles, ns, p->gtc_part, s);
        fkk::launch_gram_tc_reduce(p->gtc_part, p->gtc_ntiles, ns, M, p->gtc_tile_of, p->gtc_nTj, p->G, sh > 0, s);
      }
    } else {
      const int ns = std::min(p->gram_nsplit_cap, fkk::gram_num_splits(std::max<int64_t>(r1 - r0, 1), M));
      fkk::launch_gram_simt(p->A + r0 * (int64_t)M, r1 - r0, M, p->gram_part, ns, s);
      fkk::launch_gram_reduce(p->gram_part, ns, M, p->G, sh > 0, s);
    }
  }
  p->coll->allreduce_sum_f64(p->G, (size_t)M * M);
  if (p->d.f_mode == FKK_F_EQ9) fkk::launch_scale_gram(p->G, p->f64, M, s);
  p->mark("gram");
  // eig on the GPU (fp64): Householder tridiagonalisation, bisection, inverse iteration
  fkk::launch_eig_topk(p->G, M, k, p->eig_work, p->V64, p->lam_d, p->flags, s);
  std::vector<double> hl(k);
  FKK_CUDA_CHECK(cudaMemcpyAsync(hl.data(), p->lam_d, k * sizeof(double), cudaMemcpyDeviceToHost, s));
  p->check_flags_sync(true);
  p->h_s.assign(k, 0.0);
  for (int i = 0; i < k; ++i) {
    if (!std::isfinite(hl[i])) throw Status(FKK_ERR_NUMERICAL, "eigensolver produced a non-finite eigenvalue");
    p->h_s[i] = std::sqrt(std::max(hl[i], 0.0));
  }
  p->mark("eig");
}

// F5..F11 given V64 (device) and s (host); q computed unless given (h_q != nullptr).
void transform_rest(fkk_plan* p, const void* cube, int64_t n_rows, int64_t row0, const int64_t* h_q_in, int nq_in,
                    void* d_out) {
  cudaStream_t s = p->stream;
  const int M = p->M, k = p->k, kp = p->kp;
  // W = D_f V (fp32 for the CUDA-core variant; a tf32 hi/lo W^T image for the tensor cores)
  const bool tcg = p->d.gemm_impl == FKK_GEMM_3XTF32;
  if (tcg) fkk::launch_build_wimg(p->V64, p->f64, nullptr, M, k, kp, p->wimg, s);
  else fkk::launch_cast_w(p->V64, p->f64, nullptr, M, k, kp, p->W, s);
  const int shards = std::max(1, p->d.loopback_shards);
  std::vector<float> hv;
  std::vector<int64_t> hi;
  for (int sh = 0; sh < shards; ++sh) {
    int64_t r0, r1;
    fkk_shard_range(n_rows, shards, sh, &r0, &r1);
    if (tcg && p->a0_raw)
      fkk::launch_project_tc(static_cast<const float*>(cube) + r0 * (int64_t)M, r1 - r0, M, p->wimg, k, kp,
                             p->US + r0 * (int64_t)kp, p->ext_val, p->ext_idx, row0 + r0, 1, s, p->inv_ref,
                             (float)p->d.ratio_floor);
    else if (tcg)
      fkk::launch_project_tc(p->A + r0 * (int64_t)M, r1 - r0, M, p->wimg, k, kp, p->US + r0 * (int64_t)kp, p->ext_val,
                             p->ext_idx, row0 + r0, 1, s);
    else
      fkk::launch_project_simt(p->A + r0 * (int64_t)M, r1 - r0, M, p->W, k, kp, p->US + r0 * (int64_t)kp, p->ext_val,
                               p->ext_idx, row0 + r0, s);
    if (r1 > r0)
      fkk::launch_extremes_reduce(p->ext_val, p->ext_idx, fkk::project_num_blocks(r1 - r0), k,
                                  p->ext_out_val + (size_t)sh * k * 2, p->ext_out_idx + (size_t)sh * k * 2, s);
    else {
      std::vector<float> ev(k * 2);
      std::vector<int64_t> ei(k * 2, INT64_MAX);
      for (int c = 0; c < k; ++c) { ev[2 * c] = -INFINITY; ev[2 * c + 1] = INFINITY; }
      FKK_CUDA_CHECK(cudaMemcpyAsync(p->ext_out_val + (size_t)sh * k * 2, ev.data(), ev.size() * 4, cudaMemcpyHostToDevice, s));
      FKK_CUDA_CHECK(cudaMemcpyAsync(p->ext_out_idx + (size_t)sh * k * 2, ei.data(), ei.size() * 8, cudaMemcpyHostToDevice, s));
      FKK_CUDA_CHECK(cudaStreamSynchronize(s));
    }
  }
  p->mark("project");
  std::vector<int64_t> q;
  if (h_q_in) {
    q.assign(h_q_in, h_q_in + nq_in);
  } else {
    // merge the per-shard (and per-rank) extremes into q (reading A12; step 4 of exchange.h)
    const size_t per = (size_t)k * 2;
    hv.resize(per * shards);
    hi.resize(per * shards);
    FKK_CUDA_CHECK(cudaMemcpyAsync(hv.data(), p->ext_out_val, hv.size() * 4, cudaMemcpyDeviceToHost, s));
    FKK_CUDA_CHECK(cudaMemcpyAsync(hi.data(), p->ext_out_idx, hi.size() * 8, cudaMemcpyDeviceToHost, s));
    FKK_CUDA_CHECK(cudaStreamSynchronize(s));
    q = fkk::exchange_extremes(*p->coll, hv.data(), hi.data(), shards, k);
  }
  const int nq = (int)q.size();
  if (nq < 1 || nq > p->nq_cap()) throw Status(FKK_ERR_INVALID_ARG, "q must have 1..2k entries");
  p->h_q = q;
  // X = US[q] (rows owned by this rank; others contribute zeros and are summed over ranks)
  const std::vector<int64_t> ql = fkk::local_rows(q, row0, n_rows);   // step 5 of exchange.h
  FKK_CUDA_CHECK(cudaMemcpyAsync(p->q_dev, ql.data(), nq * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  fkk::launch_gather_rows(p->US, k, kp, p->q_dev, nq, p->X, s);
  FKK_CUDA_CHECK(cudaStreamSynchronize(s));   // ql is a host vector
  p->coll->allreduce_sum_f64(p->X, (size_t)nq * k);
  p->mark("select_q");
  // ---- basis (F6..F10), fp64
  fkk::launch_vt_over_f(p->V64, p->f64, M, k, p->Vt_f, s);
  fkk::launch_hilbert_rows_f64(p->Vt_f, k, M, M, p->Hv, p->L, p->pad_zero, p->tw64, s);          // Eq. 11
  fkk::launch_dgemm_small(nq, M, k, p->X, k, 0, p->Hv, M, 0, p->P, M, 0.0, s);                    // Eq. 16 argument
  fkk::launch_als_rows(p->P, 1, nq, M, p->d.als_lambda, p->d.als_p, p->d.als_iters, p->Phi_err, 1, s);                                                         // D{.}
  fkk::launch_dgemm_small(k, k, nq, p->X, k, 1, p->X, k, 0, p->XtX, k, 0.0, s);                   // X^T X
  fkk::launch_dgemm_small(k, M, nq, p->X, k, 1, p->Phi_err, M, 0, p->XtPhi, M, 0.0, s);           // X^T Phi_err
  fkk::launch_ridge(p->XtX, k, p->XtPhi, M, p->d.ridge_rel, p->Phi_pec, p->lam, p->ridge_work, p->flags, s);  // Eq. 17
  fkk::launch_hilbert_rows_f64(p->Phi_pec, k, M, M, p->HPhi, p->L, p->pad_zero, p->tw64, s);      // Eq. 18
  fkk::launch_add_f64(p->Vt_f, p->HPhi, p->tmp, (int64_t)k * M, s);
  fkk::launch_sg_rows_f64(p->tmp, k, M, p->sg_half, p->Vsec, s);                                  // Eq. 22
  fkk::launch_assemble_B(p->Vt_f, p->HPhi, p->Vsec, p->Hv, p->Phi_pec, k, M, p->Bi, s);           // Eq. 23
  if (p->d.gemm_impl == FKK_GEMM_3XTF32) fkk::launch_build_bimg(p->Bi, k, M, p->bimg, s);
  p->mark("basis");
  // ---- reconstruction (F11)
  if (p->d.gemm_impl == FKK_GEMM_3XTF32)
    fkk::launch_reconstruct_tc(p->US, n_rows, k, kp, p->bimg, M, d_out, p->d.out_layout == FKK_OUT_IMAG_F32, s);
  else
    fkk::launch_reconstruct_simt(p->US, n_rows, k, kp, p->Bi, M, d_out, p->d.out_layout == FKK_OUT_IMAG_F32, s);
  p->mark("reconstruct");
  p->last_rows = n_rows;
  p->last_row0 = row0;
  p->have_transform = true;
}

fkk_basis* export_basis(fkk_plan* p) {
  auto b = std::make_unique<fkk_basis>();
  cudaStream_t s = p->stream;
  const int M = p->M, k = p->k, kp = p->kp;
  b->M = M; b->k = k; b->kp = kp; b->L = p->L; b->pad = p->pad_zero; b->device = p->d.device;
  b->ratio_floor = p->d.ratio_floor;
  b->s = p->h_s;
  b->inv_ref = dalloc<float>(M);
  b->ref64 = dalloc<double>(M);
  b->f64 = dalloc<double>(M);
  b->W = dalloc<float>((size_t)M * kp);
  b->Bi = dalloc<float>((size_t)k * M * 2);
  b->V64 = dalloc<double>((size_t)M * k);
  b->bimg = dalloc<float>(fkk::reconstruct_tc_bimg_floats(k, M));
  if (p->d.gemm_impl == FKK_GEMM_3XTF32) {
    FKK_CUDA_CHECK(cudaMemcpyAsync(b->bimg, p->bimg, fkk::reconstruct_tc_bimg_floats(k, M) * sizeof(float),
                                   cudaMemcpyDeviceToDevice, s));
    b->bimg_valid = true;
  }
  FKK_CUDA_CHECK(cudaMemcpyAsync(b->inv_ref, p->inv_ref, M * sizeof(float), cudaMemcpyDeviceToDevice, s));
  FKK_CUDA_CHECK(cudaMemcpyAsync(b->ref64, p->ref64, M * sizeof(double), cudaMemcpyDeviceToDevice, s));
  FKK_CUDA_CHECK(cudaMemcpyAsync(b->f64, p->f64, M * sizeof(double), cudaMemcpyDeviceToDevice, s));
  FKK_CUDA_CHECK(cudaMemcpyAsync(b->Bi, p->Bi, (size_t)k * M * 2 * sizeof(float), cudaMemcpyDeviceToDevice, s));
  FKK_CUDA_CHECK(cudaMemcpyAsync(b->V64, p->V64, (size_t)M * k * sizeof(double), cudaMemcpyDeviceToDevice, s));
  // W_ml = D_f V diag(s^2/(s^2 + lam_ml)), lam_ml = ml_ridge_rel * s_1^2 (Eq. 25 closed form)
  std::vector<double> c(k);
  const double lam_ml = p->d.ml_ridge_rel * (k > 0 ? p->h_s[0] * p->h_s[0] : 0.0);
  for (int i = 0; i < k; ++i) {
    const double s2 = p->h_s[i] * p->h_s[i];
    c[i] = s2 + lam_ml > 0 ? s2 / (s2 + lam_ml) : 0.0;
  }
  double* dc = dalloc<double>(k);
  FKK_CUDA_CHECK(cudaMemcpyAsync(dc, c.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  fkk::launch_cast_w(p->V64, p->f64, dc, M, k, kp, b->W, s);
  b->wimg = dalloc<float>(fkk::project_tc_wimg_floats(M, kp));
  fkk::launch_build_wimg(p->V64, p->f64, dc, M, k, kp, b->wimg, s);
  FKK_CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(dc);
  return b.release();
}

fkk_status fail(fkk_plan* p, int code, const std::string& msg) {
  if (p) p->err = msg;
  return (fkk_status)code;
}

template <typename F>
fkk_status guarded(fkk_plan* p, F&& f) {
  if (!p) return FKK_ERR_INVALID_ARG;
  try {
    p->err.clear();
    f();
    return FKK_OK;
  } catch (const Status& e) {
    p->nvtx_pop_all();
    return fail(p, e.code, e.what());
  } catch (const std::exception& e) {
    p->nvtx_pop_all();
    return fail(p, FKK_ERR_STATE, e.what());
  }
}

void direct_run(fkk_plan* p, const void* d_icars, int64_t n_rows, const void* d_iref, void* d_out) {
  cudaStream_t s = p->stream;
  const int M = p->M;
  if (p->L > 4096) throw Status(FKK_ERR_NOT_IMPLEMENTED, "direct path: FFT length above 4096 (M <= 2048)");
  p->ensure_direct();
  fkk::launch_prep_ref(d_iref, p->in_f64, M, p->inv_ref, p->ref64, p->flags, s);
  const size_t oel = p->d.out_layout == FKK_OUT_IMAG_F32 ? 4 : 8;
  for (int64_t b0 = 0; b0 < n_rows; b0 += p->direct_batch) {
    const int64_t nb = std::min<int64_t>(p->direct_batch, n_rows - b0);
    const char* in = static_cast<const char*>(d_icars) + (size_t)b0 * M * p->in_elem;
    char* out = static_cast<char*>(d_out) + (size_t)b0 * M * oel;
    fkk::launch_direct_phase(in, p->in_f64, nb, M, p->inv_ref, p->ref64, (float)p->d.ratio_floor, p->L, p->tw32,
                             p->pmap, p->phi, p->flags, s);
    p->mark("kk_phase");
    fkk::launch_als_rows(p->phi, 0, nb, M, p->d.als_lambda, p->d.als_p, p->d.als_iters, p->phierr, 0, s, p->als_solves, p->als_ctr);
    p->mark("als");
    fkk::launch_direct_finish(in, p->in_f64, nb, M, p->inv_ref, p->ref64, (float)p->d.ratio_floor, p->L, p->tw32,
                              p->pmap, p->phi, p->phierr, p->sg_half, out, p->d.out_layout == FKK_OUT_IMAG_F32, s);
    p->mark("pec_sec");
  }
}

void apply_run(fkk_plan* p, fkk_basis* b, const void* d_icars, int64_t n_rows, void* d_out) {
  if (b->M != p->M || b->L != p->L || b->pad != p->pad_zero || b->k > p->k)
    throw Status(FKK_ERR_INCOMPATIBLE_BASIS, "trained basis M/L/pad/k incompatible with the plan");
  cudaStream_t s = p->stream;
  const int M = p->M;
  const bool tcg = p->d.gemm_impl == FKK_GEMM_3XTF32;
  if (tcg && !p->in_f64 && fkk::project_raw_ok(M, b->kp)) {
    // F12 as two streaming kernels: the projection forms A0 = 1/2 ln(max(I/I_ref, floor)) from the raw
    // cube in its converter warps (no A0 round trip through HBM), US_new = A0 W (W = D_f V diag(s^2 /
    // (s^2 + lam_ml)), Eq. 25), then the reconstruction with the trained B (Eq. 23)
    fkk::launch_project_tc(static_cast<const float*>(d_icars), n_rows, M, b->wimg, b->k, b->kp, p->US, p->ext_val,
                           p->ext_idx, 0, 0, s, b->inv_ref, (float)b->ratio_floor);
    p->mark("project");
  } else {
    fkk::launch_logratio(d_icars, p->in_f64, n_rows, M, b->inv_ref, b->ref64, (float)b->ratio_floor, p->A, p->flags, s);
    p->mark("logratio");
    if (tcg)
      fkk::launch_project_tc(p->A, n_rows, M, b->wimg, b->k, b->kp, p->US, p->ext_val, p->ext_idx, 0, 0, s);
    else
      fkk::launch_project_simt(p->A, n_rows, M, b->W, b->k, b->kp, p->US, p->ext_val, p->ext_idx, 0, s);
    p->mark("project");
  }
  if (tcg) {
    if (!b->bimg_valid) { fkk::launch_build_bimg(b->Bi, b->k, M, b->bimg, s); b->bimg_valid = true; }
    fkk::launch_reconstruct_tc(p->US, n_rows, b->k, b->kp, b->bimg, M, d_out, p->d.out_layout == FKK_OUT_IMAG_F32, s);
  } else {
    fkk::launch_reconstruct_simt(p->US, n_rows, b->k, b->kp, b->Bi, M, d_out, p->d.out_layout == FKK_OUT_IMAG_F32, s);
  }
  p->mark("reconstruct");
}

void* ensure_dev(void*& buf, size_t& have, size_t need) {
  if (have < need) {
    if (buf) cudaFree(buf);
    buf = dalloc<char>(need);
    have = need;
  }
  return buf;
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------------
extern "C" {

void fkk_plan_desc_init(fkk_plan_desc* d, int32_t n_freq, int32_t rank_k, int64_t max_rows) {
  if (!d) return;
  std::memset(d, 0, sizeof(*d));
  d->n_freq = n_freq;
  d->rank_k = rank_k;
  d->max_rows = max_rows;
  d->fft_len = 0;
  d->pad_mode = FKK_PAD_REFLECT;
  d->ratio_floor = 1e-6;
  d->f_mode = FKK_F_ONE;
  d->f_alpha = 0.0;
  d->f_sigma_g = 1.0;
  d->als_lambda = 1e4;
  d->als_p = 1e-3;
  d->als_iters = 10;
  d->sg_window = 0;
  d->sg_order = 2;
  d->ridge_rel = 1e-3;
  d->ml_ridge_rel = 0.0;
  d->gemm_impl = FKK_GEMM_3XTF32;
  d->out_layout = FKK_OUT_COMPLEX64;
  d->in_dtype = FKK_IN_F32;
  d->device = 0;
  d->world_size = 1;
  d->rank = 0;
  d->nccl_id = nullptr;
  d->loopback_shards = 0;
  d->svd_mode = FKK_SVD_GRAM;
  d->rf_oversample = 10;
  d->rf_power_iters = 1;
  d->rf_seed = 0;
}

fkk_status fkk_get_nccl_unique_id(uint8_t out[128]) {
  if (!out) return FKK_ERR_INVALID_ARG;
  std::string e;
  if (!g_nccl.load(e)) return FKK_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return FKK_ERR_NCCL;
  std::memcpy(out, &id, 128);
  return FKK_OK;
}

static thread_local std::string g_create_err;

fkk_status fkk_plan_create(const fkk_plan_desc* d, fkk_plan_t* out) {
  if (!out) return FKK_ERR_INVALID_ARG;
  *out = nullptr;
  auto p = std::make_unique<fkk_plan>();
  try {
    create_plan(d, p.get());
  } catch (const Status& e) {
    g_create_err = e.what();
    return (fkk_status)e.code;
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return FKK_ERR_STATE;
  }
  *out = p.release();
  return FKK_OK;
}

fkk_status fkk_plan_destroy(fkk_plan_t p) {
  delete p;
  return FKK_OK;
}

const char* fkk_last_error(fkk_plan_t p) { return p ? p->err.c_str() : g_create_err.c_str(); }

fkk_status fkk_plan_set_stream(fkk_plan_t p, void* cuda_stream) {
  return guarded(p, [&] {
    if (p->stream == static_cast<cudaStream_t>(cuda_stream) && !p->own_stream) return;
    if (p->own_stream && p->stream) { FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream)); cudaStreamDestroy(p->stream); }
    // NULL selects the legacy default stream (what torch's default stream handle 0 denotes)
    p->stream = static_cast<cudaStream_t>(cuda_stream);
    p->own_stream = false;
  });
}

fkk_status fkk_plan_sync(fkk_plan_t p) {
  return guarded(p, [&] { p->check_flags_sync(); });
}

fkk_status fkk_svd(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref, float* d_V_out,
                   double* h_s_out) {
  return guarded(p, [&] {
    check_cube_args(p, d_icars, n_rows, d_iref, d_V_out);
    if (!h_s_out) throw Status(FKK_ERR_INVALID_ARG, "h_s_out is NULL");
    p->begin_call("fkk_svd");
    int64_t row0, ng;
    exchange_rows(p, n_rows, row0, ng);
    if (ng < p->k) throw Status(FKK_ERR_INVALID_ARG, "rank_k exceeds the global number of spectra");
    svd_stage(p, d_icars, n_rows, d_iref, ng);
    // fp32 column-major copy of V (the f-unscaled right singular vectors)
    std::vector<double> hv((size_t)p->M * p->k);
    FKK_CUDA_CHECK(cudaMemcpyAsync(hv.data(), p->V64, hv.size() * 8, cudaMemcpyDeviceToHost, p->stream));
    FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream));
    std::vector<float> hf(hv.begin(), hv.end());
    FKK_CUDA_CHECK(cudaMemcpyAsync(d_V_out, hf.data(), hf.size() * 4, cudaMemcpyHostToDevice, p->stream));
    FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream));
    std::copy(p->h_s.begin(), p->h_s.end(), h_s_out);
    p->end_call();
  });
}

fkk_status fkk_transform(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref, void* d_out,
                         fkk_basis_t* basis_out) {
  return guarded(p, [&] {
    check_cube_args(p, d_icars, n_rows, d_iref, d_out);
    if (basis_out) *basis_out = nullptr;
    p->begin_call("fkk_transform");
    int64_t row0, ng;
    exchange_rows(p, n_rows, row0, ng);
    if (ng < p->k) throw Status(FKK_ERR_INVALID_ARG, "rank_k exceeds the global number of spectra");
    p->last_global_rows = ng;
    svd_stage(p, d_icars, n_rows, d_iref, ng);
    transform_rest(p, d_icars, n_rows, row0, nullptr, 0, d_out);
    p->check_flags_sync(true);
    if (basis_out) *basis_out = export_basis(p);
    p->end_call();
  });
}

fkk_status fkk_transform_from(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref, const float* d_V,
                              const double* h_s, const int64_t* h_q, int32_t nq, void* d_out) {
  return guarded(p, [&] {
    check_cube_args(p, d_icars, n_rows, d_iref, d_out);
    if (!d_V || !h_s || !h_q || nq < 1 || nq > p->nq_cap()) throw Status(FKK_ERR_INVALID_ARG, "bad V/s/q");
    p->begin_call("fkk_transform_from");
    int64_t row0, ng;
    exchange_rows(p, n_rows, row0, ng);
    cudaStream_t s = p->stream;
    const int M = p->M, k = p->k;
    fkk::launch_prep_ref(d_iref, p->in_f64, M, p->inv_ref, p->ref64, p->flags, s);
    fkk::launch_logratio(d_icars, p->in_f64, n_rows, M, p->inv_ref, p->ref64, (float)p->d.ratio_floor, p->A, p->flags, s);
    p->a0_raw = false;   // A0 materialised here
    if (p->d.f_mode == FKK_F_EQ9) {
      FKK_CUDA_CHECK(cudaMemsetAsync(p->colsum, 0, M * sizeof(double), s));
      fkk::launch_colsum(d_icars, p->in_f64, n_rows, M, p->colsum, s);
      p->coll->allreduce_sum_f64(p->colsum, M);
      fkk::launch_noise_scale_from_sums(p->colsum, M, 1.0 / (double)std::max<int64_t>(ng, 1), p->d.f_alpha, p->d.f_sigma_g, p->f64, p->f32, s);
    } else {
      fkk::launch_fill(p->f64, 1.0, M, s);
      fkk::launch_fill_f(p->f32, 1.0f, M, s);
    }
    std::vector<float> hv((size_t)M * k);
    FKK_CUDA_CHECK(cudaMemcpyAsync(hv.data(), d_V, hv.size() * 4, cudaMemcpyDeviceToHost, s));
    FKK_CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<double> hd(hv.begin(), hv.end());
    FKK_CUDA_CHECK(cudaMemcpyAsync(p->V64, hd.data(), hd.size() * 8, cudaMemcpyHostToDevice, s));
    FKK_CUDA_CHECK(cudaStreamSynchronize(s));
    p->h_s.assign(h_s, h_s + k);
    transform_rest(p, d_icars, n_rows, row0, h_q, nq, d_out);
    p->check_flags_sync(true);
    p->end_call();
  });
}

fkk_status fkk_apply_trained_basis(fkk_plan_t p, fkk_basis_t b, const void* d_icars, int64_t n_rows, void* d_out) {
  return guarded(p, [&] {
    if (!b) throw Status(FKK_ERR_INVALID_ARG, "basis is NULL");
    check_cube_args(p, d_icars, n_rows, b->ref64, d_out);
    p->begin_call("fkk_apply_trained_basis");
    apply_run(p, b, d_icars, n_rows, d_out);
    p->end_call();
  });
}

fkk_status kk_direct_batch(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref, void* d_out) {
  return guarded(p, [&] {
    check_cube_args(p, d_icars, n_rows, d_iref, d_out);
    p->begin_call("kk_direct_batch");
    direct_run(p, d_icars, n_rows, d_iref, d_out);
    p->end_call();
  });
}

// Conventional workflow with SVD denoise (Fig. 1(a); reading A26):
// rank-k_keep SVD of the RAW cube through the same pre-split Gram + GPU eigensolver + TMA projection, the
// denoised cube I_k = US . V^T by the reconstruction GEMM in linear mode (into the plan's N x M
// workspace), then the direct KK + PEC + SEC of every denoised spectrum.  Local (single rank).
fkk_status fkk_conventional(fkk_plan_t p, const void* d_icars, int64_t n_rows, const void* d_iref, int32_t k_keep,
                            void* d_out) {
  return guarded(p, [&] {
    check_cube_args(p, d_icars, n_rows, d_iref, d_out);
    if (k_keep < 1 || k_keep > p->k) throw Status(FKK_ERR_INVALID_ARG, "k_keep must be in [1, rank_k]");
    if (p->in_f64 || !p->apre || p->d.gemm_impl != FKK_GEMM_3XTF32 || p->d.world_size != 1 ||
        !fkk::project_raw_ok(p->M, p->kp))
      throw Status(FKK_ERR_NOT_IMPLEMENTED,
                   "conventional workflow: f32 input, tensor-core path (pre-split Gram, TMA projection), one rank");
    if (n_rows < 1) throw Status(FKK_ERR_INVALID_ARG, "n_rows must be >= 1");
    p->begin_call("fkk_conventional");
    cudaStream_t s = p->stream;
    const int M = p->M, k = p->k, kp = p->kp;
    fkk::launch_prep_ref(d_iref, p->in_f64, M, p->inv_ref, p->ref64, p->flags, s);
    // Gram of the raw cube (image with raw = 1) and the eigensolver
    fkk::launch_logratio_pre(static_cast<const float*>(d_icars), n_rows, M, p->apre_blocks, p->inv_ref,
                             (float)p->d.ratio_floor, nullptr, p->apre, p->flags, s, 1);
    gram_from_image(p, n_rows, n_rows, false, s);
    p->mark("gram");
    fkk::launch_eig_topk(p->G, M, k, p->eig_work, p->V64, p->lam_d, p->flags, s);
    p->check_flags_sync();
    p->mark("eig");
    // US = I V_k (the projection on the raw cube, no log), I_k = US V_k^T (linear reconstruction)
    fkk::launch_fill(p->f64, 1.0, M, s);
    fkk::launch_build_wimg(p->V64, p->f64, nullptr, M, k_keep, kp, p->wimg, s);
    fkk::launch_project_tc(static_cast<const float*>(d_icars), n_rows, M, p->wimg, k_keep, kp, p->US, p->ext_val,
                           p->ext_idx, 0, 0, s);
    fkk::launch_bi_linear(p->V64, k_keep, M, p->Bi, s);
    fkk::launch_build_bimg(p->Bi, k_keep, M, p->bimg, s);
    fkk::launch_reconstruct_tc(p->US, n_rows, k_keep, kp, p->bimg, M, p->A, 2, s);
    p->mark("denoise");
    // conventional KK + PEC + SEC on the denoised cube
    direct_run(p, p->A, n_rows, d_iref, d_out);
    p->end_call();
  });
}

fkk_status fkk_transform_host(fkk_plan_t p, const void* h_icars, int64_t n_rows, const void* h_iref, void* h_out,
                              fkk_basis_t* basis_out) {
  return guarded(p, [&] {
    if (!h_icars || !h_iref || !h_out) throw Status(FKK_ERR_INVALID_ARG, "NULL host buffer");
    if (n_rows < 0 || n_rows > p->d.max_rows) throw Status(FKK_ERR_INVALID_ARG, "n_rows must be in [0, max_rows]");
    const size_t in_bytes = (size_t)n_rows * p->M * p->in_elem;
    const size_t out_bytes = (size_t)n_rows * p->M * (p->d.out_layout == FKK_OUT_IMAG_F32 ? 4 : 8);
    void* din = ensure_dev(p->d_in_cube, p->d_in_cube_bytes, in_bytes);
    void* dout = ensure_dev(p->d_out_cube, p->d_out_cube_bytes, out_bytes);
    if (!p->d_ref_buf) p->d_ref_buf = dalloc<double>(p->M);
    FKK_CUDA_CHECK(cudaMemcpyAsync(din, h_icars, in_bytes, cudaMemcpyHostToDevice, p->stream));
    FKK_CUDA_CHECK(cudaMemcpyAsync(p->d_ref_buf, h_iref, (size_t)p->M * p->in_elem, cudaMemcpyHostToDevice, p->stream));
    fkk_status st = fkk_transform(p, din, n_rows, p->d_ref_buf, dout, basis_out);
    if (st != FKK_OK) throw Status(st, p->err);
    FKK_CUDA_CHECK(cudaMemcpyAsync(h_out, dout, out_bytes, cudaMemcpyDeviceToHost, p->stream));
    FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream));
  });
}

// Host cubes streamed through the transform: cube i+1's host->device copy and cube i-1's device->host
// copy (copy streams s_in / s_out, two device buffer pairs) overlap cube i's transform, and cube i's
// device->host copy overlaps cube i+2's host->device copy (the link is full duplex).  Every cube gets
// its own transform (Gram, eigensolve, basis, K), exactly as fkk_transform_host.
fkk_status fkk_transform_host_stream(fkk_plan_t p, const void* const* h_icars, int32_t n_cubes, int64_t n_rows,
                                     const void* h_iref, void* const* h_out, float* h_cube_ms) {
  return guarded(p, [&] {
    if (!h_icars || !h_iref || !h_out || n_cubes < 0) throw Status(FKK_ERR_INVALID_ARG, "NULL argument");
    for (int i = 0; i < n_cubes; ++i)
      if (!h_icars[i] || !h_out[i]) throw Status(FKK_ERR_INVALID_ARG, "NULL host cube");
    if (n_rows < 1 || n_rows > p->d.max_rows) throw Status(FKK_ERR_INVALID_ARG, "n_rows must be in [1, max_rows]");
    const int M = p->M;
    const size_t in_b = (size_t)n_rows * M * p->in_elem;
    const size_t out_b = (size_t)n_rows * M * (p->d.out_layout == FKK_OUT_IMAG_F32 ? 4 : 8);
    if (p->cube_in_bytes < in_b || p->cube_out_bytes < out_b) {
      for (void*& b : p->cube_bufs) if (b) { cudaFree(b); b = nullptr; }
      for (int i = 0; i < 2; ++i) {
        p->cube_bufs[i] = dalloc<char>(in_b);
        p->cube_bufs[2 + i] = dalloc<char>(out_b);
      }
      p->cube_in_bytes = in_b;
      p->cube_out_bytes = out_b;
    }
    if (!p->s_in) FKK_CUDA_CHECK(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
    if (!p->s_out) FKK_CUDA_CHECK(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
    if (!p->d_ref_buf) p->d_ref_buf = dalloc<double>(p->M);
    FKK_CUDA_CHECK(cudaMemcpyAsync(p->d_ref_buf, h_iref, (size_t)M * p->in_elem, cudaMemcpyHostToDevice, p->stream));
    std::vector<cudaEvent_t> ev(4 * (size_t)std::max(n_cubes, 1));
    for (auto& e : ev) FKK_CUDA_CHECK(cudaEventCreate(&e));
    // ev[4i]: H2D start, ev[4i+1]: H2D done, ev[4i+2]: transform done, ev[4i+3]: D2H done
    auto h2d = [&](int i) {
      if (i >= 2) FKK_CUDA_CHECK(cudaStreamWaitEvent(p->s_in, ev[4 * (i - 2) + 2], 0));   // slot's last reader
      FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i], p->s_in));
      FKK_CUDA_CHECK(cudaMemcpyAsync(p->cube_bufs[i & 1], h_icars[i], in_b, cudaMemcpyHostToDevice, p->s_in));
      FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i + 1], p->s_in));
    };
    try {
      if (n_cubes > 0) h2d(0);
      for (int i = 0; i < n_cubes; ++i) {
        if (i + 1 < n_cubes) h2d(i + 1);   // enqueued before the transform blocks the host
        FKK_CUDA_CHECK(cudaStreamWaitEvent(p->stream, ev[4 * i + 1], 0));
        if (i >= 2) FKK_CUDA_CHECK(cudaStreamWaitEvent(p->stream, ev[4 * (i - 2) + 3], 0));   // output slot drained
        const fkk_status st = fkk_transform(p, p->cube_bufs[i & 1], n_rows, p->d_ref_buf, p->cube_bufs[2 + (i & 1)], nullptr);
        if (st != FKK_OK) throw Status(st, p->err);
        FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i + 2], p->stream));
        FKK_CUDA_CHECK(cudaStreamWaitEvent(p->s_out, ev[4 * i + 2], 0));
        FKK_CUDA_CHECK(cudaMemcpyAsync(h_out[i], p->cube_bufs[2 + (i & 1)], out_b, cudaMemcpyDeviceToHost, p->s_out));
        FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i + 3], p->s_out));
      }
      FKK_CUDA_CHECK(cudaStreamSynchronize(p->s_out));
      FKK_CUDA_CHECK(cudaStreamSynchronize(p->s_in));
      FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream));
      if (h_cube_ms)
        for (int i = 0; i < n_cubes; ++i) FKK_CUDA_CHECK(cudaEventElapsedTime(h_cube_ms + i, ev[4 * i], ev[4 * i + 3]));
    } catch (...) {
      cudaStreamSynchronize(p->s_in);
      cudaStreamSynchronize(p->s_out);
      cudaStreamSynchronize(p->stream);
      for (auto& e : ev) cudaEventDestroy(e);
      throw;
    }
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

fkk_status kk_direct_batch_host(fkk_plan_t p, const void* h_icars, int64_t n_rows, const void* h_iref, void* h_out) {
  return guarded(p, [&] {
    if (!h_icars || !h_iref || !h_out) throw Status(FKK_ERR_INVALID_ARG, "NULL host buffer");
    if (n_rows < 0 || n_rows > p->d.max_rows) throw Status(FKK_ERR_INVALID_ARG, "n_rows must be in [0, max_rows]");
    const size_t in_bytes = (size_t)n_rows * p->M * p->in_elem;
    const size_t out_bytes = (size_t)n_rows * p->M * (p->d.out_layout == FKK_OUT_IMAG_F32 ? 4 : 8);
    void* din = ensure_dev(p->d_in_cube, p->d_in_cube_bytes, in_bytes);
    void* dout = ensure_dev(p->d_out_cube, p->d_out_cube_bytes, out_bytes);
    if (!p->d_ref_buf) p->d_ref_buf = dalloc<double>(p->M);
    FKK_CUDA_CHECK(cudaMemcpyAsync(din, h_icars, in_bytes, cudaMemcpyHostToDevice, p->stream));
    FKK_CUDA_CHECK(cudaMemcpyAsync(p->d_ref_buf, h_iref, (size_t)p->M * p->in_elem, cudaMemcpyHostToDevice, p->stream));
    fkk_status st = kk_direct_batch(p, din, n_rows, p->d_ref_buf, dout);
    if (st != FKK_OK) throw Status(st, p->err);
    FKK_CUDA_CHECK(cudaMemcpyAsync(h_out, dout, out_bytes, cudaMemcpyDeviceToHost, p->stream));
    p->check_flags_sync();
  });
}

fkk_status fkk_apply_trained_basis_host(fkk_plan_t p, fkk_basis_t b, const void* h_icars, int64_t n_rows, void* h_out) {
  return guarded(p, [&] {
    if (!b || !h_icars || !h_out) throw Status(FKK_ERR_INVALID_ARG, "NULL argument");
    if (n_rows < 0 || n_rows > p->d.max_rows) throw Status(FKK_ERR_INVALID_ARG, "n_rows must be in [0, max_rows]");
    const size_t in_bytes = (size_t)n_rows * p->M * p->in_elem;
    const size_t out_bytes = (size_t)n_rows * p->M * (p->d.out_layout == FKK_OUT_IMAG_F32 ? 4 : 8);
    void* din = ensure_dev(p->d_in_cube, p->d_in_cube_bytes, in_bytes);
    void* dout = ensure_dev(p->d_out_cube, p->d_out_cube_bytes, out_bytes);
    FKK_CUDA_CHECK(cudaMemcpyAsync(din, h_icars, in_bytes, cudaMemcpyHostToDevice, p->stream));
    fkk_status st = fkk_apply_trained_basis(p, b, din, n_rows, dout);
    if (st != FKK_OK) throw Status(st, p->err);
    FKK_CUDA_CHECK(cudaMemcpyAsync(h_out, dout, out_bytes, cudaMemcpyDeviceToHost, p->stream));
    p->check_flags_sync();
  });
}

// ML apply of a host-resident cube streamed in batches: batch i's host->device copy,
// apply (projection + reconstruction on the plan stream) and device->host copy run on three streams
// with two device buffer pairs, so the copies of neighbouring batches overlap the compute.
// h_batch_ms (nullable): per-batch end-to-end latency, first H2D start to last D2H end.
fkk_status fkk_apply_trained_basis_stream(fkk_plan_t p, fkk_basis_t b, const void* h_icars, int64_t n_rows,
                                          int64_t batch, void* h_out, float* h_batch_ms) {
  return guarded(p, [&] {
    if (!b || !h_icars || !h_out) throw Status(FKK_ERR_INVALID_ARG, "NULL argument");
    if (batch < 1 || batch > p->d.max_rows) throw Status(FKK_ERR_INVALID_ARG, "batch must be in [1, max_rows]");
    if (n_rows < 0) throw Status(FKK_ERR_INVALID_ARG, "n_rows must be >= 0");
    const int M = p->M;
    const size_t oel = p->d.out_layout == FKK_OUT_IMAG_F32 ? 4 : 8;
    const size_t in_b = (size_t)batch * M * p->in_elem, out_b = (size_t)batch * M * oel;
    if (!p->stream_bufs[0]) {
      for (int i = 0; i < 2; ++i) {
        p->stream_bufs[i] = dalloc<char>(in_b);
        p->stream_bufs[2 + i] = dalloc<char>(out_b);
      }
      p->stream_in_bytes = in_b;
      p->stream_out_bytes = out_b;
      FKK_CUDA_CHECK(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
      FKK_CUDA_CHECK(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
    }
    if (p->stream_in_bytes < in_b || p->stream_out_bytes < out_b)
      throw Status(FKK_ERR_INVALID_ARG, "batch larger than the first streaming call's batch");
    p->begin_call("fkk_apply_trained_basis_stream");
    const int64_t nb = (n_rows + batch - 1) / batch;
    std::vector<cudaEvent_t> ev(4 * std::max<int64_t>(nb, 1));
    for (auto& e : ev) FKK_CUDA_CHECK(cudaEventCreate(&e));
    // ev[4i]: H2D start, ev[4i+1]: H2D done, ev[4i+2]: apply done, ev[4i+3]: D2H done
    try {
      for (int64_t i = 0; i < nb; ++i) {
        const int64_t r0 = i * batch, rows = std::min(batch, n_rows - r0);
        const int slot = (int)(i & 1);
        if (i >= 2) {   // the slot's previous batch: its apply read the input, its D2H read the output
          FKK_CUDA_CHECK(cudaStreamWaitEvent(p->s_in, ev[4 * (i - 2) + 2], 0));
        }
        FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i], p->s_in));
        FKK_CUDA_CHECK(cudaMemcpyAsync(p->stream_bufs[slot], static_cast<const char*>(h_icars) + (size_t)r0 * M * p->in_elem,
                                       (size_t)rows * M * p->in_elem, cudaMemcpyHostToDevice, p->s_in));
        FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i + 1], p->s_in));
        FKK_CUDA_CHECK(cudaStreamWaitEvent(p->stream, ev[4 * i + 1], 0));
        if (i >= 2) FKK_CUDA_CHECK(cudaStreamWaitEvent(p->stream, ev[4 * (i - 2) + 3], 0));
        apply_run(p, b, p->stream_bufs[slot], rows, p->stream_bufs[2 + slot]);
        FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i + 2], p->stream));
        FKK_CUDA_CHECK(cudaStreamWaitEvent(p->s_out, ev[4 * i + 2], 0));
        FKK_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(h_out) + (size_t)r0 * M * oel, p->stream_bufs[2 + slot],
                                       (size_t)rows * M * oel, cudaMemcpyDeviceToHost, p->s_out));
        FKK_CUDA_CHECK(cudaEventRecord(ev[4 * i + 3], p->s_out));
      }
      FKK_CUDA_CHECK(cudaStreamSynchronize(p->s_out));
      FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream));
      if (h_batch_ms)
        for (int64_t i = 0; i < nb; ++i) FKK_CUDA_CHECK(cudaEventElapsedTime(h_batch_ms + i, ev[4 * i], ev[4 * i + 3]));
    } catch (...) {
      cudaStreamSynchronize(p->s_in);
      cudaStreamSynchronize(p->s_out);
      cudaStreamSynchronize(p->stream);
      for (auto& e : ev) cudaEventDestroy(e);
      throw;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    p->check_flags_sync();
    p->end_call();
  });
}

fkk_status fkk_basis_destroy(fkk_basis_t b) {
  delete b;
  return FKK_OK;
}

fkk_status fkk_basis_info(fkk_basis_t b, int32_t* n_freq, int32_t* rank_k, int32_t* fft_len) {
  if (!b) return FKK_ERR_INVALID_ARG;
  if (n_freq) *n_freq = b->M;
  if (rank_k) *rank_k = b->k;
  if (fft_len) *fft_len = b->L;
  return FKK_OK;
}

size_t fkk_stage_size(fkk_plan_t p, int32_t stage) {
  if (!p) return 0;
  const size_t M = p->M, k = p->k, nq = p->h_q.size();
  switch (stage) {
    case FKK_STAGE_G: return M * M * 8;
    case FKK_STAGE_S: return k * 8;
    case FKK_STAGE_V: return M * k * 8;
    case FKK_STAGE_US: return (size_t)p->last_rows * k * 4;
    case FKK_STAGE_Q: return nq * 8;
    case FKK_STAGE_HV: case FKK_STAGE_PHI_PEC: case FKK_STAGE_V_SEC: return k * M * 8;
    case FKK_STAGE_PHI_ERR: return nq * M * 8;
    case FKK_STAGE_B: return k * M * 2 * 4;
    case FKK_STAGE_LAMBDA: return 8;
    case FKK_STAGE_F: return M * 8;
    default: return 0;
  }
}

fkk_status fkk_get_stage(fkk_plan_t p, int32_t stage, void* dst, size_t bytes, int32_t dst_is_device) {
  return guarded(p, [&] {
    if (!dst) throw Status(FKK_ERR_INVALID_ARG, "dst is NULL");
    const size_t n = std::min(bytes, fkk_stage_size(p, stage));
    const void* src = nullptr;
    bool host_src = false;
    switch (stage) {
      case FKK_STAGE_G: src = p->G; break;
      case FKK_STAGE_S: src = p->h_s.data(); host_src = true; break;
      case FKK_STAGE_V: src = p->V64; break;
      case FKK_STAGE_US: src = p->US; break;
      case FKK_STAGE_Q: src = p->h_q.data(); host_src = true; break;
      case FKK_STAGE_HV: src = p->Hv; break;
      case FKK_STAGE_PHI_ERR: src = p->Phi_err; break;
      case FKK_STAGE_PHI_PEC: src = p->Phi_pec; break;
      case FKK_STAGE_V_SEC: src = p->Vsec; break;
      case FKK_STAGE_B: src = p->Bi; break;
      case FKK_STAGE_LAMBDA: src = p->lam; break;
      case FKK_STAGE_F: src = p->f64; break;
      default: throw Status(FKK_ERR_INVALID_ARG, "unknown stage");
    }
    cudaMemcpyKind kind = host_src ? (dst_is_device ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost)
                                   : (dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
    if (stage == FKK_STAGE_US) {   // stored with row stride kp
      const size_t rows = n / ((size_t)p->k * 4);
      if (rows) FKK_CUDA_CHECK(cudaMemcpy2DAsync(dst, (size_t)p->k * 4, src, (size_t)p->kp * 4, (size_t)p->k * 4, rows, kind, p->stream));
    } else {
      FKK_CUDA_CHECK(cudaMemcpyAsync(dst, src, n, kind, p->stream));
    }
    FKK_CUDA_CHECK(cudaStreamSynchronize(p->stream));
  });
}

fkk_status fkk_enable_timing(fkk_plan_t p, int32_t on) {
  if (!p) return FKK_ERR_INVALID_ARG;
  p->timing = on != 0;
  return FKK_OK;
}

int32_t fkk_stage_times(fkk_plan_t p, const char** names, float* ms, int32_t cap) {
  if (!p) return 0;
  int32_t n = std::min<int32_t>(cap, (int32_t)p->t_ms.size());
  for (int32_t i = 0; i < n; ++i) {
    if (names) names[i] = p->t_names[i].c_str();
    if (ms) ms[i] = p->t_ms[i];
  }
  return n;
}

int64_t fkk_last_launch_count(fkk_plan_t p) { return p ? p->launches : 0; }

int64_t fkk_debug_als_solves(fkk_plan_t p) {
  if (!p || !p->als_solves) return 0;
  int v = 0;
  if (cudaStreamSynchronize(p->stream) != cudaSuccess) return -1;
  if (cudaMemcpy(&v, p->als_solves, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  cudaMemset(p->als_solves, 0, sizeof(int));
  return v;
}

fkk_status fkk_debug_tc_mma(int32_t mode, const float* d_A, const float* d_B, float* d_D, int32_t N) {
  if (!d_A || !d_B || !d_D || N < 16 || N > 256 || N % 16) return FKK_ERR_INVALID_ARG;
  try {
    fkk::launch_tc_selftest(mode, d_A, d_B, d_D, N, nullptr);
    FKK_CUDA_CHECK(cudaDeviceSynchronize());
    return FKK_OK;
  } catch (const Status& e) {
    g_create_err = e.what();
    return (fkk_status)e.code;
  }
}

fkk_status fkk_debug_eig_topk(const double* d_G, int32_t M, int32_t k, double* d_V, double* d_lam) {
  if (!d_G || !d_V || !d_lam || M < 3 || k < 1 || k > M) return FKK_ERR_INVALID_ARG;
  double* work = nullptr;
  int* flags = nullptr;
  try {
    work = dalloc<double>(fkk::eig_workspace_doubles(M, k));
    flags = dalloc<int>(1);
    FKK_CUDA_CHECK(cudaMemset(flags, 0, sizeof(int)));
    fkk::launch_eig_topk(d_G, M, k, work, d_V, d_lam, flags, nullptr);
    FKK_CUDA_CHECK(cudaDeviceSynchronize());
    int hf = 0;
    FKK_CUDA_CHECK(cudaMemcpy(&hf, flags, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(work);
    cudaFree(flags);
    return hf ? FKK_ERR_NUMERICAL : FKK_OK;
  } catch (const Status& e) {
    g_create_err = e.what();
    cudaFree(work);
    cudaFree(flags);
    return (fkk_status)e.code;
  }
}

int32_t fkk_debug_eig_path(int32_t M) { return fkk::eig_path_rows_resident(M); }

fkk_status fkk_debug_tridiag(const double* d_G, int32_t M, double* d_det) {
  if (!d_G || !d_det || M < 3) return FKK_ERR_INVALID_ARG;
  try {
    fkk::debug_tridiag(d_G, M, d_det);
    return FKK_OK;
  } catch (const Status& e) {
    g_create_err = e.what();
    return (fkk_status)e.code;
  }
}

fkk_status fkk_host_eig_topk(const double* G, int32_t M, int32_t k, double* V, double* lam) {
  if (!G || !V || !lam || M < 1 || k < 1 || k > M) return FKK_ERR_INVALID_ARG;
  try {
    return fkk::host_eig_topk(G, M, k, V, lam) == 0 ? FKK_OK : FKK_ERR_NUMERICAL;
  } catch (...) {
    return FKK_ERR_NUMERICAL;
  }
}

void fkk_shard_range(int64_t n_global, int32_t world, int32_t rank, int64_t* row0, int64_t* row1) {
  if (world < 1) world = 1;
  const int64_t base = n_global / world, rem = n_global % world;
  const int64_t r0 = rank * base + std::min<int64_t>(rank, rem);
  const int64_t len = base + (rank < rem ? 1 : 0);
  if (row0) *row0 = r0;
  if (row1) *row1 = r0 + len;
}

int32_t fkk_merge_extremes(const float* vals, const int64_t* idx, int32_t world, int32_t k, int64_t* q_out) {
  std::vector<int64_t> q;
  q.reserve(2 * k);
  for (int c = 0; c < k; ++c) {
    float bM = -INFINITY, bm = INFINITY;
    int64_t iM = INT64_MAX, im = INT64_MAX;
    for (int r = 0; r < world; ++r) {
      const size_t o = ((size_t)r * k + c) * 2;
      if (idx[o] != INT64_MAX && (vals[o] > bM || (vals[o] == bM && idx[o] < iM))) { bM = vals[o]; iM = idx[o]; }
      if (idx[o + 1] != INT64_MAX && (vals[o + 1] < bm || (vals[o + 1] == bm && idx[o + 1] < im))) { bm = vals[o + 1]; im = idx[o + 1]; }
    }
    if (iM != INT64_MAX) q.push_back(iM);
    if (im != INT64_MAX) q.push_back(im);
  }
  std::sort(q.begin(), q.end());
  q.erase(std::unique(q.begin(), q.end()), q.end());
  std::copy(q.begin(), q.end(), q_out);
  return (int32_t)q.size();
}

}  // extern "C"
