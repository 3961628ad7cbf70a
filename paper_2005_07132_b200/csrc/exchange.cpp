// Collective sequence of the pixel-sharded transform (exchange.h) and its host-callback backend, the
// C-ABI self-test fkk_exchange_selftest that the 2-rank gloo test drives on CPU.
#include "exchange.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "../../include/fkk.h"
#include "fkk_internal.h"

namespace fkk {

void exchange_rows(Collectives& c, int64_t n_rows, int64_t* row0, int64_t* n_global) {
  std::vector<int64_t> all(c.world);
  c.allgather_host(&n_rows, all.data(), sizeof(int64_t));
  int64_t r0 = 0, ng = 0;
  for (int r = 0; r < c.world; ++r) {
    if (r < c.rank) r0 += all[r];
    ng += all[r];
  }
  *row0 = r0;
  *n_global = ng;
}

std::vector<int64_t> exchange_extremes(Collectives& c, const float* vals, const int64_t* idx, int shards, int k) {
  const size_t per = (size_t)shards * k * 2;
  std::vector<float> av(per * c.world);
  std::vector<int64_t> ai(per * c.world);
  c.allgather_host(vals, av.data(), per * sizeof(float));
  c.allgather_host(idx, ai.data(), per * sizeof(int64_t));
  std::vector<int64_t> q(2 * (size_t)k);
  const int nq = fkk_merge_extremes(av.data(), ai.data(), shards * c.world, k, q.data());
  q.resize(nq);
  return q;
}

std::vector<int64_t> local_rows(const std::vector<int64_t>& q, int64_t row0, int64_t n_rows) {
  std::vector<int64_t> ql(q.size());
  for (size_t i = 0; i < q.size(); ++i) ql[i] = (q[i] >= row0 && q[i] < row0 + n_rows) ? q[i] - row0 : -1;
  return ql;
}

namespace {

struct HostCallbackCollectives : Collectives {
  const fkk_host_collectives* cb;
  explicit HostCallbackCollectives(const fkk_host_collectives* c) : cb(c) {
    world = c->world_size;
    rank = c->rank;
  }
  void check(int rc, const char* what) {
    if (rc != 0) throw Status(FKK_ERR_NCCL, std::string("host collective failed: ") + what);
  }
  void allgather_host(const void* send, void* recv, size_t bytes) override {
    check(cb->allgather(cb->ctx, send, recv, bytes), "allgather");
  }
  void allreduce_sum_f64(double* data, size_t n) override { check(cb->allreduce_sum_f64(cb->ctx, data, n), "allreduce_sum_f64"); }
  void allreduce_max_i32(int* data, size_t n) override { check(cb->allreduce_max_i32(cb->ctx, data, n), "allreduce_max_i32"); }
  void sync() override {}
};

}  // namespace
}  // namespace fkk

extern "C" {

// The sequence of the sharded transform on host data (no GPU): steps 1, 3, 4, 5, 6 of exchange.h with
// the same functions the NCCL path calls.  In: this rank's n_rows, local Gram partial G (M x M, summed
// in place), local extremes [shards][k][2] (value, global pixel), US_local (n_rows x k row-major),
// local error flags.  Out: row0, N, G (global), q (<= 2k entries), X = US[q] (nq x k, global), flags.
fkk_status fkk_exchange_selftest(const fkk_host_collectives* comm, int64_t n_rows, int32_t M, int32_t k, int32_t shards,
                                 double* G, const float* ext_val, const int64_t* ext_idx, const float* US_local,
                                 int32_t* flags, int64_t* row0_out, int64_t* n_global_out, int64_t* q_out,
                                 int32_t* nq_out, double* X_out) {
  if (!comm || !G || !ext_val || !ext_idx || !flags || !row0_out || !n_global_out || !q_out || !nq_out || !X_out ||
      (n_rows > 0 && !US_local) || M < 1 || k < 1 || shards < 1)
    return FKK_ERR_INVALID_ARG;
  try {
    fkk::HostCallbackCollectives c(comm);
    int64_t row0 = 0, ng = 0;
    fkk::exchange_rows(c, n_rows, &row0, &ng);                                   // 1
    c.allreduce_sum_f64(G, (size_t)M * M);                                       // 3
    const std::vector<int64_t> q = fkk::exchange_extremes(c, ext_val, ext_idx, shards, k);   // 4
    const std::vector<int64_t> ql = fkk::local_rows(q, row0, n_rows);            // 5
    for (size_t i = 0; i < q.size(); ++i)
      for (int c2 = 0; c2 < k; ++c2) X_out[i * k + c2] = ql[i] >= 0 ? (double)US_local[ql[i] * k + c2] : 0.0;
    c.allreduce_sum_f64(X_out, q.size() * (size_t)k);
    c.allreduce_max_i32(flags, 1);                                               // 6
    c.sync();
    *row0_out = row0;
    *n_global_out = ng;
    std::copy(q.begin(), q.end(), q_out);
    *nq_out = (int32_t)q.size();
    return FKK_OK;
  } catch (const fkk::Status& e) {
    return (fkk_status)e.code;
  }
}

}  // extern "C"
