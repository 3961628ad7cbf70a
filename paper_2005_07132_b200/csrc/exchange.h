// The collective sequence of the pixel-sharded fKK-EC transform,
// written once against an abstract set of collectives:
//   1. row counts      : allgather of n_rows            -> this rank's global row offset, N
//   2. noise scale     : allreduce(sum) of column sums  (f_mode = eq9, Eq. 9)
//   3. Gram / A^T Y    : allreduce(sum) of the fp64 partial products
//   4. extremes        : allgather of the per-shard column argmax / argmin -> q (reading A12)
//   5. X = US[q]       : allreduce(sum) of the rows this rank owns (zeros elsewhere)
//   6. error flags     : allreduce(max) of the device error word before any host check
// Every rank issues them in this order.  Small control data (1, 4) travel as HOST buffers; bulk data
// (2, 3, 5, 6) stays in the backend's data memory (device for NCCL, host for the callback backend
// the CPU tests drive through fkk_exchange_selftest).
#pragma once
#include <stdint.h>

#include <vector>

namespace fkk {

struct Collectives {
  int world = 1, rank = 0;
  virtual ~Collectives() = default;
  virtual void allgather_host(const void* send, void* recv, size_t bytes) = 0;   // recv: world x bytes
  virtual void allreduce_sum_f64(double* data, size_t n) = 0;
  virtual void allreduce_max_i32(int* data, size_t n) = 0;
  virtual void sync() = 0;   // the data collectives enqueued so far are complete
};

// step 1
void exchange_rows(Collectives& c, int64_t n_rows, int64_t* row0, int64_t* n_global);
// step 4: local (per virtual shard) extremes [shards][k][2] (value, global index) -> sorted unique q
std::vector<int64_t> exchange_extremes(Collectives& c, const float* vals, const int64_t* idx, int shards, int k);
// step 5 helper: local row of each q entry (-1 if another rank owns it)
std::vector<int64_t> local_rows(const std::vector<int64_t>& q, int64_t row0, int64_t n_rows);

}  // namespace fkk
