// TMA tensor maps (host) and bulk-tensor copies (device) for the tcgen05 kernels.  The tensor map
// is encoded on the host with the driver's cuTensorMapEncodeTiled (resolved once through
// cudaGetDriverEntryPoint, so the library needs no -lcuda) and passed by value as a
// __grid_constant__ kernel parameter.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fkk {
namespace tma {

// 2-D fp32 tensor [rows][cols] (row pitch `pitch_bytes`, multiple of 16), box [box_rows][box_cols],
// swizzle = 0 (none), 64 or 128 (bytes).  Throws fkk::Status on failure.
CUtensorMap make_2d_f32(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_bytes, uint32_t box_rows,
                        uint32_t box_cols, int swizzle);

#if defined(__CUDACC__)
// smem -> global 2-D tile store, bulk-group completion (cp.async.bulk.wait_group[.read])
__device__ __forceinline__ void store_2d(const CUtensorMap* map, uint32_t smem_addr, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_addr), "r"(x), "r"(y)
               : "memory");
}
// global -> smem 2-D tile load, completion on an mbarrier (transaction bytes)
__device__ __forceinline__ void load_2d(const CUtensorMap* map, uint32_t smem_addr, uint32_t mbar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_addr),
      "l"(map), "r"(mbar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
#endif

}  // namespace tma
}  // namespace fkk
