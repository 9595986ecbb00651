// Partitioned (on-chip) direct solvers -- placeholder until the kernels land.
#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {

size_t part_workspace_bytes(int, int64_t, int64_t) { return 0; }

int ntdm_part(const double *, const double *, const double *, const double *, double *, double *,
              int32_t *, int32_t *, int64_t, int64_t, int64_t, int, cudaStream_t) {
  bxh::set_error("bx_ntdm_f64: BX_ALGO_PARTITIONED not built yet");
  return BX_ERR_UNSUPPORTED;
}

int penta_part(bool, const double *, const double *, const double *, const double *,
               const double *, const double *, double *, double *, int32_t *, int32_t *,
               int64_t *, int64_t, int64_t, int64_t, int, cudaStream_t) {
  bxh::set_error("BX_ALGO_PARTITIONED not built yet");
  return BX_ERR_UNSUPPORTED;
}

size_t other_workspace_bytes(int, int64_t, int64_t) { return 0; }

}  // namespace bx
