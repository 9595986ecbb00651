// Internal launcher declarations shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace bx {

// bx_direct_seq.cu
void ntdm_seq(const double *d, const double *e, const double *f, const double *b, double *x,
              double *ws, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld,
              int layout, cudaStream_t stream);
void penta_seq(bool mod, const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, double *ws, int32_t *st,
               int32_t *ix, int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout,
               cudaStream_t stream);
void residual_inf(int bw, const double *c, const double *d, const double *e, const double *f,
                  const double *g, const double *x, const double *b, double *out, int64_t batch,
                  int64_t n, int64_t ld, int layout, cudaStream_t stream);

// bx_direct_part.cu
size_t part_workspace_bytes(int bandwidth, int64_t batch, int64_t n);
int ntdm_part(const double *d, const double *e, const double *f, const double *b, double *x,
              double *ws, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld,
              int layout, cudaStream_t stream);
int penta_part(bool mod, const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, double *ws, int32_t *st,
               int32_t *ix, int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout,
               cudaStream_t stream);

// workspace of the non-direct solvers (bx_api.cu dispatch)
size_t other_workspace_bytes(int solver, int64_t batch, int64_t n);

}  // namespace bx
