// Shared device helpers for the bandix_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bandix_b200.h"

namespace bx {

// ---- element addressing for the two layouts of the C ABI ------------------
// Interleaved: (row i, system s) at i*ld + s (system fastest; coalesced when
// consecutive lanes own consecutive systems).  System-major: s*ld + i.
struct Interleaved {
  int64_t ld;
  __device__ __forceinline__ int64_t operator()(int64_t i, int64_t s) const { return i * ld + s; }
};
struct SystemMajor {
  int64_t ld;
  __device__ __forceinline__ int64_t operator()(int64_t i, int64_t s) const { return s * ld + i; }
};

// Workspace rows are always interleaved with ld = batch, so a warp's 32
// consecutive systems touch one 256-byte segment per row.
struct Scratch {
  int64_t batch;
  __device__ __forceinline__ int64_t operator()(int64_t i, int64_t s) const { return i * batch + s; }
};

__device__ __forceinline__ double ldg(const double *p) { return __ldg(p); }

// Single-rounding IEEE binary64 operations.  The parity kernels use these
// explicitly so that no multiply-subtract pair can be contracted into an FMA:
// the reference evaluates every operation with one rounding (CPython float),
// and bit parity depends on it.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ void set_status(int32_t *status, int32_t *index, int64_t s, int32_t st,
                                           int32_t idx) {
  if (status) status[s] = st;
  if (index) index[s] = idx;
}

}  // namespace bx

// Host-side error plumbing (bx_api.cu).
namespace bxh {
void set_error(const char *fmt, ...);
int check_launch(const char *what);
}  // namespace bxh
