// common.cuh — device-side helpers shared by the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "layout.h"

namespace hg {

// ------------------------------------------------------------------ batch view
struct BatchView {
  int B, N, E, F0, Fe;
  const int *gp;
  const float *y;
  const int *rowptr;
  const int *col;
  const float *x;
  const float *ea;
  const uint8_t *slot;
};

__device__ __forceinline__ BatchView load_batch(const uint8_t *blob) {
  BatchView v;
  const int *h = reinterpret_cast<const int *>(blob);
  v.B = h[0]; v.N = h[1]; v.E = h[2]; v.F0 = h[3]; v.Fe = h[4];
  const BatchOffsets o = batch_offsets(v.B, v.N, v.E, v.F0, v.Fe);
  v.gp = reinterpret_cast<const int *>(blob + o.graph_ptr);
  v.y = reinterpret_cast<const float *>(blob + o.y);
  v.rowptr = reinterpret_cast<const int *>(blob + o.rowptr);
  v.col = reinterpret_cast<const int *>(blob + o.col);
  v.x = reinterpret_cast<const float *>(blob + o.x);
  v.ea = reinterpret_cast<const float *>(blob + o.eattr);
  v.slot = blob + o.slot;
  return v;
}

__device__ __forceinline__ int batch_N(const uint8_t *blob) { return reinterpret_cast<const int *>(blob)[1]; }

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
constexpr int kSMs = 148;


__device__ __forceinline__ float4 ldg4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }

}  // namespace hg
