// common.cuh — device-side helpers shared by the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "layout.h"

namespace hg {

// ------------------------------------------------------------------ batch view
struct BatchView {
  int B, N, E, F0, Fe;
  const int *gp;
  const float *y, *y_node;
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
  v.y_node = reinterpret_cast<const float *>(blob + o.y_node);
  v.rowptr = reinterpret_cast<const int *>(blob + o.rowptr);
  v.col = reinterpret_cast<const int *>(blob + o.col);
  v.x = reinterpret_cast<const float *>(blob + o.x);
  v.ea = reinterpret_cast<const float *>(blob + o.eattr);
  v.slot = blob + o.slot;
  return v;
}

__device__ __forceinline__ int batch_N(const uint8_t *blob) { return reinterpret_cast<const int *>(blob)[1]; }

inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// ------------------------------------------------ launches
// launch priority: kernels enqueued while g_low_prio is set (side-stream weight
// gradients) get the device's lowest priority, all others its highest
extern bool g_low_prio;
extern int g_prio_lo, g_prio_hi;
// Every kernel starts with pdl_enter() (griddepcontrol.wait / launch_dependents): a no-op
// under plain stream ordering, it makes the kernels safe to launch with programmatic
// dependent launch (measured slower for this step, round 2 again: config B 268k vs 314k graphs/s,
// D 367k vs 377k, profiles/r02_pdl_rejected_*.json; so it is not enabled).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args &&...args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = g_low_prio ? g_prio_lo : g_prio_hi;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
constexpr int kSMs = 148;


__device__ __forceinline__ float4 ldg4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }

}  // namespace hg
