// layout.h — packed-batch blob layout (include/hgnn.h) shared by
// the host packer and the device kernels. Pure integer arithmetic.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HG_HD __host__ __device__ __forceinline__
#else
#define HG_HD inline
#endif

namespace hg {

constexpr int kHeaderInts = 16;

HG_HD int64_t align16(int64_t v) { return (v + 15) & ~int64_t(15); }
HG_HD int64_t align256(int64_t v) { return (v + 255) & ~int64_t(255); }

struct BatchOffsets {
  int64_t graph_ptr, y, y_node, rowptr, col, x, eattr, slot, total;
};

// offsets of each array inside a batch blob with B graphs, N nodes, E edges
HG_HD BatchOffsets batch_offsets(int64_t B, int64_t N, int64_t E, int64_t F0, int64_t Fe) {
  BatchOffsets o;
  int64_t p = kHeaderInts * 4;
  o.graph_ptr = p; p = align16(p + 4 * (B + 1));
  o.y = p;         p = align16(p + 4 * B);
  o.y_node = p;    p = align16(p + 4 * N);
  o.rowptr = p;    p = align16(p + 4 * (N + 1));
  o.col = p;       p = align16(p + 4 * E);
  o.x = p;         p = align16(p + 4 * N * F0);
  o.eattr = p;     p = align16(p + 4 * E * Fe);
  o.slot = p;      p = align16(p + E);
  o.total = p;
  return o;
}

}  // namespace hg
