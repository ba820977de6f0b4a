// internal.h — declarations shared by the host (host.cpp) and device (ctx.cu)
// translation units of libhgnn. Not part of the public ABI.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "hgnn.h"

namespace hg {

hg_status fail(hg_status st, const char *fmt, ...);
uint64_t splitmix64(uint64_t x);

struct TensorInfo {
  std::string name;
  int rows = 0, cols = 0, fan_in = 0, fan_out = 0;
  int64_t offset = 0;  // in floats, into the flat parameter arena
};
std::vector<TensorInfo> param_layout(const hg_config &c);
int64_t param_total(const std::vector<TensorInfo> &v);
hg_status check_config(const hg_config *c);
void init_params_host(const hg_config &c, uint64_t seed, float *dst);

}  // namespace hg

// Table-1 store: global arrays + per-graph offsets, plus the
// derived per-edge slot (position of src inside dst's neighbour row).
struct hg_store;
namespace hg {
hg_status store_finish(hg_store *s, int32_t threads);  // host.cpp
}
struct hg_store {
  int64_t G = 0, N = 0, E = 0;
  int32_t F0 = 0, Fe = 0;
  const int64_t *no = nullptr, *eo = nullptr;
  const float *x = nullptr, *ea = nullptr, *y = nullptr;
  const int32_t *src = nullptr, *dst = nullptr;
  std::vector<int64_t> own_no, own_eo;
  std::vector<float> own_x, own_ea, own_y;
  std::vector<int32_t> own_ei;
  std::vector<uint8_t> slot;
  int32_t max_nodes = 0, max_deg = 0;
};
