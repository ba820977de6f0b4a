// internal.h — declarations shared by the host (host.cpp) and device (ctx.cu)
// translation units of libhgnn. Not part of the public ABI.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "hgnn.h"

namespace hg {

// CRC-32C (Castagnoli), container.cpp
uint32_t crc32c(const void *data, size_t n, uint32_t crc = 0);


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

// Channel padding (SURVEY §8(d) "Padding hazard"; paper widths H = 55, 200 at
// PAPER.md:315, 318). A hidden width that is not a multiple of the tensor-core tile
// (kChannelTile = 128) runs internally at Hp = roundup(H, 128), fc_hidden == H padded alike. The padded parameter entries are zero and stay zero
// (their gradients are exactly zero: the aggregation kernel writes zero aggregates
// for padded channels, see launch_agg_fwd), so the padded model computes the
// logical one exactly. The public arena (hg_param_info, get/set) stays logical.
constexpr int kChannelTile = 128;
constexpr int kClassSlots = 32;  // degree-class slots at most (kernels.h kMaxClasses)
constexpr int HG_FLAGS_KNOWN = HG_FLAG_TF32 | HG_FLAG_SELF_TERM | HG_FLAG_NODE_HEAD;
int scaler_mask(const hg_config &c);  // c.scalers, or the default identity | amplification | attenuation
int n_scalers(const hg_config &c);
bool self_term(const hg_config &c);
hg_config padded_config(const hg_config &c);
// degree classes a ctx of this configuration holds: min(max_degree + 1, kClassSlots); a batch
// with more distinct node degrees is rejected when it is packed (HG_E_DEGREE)
int class_slots(const hg_config &c);
// validate a packed blob (include/hgnn.h layout) against a configuration: header, capacities,
// offsets, node degrees and distinct-degree count (hg_upload_packed)
hg_status check_blob(const void *blob, size_t bytes, const hg_config &cfg);
bool config_is_padded(const hg_config &c);
// scatter a logical arena (layout of `logical`) into a zeroed padded arena
// (layout of padded_config(logical)), or gather it back
void arena_pad(const hg_config &logical, const float *src, float *dst);
void arena_unpad(const hg_config &logical, const float *src, float *dst);

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
  const float *x = nullptr, *ea = nullptr, *y = nullptr, *yn = nullptr;  // yn: node targets or null
  const int32_t *src = nullptr, *dst = nullptr;
  std::vector<int64_t> own_no, own_eo;
  std::vector<float> own_x, own_ea, own_y, own_yn;
  std::vector<int32_t> own_ei;
  std::vector<uint8_t> slot;
  const uint8_t *slotp = nullptr;  // = slot.data(), or the shared-memory copy (hg_store_open_shared)
  void *shm_base = nullptr;        // POSIX shared-memory mapping of a shared store (shm.cpp)
  size_t shm_bytes = 0;
  bool shm_pinned = false;         // the mapping is cudaHostRegister-ed
  ~hg_store();
  int32_t max_nodes = 0, max_deg = 0;
};
