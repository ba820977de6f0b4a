// host.cpp — host side of the C-ABI: error reporting, the Table-1 graph store
// (PAPER.md:183-190, 232-253), sharding, the host collate
// (SPEC.md:275-283), the degree statistic and the parameter
// layout / counter-based initialisation.
// No CUDA in this translation unit: these calls work on a machine without a GPU.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hgnn.h"
#include "internal.h"
#include "layout.h"

namespace hg {

static thread_local std::string t_err;

hg_status fail(hg_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return st;
}

// threads of one collation (hg_pack / hg_pack_host): hg_pack_threads_set, default 4
static std::atomic<int> g_pack_threads{4};
static int hg_pack_threads() { return g_pack_threads.load(); }

static int hw_threads(int32_t t) {
  if (t > 0) return t;
  unsigned n = std::thread::hardware_concurrency();
  return n ? (int)n : 1;
}

template <class F>
static void parallel_for(int64_t n, int threads, F fn) {
  threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n));
  if (threads == 1) {
    fn(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    int64_t a = t * chunk, b = std::min<int64_t>(n, a + chunk);
    if (a >= b) break;
    th.emplace_back(fn, a, b, t);
  }
  for (auto &x : th) x.join();
}

uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------------ params
std::vector<TensorInfo> param_layout(const hg_config &c) {
  std::vector<TensorInfo> v;
  const int H = c.hidden, Fe = c.f_edge, Hf = c.fc_hidden;
  int64_t off = 0;
  auto add = [&](const std::string &name, int rows, int cols, int fi, int fo) {
    TensorInfo t;
    t.name = name; t.rows = rows; t.cols = cols; t.fan_in = fi; t.fan_out = fo; t.offset = off;
    off += ((int64_t)rows * cols + 63) / 64 * 64;  // 256-byte aligned tensors
    v.push_back(t);
  };
  const int S = n_scalers(c);
  const bool st = self_term(c);
  for (int l = 0; l < c.layers; ++l) {
    const int Fl = l == 0 ? c.f_node : H;
    std::string p = "conv" + std::to_string(l) + ".";
    const int fm = (st ? 2 * Fl : Fl) + Fe, fu = 4 * S * H + (st ? Fl : 0);  // fans of M, [U | U_x]
    add(p + "M_x", H, Fl, fm, H);
    if (st) add(p + "M_s", H, Fl, fm, H);
    add(p + "M_e", H, Fe, fm, H);
    add(p + "b_M", 1, H, 0, 0);
    add(p + "U", H, 4 * S * H, fu, H);
    if (st) add(p + "U_x", H, Fl, fu, H);
    add(p + "b_U", 1, H, 0, 0);
  }
  add("head.W1", Hf, H, H, Hf);
  add("head.b1", 1, Hf, 0, 0);
  add("head.W2", 1, Hf, Hf, 1);
  add("head.b2", 1, 1, 0, 0);
  if (c.flags & HG_FLAG_NODE_HEAD) {  // node-level head (reading R-node-head): the graph head's shape
    add("head_n.W1", Hf, H, H, Hf);
    add("head_n.b1", 1, Hf, 0, 0);
    add("head_n.W2", 1, Hf, Hf, 1);
    add("head_n.b2", 1, 1, 0, 0);
  }
  return v;
}

int64_t param_total(const std::vector<TensorInfo> &v) {
  const TensorInfo &t = v.back();
  return t.offset + ((int64_t)t.rows * t.cols + 63) / 64 * 64;
}

hg_status check_config(const hg_config *c) {
  if (!c) return fail(HG_E_INVALID, "null config");
  if (c->f_node < 1 || c->f_edge < 1 || c->layers < 1 || c->fc_hidden < 1)
    return fail(HG_E_INVALID, "config widths must be positive");
  if (c->hidden < 1 || c->hidden > 1024)
    return fail(HG_E_INVALID, "hidden must be in [1, 1024] (got %d)", c->hidden);
  if (c->fc_hidden > 1024) return fail(HG_E_INVALID, "fc_hidden must be <= 1024");
  if (c->f_edge > 8) return fail(HG_E_INVALID, "f_edge must be <= 8");
  if (c->max_graphs < 1 || c->max_nodes < 1 || c->max_edges < 0 || c->n_slots < 1)
    return fail(HG_E_INVALID, "capacities must be positive");
  if (!(c->delta > 0.0)) return fail(HG_E_INVALID, "delta must be > 0 (SPEC.md:329)");
  if (!(c->var_floor > 0.0f)) return fail(HG_E_INVALID, "var_floor must be > 0");
  if (c->max_degree < 0 || c->max_degree > HG_MAX_DEGREE) return fail(HG_E_INVALID, "max_degree out of range");
  if (c->flags & ~HG_FLAGS_KNOWN) return fail(HG_E_INVALID, "unknown flags 0x%x", c->flags);
  const int sm = scaler_mask(*c);
  if (sm & ~31) return fail(HG_E_INVALID, "unknown scaler bits 0x%x", c->scalers);
  if (!(sm & HG_SCALER_IDENTITY)) return fail(HG_E_INVALID, "the identity scaler is required (SPEC.md:327)");
  if ((sm & (HG_SCALER_LINEAR | HG_SCALER_INVERSE_LINEAR)) && !(c->delta_lin > 0.0))
    return fail(HG_E_INVALID, "delta_lin must be > 0 with the linear scalers");
  if ((c->flags & HG_FLAG_NODE_HEAD) && !(c->node_weight >= 0.f))
    return fail(HG_E_INVALID, "node_weight must be >= 0");
  if ((c->flags & HG_FLAG_NODE_HEAD) && c->fc_hidden != c->hidden && c->fc_hidden % 128)
    return fail(HG_E_INVALID, "the node-level head needs fc_hidden == hidden or a multiple of 128");
  if (self_term(*c) && c->f_node > c->hidden)
    return fail(HG_E_INVALID, "the self-term variant needs f_node <= hidden (got %d > %d)", c->f_node, c->hidden);
  return HG_OK;
}

int scaler_mask(const hg_config &c) {
  return c.scalers ? c.scalers : (HG_SCALER_IDENTITY | HG_SCALER_AMPLIFICATION | HG_SCALER_ATTENUATION);
}
int n_scalers(const hg_config &c) { return __builtin_popcount((unsigned)scaler_mask(c) & 31u); }
bool self_term(const hg_config &c) { return (c.flags & HG_FLAG_SELF_TERM) != 0; }

bool config_is_padded(const hg_config &c) { return c.hidden % kChannelTile != 0; }

hg_config padded_config(const hg_config &c) {
  if (!config_is_padded(c)) return c;
  hg_config p = c;
  const int q = kChannelTile;
  p.hidden = (c.hidden + q - 1) / q * q;
  if (c.fc_hidden == c.hidden) p.fc_hidden = p.hidden;
  return p;
}

// Per tensor: logical [R, nb*W] -> padded [Rp, nb*Wp]; column j = q*W + c maps to
// q*Wp + c (nb = 12 column blocks for U: (s*4+a)*H + c), rows r -> r.
static void arena_map(const hg_config &logical, const float *src, float *dst, bool to_padded) {
  const hg_config pc = padded_config(logical);
  const auto ll = param_layout(logical), lp = param_layout(pc);
  for (size_t t = 0; t < ll.size(); ++t) {
    const TensorInfo &a = ll[t], &b = lp[t];
    const int nb = a.name.size() >= 2 && a.name.compare(a.name.size() - 2, 2, ".U") == 0 ? 4 * n_scalers(logical) : 1;
    const int W = a.cols / nb, Wp = b.cols / nb;
    for (int r = 0; r < a.rows; ++r)
      for (int q = 0; q < nb; ++q)
        for (int c = 0; c < W; ++c) {
          const int64_t li = a.offset + (int64_t)r * a.cols + (int64_t)q * W + c;
          const int64_t pi = b.offset + (int64_t)r * b.cols + (int64_t)q * Wp + c;
          if (to_padded) dst[pi] = src[li];
          else dst[li] = src[pi];
        }
  }
}
void arena_pad(const hg_config &logical, const float *src, float *dst) { arena_map(logical, src, dst, true); }
void arena_unpad(const hg_config &logical, const float *src, float *dst) { arena_map(logical, src, dst, false); }

void init_params_host(const hg_config &c, uint64_t seed, float *dst) {
  auto lay = param_layout(c);
  std::memset(dst, 0, sizeof(float) * param_total(lay));
  for (size_t t = 0; t < lay.size(); ++t) {
    const TensorInfo &ti = lay[t];
    if (ti.fan_in == 0) continue;  // biases: zero
    const double a = std::sqrt(6.0 / (double)(ti.fan_in + ti.fan_out));
    const int64_t n = (int64_t)ti.rows * ti.cols;
    const uint64_t tk = (uint64_t)t * 0x9E3779B97F4A7C15ULL;
    for (int64_t e = 0; e < n; ++e) {
      uint64_t key = seed ^ tk ^ ((uint64_t)e * 0xD1B54A32D192ED03ULL);
      double u = (double)(splitmix64(key) >> 11) * (1.0 / 9007199254740992.0);
      dst[ti.offset + e] = (float)((2.0 * u - 1.0) * a);
    }
  }
}

}  // namespace hg

namespace hg {
// validate a store whose array pointers are set and compute slot / max stats
// (shared by hg_store_create and the container readers); on failure the caller
// deletes s.
int class_slots(const hg_config &c) {
  const int dmax = c.max_degree > 0 ? c.max_degree : HG_MAX_DEGREE;
  return std::min(dmax + 1, kClassSlots);
}

hg_status check_blob(const void *blob, size_t bytes, const hg_config &cfg) {
  const int32_t *h = (const int32_t *)blob;
  const int32_t B = h[0], N = h[1], E = h[2];
  if (B < 1) return fail(HG_E_EMPTY, "EmptyBatch");
  if (B > cfg.max_graphs || N > cfg.max_nodes || E > cfg.max_edges || N < 0 || E < 0)
    return fail(HG_E_CAPACITY, "blob exceeds ctx capacity");
  if (h[3] != cfg.f_node || h[4] != cfg.f_edge) return fail(HG_E_SHAPE, "blob feature widths differ");
  const BatchOffsets o = batch_offsets(B, N, E, h[3], h[4]);
  if (bytes < (size_t)o.total) return fail(HG_E_SHAPE, "blob shorter than its header implies");
  const int32_t *rp = (const int32_t *)((const uint8_t *)blob + o.rowptr);
  const int32_t *col = (const int32_t *)((const uint8_t *)blob + o.col);
  const int32_t *gp = (const int32_t *)((const uint8_t *)blob + o.graph_ptr);
  if (gp[0] != 0 || gp[B] != N || rp[0] != 0 || rp[N] != E) return fail(HG_E_SHAPE, "blob offsets inconsistent");
  for (int32_t g = 0; g < B; ++g)
    if (gp[g + 1] <= gp[g]) return fail(HG_E_EMPTY, "EmptyGraphSlot in blob");
  const int maxdeg = cfg.max_degree > 0 ? cfg.max_degree : HG_MAX_DEGREE;
  uint64_t bits[2] = {0, 0};
  for (int32_t i = 0; i < N; ++i) {
    const int32_t d = rp[i + 1] - rp[i];
    if (d < 0 || d > maxdeg) return fail(HG_E_DEGREE, "blob node %d has degree %d", i, d);
    bits[d >> 6] |= 1ull << (d & 63);
  }
  for (int32_t k = 0; k < E; ++k)
    if (col[k] < 0 || col[k] >= N) return fail(HG_E_RANGE, "blob edge %d endpoint out of range", k);
  const int ndeg = __builtin_popcountll(bits[0]) + __builtin_popcountll(bits[1]);
  if (ndeg > class_slots(cfg))
    return fail(HG_E_DEGREE, "batch has %d distinct node degrees > %d degree-class slots", ndeg, class_slots(cfg));
  return HG_OK;
}

hg_status store_finish(hg_store *s, int32_t threads) {
  const int64_t G = s->G;
  // offsets first, serially: every later (parallel) pass indexes the arrays through them
  if (s->no[0] != 0 || s->eo[0] != 0 || s->no[G] != s->N || s->eo[G] != s->E)
    return fail(HG_E_SHAPE, "offsets must start at 0 and end at the totals");
  for (int64_t g = 0; g < G; ++g)
    if (s->no[g + 1] < s->no[g] || s->eo[g + 1] < s->eo[g] || s->no[g + 1] > s->N || s->eo[g + 1] > s->E)
      return fail(HG_E_SHAPE, "store graph %lld: offsets not non-decreasing within the totals", (long long)g);
  s->slot.assign((size_t)s->E, 0);
  const int nt = hw_threads(threads);
  std::vector<hg_status> st(nt, HG_OK);
  std::vector<int64_t> bad(nt, -1);
  std::vector<int32_t> mxn(nt, 0), mxd(nt, 0);
  parallel_for(G, nt, [&](int64_t g0, int64_t g1, int t) {
    std::vector<int32_t> rs;
    for (int64_t g = g0; g < g1 && st[t] == HG_OK; ++g) {
      const int64_t n0 = s->no[g], n1 = s->no[g + 1], e0 = s->eo[g], e1 = s->eo[g + 1];
      const int64_t n = n1 - n0;
      if (n < 1) { st[t] = HG_E_EMPTY; bad[t] = g; break; }
      if (e1 < e0 || n1 < n0) { st[t] = HG_E_SHAPE; bad[t] = g; break; }
      mxn[t] = std::max<int32_t>(mxn[t], (int32_t)n);
      {  // fault in this graph's node-feature pages now (a borrowed, memory-mapped store would
         // otherwise page-fault inside every later collation)
        volatile float sink = 0.f;
        const float *xa = s->x + n0 * s->F0;
        const int64_t nx = n * s->F0;
        for (int64_t q = 0; q < nx; q += 1024) sink = sink + xa[q];
        sink = sink + xa[nx - 1];
        (void)sink;
      }
      rs.assign((size_t)n + 1, 0);
      for (int64_t k = e0; k < e1; ++k) {
        const int32_t a = s->src[k], b = s->dst[k];
        if (a < 0 || a >= n || b < 0 || b >= n) { st[t] = HG_E_RANGE; bad[t] = g; break; }
        if (k > e0) {
          const int32_t pa = s->src[k - 1], pb = s->dst[k - 1];
          if (a < pa || (a == pa && b <= pb)) { st[t] = HG_E_UNSORTED; bad[t] = g; break; }
        }
        rs[a + 1]++;
      }
      if (st[t] != HG_OK) break;
      for (int64_t i = 0; i < n; ++i) {
        if (rs[i + 1] > HG_MAX_DEGREE) { st[t] = HG_E_DEGREE; bad[t] = g; break; }
        mxd[t] = std::max<int32_t>(mxd[t], rs[i + 1]);
        rs[i + 1] += rs[i];
      }
      if (st[t] != HG_OK) break;
      for (int64_t k = e0; k < e1; ++k) {
        const int32_t r = s->src[k], c = s->dst[k];
        // row c = edges with src == c, dst ascending: binary search for r
        const int32_t *lo = s->dst + e0 + rs[c], *hi = s->dst + e0 + rs[c + 1];
        const int32_t *p = std::lower_bound(lo, hi, r);
        if (p == hi || *p != r) { st[t] = HG_E_ASYMMETRIC; bad[t] = g; break; }
        const int64_t kk = p - s->dst;
        if (std::memcmp(s->ea + kk * s->Fe, s->ea + k * s->Fe, sizeof(float) * s->Fe) != 0) {
          st[t] = HG_E_ASYMMETRIC; bad[t] = g; break;
        }
        s->slot[k] = (uint8_t)(p - lo);
      }
    }
  });
  for (int t = 0; t < nt; ++t) {
    if (st[t] != HG_OK) {
      int64_t g = bad[t];
      const char *what = st[t] == HG_E_EMPTY ? "empty graph (SPEC.md:356)"
                         : st[t] == HG_E_RANGE ? "edge endpoint out of range"
                         : st[t] == HG_E_UNSORTED ? "edges not sorted by (src,dst)"
                         : st[t] == HG_E_DEGREE ? "degree exceeds HG_MAX_DEGREE"
                         : st[t] == HG_E_ASYMMETRIC ? "edge list not symmetric with identical attributes"
                                                     : "bad offsets";
      return fail(st[t], "store graph %lld: %s", (long long)g, what);
    }
    s->max_nodes = std::max(s->max_nodes, mxn[t]);
    s->max_deg = std::max(s->max_deg, mxd[t]);
  }
  s->slotp = s->slot.data();
  return HG_OK;
}
}  // namespace hg

using namespace hg;

extern "C" {

const char *hg_last_error(void) { return hg::t_err.c_str(); }
int32_t hg_abi_version(void) { return HG_ABI_VERSION; }

hg_status hg_store_create(const hg_store_desc *d, int32_t copy, int32_t threads, hg_store **out) {
  if (!d || !out) return fail(HG_E_INVALID, "null argument");
  *out = nullptr;
  if (d->num_graphs < 1) return fail(HG_E_EMPTY, "store has no graphs");
  if (d->num_nodes < 0 || d->num_edges < 0 || d->f_node < 1 || d->f_edge < 1)
    return fail(HG_E_INVALID, "bad sizes");
  if (!d->node_offset || !d->edge_offset || !d->x || !d->y || (d->num_edges && (!d->edge_index || !d->edge_attr)))
    return fail(HG_E_INVALID, "null array");
  const int64_t G = d->num_graphs;
  if (d->node_offset[0] != 0 || d->edge_offset[0] != 0 || d->node_offset[G] != d->num_nodes ||
      d->edge_offset[G] != d->num_edges)
    return fail(HG_E_SHAPE, "offsets must start at 0 and end at the totals");
  hg_store *s = new hg_store();
  s->G = G; s->N = d->num_nodes; s->E = d->num_edges; s->F0 = d->f_node; s->Fe = d->f_edge;
  if (copy) {
    s->own_no.assign(d->node_offset, d->node_offset + G + 1);
    s->own_eo.assign(d->edge_offset, d->edge_offset + G + 1);
    s->own_x.assign(d->x, d->x + s->N * s->F0);
    s->own_ea.assign(d->edge_attr, d->edge_attr + s->E * s->Fe);
    s->own_y.assign(d->y, d->y + G);
    if (d->y_node) s->own_yn.assign(d->y_node, d->y_node + s->N);
    s->own_ei.assign(d->edge_index, d->edge_index + 2 * s->E);
    s->no = s->own_no.data(); s->eo = s->own_eo.data(); s->x = s->own_x.data();
    s->ea = s->own_ea.data(); s->y = s->own_y.data();
    s->yn = d->y_node ? s->own_yn.data() : nullptr;
    s->src = s->own_ei.data(); s->dst = s->own_ei.data() + s->E;
  } else {
    s->no = d->node_offset; s->eo = d->edge_offset; s->x = d->x; s->ea = d->edge_attr; s->y = d->y;
    s->yn = d->y_node;
    s->src = d->edge_index; s->dst = d->edge_index + s->E;
  }
  hg_status fst = store_finish(s, threads);
  if (fst != HG_OK) {
    delete s;
    return fst;
  }
  *out = s;
  return HG_OK;
}

hg_status hg_store_destroy(hg_store *s) {
  delete s;
  return HG_OK;
}

hg_status hg_store_stats(const hg_store *s, int64_t *graphs, int64_t *nodes, int64_t *edges,
                         int32_t *max_nodes_per_graph, int32_t *max_degree) {
  if (!s) return fail(HG_E_INVALID, "null store");
  if (graphs) *graphs = s->G;
  if (nodes) *nodes = s->N;
  if (edges) *edges = s->E;
  if (max_nodes_per_graph) *max_nodes_per_graph = s->max_nodes;
  if (max_degree) *max_degree = s->max_deg;
  return HG_OK;
}

hg_status hg_degree_stat(const hg_store *s, const int64_t *ids, int64_t n, double *delta) {
  if (!s || !delta) return fail(HG_E_INVALID, "null argument");
  if (!ids) n = s->G;
  if (n < 1) return fail(HG_E_EMPTY, "no graphs");
  double tot = 0.0;
  int64_t cnt = 0;
  std::vector<int32_t> deg;
  for (int64_t q = 0; q < n; ++q) {
    const int64_t g = ids ? ids[q] : q;
    if (g < 0 || g >= s->G) return fail(HG_E_RANGE, "graph id %lld out of range", (long long)g);
    const int64_t nn = s->no[g + 1] - s->no[g];
    deg.assign((size_t)nn, 0);
    for (int64_t k = s->eo[g]; k < s->eo[g + 1]; ++k) deg[s->dst[k]]++;  // in-degree
    double part = 0.0;
    for (int64_t i = 0; i < nn; ++i) part += std::log((double)deg[i] + 1.0);
    tot += part;
    cnt += nn;
  }
  *delta = tot / (double)cnt;
  return HG_OK;
}

hg_status hg_degree_stat_linear(const hg_store *s, const int64_t *ids, int64_t n, double *delta_lin) {
  if (!s || !delta_lin) return fail(HG_E_INVALID, "null argument");
  if (!ids) n = s->G;
  if (n < 1) return fail(HG_E_EMPTY, "no graphs");
  int64_t ne = 0, nn = 0;
  for (int64_t q = 0; q < n; ++q) {
    const int64_t g = ids ? ids[q] : q;
    if (g < 0 || g >= s->G) return fail(HG_E_RANGE, "graph id %lld out of range", (long long)g);
    ne += s->eo[g + 1] - s->eo[g];  // symmetric edge lists: sum of in-degrees = directed edges
    nn += s->no[g + 1] - s->no[g];
  }
  *delta_lin = (double)ne / (double)nn;
  return HG_OK;
}

hg_status hg_shard(uint64_t seed, int64_t epoch, int32_t rank, int32_t world, int64_t n,
                   int64_t *ids_out, int64_t *n_out) {
  if (world < 1 || rank < 0 || rank >= world) return fail(HG_E_INVALID, "rank/world out of range");
  if (n < 0 || !ids_out || !n_out) return fail(HG_E_INVALID, "bad arguments");
  std::vector<std::pair<uint64_t, int64_t>> keys((size_t)n);
  const uint64_t base = seed ^ ((uint64_t)epoch * 0x9E3779B97F4A7C15ULL);
  for (int64_t i = 0; i < n; ++i) keys[i] = {splitmix64(base ^ ((uint64_t)i * 0xD1B54A32D192ED03ULL)), i};
  std::sort(keys.begin(), keys.end());
  const int64_t per = n / world;
  for (int64_t q = 0; q < per; ++q) ids_out[q] = keys[(size_t)(q * world + rank)].second;
  *n_out = per;
  return HG_OK;
}

hg_status hg_batch_offsets_get(int32_t B, int32_t N, int32_t E, int32_t f_node, int32_t f_edge,
                               hg_batch_offsets *off) {
  if (!off || B < 0 || N < 0 || E < 0) return fail(HG_E_INVALID, "bad arguments");
  BatchOffsets o = batch_offsets(B, N, E, f_node, f_edge);
  off->graph_ptr = o.graph_ptr; off->y = o.y; off->y_node = o.y_node; off->rowptr = o.rowptr; off->col = o.col;
  off->x = o.x; off->eattr = o.eattr; off->slot = o.slot; off->total = o.total;
  return HG_OK;
}

hg_status hg_pack_host(const hg_store *s, const int64_t *ids, int32_t B, const hg_config *cfg,
                       void *dst, size_t cap, size_t *used) {
  if (!s || !cfg || !dst) return fail(HG_E_INVALID, "null argument");
  if (B <= 0 || !ids) return fail(HG_E_EMPTY, "EmptyBatch (SPEC.md:279)");
  if (cfg->f_node != s->F0 || cfg->f_edge != s->Fe)
    return fail(HG_E_SHAPE, "feature widths (%d,%d) differ from the store's (%d,%d)", cfg->f_node,
                cfg->f_edge, s->F0, s->Fe);
  if (B > cfg->max_graphs) return fail(HG_E_CAPACITY, "B=%d exceeds max_graphs=%d", B, cfg->max_graphs);
  int64_t N = 0, E = 0;
  for (int32_t b = 0; b < B; ++b) {
    const int64_t g = ids[b];
    if (g < 0 || g >= s->G) return fail(HG_E_RANGE, "graph id %lld out of range", (long long)g);
    N += s->no[g + 1] - s->no[g];
    E += s->eo[g + 1] - s->eo[g];
  }
  if (N > cfg->max_nodes || E > cfg->max_edges)
    return fail(HG_E_CAPACITY, "batch N=%lld E=%lld exceeds capacity (%d, %d)", (long long)N, (long long)E,
                cfg->max_nodes, cfg->max_edges);
  const BatchOffsets o = batch_offsets(B, N, E, s->F0, s->Fe);
  if ((size_t)o.total > cap) return fail(HG_E_CAPACITY, "destination too small (%lld bytes needed)", (long long)o.total);
  uint8_t *base = (uint8_t *)dst;
  int32_t *hdr = (int32_t *)base;
  std::memset(hdr, 0, kHeaderInts * 4);
  hdr[0] = B; hdr[1] = (int32_t)N; hdr[2] = (int32_t)E; hdr[3] = s->F0; hdr[4] = s->Fe;
  int32_t *gp = (int32_t *)(base + o.graph_ptr);
  float *y = (float *)(base + o.y);
  float *yn = (float *)(base + o.y_node);
  int32_t *rp = (int32_t *)(base + o.rowptr);
  int32_t *col = (int32_t *)(base + o.col);
  float *x = (float *)(base + o.x);
  float *ea = (float *)(base + o.eattr);
  uint8_t *sl = base + o.slot;
  const int maxdeg = cfg->max_degree > 0 ? cfg->max_degree : HG_MAX_DEGREE;
  // graph b's node / edge offsets in the batch (prefix sums), then the graphs are
  // collated independently (in parallel: hg_pack_threads()); the bytes do not
  // depend on the thread count
  thread_local std::vector<int64_t> nbo, ebo;
  nbo.resize((size_t)B + 1);
  ebo.resize((size_t)B + 1);
  nbo[0] = ebo[0] = 0;
  for (int32_t b = 0; b < B; ++b) {
    const int64_t g = ids[b];
    nbo[b + 1] = nbo[b] + (s->no[g + 1] - s->no[g]);
    ebo[b + 1] = ebo[b] + (s->eo[g + 1] - s->eo[g]);
  }
  gp[0] = 0;
  rp[0] = 0;
  int32_t bad_b = -1;  // first offending graph in batch order
  int64_t bad_deg = 0;
  const int64_t *nbp = nbo.data(), *ebp = ebo.data();
  // degrees present in the batch (bitset over 0..HG_MAX_DEGREE): one degree class each
  thread_local std::vector<uint64_t> dbits;
  dbits.assign(2 * (size_t)B, 0);
  uint64_t *dbp = dbits.data();
#pragma omp parallel for num_threads(hg_pack_threads()) schedule(static) if (B >= 32)
  for (int32_t b = 0; b < B; ++b) {
    const int64_t g = ids[b], nb = nbp[b], eb = ebp[b];
    const int64_t n0 = s->no[g], n = s->no[g + 1] - n0, e0 = s->eo[g], e = s->eo[g + 1] - e0;
    y[b] = s->y[g];
    if (s->yn) std::memcpy(yn + nb, s->yn + n0, sizeof(float) * n);
    else std::memset(yn + nb, 0, sizeof(float) * n);
    std::memcpy(x + nb * s->F0, s->x + n0 * s->F0, sizeof(float) * n * s->F0);
    std::memcpy(ea + eb * s->Fe, s->ea + e0 * s->Fe, sizeof(float) * e * s->Fe);
    std::memcpy(sl + eb, s->slotp + e0, (size_t)e);
    // CSR row i (destination) = edges with src == i (symmetric store):
    // in-neighbours are their dst values, already ascending.
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t kstart = k;
      while (k < e && s->src[e0 + k] == i) {
        col[eb + k] = (int32_t)(s->dst[e0 + k] + nb);
        ++k;
      }
      if (k - kstart > maxdeg) {
#pragma omp critical
        if (bad_b < 0 || b < bad_b) { bad_b = b; bad_deg = k - kstart; }
      } else {
        const int64_t d = k - kstart;
        dbp[2 * b + (d >> 6)] |= 1ull << (d & 63);
      }
      rp[nb + i + 1] = (int32_t)(eb + k);
    }
    gp[b + 1] = (int32_t)(nb + n);
  }
  if (bad_b >= 0)
    return fail(HG_E_CAPACITY, "graph %lld has a node of degree %lld > max_degree %d", (long long)ids[bad_b],
                (long long)bad_deg, maxdeg);
  uint64_t d0 = 0, d1 = 0;
  for (int32_t b = 0; b < B; ++b) {
    d0 |= dbp[2 * b];
    d1 |= dbp[2 * b + 1];
  }
  const int ndeg = __builtin_popcountll(d0) + __builtin_popcountll(d1);
  if (ndeg > class_slots(*cfg))
    return fail(HG_E_DEGREE, "batch has %d distinct node degrees > %d degree-class slots", ndeg, class_slots(*cfg));
  if (used) *used = (size_t)o.total;
  return HG_OK;
}

hg_status hg_pack_threads_set(int32_t threads) {
  if (threads < 1 || threads > 1024) return fail(HG_E_INVALID, "threads must be in [1, 1024]");
  g_pack_threads.store(threads);
  return HG_OK;
}

hg_status hg_config_internal(const hg_config *c, hg_config *out) {
  hg_status st = check_config(c);
  if (st) return st;
  if (!out) return fail(HG_E_INVALID, "null output");
  *out = padded_config(*c);
  return HG_OK;
}

hg_status hg_param_layout(const hg_config *c, int32_t *n_tensors, int64_t *n_elems) {
  hg_status st = check_config(c);
  if (st) return st;
  auto lay = param_layout(*c);
  if (n_tensors) *n_tensors = (int32_t)lay.size();
  if (n_elems) *n_elems = param_total(lay);
  return HG_OK;
}

hg_status hg_param_layout_info(const hg_config *c, int32_t i, const char **name, int64_t *offset,
                               int32_t *rows, int32_t *cols) {
  hg_status st = check_config(c);
  if (st) return st;
  static thread_local std::vector<TensorInfo> lay;
  lay = param_layout(*c);
  if (i < 0 || i >= (int32_t)lay.size()) return fail(HG_E_RANGE, "tensor index out of range");
  if (name) *name = lay[i].name.c_str();
  if (offset) *offset = lay[i].offset;
  if (rows) *rows = lay[i].rows;
  if (cols) *cols = lay[i].cols;
  return HG_OK;
}

hg_status hg_params_init_host(const hg_config *c, uint64_t seed, float *dst) {
  hg_status st = check_config(c);
  if (st) return st;
  if (!dst) return fail(HG_E_INVALID, "null destination");
  init_params_host(*c, seed, dst);
  return HG_OK;
}

}  // extern "C"
