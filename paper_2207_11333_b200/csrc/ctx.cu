// ctx.cu — device context of the C-ABI: workspace plan, batch slots with an
// async H2D ring, the per-step kernel sequence (forward / backward / step),
// NCCL gradient averaging and CUDA-graph capture of a
// whole training step.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <cstring>
#include <string>
#include <vector>

#include "hgnn.h"
#include "internal.h"
#include "nvtx3/nvToolsExt.h"
#include "kernels.h"
#include "layout.h"

using namespace hg;
static_assert(kClassSlots == kMaxClasses, "degree-class slots (internal.h) == kernels.h");

namespace {

struct Plan {
  size_t params = 0, grads = 0, m = 0, v = 0, adam = 0, loss = 0;
  std::vector<size_t> slot;
  size_t blob_max = 0;
  std::vector<size_t> P, A, arg, X;  // X[l] = output of layer l (X_{l+1})
  size_t dA = 0;
  // per layer l: dZ[l] = dL/dX_l (degree-sorted rows), dP[l] and the dM_e block partials --
  // one buffer per layer so the side-stream readers never hold up the main chain (no
  // write-after-read waits)
  std::vector<size_t> dZ, dPl, pagg;
  size_t G = 0, hpre = 0, dhid = 0, yhat = 0, dy = 0, sqerr = 0;
  size_t part = 0, part2 = 0, part3 = 0, part2b = 0;  // split partials: spare, Gram (dU), dM_x, layer 0's Gram
  size_t eval_acc = 0;
  size_t u_off = 0, ux_off = 0;
  int cmax = 0;  // degree-class slots
  // per slot (computed when the slot's batch is uploaded, on the copy stream): the degree
  // sort's perm / pos, class table, GEMM tiles, Gram splits, per-graph ranges, node scalers
  std::vector<size_t> perm, pos, deginfo, tiles, splits, gslice, amp, att;
  size_t Wf = 0, WbT = 0;
  // residuals w - trunc19(w) of the weight operands (activations' lo terms are derived in
  // shared memory by the GEMM kernels)
  size_t Wf_lo = 0, WbT_lo = 0, ones = 0, xpad = 0;
  std::vector<size_t> Xs;          // per layer: X_l in degree-sorted rows (fused dX->dA path)
  std::vector<size_t> Xmask;       // per layer: ReLU mask bits of X_l, sorted rows, [N][H/32]
  size_t Mx_lo = 0, MxT = 0, MxT_lo = 0, mx_off = 0;
  size_t p2p = 0;  // P2PDev flags of the peer-memory gradient exchange
  size_t dm_scratch = 0;
  size_t nh_hpre = 0, nh_yn = 0, nh_sq = 0, nh_dyn = 0, nh_dhn = 0, nh_part = 0;  // node-level head
  size_t total = 0;
};

Plan make_plan(const hg_config &c) {
  Plan p;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = (size_t)align256((int64_t)(off + bytes));
    return o;
  };
  const auto lay = param_layout(c);
  const size_t PB = sizeof(float) * (size_t)param_total(lay);
  const size_t N = c.max_nodes, H = c.hidden, B = c.max_graphs, Hf = c.fc_hidden;
  Caps caps{c.max_graphs, c.max_nodes, c.max_edges, c.f_node, c.f_edge, c.hidden, c.fc_hidden};
  caps.S = n_scalers(c);
  caps.self_t = self_term(c) ? 1 : 0;
  const size_t KA = caps.KA(), PW = caps.PW();
  p.params = take(PB);
  p.grads = take(PB);
  p.m = take(PB);
  p.v = take(PB);
  p.adam = take(sizeof(AdamDev));
  p.p2p = take(sizeof(P2PDev));
  p.loss = take(sizeof(float) * 4);
  p.eval_acc = take(sizeof(double) * 4);  // evaluation sums: sq err, abs err, graphs
  p.blob_max = (size_t)batch_offsets(c.max_graphs, c.max_nodes, c.max_edges, c.f_node, c.f_edge).total;
  for (int s = 0; s < c.n_slots; ++s) p.slot.push_back(take(p.blob_max));
  for (int l = 0; l < c.layers; ++l) {
    p.P.push_back(take(sizeof(float) * N * PW));
    p.A.push_back(take(sizeof(float) * N * KA));
    p.arg.push_back(take(N * 2 * H));
    p.X.push_back(take(sizeof(float) * N * H));
  }
  const size_t Fmax = std::max<size_t>(H, c.f_node);
  for (int l = 0; l < c.layers; ++l) {
    p.dZ.push_back(take(sizeof(float) * N * Fmax));
    p.dPl.push_back(take(sizeof(float) * N * PW));
  }
  p.dA = take(sizeof(float) * N * KA);
  p.G = take(sizeof(float) * B * H);
  p.hpre = take(sizeof(float) * B * Hf);
  p.dhid = take(sizeof(float) * B * Hf);
  p.yhat = take(sizeof(float) * B);
  p.dy = take(sizeof(float) * B);
  p.sqerr = take(sizeof(float) * B);
  p.cmax = tc_num_classes(c.max_degree);
  p.u_off = take(sizeof(int64_t) * (size_t)c.layers);
  p.ux_off = take(sizeof(int64_t) * (size_t)c.layers);
  for (int s = 0; s < c.n_slots; ++s) {
    p.perm.push_back(take(sizeof(int) * N));
    p.pos.push_back(take(sizeof(int) * N));
    p.deginfo.push_back(take(sizeof(DegInfo)));
    p.gslice.push_back(take(sizeof(int4) * B));
    p.tiles.push_back(take(sizeof(int4) * (size_t)tc_max_tiles(caps, p.cmax)));
    p.splits.push_back(take(sizeof(int4) * (size_t)tc_max_splits(caps, p.cmax)));
    p.amp.push_back(take(sizeof(float) * N));
    p.att.push_back(take(sizeof(float) * N));
  }
  p.Wf = take(sizeof(float) * (size_t)c.layers * p.cmax * H * KA);
  p.WbT = take(sizeof(float) * (size_t)c.layers * p.cmax * H * KA);
  p.Wf_lo = take(sizeof(float) * (size_t)c.layers * p.cmax * H * KA);
  p.WbT_lo = take(sizeof(float) * (size_t)c.layers * p.cmax * H * KA);
  for (int l = 0; l < c.layers; ++l) {
    p.Xs.push_back(take(sizeof(float) * N * H));
    p.Xmask.push_back(take(sizeof(uint32_t) * N * ((H + 31) / 32)));
  }
  p.ones = take(sizeof(float) * N * 32);  // B operand of the column-sum tiles
  p.xpad = take(sizeof(float) * N * pad_x0_width(c.f_node));  // layer-0 features for the TMA dM_x Gram
  p.Mx_lo = take(sizeof(float) * (size_t)std::max(1, c.layers - 1) * PW * H);
  p.MxT = take(sizeof(float) * (size_t)std::max(1, c.layers - 1) * PW * H);
  p.MxT_lo = take(sizeof(float) * (size_t)std::max(1, c.layers - 1) * PW * H);
  p.mx_off = take(sizeof(int64_t) * (size_t)c.layers);
  size_t pf = std::max({mn_gram_partial_floats(caps, p.cmax), mn_dmx_partial_floats(caps, H),
                        mn_dmx_partial_floats(caps, c.f_node)});
  if (c.flags & HG_FLAG_NODE_HEAD) {
    pf = std::max(pf, mn_dmx_partial_floats(caps, H, Hf));  // (the node head's W1n Gram)
    p.nh_hpre = take(sizeof(float) * N * Hf);
    p.nh_dhn = take(sizeof(float) * N * Hf);
    p.nh_yn = take(sizeof(float) * N);
    p.nh_sq = take(sizeof(float) * N);
    p.nh_dyn = take(sizeof(float) * N);
    p.nh_part = take(sizeof(float) * node_head_partial_floats(caps));
  }
  p.part = take(sizeof(float) * 4);
  p.part2 = take(sizeof(float) * pf);
  p.part2b = take(sizeof(float) * pf);
  p.part3 = take(sizeof(float) * pf);
  for (int l = 0; l < c.layers; ++l) p.pagg.push_back(take(sizeof(float) * agg_bwd_partial_floats(caps)));
  p.dm_scratch = take(sizeof(float) * agg_bwd_dm_floats(caps));  // graphs too large to stage (agg.cu)
  p.total = off;
  return p;
}

}  // namespace

struct hg_ctx {
  hg_config cfg{};    // internal (padded) configuration the kernels run
  hg_config cfg_l{};  // the caller's configuration (logical widths)
  bool padded = false;
  Caps caps{};
  Plan plan;
  std::vector<TensorInfo> lay, lay_l;  // device arena layout / public (logical) layout
  int64_t n_params = 0, n_params_l = 0;
  int device = 0;
  uint8_t *ws = nullptr;
  cudaStream_t stream = nullptr, copy_stream = nullptr, cap_stream = nullptr;
  std::vector<void *> staging;
  std::vector<cudaEvent_t> copy_done, compute_done;
  std::vector<cudaGraphExec_t> graphs;
  std::vector<int64_t> graph_kernels;
  std::vector<hg_adamw> graph_hyper;
  std::vector<cudaGraphExec_t> eval_graphs;  // forward + metric accumulation per slot
  std::vector<int64_t> eval_kernels;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  cudaStream_t comm_stream = nullptr;           // bucketed allreduce overlapping the backward
  std::vector<cudaEvent_t> bucket_ready;         // per bucket (head, conv L-1 .. conv 0)
  cudaEvent_t comm_done = nullptr;
  cudaStream_t side_stream = nullptr, side2_stream = nullptr;  // weight-gradient GEMMs beside the critical chain
  cudaStream_t side3_stream = nullptr;  // layer 0's Gram (its own stream: it need not queue behind layer 1's)
  cudaStream_t adam_stream = nullptr;  // early AdamW of layers >= 1 (must not delay layer 0's side-stream work)
  bool p2p = false;                        // captured steps exchange over peer memory (hg_p2p_open)
  bool mv_sharded = false;                 // Adam moments valid on this rank's shard only (after p2p steps)
  uint8_t *peer_ws[kP2PMaxWorld] = {};     // every rank's workspace ([rank] = ws)
  void *peer_base[kP2PMaxWorld] = {};      // opened IPC mappings (closed at destroy)
  unsigned long long timeout_ns = 0;       // fail-stop bound of device flag waits and hg_sync (0 = none)
  std::vector<cudaEvent_t> ev_dz, ev_gram, ev_dp, ev_side, ev_dx, ev_upd, ev_pl;  // per layer fork / join points
  cudaEvent_t ev_head = nullptr, ev_prep = nullptr, ev_start = nullptr, ev_prepmx = nullptr, ev_prepw = nullptr,
              ev_ar1 = nullptr, ev_adam = nullptr;
  float *loss_ring = nullptr;  // pinned and mapped, HG_LOSS_RING entries
  float *loss_ring_dev = nullptr;  // its device address
  cudaEvent_t loss_ev[HG_LOSS_RING] = {};
  int64_t launches = 0;
  bool dxda = false;    // fused dX -> dA backward kernel (H == 128)
  hg_status sticky = HG_OK;
  std::string sticky_msg;

  float *f(size_t off) const { return reinterpret_cast<float *>(ws + off); }
  uint8_t *b(size_t off) const { return ws + off; }
  float *param(const std::string &name) const {
    for (auto &t : lay)
      if (t.name == name) return f(plan.params) + t.offset;
    return nullptr;
  }
  float *grad(const std::string &name) const {
    for (auto &t : lay)
      if (t.name == name) return f(plan.grads) + t.offset;
    return nullptr;
  }
};

namespace {

hg_status cuda_fail(hg_ctx *x, cudaError_t e, const char *what) {
  hg_status st = fail(HG_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  if (x) {
    x->sticky = HG_E_CUDA;
    x->sticky_msg = hg_last_error();
  }
  return st;
}

#define CK(x, call)                                   \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(x, e_, #call); \
  } while (0)

hg_status nccl_fail(hg_ctx *x, ncclResult_t r, const char *what) {
  hg_status st = fail(HG_E_NCCL, "%s: %s", what, ncclGetErrorString(r));
  if (x) {
    x->sticky = HG_E_NCCL;
    x->sticky_msg = hg_last_error();
  }
  return st;
}

hg_status usable(hg_ctx *x) {
  if (!x) return fail(HG_E_INVALID, "null ctx");
  if (x->sticky != HG_OK) return fail(HG_E_STATE, "ctx unusable after earlier failure: %s", x->sticky_msg.c_str());
  return HG_OK;
}

hg_status check_slot(hg_ctx *x, int32_t slot) {
  if (slot < 0 || slot >= x->cfg.n_slots) return fail(HG_E_RANGE, "slot %d out of range", slot);
  return HG_OK;
}

std::string lname(int l, const char *t) { return "conv" + std::to_string(l) + "." + t; }

// Instrumented (non-graph) mode: CUDA events around every kernel-class call
// (SURVEY §5 "phase timings"; SPEC.md:429-432 PhaseTimings).
struct Prof {
  cudaStream_t st;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  std::vector<int64_t> launches;
  Prof(cudaStream_t s) : st(s), launches(HG_PHASE_COUNT, 0) {}
  ~Prof() {
    for (auto &m : marks) {
      cudaEventDestroy(m.second.first);
      cudaEventDestroy(m.second.second);
    }
  }
};

template <class F>
void phase(Prof *pr, int ph, F &&fn) {
  if (!pr) {
    fn();
    return;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // external event nodes: the graph replay records them, so they can be timed
  cudaEventRecordWithFlags(a, pr->st, cudaEventRecordExternal);
  const int64_t l0 = launches_so_far();
  fn();
  pr->launches[ph] += launches_so_far() - l0;
  cudaEventRecordWithFlags(b, pr->st, cudaEventRecordExternal);
  pr->marks.push_back({ph, {a, b}});
}

hg_status enqueue_bucket(hg_ctx *x, cudaStream_t st, int b);
std::pair<int64_t, int64_t> bucket_range(hg_ctx *x, int b);
int bucket_count(const hg_ctx *x);
int bucket_closed_by(const hg_ctx *x, int l);

// ---- the step's kernel sequence (enqueue only) ----
// The batch's degree classes (stable sort by degree, class table with the configured scalers,
// GEMM tiles, Gram splits, per-graph ranges): a property of the packed batch like its
// reverse-edge slots, computed once per upload on the copy stream (one CTA beside the running
// step) into the slot's buffers instead of at the head of every step's critical chain. High
// priority: the next step waits for it, and at low priority the running step's kernels kept
// it off the SMs until that step ended.
void enqueue_degsort(hg_ctx *x, int slot, cudaStream_t st) {
  const Plan &p = x->plan;
  const hg_config &c = x->cfg;
  g_low_prio = false;
  launch_degsort(st, x->b(p.slot[slot]), c.delta, p.cmax, x->f(p.amp[slot]), x->f(p.att[slot]),
                 reinterpret_cast<int *>(x->b(p.perm[slot])), reinterpret_cast<DegInfo *>(x->b(p.deginfo[slot])),
                 reinterpret_cast<int4 *>(x->b(p.tiles[slot])), reinterpret_cast<int4 *>(x->b(p.splits[slot])),
                 reinterpret_cast<int *>(x->b(p.pos[slot])), reinterpret_cast<int4 *>(x->b(p.gslice[slot])),
                 scaler_mask(c), c.delta_lin, gram_ks(x->caps), x->caps.maxN);
  g_low_prio = false;
}

// node-level head (HG_FLAG_NODE_HEAD): forward, and with bwd its gradient into dZ_L (after the
// graph head wrote dZ_L), dyn and dhn for its parameter gradients (enqueue_node_head_grads)
void enqueue_node_head(hg_ctx *x, cudaStream_t st, int slot, bool bwd) {
  const Plan &p = x->plan;
  const int L = x->cfg.layers;
  launch_node_head(st, x->caps, x->b(p.slot[slot]), x->f(p.X[L - 1]), x->param("head_n.W1"), x->param("head_n.b1"),
                   x->param("head_n.W2"), x->param("head_n.b2"), x->cfg.node_weight, x->f(p.nh_hpre), x->f(p.nh_yn),
                   x->f(p.nh_sq), x->f(p.nh_dyn), x->f(p.nh_dhn), x->f(p.dZ[L - 1]),
                   reinterpret_cast<const int *>(x->b(p.pos[slot])), bwd);
}
void enqueue_node_head_grads(hg_ctx *x, cudaStream_t st, int slot, float *part) {
  const Plan &p = x->plan;
  const uint8_t *blob = x->b(p.slot[slot]);
  const int L = x->cfg.layers, H = x->cfg.hidden, Hf = x->cfg.fc_hidden;
  // dW1n = dhn^T X_L and db1n = sum dhn: the MN-major Gram over nodes (rows = Hf)
  launch_mn_dMx(st, x->caps, blob, x->f(p.nh_dhn), x->f(p.X[L - 1]), H, H, x->f(p.ones), part,
                x->grad("head_n.W1"), x->grad("head_n.b1"), Hf);
  // dW2n = sum dyn ReLU(hpre), db2n = sum dyn (b2n follows W2n in the arena: Hf % 64 == 0)
  launch_node_head_w2(st, x->caps, blob, x->f(p.nh_hpre), x->f(p.nh_dyn), x->f(p.nh_part));
  launch_reduce_cols(st, x->f(p.nh_part), node_head_chunks(x->caps), Hf + 4, Hf + 4, x->grad("head_n.W2"));
}

void enqueue_forward(hg_ctx *x, cudaStream_t st, int slot, Prof *pr = nullptr, bool fuse_head_bwd = false) {
  const hg_config &c = x->cfg;
  g_gemm_passes = (c.flags & HG_FLAG_TF32) ? 1 : 3;
  const Plan &p = x->plan;
  const uint8_t *blob = x->b(p.slot[slot]);
  const int *pos = reinterpret_cast<const int *>(x->b(p.pos[slot]));  // sorted A / dZ rows
  const DegInfo *dinfo = reinterpret_cast<const DegInfo *>(x->b(p.deginfo[slot]));
  const size_t HH = (size_t)c.hidden * c.hidden;
  // The batch's degree classes were computed when it was uploaded (enqueue_degsort, copy
  // stream). The class-weight / M_x preparation runs on side stream 2, concurrent with layer
  // 0's projection; the main chain joins the class weights before layer 0's update and M_x
  // before layer 1's projection.
  const bool fork = !pr && x->side_stream != nullptr;
  cudaStream_t wst = fork ? x->side2_stream : st;
  // the prep branch is enqueued after layer 0's projection so that the main chain is the
  // sort's first successor in the graph (measured: the other successor starts later)
  auto enqueue_prep = [&] {
    // (forked after layer 0's projection, ev_start, and enqueued after layer 0's aggregation so
    // that the main chain is the projection's first successor in the graph: a second root
    // branch, or the prep branch as the first successor, measured starting the other late)
    if (fork) cudaStreamWaitEvent(wst, x->ev_start, 0);
    phase(pr, HG_PHASE_SCALERS, [&] {  // (class weights belong with the scalers)
      // layer 0's weights first, at high priority (update_0 waits for them: at low priority they
      // ran only after agg_0 had drained); the rest at low priority
      g_low_prio = false;
      const int64_t *uo = reinterpret_cast<const int64_t *>(x->b(p.u_off));
      const int64_t *uxo = reinterpret_cast<const int64_t *>(x->b(p.ux_off));
      launch_prep_W2(wst, x->caps, x->f(p.params), uo, uxo, 0, 1, p.cmax, dinfo, x->f(p.Wf), x->f(p.Wf_lo),
                     x->f(p.WbT), x->f(p.WbT_lo));
      if (fork) cudaEventRecord(x->ev_prep, wst);
      g_low_prio = fork;
      launch_prep_Mx(wst, x->caps, x->f(p.params), reinterpret_cast<const int64_t *>(x->b(p.mx_off)), c.layers,
                     x->f(p.Mx_lo), x->f(p.MxT), x->f(p.MxT_lo));
      if (fork) cudaEventRecord(x->ev_prepmx, wst);
      launch_pad_x0(wst, x->caps, blob, x->f(p.xpad), x->dxda ? pos : nullptr);
      if (fork) cudaEventRecord(x->ev_prepw, wst);
      g_low_prio = false;
    });
  };
  for (int l = 0; l < c.layers; ++l) {
    const int F = l == 0 ? c.f_node : c.hidden;
    if (fork && l == 1) cudaStreamWaitEvent(st, x->ev_prepmx, 0);
    phase(pr, HG_PHASE_PROJ, [&] {
      if (l > 0)
        launch_d_proj(st, x->caps, blob, x->f(p.X[l - 1]), F, x->param(lname(l, "M_x")),
                      x->f(p.Mx_lo) + (size_t)(l - 1) * HH * (x->caps.self_t ? 2 : 1), x->f(p.P[l]));
      else
        launch_proj(st, x->caps, blob, nullptr, F, x->param(lname(l, "M_x")), x->f(p.P[l]));
    });
    if (fork && l == 0) cudaEventRecord(x->ev_start, st);
    phase(pr, HG_PHASE_AGG_FWD, [&] {
      launch_agg_fwd(st, x->caps, blob, reinterpret_cast<const int4 *>(x->b(p.gslice[slot])), x->f(p.P[l]),
                     x->param(lname(l, "M_e")), x->param(lname(l, "b_M")),
                     c.var_floor, x->f(p.A[l]), x->b(p.arg[l]), pos, l == 0 ? nullptr : x->f(p.X[l - 1]), F);
    });
    if (l == 0) enqueue_prep();
    if (fork && l == 0) cudaStreamWaitEvent(st, x->ev_prep, 0);
    if (fork && l == 1) cudaStreamWaitEvent(st, x->ev_prepw, 0);
    if (fork && l >= 1) cudaStreamWaitEvent(st, x->ev_pl[l], 0);
    phase(pr, HG_PHASE_UPDATE, [&] {
      const bool keep_sorted = x->dxda && l + 1 < c.layers;  // X_l operands of the fused dX -> dA kernel
      const size_t wl = (size_t)l * p.cmax * c.hidden * x->caps.KA();  // layer l's class weights
      launch_d_update_cls(st, x->caps, p.cmax, x->f(p.A[l]), reinterpret_cast<const int *>(x->b(p.perm[slot])),
                          dinfo, reinterpret_cast<const int4 *>(x->b(p.tiles[slot])), x->f(p.Wf) + wl,
                          x->f(p.Wf_lo) + wl,
                          x->param(lname(l, "b_U")), x->f(p.X[l]),
                          keep_sorted ? x->f(p.Xs[l]) : nullptr,
                          keep_sorted ? reinterpret_cast<uint32_t *>(x->b(p.Xmask[l])) : nullptr);
    });
    if (l + 1 < c.layers) {
      // layer l+1's class weights, on side stream 2 once update_l is done: they run beside
      // proj_{l+1} / agg_{l+1} instead of beside update_l, whose persistent TMA CTAs need whole
      // SMs (timeline, config B: all layers' weights prepared beside update_0 made it 30 us
      // instead of 16)
      if (fork) {
        cudaEventRecord(x->ev_upd[l], st);
        cudaStreamWaitEvent(wst, x->ev_upd[l], 0);
      }
      phase(pr, HG_PHASE_SCALERS, [&] {
        g_low_prio = fork;
        launch_prep_W2(wst, x->caps, x->f(p.params), reinterpret_cast<const int64_t *>(x->b(p.u_off)),
                       reinterpret_cast<const int64_t *>(x->b(p.ux_off)), l + 1, l + 2, p.cmax, dinfo, x->f(p.Wf),
                       x->f(p.Wf_lo), x->f(p.WbT), x->f(p.WbT_lo));
        g_low_prio = false;
      });
      if (fork) cudaEventRecord(x->ev_pl[l + 1], wst);
    }
  }
  if (fork && c.layers < 2) cudaStreamWaitEvent(st, x->ev_prepw, 0);  // join side stream 2
  phase(pr, HG_PHASE_HEAD_FWD, [&] {
    const bool nh = (c.flags & HG_FLAG_NODE_HEAD) != 0;
    if (fuse_head_bwd) {
      launch_head_fused(st, x->caps, blob, x->f(p.X[c.layers - 1]), x->param("head.W1"), x->param("head.b1"),
                        x->param("head.W2"), x->param("head.b2"), x->f(p.G), x->f(p.hpre), x->f(p.yhat),
                        x->f(p.sqerr), x->f(p.loss), x->f(p.dy), x->f(p.dhid), x->f(p.dZ[c.layers - 1]), pos);
      if (nh) enqueue_node_head(x, st, slot, true);  // (adds its part of dZ_L after the graph head's)
      // the loss value is an output only: reduce it on the side stream (joined at the end of the backward)
      if (fork) {
        cudaEventRecord(x->ev_head, st);
        cudaStreamWaitEvent(x->side_stream, x->ev_head, 0);
      }
      launch_loss(fork ? x->side_stream : st, blob, x->f(p.sqerr), x->f(p.loss), nh ? x->f(p.nh_sq) : nullptr,
                  c.node_weight);
    } else {
      if (nh) enqueue_node_head(x, st, slot, false);
      launch_head_fwd(st, x->caps, blob, x->f(p.X[c.layers - 1]), x->param("head.W1"), x->param("head.b1"),
                      x->param("head.W2"), x->param("head.b2"), x->f(p.G), x->f(p.hpre), x->f(p.yhat),
                      x->f(p.sqerr), x->f(p.loss), nh ? x->f(p.nh_sq) : nullptr, c.node_weight);
    }
  });
}

void enqueue_step(hg_ctx *x, cudaStream_t st, const hg_adamw &h, Prof *pr, int64_t b, int64_t e, bool advance);
int64_t layer1_offset(const hg_ctx *x);
void enqueue_backward(hg_ctx *x, cudaStream_t st, int slot, Prof *pr = nullptr, bool head_done = false,
                      bool overlap_allreduce = false, const hg_adamw *early_adamw = nullptr) {
  const hg_config &c = x->cfg;
  g_gemm_passes = (c.flags & HG_FLAG_TF32) ? 1 : 3;
  const Plan &p = x->plan;
  const uint8_t *blob = x->b(p.slot[slot]);
  const int *pos = reinterpret_cast<const int *>(x->b(p.pos[slot]));  // sorted A / dZ rows
  const size_t HH = (size_t)c.hidden * c.hidden;
  const bool fork = !pr && x->side_stream != nullptr;
  cudaStream_t side = fork ? x->side_stream : st, side2 = fork ? x->side2_stream : st;
  auto rec = [&](cudaEvent_t ev, cudaStream_t s) { if (fork) cudaEventRecord(ev, s); };
  auto wait = [&](cudaStream_t s, cudaEvent_t ev) { if (fork) cudaStreamWaitEvent(s, ev, 0); };
  bool adam_forked = false;
  phase(pr, HG_PHASE_HEAD_BWD, [&] {
    if (!head_done) {  // dZ of the last layer on the main stream
      launch_head_bwd(st, x->caps, blob, x->f(p.X[c.layers - 1]), x->param("head.W1"), x->param("head.W2"),
                      x->f(p.G), x->f(p.hpre), x->f(p.yhat), x->f(p.dy), x->f(p.dhid), x->f(p.dZ[c.layers - 1]),
                      x->grad("head.W1"), x->grad("head.b1"), x->grad("head.W2"), x->grad("head.b2"), false, pos,
                      false);
      if (c.flags & HG_FLAG_NODE_HEAD) enqueue_node_head(x, st, slot, true);
    }
    rec(x->ev_head, st);
    wait(side, x->ev_head);
    g_low_prio = fork;
    // head parameter gradients: off the critical chain
    launch_head_grads(side, x->caps, blob, x->f(p.G), x->f(p.hpre), x->f(p.dy), x->f(p.dhid), x->grad("head.W1"),
                      x->grad("head.b1"), x->grad("head.W2"), x->grad("head.b2"));
    if (c.flags & HG_FLAG_NODE_HEAD) enqueue_node_head_grads(x, side, slot, x->f(p.part2));
    g_low_prio = false;
  });
  const int *perm = reinterpret_cast<const int *>(x->b(p.perm[slot]));
  const DegInfo *dinfo = reinterpret_cast<const DegInfo *>(x->b(p.deginfo[slot]));
  const int4 *tiles = reinterpret_cast<const int4 *>(x->b(p.tiles[slot]));
  // Weight-gradient GEMMs (dU / db_U from the class Gram, dM_x / db_M) feed only the
  // exchange and AdamW, so they run on low-priority side streams while the main stream
  // walks the critical chain dA -> agg_bwd -> dX of each layer.
  // Hazards: dX_l overwrites the dZ buffer Gram_{l+1} read; agg_bwd_l overwrites the dP
  // dM_x(l+1) read -> one buffer per layer (Plan), so no write-after-read waits.
  float *part_dU = x->f(p.part2), *part_dMx = x->f(p.part3);  // (one per side stream)
  for (int l = c.layers - 1; l >= 0; --l) {
    float *dZ = x->f(p.dZ[l]);
    float *dP = x->f(p.dPl[l]), *pagg = x->f(p.pagg[l]);
    // ---- side: Gram (dU, db_U) as soon as dZ_l is ready (layer 0's on a stream of its own:
    // behind layer 1's Gram and reduction it started ~18 us after dZ_0, in the step's tail)
    cudaStream_t gs = (fork && l == 0) ? x->side3_stream : side;
    rec(x->ev_dz[l], st);
    wait(gs, x->ev_dz[l]);
    g_low_prio = fork;
    phase(pr, HG_PHASE_DU, [&] {  // (side stream 1)
      // layer 0's Gram ends the step (only agg_bwd_0 and dM_x0 run beside it): every SM
      g_mn_grid_override = l == 0 ? kNumSMs : 0;
      launch_mn_dU_cls(gs, x->caps, p.cmax, dZ, x->f(p.A[l]), x->f(p.ones), dinfo,
                       reinterpret_cast<const int4 *>(x->b(p.splits[slot])), gs == side ? part_dU : x->f(p.part2b),
                       x->grad(lname(l, "U")),
                       x->grad(lname(l, "b_U")), x->caps.self_t ? x->grad(lname(l, "U_x")) : nullptr,
                       l == 0 ? c.f_node : c.hidden);
      g_mn_grid_override = 0;
    });
    rec(x->ev_gram[l], gs);
    g_low_prio = false;
    // ---- main: dA, aggregation backward
    phase(pr, HG_PHASE_DA, [&] {
      if (!(x->dxda && l + 1 < c.layers))  // (else dA_l came with dZ_l from layer l+1's fused dX -> dA)
        launch_d_dA_cls(st, x->caps, p.cmax, dZ, perm, dinfo, tiles,
                        x->f(p.WbT) + (size_t)l * p.cmax * c.hidden * x->caps.KA(),
                        x->f(p.WbT_lo) + (size_t)l * p.cmax * c.hidden * x->caps.KA(), x->f(p.dA));
    });
    phase(pr, HG_PHASE_AGG_BWD, [&] {
      launch_agg_bwd(st, x->caps, blob, reinterpret_cast<const int4 *>(x->b(p.gslice[slot])), x->f(p.P[l]),
                     x->param(lname(l, "M_e")), x->param(lname(l, "b_M")),
                     x->f(p.A[l]), x->b(p.arg[l]), x->f(p.dA), dP, pagg, pos, x->dxda ? pos : nullptr,
                     x->f(p.dm_scratch));
    });
    const int F = l == 0 ? c.f_node : c.hidden;
    // ---- side stream 2: dM_e, dM_x, db_M once dP_l is ready; with Gram_l done, layer l is complete
    rec(x->ev_dp[l], st);
    wait(side2, x->ev_dp[l]);
    g_low_prio = fork;
    phase(pr, HG_PHASE_DMX, [&] {
      // layer 0 on one GPU: off the step's final dM_x chain, on the idle AdamW stream (with W > 1
      // the conv0 bucket's allreduce is enqueued on side stream 2 and must follow dM_e)
      if (l == 0 && adam_forked && !x->comm) {
        wait(x->adam_stream, x->ev_dp[0]);
        launch_reduce_dMe(x->adam_stream, x->caps, pagg, x->grad(lname(l, "M_e")), x->grad(lname(l, "b_M")));
        rec(x->ev_adam, x->adam_stream);
      } else {
        launch_reduce_dMe(side2, x->caps, pagg, x->grad(lname(l, "M_e")), x->grad(lname(l, "b_M")));
      }
      // MN-major TMA Gram dM_x = dP^T X (db_M comes from the aggregation partials);
      // fused dX -> dA path: dP rows are degree-sorted, so X comes in sorted rows too
      const float *Xg = l > 0 ? x->f(x->dxda ? p.Xs[l - 1] : p.X[l - 1]) : x->f(p.xpad);
      g_mn_grid_override = l == 0 ? kNumSMs : 0;  // layer 0's dM_x runs after the last main-chain kernel
      launch_mn_dMx(side2, x->caps, blob, dP, Xg, F, l > 0 ? F : pad_x0_width(c.f_node), x->f(p.ones), part_dMx,
                    x->grad(lname(l, "M_x")), nullptr);
      g_mn_grid_override = 0;
    });
    g_low_prio = false;
    const int bk = bucket_closed_by(x, l);
    if (overlap_allreduce && bk >= 0) {  // conv l's gradients complete: its bucket may go
      wait(side2, x->ev_gram[l]);
      enqueue_bucket(x, side2, bk);
      if (x->comm && l == 1) rec(x->ev_ar1, x->comm_stream);  // layers >= 1 averaged
    }
    rec(x->ev_side[l], side2);
    // ---- main: dX into dZ[l-1]
    if (l > 0) {
      float *dZn = x->f(p.dZ[l - 1]);
      phase(pr, HG_PHASE_DX, [&] {
        if (x->dxda)
          launch_dxda(st, x->caps, p.cmax, dP, x->f(p.MxT) + (size_t)(l - 1) * HH,
                      x->f(p.MxT_lo) + (size_t)(l - 1) * HH, x->f(p.WbT) + (size_t)(l - 1) * p.cmax * 4 * HH,
                      x->f(p.WbT_lo) + (size_t)(l - 1) * p.cmax * 4 * HH, perm, dinfo, tiles,
                      reinterpret_cast<const uint32_t *>(x->b(p.Xmask[l - 1])), dZn, x->f(p.dA));
        else
          launch_d_dX(st, x->caps, blob, dP, x->f(p.MxT) + (size_t)(l - 1) * HH * (x->caps.self_t ? 2 : 1),
                      x->f(p.MxT_lo) + (size_t)(l - 1) * HH * (x->caps.self_t ? 2 : 1), F, x->f(p.X[l - 1]), dZn, pos,
                      x->caps.self_t ? x->f(p.dA) + 4 * c.hidden : nullptr);
      });
      if (early_adamw && fork && l == 1) {
        // every parameter of layers >= 1 and the head is final (and averaged) and no longer
        // read by this step (dX_1 was the last reader): update them now, off the critical
        // chain; conv0's parameters follow after the backward (that launch advances the step)
        // (own stream: on side stream 2 it delayed layer 0's dM_x chain at the step's end)
        cudaStream_t as = x->adam_stream;
        rec(x->ev_dx[1], st);
        wait(as, x->ev_dx[1]);
        wait(as, x->ev_gram[1]);
        wait(as, x->ev_side[1]);
        if (x->comm) wait(as, x->ev_ar1);  // (layer 1 closes a bucket)
        g_low_prio = true;
        enqueue_step(x, as, *early_adamw, nullptr, layer1_offset(x), -1, false);
        g_low_prio = false;
        rec(x->ev_adam, as);
        adam_forked = true;
      }
    }
  }
  // join: every gradient is complete on the main stream (layer 0's Gram runs on its own stream,
  // so the side stream's last Gram, layer 1's, is joined explicitly)
  wait(st, x->ev_gram[0]);
  if (c.layers > 1) wait(st, x->ev_gram[1]);
  wait(st, x->ev_side[0]);
  if (adam_forked) wait(st, x->ev_adam);
}

// Gradient buckets in backward order. Bucket 0 holds the head and the first groups[0]
// conv layers (L-1, L-2, ...), bucket k the next groups[k] layers; a bucket is averaged on
// the comm stream once its lowest layer's gradients are final. Layer pairs, the last two
// layers alone (measured best at 2 GPUs, config B). Buckets are contiguous
// ranges of the flat arena and together cover it exactly (hg_bucket_layout, tested).
std::vector<int> bucket_groups_for(int L) {
  std::vector<int> g;
  int rest = L;
  while (rest > 2) {
    const int v = std::min(2, rest - 2);
    g.push_back(v);
    rest -= v;
  }
  while (rest-- > 0) g.push_back(1);
  return g;
}
std::vector<int> bucket_groups(const hg_ctx *x) { return bucket_groups_for(x->cfg.layers); }
int bucket_count(const hg_ctx *x) { return (int)bucket_groups(x).size(); }
// bucket that completes when layer l's gradients are final, or -1
int bucket_closed_by(const hg_ctx *x, int l) {
  const auto g = bucket_groups(x);
  int top = x->cfg.layers;  // layers [top - g[k], top) belong to bucket k
  for (int k = 0; k < (int)g.size(); ++k) {
    top -= g[k];
    if (l == top) return k;
  }
  return -1;
}
// float range [beg, end) of bucket b in the arena layout `lay` (n = arena floats)
std::pair<int64_t, int64_t> bucket_range_of(const std::vector<TensorInfo> &lay, int64_t n, int L, int b) {
  auto off = [&](const std::string &name) {
    for (auto &t : lay)
      if (t.name == name) return t.offset;
    return (int64_t)-1;
  };
  const auto g = bucket_groups_for(L);
  int top = L;
  for (int k = 0; k < b; ++k) top -= g[k];
  const int lo = top - g[b];
  const int64_t beg = off(lname(lo, "M_x"));
  const int64_t end = b == 0 ? n : off(lname(top, "M_x"));
  return {beg, end};
}
std::pair<int64_t, int64_t> bucket_range(hg_ctx *x, int b) {
  return bucket_range_of(x->lay, x->n_params, x->cfg.layers, b);
}

// enqueue the average of bucket b on the comm stream once the compute stream reaches this point
hg_status enqueue_bucket(hg_ctx *x, cudaStream_t st, int b) {
  if (!x->comm) return HG_OK;
  auto r = bucket_range(x, b);
  cudaError_t e;
  if ((e = cudaEventRecord(x->bucket_ready[b], st)) != cudaSuccess) return cuda_fail(x, e, "cudaEventRecord");
  if ((e = cudaStreamWaitEvent(x->comm_stream, x->bucket_ready[b], 0)) != cudaSuccess)
    return cuda_fail(x, e, "cudaStreamWaitEvent");
  float *g = x->f(x->plan.grads) + r.first;
  ncclResult_t nr = ncclAllReduce(g, g, (size_t)(r.second - r.first), ncclFloat32, ncclAvg, x->comm, x->comm_stream);
  if (nr != ncclSuccess) return nccl_fail(x, nr, "ncclAllReduce");
  return HG_OK;
}

// join: the compute stream waits for every bucket's average
hg_status join_buckets(hg_ctx *x, cudaStream_t st) {
  if (!x->comm) return HG_OK;
  cudaError_t e;
  if ((e = cudaEventRecord(x->comm_done, x->comm_stream)) != cudaSuccess) return cuda_fail(x, e, "cudaEventRecord");
  if ((e = cudaStreamWaitEvent(st, x->comm_done, 0)) != cudaSuccess) return cuda_fail(x, e, "cudaStreamWaitEvent");
  return HG_OK;
}

hg_status enqueue_allreduce(hg_ctx *x, cudaStream_t st) {
  if (!x->comm) return HG_OK;
  ncclResult_t r = ncclAllReduce(x->f(x->plan.grads), x->f(x->plan.grads), (size_t)x->n_params, ncclFloat32, ncclAvg,
                                 x->comm, st);
  if (r != ncclSuccess) return nccl_fail(x, r, "ncclAllReduce");
  return HG_OK;
}

// AdamW over parameters [b, e) of the flat arena (default: all); `advance` = this launch
// is the step's last and advances the step counter
void enqueue_step(hg_ctx *x, cudaStream_t st, const hg_adamw &h, Prof *pr = nullptr, int64_t b = 0, int64_t e = -1,
                  bool advance = true) {
  const Plan &p = x->plan;
  if (e < 0) e = x->n_params;
  phase(pr, HG_PHASE_ADAMW, [&] {
    launch_adamw(st, x->f(p.params) + b, x->f(p.grads) + b, x->f(p.m) + b, x->f(p.v) + b, e - b,
                 reinterpret_cast<AdamDev *>(x->b(p.adam)), h.lr, h.beta1, h.beta2, h.eps, h.weight_decay, advance);
  });
}
// peer-memory exchange arguments; peers = every rank's workspace (mapped or, emulated, local)
P2PArgs p2p_args_of(hg_ctx *x, uint8_t *const *peers, int world, int rank, const hg_adamw &h) {
  P2PArgs a{};
  const Plan &p = x->plan;
  for (int q = 0; q < world; ++q) {
    a.params[q] = reinterpret_cast<float *>(peers[q] + p.params);
    a.grads[q] = reinterpret_cast<const float *>(peers[q] + p.grads);
    a.dev[q] = reinterpret_cast<P2PDev *>(peers[q] + p.p2p);
    a.m_all[q] = reinterpret_cast<const float *>(peers[q] + p.m);
    a.v_all[q] = reinterpret_cast<const float *>(peers[q] + p.v);
  }
  a.m = x->f(p.m);
  a.v = x->f(p.v);
  a.ad = reinterpret_cast<AdamDev *>(x->b(p.adam));
  a.world = world;
  a.rank = rank;
  a.n4 = x->n_params / 4;
  a.timeout_ns = x->timeout_ns;
  a.lr = h.lr; a.beta1 = h.beta1; a.beta2 = h.beta2; a.eps = h.eps; a.wd = h.weight_decay;
  return a;
}
P2PArgs p2p_args(hg_ctx *x, const hg_adamw &h) { return p2p_args_of(x, x->peer_ws, x->world, x->rank, h); }
int64_t layer1_offset(const hg_ctx *x) {  // start of conv1's parameters (conv0's come first)
  for (auto &t : x->lay)
    if (t.name == lname(1, "M_x")) return t.offset;
  return x->n_params;
}

hg_status after_enqueue(hg_ctx *x, const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(x, e, what);
  return HG_OK;
}

// moments sharded by earlier peer-memory steps: gather the peers' shards (stream-ordered
// after the last exchange, whose final done-wait guarantees the peers' shards are written)
hg_status gather_moments(hg_ctx *x) {
  if (!x->mv_sharded) return HG_OK;
  launch_p2p_gather_moments(x->stream, p2p_args(x, hg_adamw{}));
  x->launches += 1;
  hg_status st = after_enqueue(x, "moment gather");
  if (st == HG_OK) x->mv_sharded = false;
  return st;
}

}  // namespace

// ---------------------------------------------------------------- checkpoint
// Little-endian file: "HGNNCKPT" | u32 version | the model part of hg_config | u32 n_tensors |
// per tensor (u16 name length, name, i64 offset, i32 rows, i32 cols) | i64 n_elems |
// f32 params[n] | i64 Adam step | f32 m[n] | f32 v[n] | u32 CRC-32C of everything before it.
namespace hg {
namespace {
constexpr char kCkptMagic[8] = {'H', 'G', 'N', 'N', 'C', 'K', 'P', 'T'};
constexpr uint32_t kCkptVersion = 1;
struct CkptModel {  // the configuration fields that fix the parameter layout and the arithmetic
  int32_t f_node, f_edge, hidden, layers, fc_hidden, flags, scalers, pad;
  double delta, delta_lin;
  float var_floor, node_weight;
};
CkptModel ckpt_model(const hg_config &c) {
  CkptModel m{};
  m.f_node = c.f_node; m.f_edge = c.f_edge; m.hidden = c.hidden; m.layers = c.layers; m.fc_hidden = c.fc_hidden;
  m.flags = c.flags; m.scalers = c.scalers; m.delta = c.delta; m.delta_lin = c.delta_lin;
  m.var_floor = c.var_floor; m.node_weight = c.node_weight;
  return m;
}
template <class T>
void put(std::vector<uint8_t> &b, const T &v) {
  const uint8_t *p = reinterpret_cast<const uint8_t *>(&v);
  b.insert(b.end(), p, p + sizeof(T));
}
void put_bytes(std::vector<uint8_t> &b, const void *p, size_t n) {
  b.insert(b.end(), (const uint8_t *)p, (const uint8_t *)p + n);
}
struct Reader {
  const std::vector<uint8_t> &b;
  size_t at = 0;
  bool ok = true;
  template <class T>
  T get() {
    T v{};
    if (at + sizeof(T) > b.size()) { ok = false; return v; }
    std::memcpy(&v, b.data() + at, sizeof(T));
    at += sizeof(T);
    return v;
  }
  const uint8_t *bytes(size_t n) {
    if (at + n > b.size()) { ok = false; return nullptr; }
    const uint8_t *p = b.data() + at;
    at += n;
    return p;
  }
};
}  // namespace
}  // namespace hg

namespace hg {
// NVTX range over one public call (SURVEY §5 tracing): shows the host API calls on an nsys /
// ncu timeline beside the kernels; a no-op unless a tool is attached
struct Range {
  explicit Range(const char *name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};
}  // namespace hg

extern "C" {

hg_status hg_workspace_bytes(const hg_config *c, size_t *bytes) {
  hg_status st = check_config(c);
  if (st) return st;
  if (!bytes) return fail(HG_E_INVALID, "null output");
  *bytes = make_plan(padded_config(*c)).total;
  return HG_OK;
}

hg_status hg_ctx_create(const hg_config *c, int32_t device, void *workspace, size_t bytes, void *stream,
                        hg_ctx **out) {
  hg_status st = check_config(c);
  if (st) return st;
  if (!out || !workspace) return fail(HG_E_INVALID, "null argument");
  *out = nullptr;
  const hg_config cl = *c;
  const hg_config pc = padded_config(cl);
  c = &pc;
  Plan plan = make_plan(*c);
  if (bytes < plan.total) return fail(HG_E_CAPACITY, "workspace too small: %zu < %zu", bytes, plan.total);
  if (((uintptr_t)workspace & 255) != 0) return fail(HG_E_INVALID, "workspace must be 256-byte aligned");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
  hg_ctx *x = new hg_ctx();
  x->cfg = *c;
  x->cfg_l = cl;
  x->padded = config_is_padded(cl);
  x->caps = Caps{c->max_graphs, c->max_nodes, c->max_edges, c->f_node, c->f_edge, c->hidden, c->fc_hidden, cl.hidden};
  x->caps.S = n_scalers(*c);
  x->caps.self_t = self_term(*c) ? 1 : 0;
  x->plan = plan;
  x->lay = param_layout(*c);
  x->n_params = param_total(x->lay);
  x->lay_l = param_layout(cl);
  x->n_params_l = param_total(x->lay_l);
  x->device = device;
  x->ws = (uint8_t *)workspace;
  x->stream = (cudaStream_t)stream;
  auto bail = [&](cudaError_t err, const char *what) {
    hg_status s2 = cuda_fail(nullptr, err, what);
    hg_ctx_destroy(x);
    return s2;
  };
  if ((e = cudaStreamCreateWithFlags(&x->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return bail(e, "cudaStreamCreate");
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if ((e = cudaStreamCreateWithPriority(&x->cap_stream, cudaStreamNonBlocking, prio_hi)) != cudaSuccess)
    return bail(e, "cudaStreamCreate");
  if ((e = cudaStreamCreateWithPriority(&x->side_stream, cudaStreamNonBlocking, prio_lo)) != cudaSuccess)
    return bail(e, "cudaStreamCreate");
  if ((e = cudaStreamCreateWithPriority(&x->side3_stream, cudaStreamNonBlocking, prio_lo)) != cudaSuccess)
    return bail(e, "cudaStreamCreate");
  if ((e = cudaStreamCreateWithPriority(&x->side2_stream, cudaStreamNonBlocking, prio_lo)) != cudaSuccess)
    return bail(e, "cudaStreamCreate");
  if ((e = cudaStreamCreateWithPriority(&x->adam_stream, cudaStreamNonBlocking, prio_lo)) != cudaSuccess)
    return bail(e, "cudaStreamCreate");
  g_prio_lo = prio_lo;
  g_prio_hi = prio_hi;
  for (cudaEvent_t *ev : {&x->ev_head, &x->ev_prep, &x->ev_start, &x->ev_prepmx, &x->ev_prepw, &x->ev_ar1, &x->ev_adam})
    if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "cudaEventCreate");
  if ((e = cudaHostAlloc((void **)&x->loss_ring, sizeof(float) * HG_LOSS_RING, cudaHostAllocMapped)) != cudaSuccess ||
      (e = cudaHostGetDevicePointer((void **)&x->loss_ring_dev, x->loss_ring, 0)) != cudaSuccess)
    return bail(e, "cudaHostAlloc");
  for (int i = 0; i < HG_LOSS_RING; ++i)
    if ((e = cudaEventCreateWithFlags(&x->loss_ev[i], cudaEventDisableTiming)) != cudaSuccess)
      return bail(e, "cudaEventCreate");
  for (auto *v : {&x->ev_dz, &x->ev_gram, &x->ev_dp, &x->ev_side, &x->ev_dx, &x->ev_upd, &x->ev_pl})
    for (int l = 0; l < c->layers; ++l) {
      cudaEvent_t ev;
      if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "cudaEventCreate");
      v->push_back(ev);
    }
  for (int s = 0; s < c->n_slots; ++s) {
    void *h = nullptr;
    if ((e = cudaHostAlloc(&h, plan.blob_max, cudaHostAllocDefault)) != cudaSuccess) return bail(e, "cudaHostAlloc");
    x->staging.push_back(h);
    cudaEvent_t a, b2;
    if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "cudaEventCreate");
    x->copy_done.push_back(a);
    if ((e = cudaEventCreateWithFlags(&b2, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "cudaEventCreate");
    x->compute_done.push_back(b2);
    x->graphs.push_back(nullptr);
    x->graph_kernels.push_back(0);
    x->eval_graphs.push_back(nullptr);
    x->eval_kernels.push_back(0);
    x->graph_hyper.push_back(hg_adamw{});
  }
  if ((e = cudaMemsetAsync(workspace, 0, plan.total, x->stream)) != cudaSuccess) return bail(e, "cudaMemsetAsync");
  head_configure(x->caps);
  if ((e = tcd_configure()) != cudaSuccess) return bail(e, "tcd_configure");
  if ((e = agg_configure()) != cudaSuccess) return bail(e, "agg_configure");
  if ((e = degsort_configure()) != cudaSuccess) return bail(e, "degsort_configure");
  x->dxda = dxda_supported(x->caps);  // fused dX -> dA backward: +2.3% at config B
  {
    std::vector<int64_t> uo, mo, uxo((size_t)c->layers, 0);
    for (int l = 0; l < c->layers; ++l)
      for (auto &t : x->lay) {
        if (t.name == lname(l, "U")) uo.push_back(t.offset);
        if (t.name == lname(l, "M_x")) mo.push_back(t.offset);
        if (t.name == lname(l, "U_x")) uxo[l] = t.offset;
        // the kernels read [M_x; M_s] as one 2H-row matrix (projection, dX, dM): adjacent tensors
        if (t.name == lname(l, "M_s") && t.offset != mo.back() + (int64_t)c->hidden * (l == 0 ? c->f_node : c->hidden)) {
          hg_ctx_destroy(x);
          return fail(HG_E_INVALID, "internal: M_s not adjacent to M_x");
        }
      }
    std::vector<float> one((size_t)c->max_nodes * 32, 1.0f);
    if ((e = cudaMemcpyAsync(x->b(plan.u_off), uo.data(), sizeof(int64_t) * uo.size(), cudaMemcpyHostToDevice,
                             x->stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(x->b(plan.mx_off), mo.data(), sizeof(int64_t) * mo.size(), cudaMemcpyHostToDevice,
                             x->stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(x->b(plan.ux_off), uxo.data(), sizeof(int64_t) * uxo.size(), cudaMemcpyHostToDevice,
                             x->stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(x->b(plan.ones), one.data(), sizeof(float) * one.size(), cudaMemcpyHostToDevice,
                             x->stream)) != cudaSuccess)
      return bail(e, "cudaMemcpyAsync");
    if ((e = cudaStreamSynchronize(x->stream)) != cudaSuccess) return bail(e, "cudaStreamSynchronize");
  }
  *out = x;
  return HG_OK;
}

hg_status hg_ctx_destroy(hg_ctx *x) {
  if (!x) return HG_OK;
  if (x->stream || x->copy_stream) cudaDeviceSynchronize();
  for (auto g : x->graphs)
    if (g) cudaGraphExecDestroy(g);
  for (auto g : x->eval_graphs)
    if (g) cudaGraphExecDestroy(g);
  for (auto h : x->staging) cudaFreeHost(h);
  for (auto ev : x->copy_done) cudaEventDestroy(ev);
  for (auto ev : x->compute_done) cudaEventDestroy(ev);
  if (x->copy_stream) cudaStreamDestroy(x->copy_stream);
  if (x->cap_stream) cudaStreamDestroy(x->cap_stream);
  if (x->side_stream) cudaStreamDestroy(x->side_stream);
  if (x->side2_stream) cudaStreamDestroy(x->side2_stream);
  if (x->side3_stream) cudaStreamDestroy(x->side3_stream);
  if (x->adam_stream) cudaStreamDestroy(x->adam_stream);
  for (auto *v : {&x->ev_dz, &x->ev_gram, &x->ev_dp, &x->ev_side, &x->ev_dx, &x->ev_upd, &x->ev_pl})
    for (auto ev : *v) cudaEventDestroy(ev);
  for (cudaEvent_t ev : {x->ev_head, x->ev_prep, x->ev_start, x->ev_prepmx, x->ev_prepw, x->ev_ar1, x->ev_adam})
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : x->loss_ev)
    if (ev) cudaEventDestroy(ev);
  if (x->loss_ring) cudaFreeHost(x->loss_ring);
  if (x->comm) ncclCommDestroy(x->comm);
  for (void *b : x->peer_base)
    if (b) cudaIpcCloseMemHandle(b);
  for (auto ev : x->bucket_ready) cudaEventDestroy(ev);
  if (x->comm_done) cudaEventDestroy(x->comm_done);
  if (x->comm_stream) cudaStreamDestroy(x->comm_stream);
  delete x;
  return HG_OK;
}

hg_status hg_param_count(const hg_ctx *x, int32_t *n_tensors, int64_t *n_elems) {
  if (!x) return fail(HG_E_INVALID, "null ctx");
  if (n_tensors) *n_tensors = (int32_t)x->lay_l.size();
  if (n_elems) *n_elems = x->n_params_l;
  return HG_OK;
}

hg_status hg_param_info(const hg_ctx *x, int32_t i, const char **name, int64_t *offset, int32_t *rows,
                        int32_t *cols) {
  if (!x) return fail(HG_E_INVALID, "null ctx");
  if (i < 0 || i >= (int32_t)x->lay_l.size()) return fail(HG_E_RANGE, "tensor index out of range");
  if (name) *name = x->lay_l[i].name.c_str();
  if (offset) *offset = x->lay_l[i].offset;
  if (rows) *rows = x->lay_l[i].rows;
  if (cols) *cols = x->lay_l[i].cols;
  return HG_OK;
}

static hg_status copy_arena(hg_ctx *x, void *dst, const void *src, size_t bytes, int on_device, bool to_dev) {
  cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : (to_dev ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost);
  CK(x, cudaMemcpyAsync(dst, src, bytes, k, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  return HG_OK;
}

// public (logical) arena -> device arena / device arena -> public arena; a padded
// configuration goes through host copies (parameter I/O is not on the step path)
static hg_status arena_in(hg_ctx *x, float *dev, const float *src, int on_device) {
  if (!x->padded) return copy_arena(x, dev, src, sizeof(float) * (size_t)x->n_params, on_device, true);
  std::vector<float> hl((size_t)x->n_params_l), hp((size_t)x->n_params, 0.f);
  if (on_device) {
    hg_status st = copy_arena(x, hl.data(), src, sizeof(float) * hl.size(), 0, false);
    if (st) return st;
  } else {
    std::memcpy(hl.data(), src, sizeof(float) * hl.size());
  }
  arena_pad(x->cfg_l, hl.data(), hp.data());
  return copy_arena(x, dev, hp.data(), sizeof(float) * hp.size(), 0, true);
}
static hg_status arena_out(hg_ctx *x, float *dst, const float *dev, int on_device) {
  if (!x->padded) return copy_arena(x, dst, dev, sizeof(float) * (size_t)x->n_params, on_device, false);
  std::vector<float> hl((size_t)x->n_params_l), hp((size_t)x->n_params);
  hg_status st = copy_arena(x, hp.data(), dev, sizeof(float) * hp.size(), 0, false);
  if (st) return st;
  arena_unpad(x->cfg_l, hp.data(), hl.data());
  if (!on_device) {
    std::memcpy(dst, hl.data(), sizeof(float) * hl.size());
    return HG_OK;
  }
  return copy_arena(x, dst, hl.data(), sizeof(float) * hl.size(), 0, true);
}

hg_status hg_params_init(hg_ctx *x, uint64_t seed) {
  hg_status st = usable(x);
  if (st) return st;
  std::vector<float> h((size_t)x->n_params, 0.f);
  if (x->padded) {
    std::vector<float> hl((size_t)x->n_params_l);
    init_params_host(x->cfg_l, seed, hl.data());
    arena_pad(x->cfg_l, hl.data(), h.data());
  } else {
    init_params_host(x->cfg, seed, h.data());
  }
  const size_t PB = sizeof(float) * (size_t)x->n_params;
  CK(x, cudaMemcpyAsync(x->f(x->plan.params), h.data(), PB, cudaMemcpyHostToDevice, x->stream));
  CK(x, cudaMemsetAsync(x->f(x->plan.m), 0, PB, x->stream));
  CK(x, cudaMemsetAsync(x->f(x->plan.v), 0, PB, x->stream));
  CK(x, cudaMemsetAsync(x->f(x->plan.grads), 0, PB, x->stream));
  CK(x, cudaMemsetAsync(x->b(x->plan.adam), 0, sizeof(AdamDev), x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  return HG_OK;
}

hg_status hg_params_set(hg_ctx *x, const float *src, int32_t on_device) {
  hg_status st = usable(x);
  if (st) return st;
  if (!src) return fail(HG_E_INVALID, "null source");
  return arena_in(x, x->f(x->plan.params), src, on_device);
}

hg_status hg_params_get(hg_ctx *x, float *dst, int32_t on_device) {
  hg_status st = usable(x);
  if (st) return st;
  if (!dst) return fail(HG_E_INVALID, "null destination");
  return arena_out(x, dst, x->f(x->plan.params), on_device);
}

hg_status hg_grads_get(hg_ctx *x, float *dst, int32_t on_device) {
  hg_status st = usable(x);
  if (st) return st;
  if (!dst) return fail(HG_E_INVALID, "null destination");
  return arena_out(x, dst, x->f(x->plan.grads), on_device);
}

hg_status hg_opt_state_get(hg_ctx *x, float *m, float *v, int64_t *step, int32_t on_device) {
  hg_status st = usable(x);
  if (st || (st = gather_moments(x))) return st;
  if (m && (st = arena_out(x, m, x->f(x->plan.m), on_device))) return st;
  if (v && (st = arena_out(x, v, x->f(x->plan.v), on_device))) return st;
  if (step) {
    AdamDev ad;
    CK(x, cudaMemcpyAsync(&ad, x->b(x->plan.adam), sizeof(ad), cudaMemcpyDeviceToHost, x->stream));
    CK(x, cudaStreamSynchronize(x->stream));
    *step = ad.step;
  }
  return HG_OK;
}

hg_status hg_opt_state_set(hg_ctx *x, const float *m, const float *v, int64_t step, int32_t on_device) {
  hg_status st = usable(x);
  if (st) return st;
  if (m && (st = arena_in(x, x->f(x->plan.m), m, on_device))) return st;
  if (v && (st = arena_in(x, x->f(x->plan.v), v, on_device))) return st;
  if (m && v) x->mv_sharded = false;
  AdamDev ad{step, 0, 0};
  CK(x, cudaMemcpyAsync(x->b(x->plan.adam), &ad, sizeof(ad), cudaMemcpyHostToDevice, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  return HG_OK;
}


hg_status hg_checkpoint_save(hg_ctx *x, const char *path) {
  Range nvtx_range("hg_checkpoint_save");
  hg_status st = usable(x);
  if (st) return st;
  if (!path) return fail(HG_E_INVALID, "null path");
  const int64_t n = x->n_params_l;
  std::vector<float> p(n), m(n), v(n);
  int64_t step = 0;
  if ((st = hg_params_get(x, p.data(), 0)) || (st = hg_opt_state_get(x, m.data(), v.data(), &step, 0))) return st;
  std::vector<uint8_t> b;
  put_bytes(b, kCkptMagic, 8);
  put(b, kCkptVersion);
  put(b, ckpt_model(x->cfg_l));
  put(b, (uint32_t)x->lay_l.size());
  for (const auto &t : x->lay_l) {
    put(b, (uint16_t)t.name.size());
    put_bytes(b, t.name.data(), t.name.size());
    put(b, (int64_t)t.offset);
    put(b, (int32_t)t.rows);
    put(b, (int32_t)t.cols);
  }
  put(b, n);
  put_bytes(b, p.data(), sizeof(float) * n);
  put(b, step);
  put_bytes(b, m.data(), sizeof(float) * n);
  put_bytes(b, v.data(), sizeof(float) * n);
  put(b, crc32c(b.data(), b.size()));
  const std::string tmp = std::string(path) + ".tmp";
  FILE *f = fopen(tmp.c_str(), "wb");
  if (!f) return fail(HG_E_IO, "cannot create %s", tmp.c_str());
  const bool wrote = fwrite(b.data(), 1, b.size(), f) == b.size();
  if (fclose(f) != 0 || !wrote || rename(tmp.c_str(), path) != 0) {
    remove(tmp.c_str());
    return fail(HG_E_IO, "cannot write %s", path);
  }
  return HG_OK;
}

hg_status hg_checkpoint_load(hg_ctx *x, const char *path) {
  Range nvtx_range("hg_checkpoint_load");
  hg_status st = usable(x);
  if (st) return st;
  if (!path) return fail(HG_E_INVALID, "null path");
  FILE *f = fopen(path, "rb");
  if (!f) return fail(HG_E_IO, "cannot open %s", path);
  std::vector<uint8_t> b;
  uint8_t buf[1 << 16];
  size_t k;
  while ((k = fread(buf, 1, sizeof(buf), f)) > 0) b.insert(b.end(), buf, buf + k);
  fclose(f);
  if (b.size() < 8 + 4 + sizeof(CkptModel) + 4 + 4 || std::memcmp(b.data(), kCkptMagic, 8) != 0)
    return fail(HG_E_IO, "%s: not a checkpoint", path);
  uint32_t crc;
  std::memcpy(&crc, b.data() + b.size() - 4, 4);
  if (crc != crc32c(b.data(), b.size() - 4)) return fail(HG_E_IO, "%s: checksum mismatch", path);
  b.resize(b.size() - 4);
  Reader r{b};
  r.at = 8;
  if (r.get<uint32_t>() != kCkptVersion) return fail(HG_E_IO, "%s: unsupported checkpoint version", path);
  const CkptModel cm = r.get<CkptModel>(), mine = ckpt_model(x->cfg_l);
  if (cm.f_node != mine.f_node || cm.f_edge != mine.f_edge || cm.hidden != mine.hidden || cm.layers != mine.layers ||
      cm.fc_hidden != mine.fc_hidden || (cm.flags & ~HG_FLAG_TF32) != (mine.flags & ~HG_FLAG_TF32) ||
      cm.scalers != mine.scalers)
    return fail(HG_E_SHAPE, "%s: model configuration differs from the ctx's", path);
  const uint32_t nt = r.get<uint32_t>();
  if (!r.ok || nt != x->lay_l.size()) return fail(HG_E_SHAPE, "%s: tensor count differs", path);
  for (uint32_t i = 0; i < nt; ++i) {
    const uint16_t len = r.get<uint16_t>();
    const uint8_t *nm = r.bytes(len);
    const int64_t off = r.get<int64_t>();
    const int32_t rows = r.get<int32_t>(), cols = r.get<int32_t>();
    const auto &t = x->lay_l[i];
    if (!r.ok || std::string((const char *)nm, len) != t.name || off != (int64_t)t.offset || rows != t.rows ||
        cols != t.cols)
      return fail(HG_E_SHAPE, "%s: tensor %u differs from the ctx's layout", path, i);
  }
  const int64_t n = r.get<int64_t>();
  if (!r.ok || n != x->n_params_l) return fail(HG_E_SHAPE, "%s: parameter count differs", path);
  const uint8_t *pp = r.bytes(sizeof(float) * n);
  const int64_t step = r.get<int64_t>();
  const uint8_t *mp = r.bytes(sizeof(float) * n), *vp = r.bytes(sizeof(float) * n);
  if (!r.ok || r.at != b.size() || step < 0) return fail(HG_E_IO, "%s: truncated or malformed", path);
  std::vector<float> p(n), m(n), v(n);
  std::memcpy(p.data(), pp, sizeof(float) * n);
  std::memcpy(m.data(), mp, sizeof(float) * n);
  std::memcpy(v.data(), vp, sizeof(float) * n);
  if ((st = hg_params_set(x, p.data(), 0)) || (st = hg_opt_state_set(x, m.data(), v.data(), step, 0))) return st;
  return HG_OK;
}

hg_status hg_batch_get(hg_ctx *x, int32_t slot, void *dst, size_t cap, size_t *used) {
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  if (!dst) return fail(HG_E_INVALID, "null destination");
  CK(x, cudaStreamWaitEvent(x->stream, x->copy_done[slot], 0));
  int32_t hdr[5];
  CK(x, cudaMemcpyAsync(hdr, x->b(x->plan.slot[slot]), sizeof(hdr), cudaMemcpyDeviceToHost, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  const size_t bytes = (size_t)batch_offsets(hdr[0], hdr[1], hdr[2], hdr[3], hdr[4]).total;
  if (used) *used = bytes;
  if (bytes > cap) return fail(HG_E_CAPACITY, "destination too small (%zu bytes needed)", bytes);
  CK(x, cudaMemcpyAsync(dst, x->b(x->plan.slot[slot]), bytes, cudaMemcpyDeviceToHost, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  return HG_OK;
}

hg_status hg_workspace_view(const hg_ctx *x, int32_t what, int32_t layer, int64_t *offset, int64_t *bytes) {
  if (!x || !offset || !bytes) return fail(HG_E_INVALID, "null argument");
  const hg_config &c = x->cfg;
  const Plan &p = x->plan;
  const int64_t N = c.max_nodes, H = c.hidden, B = c.max_graphs;
  const bool needs_layer = what >= 0 && what <= 3;
  if (needs_layer && (layer < 0 || layer >= c.layers)) return fail(HG_E_RANGE, "layer out of range");
  switch (what) {
    case 0: *offset = p.P[layer]; *bytes = 4 * N * x->caps.PW(); break;
    case 1: *offset = p.A[layer]; *bytes = 4 * N * x->caps.KA(); break;
    case 2: *offset = p.arg[layer]; *bytes = 2 * N * H; break;
    case 3: *offset = p.X[layer]; *bytes = 4 * N * H; break;
    case 4:
      if (layer < 0 || layer >= c.n_slots) return fail(HG_E_RANGE, "slot out of range");
      *offset = p.slot[layer]; *bytes = p.blob_max; break;
    case 5: *offset = p.yhat; *bytes = 4 * B; break;
    case 6: *offset = p.loss; *bytes = 4; break;
    case 7: *offset = p.hpre; *bytes = 4 * B * c.fc_hidden; break;
    case 8: *offset = p.params; *bytes = 4 * x->n_params; break;
    case 9: *offset = p.grads; *bytes = 4 * x->n_params; break;
    case 10:
    case 11:  // (per slot: layer = slot)
      if (layer < 0 || layer >= c.n_slots) return fail(HG_E_RANGE, "slot out of range");
      *offset = what == 10 ? p.amp[layer] : p.att[layer]; *bytes = 4 * N; break;
    case 12: if (!p.nh_yn) return fail(HG_E_RANGE, "no node head"); *offset = p.nh_yn; *bytes = 4 * N; break;
    case 13: if (!p.nh_hpre) return fail(HG_E_RANGE, "no node head"); *offset = p.nh_hpre; *bytes = 4 * N * c.fc_hidden; break;
    // (debug views, not in the header: per-layer dP, dP_lo; padded layer-0 features)
    case 100: if (layer < 0 || layer >= c.layers) return fail(HG_E_RANGE, "layer"); *offset = p.dPl[layer]; *bytes = 4 * N * x->caps.PW(); break;
    case 102: if (!p.xpad) return fail(HG_E_RANGE, "no xpad"); *offset = p.xpad; *bytes = 4 * N * pad_x0_width(c.f_node); break;
    default: return fail(HG_E_RANGE, "unknown view %d", what);
  }
  return HG_OK;
}

hg_status hg_pack(hg_ctx *x, const hg_store *s, const int64_t *ids, int32_t B, int32_t slot) {
  Range nvtx_range("hg_pack");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  // the staging buffer may still be the source of an in-flight copy
  CK(x, cudaEventSynchronize(x->copy_done[slot]));
  size_t used = 0;
  st = hg_pack_host(s, ids, B, &x->cfg, x->staging[slot], x->plan.blob_max, &used);
  if (st) return st;
  // the device slot may still be read by an earlier step
  CK(x, cudaStreamWaitEvent(x->copy_stream, x->compute_done[slot], 0));
  CK(x, cudaMemcpyAsync(x->b(x->plan.slot[slot]), x->staging[slot], used, cudaMemcpyHostToDevice, x->copy_stream));
  enqueue_degsort(x, slot, x->copy_stream);
  CK(x, cudaEventRecord(x->copy_done[slot], x->copy_stream));
  return HG_OK;
}

hg_status hg_upload_packed(hg_ctx *x, const void *blob, size_t bytes, int32_t slot) {
  Range nvtx_range("hg_upload_packed");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  if (!blob || bytes < (size_t)kHeaderInts * 4) return fail(HG_E_INVALID, "bad blob");
  if ((st = check_blob(blob, bytes, x->cfg))) return st;
  const int32_t *h = (const int32_t *)blob;
  const size_t need = (size_t)batch_offsets(h[0], h[1], h[2], h[3], h[4]).total;
  CK(x, cudaEventSynchronize(x->copy_done[slot]));
  std::memcpy(x->staging[slot], blob, need);
  CK(x, cudaStreamWaitEvent(x->copy_stream, x->compute_done[slot], 0));
  CK(x, cudaMemcpyAsync(x->b(x->plan.slot[slot]), x->staging[slot], need, cudaMemcpyHostToDevice, x->copy_stream));
  enqueue_degsort(x, slot, x->copy_stream);
  CK(x, cudaEventRecord(x->copy_done[slot], x->copy_stream));
  return HG_OK;
}

hg_status hg_forward(hg_ctx *x, int32_t slot) {
  Range nvtx_range("hg_forward");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  CK(x, cudaStreamWaitEvent(x->stream, x->copy_done[slot], 0));
  const int64_t l0 = launches_so_far();
  enqueue_forward(x, x->stream, slot);
  x->launches += launches_so_far() - l0;
  if ((st = after_enqueue(x, "forward launch"))) return st;
  // the slot's blob is read by this forward: a later hg_pack of the slot waits for it
  CK(x, cudaEventRecord(x->compute_done[slot], x->stream));
  return HG_OK;
}

// ---- evaluation path
hg_status hg_eval_reset(hg_ctx *x) {
  hg_status st = usable(x);
  if (st) return st;
  CK(x, cudaMemsetAsync(x->b(x->plan.eval_acc), 0, sizeof(double) * 4, x->stream));
  return HG_OK;
}

hg_status hg_eval_batch(hg_ctx *x, int32_t slot, int32_t graph) {
  Range nvtx_range("hg_eval_batch");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  CK(x, cudaStreamWaitEvent(x->stream, x->copy_done[slot], 0));
  const uint8_t *blob = x->b(x->plan.slot[slot]);
  double *acc = reinterpret_cast<double *>(x->b(x->plan.eval_acc));
  if (!graph) {
    const int64_t l0 = launches_so_far();
    enqueue_forward(x, x->stream, slot);
    launch_eval_accum(x->stream, blob, x->f(x->plan.yhat), acc);
    x->launches += launches_so_far() - l0;
    if ((st = after_enqueue(x, "eval launch"))) return st;
  } else {
    if (!x->eval_graphs[slot]) {
      cudaGraph_t g = nullptr;
      CK(x, cudaStreamBeginCapture(x->cap_stream, cudaStreamCaptureModeThreadLocal));
      const int64_t l0 = launches_so_far();
      enqueue_forward(x, x->cap_stream, slot);
      launch_eval_accum(x->cap_stream, blob, x->f(x->plan.yhat), acc);
      const int64_t nk = launches_so_far() - l0;
      cudaError_t e = cudaStreamEndCapture(x->cap_stream, &g);
      if (e != cudaSuccess) return cuda_fail(x, e, "cudaStreamEndCapture");
      cudaGraphExec_t ex = nullptr;
      e = cudaGraphInstantiate(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(x, e, "cudaGraphInstantiate");
      x->eval_graphs[slot] = ex;
      x->eval_kernels[slot] = nk;
    }
    CK(x, cudaGraphLaunch(x->eval_graphs[slot], x->stream));
    x->launches += x->eval_kernels[slot];
  }
  CK(x, cudaEventRecord(x->compute_done[slot], x->stream));
  return HG_OK;
}

hg_status hg_eval_result(hg_ctx *x, double *mse, double *mae, int64_t *count) {
  hg_status st = usable(x);
  if (st) return st;
  double h[4] = {0, 0, 0, 0};
  CK(x, cudaMemcpyAsync(h, x->b(x->plan.eval_acc), sizeof(h), cudaMemcpyDeviceToHost, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  const int64_t n = (int64_t)h[2];
  if (count) *count = n;
  if (n == 0) return fail(HG_E_EMPTY, "no graphs evaluated since hg_eval_reset");
  if (mse) *mse = h[0] / (double)n;
  if (mae) *mae = h[1] / (double)n;
  return HG_OK;
}

hg_status hg_eval_pairs(hg_ctx *x, int32_t slot, float *y, float *yhat, int32_t cap, int32_t *n) {
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  if (!y || !yhat || !n) return fail(HG_E_INVALID, "null argument");
  int32_t hdr[kHeaderInts];
  CK(x, cudaMemcpyAsync(hdr, x->b(x->plan.slot[slot]), sizeof(hdr), cudaMemcpyDeviceToHost, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  const int32_t B = hdr[0];
  if (B > cap) return fail(HG_E_CAPACITY, "batch has %d graphs > cap %d", B, cap);
  const BatchOffsets o = batch_offsets(hdr[0], hdr[1], hdr[2], hdr[3], hdr[4]);
  CK(x, cudaMemcpyAsync(y, x->b(x->plan.slot[slot]) + o.y, sizeof(float) * B, cudaMemcpyDeviceToHost, x->stream));
  CK(x, cudaMemcpyAsync(yhat, x->f(x->plan.yhat), sizeof(float) * B, cudaMemcpyDeviceToHost, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  *n = B;
  return HG_OK;
}

hg_status hg_backward(hg_ctx *x, int32_t slot) {
  Range nvtx_range("hg_backward");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  const int64_t l0 = launches_so_far();
  enqueue_backward(x, x->stream, slot);
  x->launches += launches_so_far() - l0;
  if ((st = after_enqueue(x, "backward launch"))) return st;
  CK(x, cudaEventRecord(x->compute_done[slot], x->stream));
  return HG_OK;
}

hg_status hg_nccl_unique_id(void *out128) {
  if (!out128) return fail(HG_E_INVALID, "null output");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id must be 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return HG_OK;
}

hg_status hg_comm_init(hg_ctx *x, const void *id128, int32_t rank, int32_t world) {
  hg_status st = usable(x);
  if (st) return st;
  if (world < 1 || rank < 0 || rank >= world) return fail(HG_E_INVALID, "bad rank/world");
  if (!id128 && world > 1) return fail(HG_E_INVALID, "null NCCL id");
  if (x->comm) return fail(HG_E_STATE, "communicator already initialised");
  x->rank = rank;
  x->world = world;
  if (!id128) return HG_OK;  // world == 1 without an id: no communicator, the exchange is a no-op
  CK(x, cudaSetDevice(x->device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&x->comm, world, id, rank);
  if (r != ncclSuccess) return nccl_fail(x, r, "ncclCommInitRank");
  CK(x, cudaStreamCreateWithFlags(&x->comm_stream, cudaStreamNonBlocking));
  for (int b = 0; b < bucket_count(x); ++b) {
    cudaEvent_t ev;
    CK(x, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    x->bucket_ready.push_back(ev);
  }
  CK(x, cudaEventCreateWithFlags(&x->comm_done, cudaEventDisableTiming));
  // graphs captured before the communicator existed do not contain the allreduce
  for (auto &g : x->graphs)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  return HG_OK;
}

hg_status hg_p2p_handle(hg_ctx *x, void *out) {
  hg_status st = usable(x);
  if (st) return st;
  if (!out) return fail(HG_E_INVALID, "null output");
  static PFN_cuMemGetAddressRange_v3020 get_range = nullptr;
  if (!get_range) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(HG_E_CUDA, "cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)x->ws) != CUDA_SUCCESS)
    return fail(HG_E_CUDA, "cuMemGetAddressRange failed on the workspace");
  cudaIpcMemHandle_t h;
  // (not sticky: an allocation without IPC support, e.g. expandable segments, only means
  // the caller keeps the NCCL exchange)
  const cudaError_t ie = cudaIpcGetMemHandle(&h, (void *)base);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    return fail(HG_E_CUDA, "cudaIpcGetMemHandle: %s (workspace not IPC-capable)", cudaGetErrorString(ie));
  }
  const int64_t off = (int64_t)((uintptr_t)x->ws - (uintptr_t)base);
  std::memcpy(out, &h, sizeof(h));
  std::memcpy((uint8_t *)out + sizeof(h), &off, sizeof(off));
  return HG_OK;
}

hg_status hg_p2p_open(hg_ctx *x, const void *all) {
  hg_status st = usable(x);
  if (st) return st;
  if (!all) {  // back to the NCCL exchange (mappings stay open until destroy)
    if ((st = gather_moments(x))) return st;  // the NCCL path's AdamW needs whole moments
    if (x->p2p)
      for (auto &g : x->graphs)
        if (g) {
          cudaGraphExecDestroy(g);
          g = nullptr;
        }
    x->p2p = false;
    return HG_OK;
  }
  if (x->world < 2 || x->world > kP2PMaxWorld) return fail(HG_E_INVALID, "p2p needs 2..8 ranks (hg_comm_init first)");
  static_assert(sizeof(cudaIpcMemHandle_t) + 8 == HG_P2P_HANDLE_BYTES, "handle size");
  CK(x, cudaSetDevice(x->device));
  for (int q = 0; q < x->world; ++q) {
    if (q == x->rank) {
      x->peer_ws[q] = x->ws;
      continue;
    }
    if (x->peer_base[q]) continue;  // already open
    cudaIpcMemHandle_t h;
    int64_t off = 0;
    const uint8_t *rec = (const uint8_t *)all + (size_t)q * HG_P2P_HANDLE_BYTES;
    std::memcpy(&h, rec, sizeof(h));
    std::memcpy(&off, rec + sizeof(h), sizeof(off));
    void *b = nullptr;
    CK(x, cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
    x->peer_base[q] = b;
    x->peer_ws[q] = (uint8_t *)b + off;
  }
  x->p2p = true;
  for (auto &g : x->graphs)  // captured graphs hold the NCCL exchange
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  return HG_OK;
}

hg_status hg_allreduce_grads(hg_ctx *x) {
  Range nvtx_range("hg_allreduce_grads");
  hg_status st = usable(x);
  if (st) return st;
  return enqueue_allreduce(x, x->stream);
}

hg_status hg_step(hg_ctx *x, const hg_adamw *h) {
  Range nvtx_range("hg_step");
  hg_status st = usable(x);
  if (st) return st;
  if (!h) return fail(HG_E_INVALID, "null hyper");
  if ((st = gather_moments(x))) return st;  // (after peer-memory steps the moments are sharded)
  const int64_t l0 = launches_so_far();
  enqueue_step(x, x->stream, *h);
  x->launches += launches_so_far() - l0;
  return after_enqueue(x, "adamw launch");
}

hg_status hg_train_step(hg_ctx *x, int32_t slot, const hg_adamw *h, int32_t graph) {
  Range nvtx_range("hg_train_step");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  if (!h) return fail(HG_E_INVALID, "null hyper");
  if (!graph) {
    if (x->p2p) return fail(HG_E_STATE, "eager steps use the NCCL exchange: hg_p2p_open(x, NULL) first");
    if ((st = hg_forward(x, slot)) || (st = hg_backward(x, slot)) || (st = hg_allreduce_grads(x)) ||
        (st = hg_step(x, h)))
      return st;
    return HG_OK;
  }
  CK(x, cudaStreamWaitEvent(x->stream, x->copy_done[slot], 0));
  if ((st = hg_capture_step(x, slot, h))) return st;
  CK(x, cudaGraphLaunch(x->graphs[slot], x->stream));
  x->launches += x->graph_kernels[slot];
  if (x->p2p) x->mv_sharded = true;
  CK(x, cudaEventRecord(x->compute_done[slot], x->stream));
  return HG_OK;
}

hg_status hg_capture_step(hg_ctx *x, int32_t slot, const hg_adamw *h) {
  Range nvtx_range("hg_capture_step");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  if (!h) return fail(HG_E_INVALID, "null hyper");
  if (x->graphs[slot] && std::memcmp(&x->graph_hyper[slot], h, sizeof(hg_adamw)) == 0) return HG_OK;
  if (x->graphs[slot]) {
    cudaGraphExecDestroy(x->graphs[slot]);
    x->graphs[slot] = nullptr;
  }
  // capture on the ctx's private stream (the caller's may be the legacy
  // default stream, which cannot be captured); replays go to the caller's stream
  cudaGraph_t g = nullptr;
  CK(x, cudaStreamBeginCapture(x->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int64_t l0 = launches_so_far();
  enqueue_forward(x, x->cap_stream, slot, nullptr, true);
  if (x->p2p) {
    // gradient average + sharded AdamW + parameter all-gather in one kernel over peer memory
    // after the backward
    enqueue_backward(x, x->cap_stream, slot, nullptr, true, false, nullptr);
    launch_p2p_exchange(x->cap_stream, p2p_args(x, *h));
    const int64_t nk = launches_so_far() - l0;
    cudaError_t e = cudaStreamEndCapture(x->cap_stream, &g);
    if (e != cudaSuccess) return cuda_fail(x, e, "cudaStreamEndCapture");
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(x, e, "cudaGraphInstantiate");
    x->graphs[slot] = ex;
    x->graph_kernels[slot] = nk;
    x->graph_hyper[slot] = *h;
    return HG_OK;
  }
  // bucketed, overlapped allreduce; AdamW of layers >= 1 and the head inside the backward
  const bool split_adamw = x->cfg.layers > 1 && x->side_stream != nullptr && (!x->comm || bucket_closed_by(x, 1) >= 0);
  enqueue_backward(x, x->cap_stream, slot, nullptr, true, true, split_adamw ? h : nullptr);
  hg_status ar = join_buckets(x, x->cap_stream);
  if (split_adamw)
    enqueue_step(x, x->cap_stream, *h, nullptr, 0, layer1_offset(x), true);  // conv0: advances the step
  else
    enqueue_step(x, x->cap_stream, *h);
  const int64_t nk = launches_so_far() - l0;
  cudaError_t e = cudaStreamEndCapture(x->cap_stream, &g);
  if (ar) {
    if (g) cudaGraphDestroy(g);
    return ar;
  }
  if (e != cudaSuccess) return cuda_fail(x, e, "cudaStreamEndCapture");
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiate(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(x, e, "cudaGraphInstantiate");
  x->graphs[slot] = ex;
  x->graph_kernels[slot] = nk;
  x->graph_hyper[slot] = *h;
  return HG_OK;
}

hg_status hg_profile_step(hg_ctx *x, int32_t slot, const hg_adamw *h, float *ms, int64_t *launches) {
  Range nvtx_range("hg_profile_step");
  hg_status st = usable(x);
  if (st || (st = check_slot(x, slot))) return st;
  if (!h || !ms) return fail(HG_E_INVALID, "null argument");
  // The step is captured with timing events between phases (single stream, no
  // side-stream overlap) and replayed as one graph, so each phase's time is its
  // kernels' device time without host launch gaps.
  if ((st = gather_moments(x))) return st;  // (the instrumented step runs the full-arena AdamW)
  Prof pr(x->cap_stream);
  CK(x, cudaStreamBeginCapture(x->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int64_t l0 = launches_so_far();
  enqueue_forward(x, x->cap_stream, slot, &pr, true);
  enqueue_backward(x, x->cap_stream, slot, &pr, true);
  hg_status ar = HG_OK;
  phase(&pr, HG_PHASE_ALLREDUCE, [&] { ar = enqueue_allreduce(x, x->cap_stream); });
  enqueue_step(x, x->cap_stream, *h, &pr);
  const int64_t nk = launches_so_far() - l0;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(x->cap_stream, &g);
  if (ar) {
    if (g) cudaGraphDestroy(g);
    return ar;
  }
  if (e != cudaSuccess) return cuda_fail(x, e, "cudaStreamEndCapture");
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(x, e, "cudaGraphInstantiate");
  x->launches += nk;
  CK(x, cudaStreamWaitEvent(x->stream, x->copy_done[slot], 0));
  e = cudaGraphLaunch(ex, x->stream);
  if (e == cudaSuccess) e = cudaEventRecord(x->compute_done[slot], x->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(x->stream);
  cudaGraphExecDestroy(ex);
  if (e != cudaSuccess) return cuda_fail(x, e, "profile graph");
  for (int i = 0; i < HG_PHASE_COUNT; ++i) ms[i] = 0.f;
  for (auto &m : pr.marks) {
    float t = 0.f;
    CK(x, cudaEventElapsedTime(&t, m.second.first, m.second.second));
    ms[m.first] += t;
  }
  if (launches)
    for (int i = 0; i < HG_PHASE_COUNT; ++i) launches[i] = pr.launches[i];
  return HG_OK;
}

hg_status hg_loss_enqueue(hg_ctx *x, int32_t i) {
  hg_status st = usable(x);
  if (st) return st;
  if (i < 0 || i >= HG_LOSS_RING) return fail(HG_E_RANGE, "loss ring index %d out of range", i);
  launch_loss_to_host(x->stream, x->f(x->plan.loss), x->loss_ring_dev + i);
  CK(x, cudaGetLastError());
  CK(x, cudaEventRecord(x->loss_ev[i], x->stream));
  return HG_OK;
}

hg_status hg_loss_fetch(hg_ctx *x, int32_t i, float *loss) {
  hg_status st = usable(x);
  if (st) return st;
  if (i < 0 || i >= HG_LOSS_RING) return fail(HG_E_RANGE, "loss ring index %d out of range", i);
  if (!loss) return fail(HG_E_INVALID, "null output");
  CK(x, cudaEventSynchronize(x->loss_ev[i]));
  *loss = x->loss_ring[i];
  return HG_OK;
}

hg_status hg_loss_get(hg_ctx *x, float *loss) {
  hg_status st = usable(x);
  if (st) return st;
  if (!loss) return fail(HG_E_INVALID, "null output");
  CK(x, cudaMemcpyAsync(loss, x->f(x->plan.loss), sizeof(float), cudaMemcpyDeviceToHost, x->stream));
  CK(x, cudaStreamSynchronize(x->stream));
  return HG_OK;
}

// wait for one stream with the fail-stop bound: poll the stream, NCCL's async error and the
// peer-exchange flag block; a failed or timed-out wait aborts the communicator (SPEC.md:459,
// 475: a dead peer fails the job instead of hanging it) and makes the ctx unusable
static hg_status wait_stream(hg_ctx *x, cudaStream_t s, const std::chrono::steady_clock::time_point &t0) {
  for (unsigned spins = 0;; ++spins) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return HG_OK;
    if (q != cudaErrorNotReady) {
      if (x->comm) {
        ncclCommAbort(x->comm);
        x->comm = nullptr;
      }
      return cuda_fail(x, q, "stream");
    }
    if (x->comm) {
      ncclResult_t ar = ncclSuccess;
      const ncclResult_t r = ncclCommGetAsyncError(x->comm, &ar);
      if (r != ncclSuccess || ar != ncclSuccess) {
        ncclCommAbort(x->comm);
        x->comm = nullptr;
        return nccl_fail(x, r != ncclSuccess ? r : ar, "NCCL async error (communicator aborted)");
      }
    }
    if (x->timeout_ns) {
      const auto el = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0);
      if ((unsigned long long)el.count() > x->timeout_ns) {
        if (x->comm) {
          ncclCommAbort(x->comm);
          x->comm = nullptr;
        }
        hg_status st = fail(HG_E_NCCL, "hg_sync timed out after %.3f s (peer not responding?)", x->timeout_ns * 1e-9);
        x->sticky = st;
        x->sticky_msg = hg_last_error();
        return st;
      }
    }
    std::this_thread::sleep_for(std::chrono::microseconds(spins < 100 ? 20 : 200));
  }
}

hg_status hg_sync(hg_ctx *x) {
  Range nvtx_range("hg_sync");
  if (!x) return fail(HG_E_INVALID, "null ctx");
  if (x->sticky != HG_OK) return fail(HG_E_STATE, "%s", x->sticky_msg.c_str());
  const auto t0 = std::chrono::steady_clock::now();
  hg_status st;
  if ((st = wait_stream(x, x->stream, t0))) return st;
  if ((st = wait_stream(x, x->copy_stream, t0))) return st;
  if (x->comm_stream && (st = wait_stream(x, x->comm_stream, t0))) return st;
  return HG_OK;
}

hg_status hg_set_timeout(hg_ctx *x, double seconds) {
  hg_status st = usable(x);
  if (st) return st;
  if (!(seconds >= 0.0) || seconds > 1e6) return fail(HG_E_INVALID, "timeout must be in [0, 1e6] s");
  x->timeout_ns = (unsigned long long)(seconds * 1e9);
  for (auto &g : x->graphs)  // captured exchanges carry the bound
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  return HG_OK;
}

hg_status hg_p2p_emulate(hg_ctx *const *ctxs, int32_t world, const hg_adamw *h) {
  if (!ctxs || !h || world < 2 || world > kP2PMaxWorld) return fail(HG_E_INVALID, "need 2..8 contexts and hyper");
  uint8_t *peers[kP2PMaxWorld] = {};
  for (int r = 0; r < world; ++r) {
    hg_status st = usable(ctxs[r]);
    if (st) return st;
    if (ctxs[r]->p2p || ctxs[r]->comm) return fail(HG_E_STATE, "emulated ranks must not hold a communicator");
    if (ctxs[r]->device != ctxs[0]->device || ctxs[r]->n_params != ctxs[0]->n_params)
      return fail(HG_E_INVALID, "emulated ranks need one device and one configuration");
    for (int q = 0; q < r; ++q)
      if (ctxs[q] == ctxs[r]) return fail(HG_E_INVALID, "context passed twice");
    peers[r] = ctxs[r]->ws;
  }
  hg_ctx *x0 = ctxs[0];
  for (int r = 0; r < world; ++r)  // every rank's backward precedes every rank's exchange
    if (r > 0) {
      CK(x0, cudaStreamSynchronize(ctxs[r]->stream));
    }
  for (int r = 0; r < world; ++r) {
    hg_ctx *x = ctxs[r];
    x->world = world;
    x->rank = r;
    for (int q = 0; q < world; ++q) x->peer_ws[q] = peers[q];
    launch_p2p_exchange_emulated(x0->stream, p2p_args(x, *h));
    x->launches += 2;
    x->mv_sharded = true;
  }
  hg_status st = after_enqueue(x0, "emulated exchange");
  if (st) return st;
  CK(x0, cudaStreamSynchronize(x0->stream));
  return HG_OK;
}

hg_status hg_exchange_time(hg_ctx *x, const hg_adamw *h, int32_t iters, float *ms) {
  hg_status st = usable(x);
  if (st) return st;
  if (!h || !ms || iters < 1) return fail(HG_E_INVALID, "bad arguments");
  if (!x->p2p && !x->comm) return fail(HG_E_STATE, "no exchange configured (hg_comm_init / hg_p2p_open)");
  cudaEvent_t a, b;
  CK(x, cudaEventCreate(&a));
  CK(x, cudaEventCreate(&b));
  CK(x, cudaStreamSynchronize(x->stream));
  CK(x, cudaEventRecord(a, x->stream));
  for (int i = 0; i < iters; ++i) {
    if (x->p2p) {
      launch_p2p_exchange(x->stream, p2p_args(x, *h));
      x->launches += 4;
      x->mv_sharded = true;
    } else if ((st = enqueue_allreduce(x, x->stream))) {
      return st;
    }
  }
  CK(x, cudaEventRecord(b, x->stream));
  if ((st = after_enqueue(x, "exchange"))) return st;
  CK(x, cudaEventSynchronize(b));
  float t = 0.f;
  CK(x, cudaEventElapsedTime(&t, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms = t / (float)iters;
  return HG_OK;
}

hg_status hg_bucket_layout(const hg_config *c, int64_t *ranges, int32_t cap, int32_t *n) {
  hg_status st = check_config(c);
  if (st) return st;
  if (!n) return fail(HG_E_INVALID, "null output");
  const hg_config pc = padded_config(*c);
  const auto lay = param_layout(pc);
  const int64_t total = param_total(lay);
  const int nb = (int)bucket_groups_for(pc.layers).size();
  *n = nb;
  if (!ranges) return HG_OK;
  if (cap < nb) return fail(HG_E_CAPACITY, "%d buckets > capacity %d", nb, cap);
  for (int b = 0; b < nb; ++b) {
    const auto r = bucket_range_of(lay, total, pc.layers, b);
    ranges[2 * b] = r.first;
    ranges[2 * b + 1] = r.second;
  }
  return HG_OK;
}

hg_status hg_launch_count(const hg_ctx *x, int64_t *count) {
  if (!x || !count) return fail(HG_E_INVALID, "null argument");
  *count = x->launches;
  return HG_OK;
}

}  // extern "C"
