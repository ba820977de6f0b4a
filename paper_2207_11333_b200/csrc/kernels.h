// kernels.h — host-side launch wrappers for the CUDA kernels of one training
// step. Every wrapper enqueues on `st` and reads the
// batch sizes (B, N, E) from the device-resident batch header, so a whole step
// is CUDA-graph capturable; grids are sized from the ctx capacities.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hg {
extern bool g_low_prio;
extern int g_prio_lo, g_prio_hi;  // launch priorities (common.cuh launch_ex)

struct Caps {
  int maxB, maxN, maxE;
  int F0, Fe, H, Hf;
  int Hl = 0;      // logical hidden width (< H when the configuration is channel-padded; 0 = H)
  int S = 3;       // degree scalers (blocks of 4H columns in U)
  int self_t = 0;  // PNA self-term variant: A rows carry x_i as a 5th block, P rows carry Q = X M_s^T
  int KA() const { return (self_t ? 5 : 4) * H; }  // width of the update GEMM's A operand
  int PW() const { return (self_t ? 2 : 1) * H; }  // width of P rows ([P | Q]) and dP rows ([dP | dQ])
};

// K1 layer 0: P[N,H] = x[N,F0] * Mx^T (SIMT; layers >= 1 use launch_d_proj)
void launch_proj(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *X, int F, const float *Mx, float *P);

// aggregation kernels (agg.cu): one CTA per graph and channel chunk, the graph staged in
// shared memory (requires c.H % 128 == 0)
cudaError_t agg_configure();  // opt-in shared memory (once, outside graph capture)
// K2: fused edge gather + message + mean/min/max/std segmented reduction; A row i is written
// at the degree-sorted row pos[i]
// (self-term: P holds [P | Q] rows, xin = the layer input rows of width Fl, null at layer 0 =
// the batch's x; A rows are KA = 5H wide with x_i in the fifth block)
void launch_agg_fwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const int4 *gslice, const float *P,
                    const float *Me, const float *bM, float var_floor, float *A, uint8_t *arg, const int *pos,
                    const float *xin = nullptr, int Fl = 0);
// K8: aggregation backward + scatter to sources (dP row j at pos[j] when dp_pos != null, else
// j; dp_pos must be pos or null); dM_e / db_M per-graph partials (launch_reduce_dMe sums them);
// dm_scratch: agg_bwd_dm_floats floats (the per-edge message gradients, L2-resident)
void launch_agg_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const int4 *gslice, const float *P,
                    const float *Me, const float *bM, const float *A, const uint8_t *arg, const float *dA, float *dP,
                    float *partial, const int *pos, const int *dp_pos, float *dm_scratch);
// dM_e and db_M = fixed-order sums of launch_agg_bwd's per-graph partials (tcmn.cu)
void launch_reduce_dMe(cudaStream_t st, const Caps &c, const float *partial, float *dMe, float *dbM);
size_t agg_bwd_partial_floats(const Caps &c);
size_t agg_bwd_dm_floats(const Caps &c);

// K4/K5: pool + head forward, loss
// (sqn != null: node-level head's per-node squared errors, added to the loss with weight w)
void launch_head_fwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                     const float *b1, const float *W2, const float *b2, float *G, float *hpre, float *yhat,
                     float *sqerr, float *loss, const float *sqn = nullptr, float w = 0.f);
// node-level head (HG_FLAG_NODE_HEAD): forward (hpre [N][Hf], yn, sqn) and, with bwd, dyn [N],
// dhn [N][Hf] and its masked contribution added into dZ_L (degree-sorted rows pos)
void launch_node_head(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                      const float *b1, const float *W2, const float *b2, float w, float *hpre, float *yn, float *sqn,
                      float *dyn, float *dhn, float *dZL, const int *pos, bool bwd);
// its W2n / b2n gradient partials over fixed node chunks ([chunks][Hf + 4]); reduce with launch_reduce_cols
void launch_node_head_w2(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *hpre, const float *dyn,
                         float *part);
size_t node_head_partial_floats(const Caps &c);
int node_head_chunks(const Caps &c);
// fixed-order column sums of `parts` rows of `stride` floats: out[e] = sum_p part[p][e], e < count
// (count % 4 == 0), tcmn.cu
void launch_reduce_cols(cudaStream_t st, const float *part, int parts, int stride, int count, float *out);
// K5+K6 fused (a training step): pool, head forward, per-graph loss terms and the
// head/pool backward down to dZ of the last layer (the loss itself: launch_loss)
void launch_head_fused(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                       const float *b1, const float *W2, const float *b2, float *G, float *hpre, float *yhat,
                       float *sqerr, float *loss, float *dy, float *dhid, float *dZL, const int *pos = nullptr);
// K6 (eager backward after a forward-only head): head + pool backward -> dZ of the last
// layer, then (with_grads) the head parameter gradients
void launch_head_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                     const float *W2, const float *G, const float *hpre, const float *yhat, float *dy,
                     float *dhid, float *dZL, float *gW1, float *gb1, float *gW2, float *gb2, bool head_done,
                     const int *pos = nullptr, bool with_grads = true);
// head parameter gradients
void launch_head_grads(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *G, const float *hpre,
                       const float *dy, const float *dhid, float *gW1, float *gb1, float *gW2, float *gb2);
// evaluation sums of one batch into acc[0..2] (fp64: squared error, absolute error, graphs)
void launch_eval_accum(cudaStream_t st, const uint8_t *blob, const float *yhat, double *acc);
// mean squared error over the batch from the per-graph terms (after launch_head_fused)
void launch_loss_to_host(cudaStream_t st, const float *loss, float *host_mapped);  // one float, mapped pinned dst
void launch_loss(cudaStream_t st, const uint8_t *blob, const float *sqerr, float *loss, const float *sqn = nullptr,
                 float w = 0.f);
void head_configure(const Caps &c);

// K10: AdamW over the flat arena
struct AdamDev {
  int64_t step;
  int32_t ticket, pad;  // blocks finished in the running k_adamw (the last one advances step)
};
// (advance: this launch covers the step's last parameter range and advances the step counter;
// ranges of one step must be launched in order on one stream)
void launch_adamw(cudaStream_t st, float *p, const float *g, float *m, float *v, int64_t n, AdamDev *ad,
                  float lr, float beta1, float beta2, float eps, float wd, bool advance = true,
                  int max_blocks = 0);

// fused gradient average + sharded AdamW + parameter all-gather over peer memory (p2p.cu)
constexpr int kP2PMaxWorld = 8;
constexpr unsigned kP2PTimeout = 1;  // P2PDev::error: a peer did not answer within the timeout
struct P2PDev {                      // in every rank's workspace; zero at ctx creation
  unsigned ready[kP2PMaxWorld];      // ready[q] = epoch: rank q's gradients of that step are complete
  unsigned done[kP2PMaxWorld];       // done[q] = epoch: rank q's shard of that step is written everywhere
  unsigned epoch;                    // steps taken through the p2p path
  unsigned ticket;                   // k_p2p_adamw's finished-block counter
  unsigned error;                    // kP2PTimeout after a timed-out wait (the kernel then traps)
  unsigned pad;
};
struct P2PArgs {
  float *params[kP2PMaxWorld];       // every rank's parameter arena ([rank] = local)
  const float *grads[kP2PMaxWorld];  // every rank's gradient arena
  P2PDev *dev[kP2PMaxWorld];         // every rank's flags
  const float *m_all[kP2PMaxWorld];  // every rank's Adam moments (moment gather)
  const float *v_all[kP2PMaxWorld];
  float *m, *v;                      // local Adam moments (the owned shard is used)
  AdamDev *ad;
  int world, rank;
  int64_t n4;                        // float4s in the flat arena
  unsigned long long timeout_ns;     // bound of every flag wait (0 = unbounded)
  float lr, beta1, beta2, eps, wd;
};
// one step's exchange: signal, wait for every ready flag, fused reduce + AdamW + all-gather of
// this rank's shard, wait for every done flag
void launch_p2p_exchange(cudaStream_t st, const P2PArgs &a);
// the same arithmetic for ranks emulated in one process on one device (hg_p2p_emulate): the
// ranks' kernels run back to back, so the flag waits are elided
void launch_p2p_exchange_emulated(cudaStream_t st, const P2PArgs &a);
// copy every peer's shard of the Adam moments into the local arrays
void launch_p2p_gather_moments(cudaStream_t st, const P2PArgs &a);

// degree classes (degsort.cu): one class per distinct degree present in the batch
constexpr int kNumSMs = 148;     // B200
constexpr int kMaxClasses = 32;  // class slots (distinct degrees per batch) at most
constexpr int kMaxScalers = 5;   // identity, amplification, attenuation, linear, inverse_linear
constexpr int kGramKS = 256;     // minimum nodes per K-split of the per-class Gram GEMM
// nodes per Gram K-split for a capacity: >= kGramKS, about 64 splits at large capacities
// (the split partials are reduced afterwards, so their number bounds that traffic)
// (32 or 128 splits measured no better at configs B and D, round 2)
inline int gram_ks(const Caps &c) {
  const int k = (c.maxN + 63) / 64;
  return k <= kGramKS ? kGramKS : (k + 31) / 32 * 32;
}
constexpr int HG_MAX_DEGREE_DEV = 127;
struct DegInfo {
  int C, T, S, overflow;  // classes, 128-row tiles, Gram splits; overflow: > cmax distinct degrees
  int deg[kMaxClasses], start[kMaxClasses], count[kMaxClasses];
  float scal[kMaxScalers][kMaxClasses];  // value of the configured scalers (U block order) per class
};
int tc_num_classes(int max_degree);  // class slots of a ctx: min(max_degree + 1, kMaxClasses)
int tc_max_tiles(const Caps &c, int cmax);
int tc_max_splits(const Caps &c, int cmax);
// stable degree sort + per-node scalers + class table / tiles / splits + per-graph node/edge
// ranges gslice[g] = (n0, n1, e0, e1); perm[r] = node at degree-sorted row r, pos = its inverse
// (smask: the configured scaler bit set, hgnn.h HG_SCALER_*; delta_lin: the linear scalers' normaliser)
void launch_degsort(cudaStream_t st, const uint8_t *blob, double delta, int cmax, float *amp, float *att, int *perm,
                    DegInfo *info, int4 *tiles, int4 *splits, int *pos, int4 *gslice, int smask, double delta_lin,
                    int ks, int maxN);
cudaError_t degsort_configure();  // opt-in shared memory for the staged degrees (outside capture)

// TMA-fed tcgen05 GEMMs (tcdirect.cu): activation operands are read once as fp32 (their tf32
// lo terms are derived in shared memory), weight operands with their lo terms (prep kernels).
// A / dZ operands of the class GEMMs are stored in degree-sorted row order (row pos[i]).
extern int g_gemm_passes;  // 3 = 3xTF32 (default), 1 = plain TF32 (HG_FLAG_TF32); set per enqueue
cudaError_t tcd_configure();
// (X1s optional: also write the output rows in degree-sorted order, X1mask their ReLU bits)
void launch_d_update_cls(cudaStream_t st, const Caps &c, int cmax, const float *A, const int *perm,
                         const DegInfo *info, const int4 *tiles, const float *Wf, const float *Wf_lo, const float *bU,
                         float *X1, float *X1s = nullptr, uint32_t *X1mask = nullptr);
void launch_d_dA_cls(cudaStream_t st, const Caps &c, int cmax, const float *dZ, const int *perm, const DegInfo *info,
                     const int4 *tiles, const float *WbT, const float *WbT_lo, float *dA);
void launch_d_proj(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *X, int F, const float *Mx,
                   const float *Mx_lo, float *P);
// (self-term: dP = [dP | dQ] rows (2H), MxT = [M_x; M_s]^T, and dXself = the dA buffer's x block
// (dA + 4H, row stride 5H) is added before the ReLU mask)
void launch_d_dX(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *MxT,
                 const float *MxT_lo, int F, const float *Xl, float *dZ, const int *pos,
                 const float *dXself = nullptr);
// fused backward (H == 128): dZ_{l-1} = (dP_l M_x) * [X_{l-1} > 0] (sorted rows) and
// dA_{l-1} = dZ_{l-1} W_c per degree-class tile; dP_s / Xs in degree-sorted row order
bool dxda_supported(const Caps &c);
void launch_dxda(cudaStream_t st, const Caps &c, int cmax, const float *dP_s, const float *MxT, const float *MxT_lo,
                 const float *WbT, const float *WbT_lo, const int *perm, const DegInfo *info, const int4 *tiles,
                 const uint32_t *Xmask, float *dZ, float *dA);
void launch_prep_Mx(cudaStream_t st, const Caps &c, const float *params, const int64_t *mx_off_dev, int L,
                    float *Mx_lo, float *MxT, float *MxT_lo);
// layers [l0, l1) of the class weights (needs the batch's class table: after launch_degsort)
// (ux_off_dev: U_x offsets per layer for the self-term variant, else null; W_c = [sum_s s(c) U_s | U_x])
void launch_prep_W2(cudaStream_t st, const Caps &c, const float *params, const int64_t *u_off_dev,
                    const int64_t *ux_off_dev, int l0, int l1, int cmax, const DegInfo *info, float *Wf, float *Wf_lo,
                    float *WbT, float *WbT_lo);

extern int g_mn_grid_override;  // tcmn.cu: grid cap override for MN Grams (0 = default)
// TMA-fed MN-major Grams (tcmn.cu): per-class-split dU / db_U and per-split dM_x / db_M,
// partials reduced in fixed order (rows of dZ / A degree-sorted)
size_t mn_gram_partial_floats(const Caps &c, int cmax);
size_t mn_dmx_partial_floats(const Caps &c, int F, int R = 0);  // (R: rows, 0 = c.PW())
// (dUx: the self-term's U_x gradient [H][Fl] from the Gram's x block, or null)
void launch_mn_dU_cls(cudaStream_t st, const Caps &c, int cmax, const float *dZ, const float *A, const float *ones,
                      const DegInfo *info, const int4 *splits, float *partial, float *dU, float *dbU, float *dUx = nullptr,
                      int Fl = 0);
// X: [maxN][Fp] (Fp >= F, 16-byte row pitch; Fp = F for hidden layers), F output columns
// (R: rows of dP = output rows, 0 = c.PW(); must be a multiple of 128)
void launch_mn_dMx(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *X, int F, int Fp,
                   const float *ones, float *partial, float *dMx,
                   float *dbM, int R = 0);  // dbM == null: no column-sum tiles (db_M comes from launch_reduce_dMe)
// layer-0 node features padded to pad_x0_width(F0) columns for the TMA path
int pad_x0_width(int F0);
void launch_pad_x0(cudaStream_t st, const Caps &c, const uint8_t *blob, float *Xp,
                   const int *pos = nullptr);  // pos: write row i at pos[i]

// process-wide count of kernels launched by the wrappers above
int64_t launches_so_far();

}  // namespace hg
