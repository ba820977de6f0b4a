// kernels.h — host-side launch wrappers for the CUDA kernels of one training
// step. Every wrapper enqueues on `st` and reads the
// batch sizes (B, N, E) from the device-resident batch header, so a whole step
// is CUDA-graph capturable; grids are sized from the ctx capacities.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hg {
extern bool g_pdl;
extern bool g_low_prio;
extern int g_prio_lo, g_prio_hi;  // launch kernels with programmatic dependent launch (common.cuh)

struct Caps {
  int maxB, maxN, maxE;
  int F0, Fe, H, Hf;
  int Hl = 0;  // logical hidden width (< H when the configuration is channel-padded; 0 = H)
};

// per-node degree scalers amp = ln(d+1)/delta, att = delta/ln(d+1) (1 for d=0)
void launch_scalers(cudaStream_t st, const Caps &c, const uint8_t *blob, double delta, float *amp, float *att);

// K1 / K9b / K3 / K7a / K7b / K9a GEMMs (SIMT fp32 v1)
// P[N,H] = X[N,F] * Mx^T
void launch_proj(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *X, int F, const float *Mx, float *P);
// X1 = ReLU(sum_s diag(s) A U_s^T + b_U)
void launch_update(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *A, const float *amp,
                   const float *att, const float *U, const float *bU, float *X1);
// dA[N,4H] = sum_s diag(s) dZ U_s
void launch_dA(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dZ, const float *amp,
               const float *att, const float *U, float *dA);
// dU[H,12H] = sum_i s_i dZ_i^T A_i ; db_U = sum_i dZ_i   (split-K partials then fixed-order reduce)
void launch_dU(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dZ, const float *A,
               const float *amp, const float *att, float *partial, float *dU, float *dbU);
// dM_x[H,F] = dP^T X ; db_M = sum_i dP_i
void launch_dMx(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *X, int F,
                float *partial, float *dMx, float *dbM);
// dZprev[N,F] = (dP Mx) * [Xl > 0]
void launch_dX(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *Mx, int F,
               const float *Xl, float *dZprev);

// K2: fused edge gather + message + mean/min/max/std segmented reduction
void launch_agg_fwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *P, const float *Me,
                    const float *bM, float var_floor, float *A, uint8_t *arg, float *A_lo = nullptr,
                    const int *pos = nullptr);  // pos: write A row i at pos[i] (degree-sorted)
// K8: aggregation backward + scatter to sources; dM_e via block partials
void launch_agg_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *P, const float *Me,
                    const float *bM, const float *A, const uint8_t *arg, const float *dA, float *dP,
                    float *partial, float *dMe, float *dP_lo = nullptr, const int *pos = nullptr,
                    const int *dp_pos = nullptr);  // dp_pos: write dP row j at dp_pos[j]
// dM_e = fixed-order sum of launch_agg_bwd's block partials (launch_agg_bwd does it when dMe != null)
// (dbM != null: also db_M = sum_j dP_j from the same partials)
void launch_reduce_dMe(cudaStream_t st, const Caps &c, const float *partial, float *dMe, float *dbM = nullptr);
size_t agg_bwd_partial_floats(const Caps &c);
size_t dU_partial_floats(const Caps &c);
size_t dMx_partial_floats(const Caps &c, int F);

// K4/K5: pool + head forward, loss
void launch_head_fwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                     const float *b1, const float *W2, const float *b2, float *G, float *hpre, float *yhat,
                     float *sqerr, float *loss);
// K5+K6 fused (a training step): pool, head forward, per-graph loss terms and the
// head/pool backward down to dZ of the last layer (the loss itself: launch_loss)
void launch_head_fused(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                       const float *b1, const float *W2, const float *b2, float *G, float *hpre, float *yhat,
                       float *sqerr, float *loss, float *dy, float *dhid, float *dZL, float *dZL_lo = nullptr,
                       const int *pos = nullptr);
// K6: head + pool backward -> dZ of the last layer (skipped if head_done), then head parameter gradients
void launch_head_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                     const float *W2, const float *G, const float *hpre, const float *yhat, float *dy,
                     float *dhid, float *dZL, float *gW1, float *gb1, float *gW2, float *gb2, bool head_done,
                     float *dZL_lo = nullptr, const int *pos = nullptr, bool with_grads = true);
// head parameter gradients only (the tail of launch_head_bwd)
void launch_head_grads(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *G, const float *hpre,
                       const float *dy, const float *dhid, float *gW1, float *gb1, float *gW2, float *gb2);
// evaluation sums of one batch into acc[0..2] (fp64: squared error, absolute error, graphs)
void launch_eval_accum(cudaStream_t st, const uint8_t *blob, const float *yhat, double *acc);
// mean squared error over the batch from the per-graph terms (after launch_head_fused)
void launch_loss(cudaStream_t st, const uint8_t *blob, const float *sqerr, float *loss);
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
struct P2PDev {                        // in every rank's workspace; zero at ctx creation
  unsigned ready[2][kP2PMaxWorld];     // ready[part][q] = epoch: rank q's gradients of that part are complete
  unsigned done[2][kP2PMaxWorld];      // done[part][q] = epoch: rank q's shard of that part is written everywhere
  unsigned epoch;                      // steps taken through the p2p path
  unsigned ticket[2];                  // k_p2p_adamw's finished-block counters
};
struct P2PArgs {
  float *params[kP2PMaxWorld];       // every rank's parameter arena ([rank] = local)
  const float *grads[kP2PMaxWorld];  // every rank's gradient arena
  P2PDev *dev[kP2PMaxWorld];         // every rank's flags
  float *m, *v;                      // local Adam moments (the owned shard is used)
  AdamDev *ad;
  int world, rank;
  int64_t n4;                        // float4s in the flat arena
  float lr, beta1, beta2, eps, wd;
};
// one exchange part (0: conv0 at the step's end, 1: layers >= 1 + head, overlapped with layer
// 0's backward) over float4 range [b4, e4): signal ready, wait for every rank's ready, fused
// reduce + AdamW + all-gather of this rank's shard (bump: first part of the step; advance:
// last part, advances the AdamW step counter); launch_p2p_wait_done: wait for every rank's
// done flag of `part` (before parameters or gradients are touched again)
void launch_p2p_part(cudaStream_t st, const P2PArgs &a, int part, int64_t b4, int64_t e4, bool bump, bool advance);
void launch_p2p_wait_done(cudaStream_t st, const P2PArgs &a, int part);

// degree classes (tcgemm.cu): one class per distinct degree present in the batch
constexpr int kMaxClasses = 16;
constexpr int kGramKS = 256;  // minimum nodes per K-split of the per-class Gram GEMM
// nodes per Gram K-split for a capacity: >= kGramKS, about 64 splits at large capacities
// (the split partials are reduced afterwards, so their number bounds that traffic)
inline int gram_ks(const Caps &c) {
  const int k = (c.maxN + 63) / 64;
  return k <= kGramKS ? kGramKS : (k + 31) / 32 * 32;
}
constexpr int HG_MAX_DEGREE_DEV = 127;
struct DegInfo {
  int C, T, S, pad;
  int deg[kMaxClasses], start[kMaxClasses], count[kMaxClasses];
  float amp[kMaxClasses], att[kMaxClasses];
};
int tc_num_classes(const Caps &c, int max_degree);  // class slots (max_degree+1) or 0 = class path off
int tc_max_tiles(const Caps &c, int cmax);
int tc_max_splits(const Caps &c, int cmax);
// stable degree sort + per-node scalers (+ class table / tiles / splits when cmax > 0)
// perm[r] = node at degree-sorted row r, pos = its inverse (pos may be null)
void launch_degsort(cudaStream_t st, const uint8_t *blob, double delta, int cmax, float *amp, float *att, int *perm,
                    DegInfo *info, int4 *tiles, int4 *splits, int *pos = nullptr, int ks = 0);

// TMA-fed tcgen05 GEMMs over pre-split operands (tcdirect.cu). A / dZ operands of
// the class GEMMs are stored in degree-sorted row order (row pos[i] for node i).
cudaError_t tcd_configure();
// (X1s, X1s_lo optional: also write the output rows in degree-sorted order)
void launch_d_update_cls(cudaStream_t st, const Caps &c, int cmax, const float *A, const float *A_lo, const int *perm,
                         const DegInfo *info, const int4 *tiles, const float *Wf, const float *Wf_lo, const float *bU,
                         float *X1, float *X1_lo, float *X1s = nullptr, float *X1s_lo = nullptr,
                         uint32_t *X1mask = nullptr);
void launch_d_dA_cls(cudaStream_t st, const Caps &c, int cmax, const float *dZ, const float *dZ_lo, const int *perm,
                     const DegInfo *info, const int4 *tiles, const float *WbT, const float *WbT_lo, float *dA);
void launch_d_proj(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *X, const float *X_lo, int F,
                   const float *Mx, const float *Mx_lo, float *P);
void launch_d_dX(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *dP_lo,
                 const float *MxT, const float *MxT_lo, int F, const float *Xl, float *dZ, float *dZ_lo,
                 const int *pos);
// fused backward (H == 128): dZ_{l-1} = (dP_l M_x) * [X_{l-1} > 0] (sorted rows, + lo) and
// dA_{l-1} = dZ_{l-1} W_c per degree-class tile; dP_s / Xs in degree-sorted row order
bool dxda_supported(const Caps &c);
void launch_dxda(cudaStream_t st, const Caps &c, int cmax, const float *dP_s, const float *dP_s_lo, const float *MxT,
                 const float *MxT_lo, const float *WbT, const float *WbT_lo, const int *perm, const DegInfo *info,
                 const int4 *tiles, const uint32_t *Xmask, float *dZ, float *dZ_lo, float *dA);
void launch_prep_Mx(cudaStream_t st, const Caps &c, const float *params, const int64_t *mx_off_dev, int L,
                    float *Mx_lo, float *MxT, float *MxT_lo);
// layers [l0, l1) of the degree-slot weights
void launch_prep_W2(cudaStream_t st, const Caps &c, const float *params, const int64_t *u_off_dev, int l0, int l1,
                    int cmax, double delta, float *Wf, float *Wf_lo, float *WbT, float *WbT_lo);

extern int g_mn_grid_override;  // tcmn.cu: grid cap override for MN Grams (0 = default)
// TMA-fed MN-major Grams (tcmn.cu): per-class-split dU / db_U and per-split dM_x / db_M,
// partials reduced in fixed order (class path; rows of dZ / A degree-sorted)
size_t mn_gram_partial_floats(const Caps &c, int cmax);
size_t mn_dmx_partial_floats(const Caps &c, int F);
void launch_mn_dU_cls(cudaStream_t st, const Caps &c, int cmax, const float *dZ, const float *dZ_lo, const float *A,
                      const float *A_lo, const float *ones, const DegInfo *info, const int4 *splits, float *partial,
                      float *dU, float *dbU);
// X: [maxN][Fp] (Fp >= F, 16-byte row pitch; Fp = F for hidden layers), F output columns
void launch_mn_dMx(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *dP_lo,
                   const float *X, const float *X_lo, int F, int Fp, const float *ones, float *partial, float *dMx,
                   float *dbM);  // dbM == null: no column-sum tiles (db_M comes from launch_reduce_dMe)
// layer-0 node features padded to pad_x0_width(F0) columns (+ tf32 residual) for the TMA path
int pad_x0_width(int F0);
void launch_pad_x0(cudaStream_t st, const Caps &c, const uint8_t *blob, float *Xp, float *Xp_lo,
                   const int *pos = nullptr);  // pos: write row i at pos[i]
int agg_bwd_partials(const Caps &c);  // number of dM_e block partials launch_agg_bwd writes

// tcgen05 3xTF32 GEMMs (tcgemm.cu); require H % 128 == 0
bool tc_supported(const Caps &c);
cudaError_t tc_configure();  // opt-in shared-memory sizes (call once, outside graph capture)
void launch_tc_update(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *A, const float *amp,
                      const float *att, const float *U, const float *bU, float *X1);
void launch_tc_dA(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dZ, const float *amp,
                  const float *att, const float *UT, float *dA);
void launch_tc_dU(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dZ, const float *A,
                  const float *amp, const float *att, float *partial, float *dU, float *dbU);
size_t tc_dU_partial_floats(const Caps &c);
bool tc_proj_ok(const Caps &c, int F);  // X rows 16-byte aligned
bool tc_dmx_ok(const Caps &c, int F);
void launch_tc_proj(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *X, int F, const float *Mx,
                    float *P);
void launch_tc_dX(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *Mx, int F,
                  const float *Xl, float *dZprev);
size_t tc_dMx_partial_floats(const Caps &c, int F);
void launch_tc_dMx(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *X, int F,
                   float *partial, float *dMx, float *dbM);
// UT[l][s*4H + n][h] = U_l[h][s*4H + n] for all layers (u_off: device array of U offsets in floats)
void launch_prep_UT(cudaStream_t st, const Caps &c, const float *params, const int64_t *u_off_dev, int L,
                    float *UT);

// process-wide count of kernels launched by the wrappers above
int64_t launches_so_far();

}  // namespace hg
