// degsort.cu — degree classes of a batch (DESIGN.md §6 "Degree-class reassociation").
//
// The PNA scalers amp = ln(d+1)/delta and att = delta/ln(d+1) (SURVEY
// C4-C5) depend only on a node's in-degree d, so for the nodes of one degree the three
// scaler blocks of U collapse into one matrix (exact reassociation of SPEC.md:347's
// U . [A || amp A || att A]):
//   Z_i   = A_i W_d^T + b_U,          W_d = U_id + amp(d) U_amp + att(d) U_att   (update)
//   dA_i  = dZ_i W_d                                                              (dA)
//   dU_s  = sum_d s(d) G_d,           G_d = dZ_d^T A_d over the class's nodes      (dU)
// One class per DISTINCT degree present in the batch (any degree <= HG_MAX_DEGREE; at most
// the ctx's class slots, checked on the host when the batch is packed). Classes are
// numbered in ascending degree order; the class-indexed weights W_c are prepared per batch
// (k_prep_W2 reads the class table). Rows are degree-sorted so every 128-row GEMM tile and
// every Gram K-split lies inside one class.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "kernels.h"

namespace hg {

extern std::atomic<int64_t> g_launches;

constexpr int kTileRows = 128;  // GEMM output tile rows (T_BM in tcdirect.cu)
constexpr int kDeg = HG_MAX_DEGREE_DEV + 1;

// One CTA of 1024 threads: stable counting sort of the nodes by degree (deterministic),
// per-node scalers, the class table, the 128-row tiles and the Gram K-splits.
// perm[r] = node at degree-sorted row r, pos[i] = its inverse.
__global__ void __launch_bounds__(1024) k_degsort(const uint8_t *__restrict__ blob, double delta, int cmax, int ks,
                                                  float *__restrict__ amp, float *__restrict__ att,
                                                  int *__restrict__ perm, DegInfo *__restrict__ info,
                                                  int4 *__restrict__ tiles, int4 *__restrict__ splits,
                                                  int *__restrict__ pos, int4 *__restrict__ gslice, int smask,
                                                  double delta_lin) {
  pdl_enter();
  __shared__ int hist[kDeg], bstart[kDeg];
  __shared__ int wcnt[32][kDeg];  // per-warp degree counts, then per-warp bases within the degree
  __shared__ float tsc[kMaxScalers][kDeg];  // scaler k (bit order) of every degree
  const BatchView b = load_batch(blob);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kDeg) {  // scalers of every degree, fp64 as the oracle, stored fp32; all 1 at d = 0
    const double d = (double)tid, ld = log(d + 1.0);
    tsc[0][tid] = 1.0f;
    tsc[1][tid] = tid ? (float)(ld / delta) : 1.0f;
    tsc[2][tid] = tid ? (float)(delta / ld) : 1.0f;
    tsc[3][tid] = tid ? (float)(d / delta_lin) : 1.0f;
    tsc[4][tid] = tid ? (float)(delta_lin / d) : 1.0f;
  }
  for (int e = tid; e < 32 * kDeg; e += blockDim.x) wcnt[e / kDeg][e % kDeg] = 0;
  // per graph (n0, n1, e0, e1): the aggregation kernels' CTAs read their graph's node and edge
  // ranges with one load instead of the dependent graph_ptr -> rowptr chain
  for (int g = tid; g < b.B; g += blockDim.x) {
    const int n0 = b.gp[g], n1 = b.gp[g + 1];
    gslice[g] = make_int4(n0, n1, b.rowptr[n0], b.rowptr[n1]);
  }
  __syncthreads();
  // warp w owns the contiguous node range [w*per, (w+1)*per), in rounds of 32 nodes; ranks
  // inside a round come from __match_any_sync (stable within the warp's range)
  const int per = (b.N + 31) / 32;
  const int w0 = warp * per, w1 = min(b.N, w0 + per);
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int d = i < w1 ? min(b.rowptr[i + 1] - b.rowptr[i], kDeg - 1) : -1;
    if (i < w1) {
      amp[i] = tsc[1][d];
      att[i] = tsc[2][d];
    }
    const unsigned mask = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(mask & ((1u << lane) - 1u));
    if (d >= 0 && rank == 0) wcnt[warp][d] += __popc(mask);
    __syncwarp();
  }
  __syncthreads();
  if (tid < kDeg) {  // per degree: total and exclusive scan over the warps in warp order
    int acc = 0;
    for (int w = 0; w < 32; ++w) {
      const int c = wcnt[w][tid];
      wcnt[w][tid] = acc;
      acc += c;
    }
    hist[tid] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    int off = 0, C = 0, T = 0, S = 0, over = 0;
    for (int d = 0; d < kDeg; ++d) {
      bstart[d] = off;
      if (hist[d] > 0) {
        if (C < cmax) {
          info->deg[C] = d;
          info->start[C] = off;
          info->count[C] = hist[d];
          for (int q = 0, k = 0; q < kMaxScalers; ++q)
            if (smask & (1 << q)) info->scal[k++][C] = tsc[q][d];
          // tiles and splits carry the class index c: the class weights W_c are indexed by it
          for (int r = 0; r < hist[d]; r += kTileRows)
            tiles[T++] = make_int4(C, off + r, min(kTileRows, hist[d] - r), 0);
          for (int r = 0; r < hist[d]; r += ks) splits[S++] = make_int4(C, off + r, min(ks, hist[d] - r), 0);
          ++C;
        } else {
          over = 1;  // more distinct degrees than class slots (hg_pack rejects such batches)
        }
      }
      off += hist[d];
    }
    info->C = C;
    info->T = T;
    info->S = S;
    info->overflow = over;
  }
  __syncthreads();
  // scatter: the same rounds again; row = degree start + warp base + running rank
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int d = i < w1 ? min(b.rowptr[i + 1] - b.rowptr[i], kDeg - 1) : -1;
    const unsigned mask = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(mask & ((1u << lane) - 1u));
    if (d >= 0) {
      const int r = bstart[d] + wcnt[warp][d] + rank;
      perm[r] = i;
      if (pos) pos[i] = r;
    }
    __syncwarp();
    if (d >= 0 && rank == 0) wcnt[warp][d] += __popc(mask);
    __syncwarp();
  }
}

int tc_num_classes(int max_degree) {
  const int dmax = max_degree > 0 ? max_degree : HG_MAX_DEGREE_DEV;
  return std::min(dmax + 1, kMaxClasses);
}
int tc_max_tiles(const Caps &c, int cmax) { return (c.maxN + kTileRows - 1) / kTileRows + cmax; }
int tc_max_splits(const Caps &c, int cmax) { return (c.maxN + gram_ks(c) - 1) / gram_ks(c) + cmax; }

void launch_degsort(cudaStream_t st, const uint8_t *blob, double delta, int cmax, float *amp, float *att, int *perm,
                    DegInfo *info, int4 *tiles, int4 *splits, int *pos, int4 *gslice, int smask, double delta_lin,
                    int ks) {
  launch_ex(k_degsort, 1, 1024, 0, st, blob, delta, cmax, ks > 0 ? ks : kGramKS, amp, att, perm, info, tiles, splits,
            pos, gslice, smask, delta_lin);
  g_launches += 1;
}

}  // namespace hg
