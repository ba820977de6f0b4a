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
                                                  double delta_lin, int deg_cap) {
  extern __shared__ uint8_t sdeg[];  // the batch's degrees (N <= deg_cap), else read from rowptr
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
  // degrees and per-node scalers in one coalesced pass (independent loads; the rounds below
  // then read shared memory instead of a dependent global chain per round)
  const bool sd = b.N <= deg_cap;
  // (four nodes per thread per round: their rowptr loads are issued before any store, so the
  // round costs one memory latency -- ncu: the one-node loop stalled on every load)
  for (int i0 = tid; i0 < b.N; i0 += 4 * blockDim.x) {
    int r0[4], r1[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      r0[u] = i < b.N ? __ldg(b.rowptr + i) : 0;
      r1[u] = i < b.N ? __ldg(b.rowptr + i + 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < b.N) {
        const int d = min(r1[u] - r0[u], kDeg - 1);
        if (sd) sdeg[i] = (uint8_t)d;
        amp[i] = tsc[1][d];
        att[i] = tsc[2][d];
      }
    }
  }
  __syncthreads();
  // warp w owns the contiguous node range [w*per, (w+1)*per), in rounds of 32 nodes; ranks
  // inside a round come from __match_any_sync (stable within the warp's range)
  const int per = (b.N + 31) / 32;
  const int w0 = warp * per, w1 = min(b.N, w0 + per);
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int d = i < w1 ? (sd ? (int)sdeg[i] : min(b.rowptr[i + 1] - b.rowptr[i], kDeg - 1)) : -1;
    const unsigned mask = __match_any_sync(0xffffffffu, d);  // (8 ballots measured slower: 43 vs 26 us at D)
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
  // class table (warp 0, 4 degrees per lane): degree starts = exclusive scan of the histogram,
  // class index = exclusive count of present degrees (at most cmax), tile and split bases =
  // exclusive scans of the classes' tile / split counts (thread 0's serial loop over the
  // degrees and the tile lists was ~10 us of the step's critical start at config B)
  __shared__ int cls_start[kMaxClasses], cls_count[kMaxClasses], cls_t0[kMaxClasses],
      cls_s0[kMaxClasses];
  __shared__ int nC;
  if (warp == 0) {
    int h[4], pres[4], nt[4], ns[4];
    int sh = 0, sp = 0, stl = 0, ssp = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int d = lane * 4 + q;
      h[q] = d < kDeg ? hist[d] : 0;
      pres[q] = h[q] > 0;
      sh += h[q];
      sp += pres[q];
    }
    // exclusive scans over the lanes: node offset and present-degree count
    int ih = sh, ip = sp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ih, o), b2 = __shfl_up_sync(0xffffffffu, ip, o);
      if (lane >= o) { ih += a; ip += b2; }
    }
    int off = ih - sh, cidx = ip - sp;
    int cl[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int d = lane * 4 + q;
      if (d < kDeg) bstart[d] = off;
      off += h[q];
      cl[q] = pres[q] ? cidx : -1;
      cidx += pres[q];
      const bool keep = cl[q] >= 0 && cl[q] < cmax;
      nt[q] = keep ? (h[q] + kTileRows - 1) / kTileRows : 0;
      ns[q] = keep ? (h[q] + ks - 1) / ks : 0;
      stl += nt[q];
      ssp += ns[q];
    }
    int it = stl, is = ssp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, it, o), b2 = __shfl_up_sync(0xffffffffu, is, o);
      if (lane >= o) { it += a; is += b2; }
    }
    int t0 = it - stl, s0 = is - ssp;
    int st = ih - sh;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int d = lane * 4 + q;
      if (cl[q] >= 0 && cl[q] < cmax) {
        const int C = cl[q];
        info->deg[C] = d;
        info->start[C] = st;
        info->count[C] = h[q];
        for (int qq = 0, k = 0; qq < kMaxScalers; ++qq)
          if (smask & (1 << qq)) info->scal[k++][C] = tsc[qq][d];
        cls_start[C] = st;
        cls_count[C] = h[q];
        cls_t0[C] = t0;
        cls_s0[C] = s0;
      }
      st += h[q];
      t0 += nt[q];
      s0 += ns[q];
    }
    if (lane == 31) {
      const int Ctot = ip;  // (inclusive count of present degrees)
      const int C = Ctot < cmax ? Ctot : cmax;
      nC = C;
      info->C = C;
      info->T = it;
      info->S = is;
      info->overflow = Ctot > cmax;  // more distinct degrees than class slots (hg_pack rejects such batches)
    }
  }
  __syncthreads();
  // tiles and splits carry the class index c: the class weights W_c are indexed by it
  for (int C = 0; C < nC; ++C) {
    const int start = cls_start[C], cnt = cls_count[C];
    const int ntl = (cnt + kTileRows - 1) / kTileRows, nsp = (cnt + ks - 1) / ks;
    for (int r = tid; r < ntl; r += blockDim.x)
      tiles[cls_t0[C] + r] = make_int4(C, start + r * kTileRows, min(kTileRows, cnt - r * kTileRows), 0);
    for (int r = tid; r < nsp; r += blockDim.x)
      splits[cls_s0[C] + r] = make_int4(C, start + r * ks, min(ks, cnt - r * ks), 0);
  }
  // scatter: the same rounds again; row = degree start + warp base + running rank
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int d = i < w1 ? (sd ? (int)sdeg[i] : min(b.rowptr[i + 1] - b.rowptr[i], kDeg - 1)) : -1;
    const unsigned mask = __match_any_sync(0xffffffffu, d);  // (8 ballots measured slower: 43 vs 26 us at D)
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

constexpr int kDegCap = 160 * 1024;  // degrees staged in shared memory up to this many nodes
static int deg_cap(int maxN) { return std::min(maxN, kDegCap); }
cudaError_t degsort_configure() {
  return cudaFuncSetAttribute(k_degsort, cudaFuncAttributeMaxDynamicSharedMemorySize, kDegCap);
}
void launch_degsort(cudaStream_t st, const uint8_t *blob, double delta, int cmax, float *amp, float *att, int *perm,
                    DegInfo *info, int4 *tiles, int4 *splits, int *pos, int4 *gslice, int smask, double delta_lin,
                    int ks, int maxN) {
  const int cap = deg_cap(maxN);
  launch_ex(k_degsort, 1, 1024, (size_t)((cap + 15) & ~15), st, blob, delta, cmax, ks > 0 ? ks : kGramKS, amp, att,
            perm, info, tiles, splits, pos, gslice, smask, delta_lin, cap);
  g_launches += 1;
}

}  // namespace hg
