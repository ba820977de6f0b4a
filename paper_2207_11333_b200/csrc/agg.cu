// agg.cu — K2 (edge gather + multi-aggregator segmented reduction) and K8 (its backward +
// scatter to the sources), SURVEY §8(a4), §8(a10).
//
// Paper passages: message passing (§3.1) with the PNA aggregators
// (PAPER.md:148), fixed by SPEC.md:347 (message M [x_j || e_ij] + b_M; aggregators mean, min,
// max, std with variance floor eps_v) and the backward SPEC.md:369-371.
//
// Molecules are graph-local and a batch's graphs are contiguous node ranges, so one CTA owns
// one graph (and one chunk of channels): every row it touches -- the CSR slice, the P rows of
// the messages' sources, the per-destination gradients -- belongs to its graph. The CTA
// stages the graph's CSR slice and P rows in shared memory with bulk async copies
// (cp.async.bulk, one mbarrier), so the rowptr -> col -> P dependency chain runs at
// shared-memory latency and HBM sees only large contiguous reads and coalesced row writes.
// A graph larger than the staging capacity runs the same arithmetic straight from global
// memory (L2), so any graph size is supported.
//
// Determinism: no atomics. Forward: one warp per destination node, fixed edge order. Backward
// (two phases in shared memory): each edge's message gradient dm_{j->i} is computed once by
// its destination's warp into a per-edge buffer, then each source sums its edges' dm in its
// row order (dP_j); dM_e / db_M are per-CTA partials reduced in fixed order afterwards.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace hg {

extern std::atomic<int64_t> g_launches;

namespace {

constexpr int kWarps = 8;            // 256 threads per CTA
constexpr int kCapNodes = 128;       // nodes of one graph staged in shared memory
constexpr int kCapEdgesFwd = 320;    // its directed edges (forward)
constexpr int kCapEdgesBwd = 256;    // (backward: each edge also holds a dm row)
constexpr int kChFwd = 128;          // channels per forward CTA (4 per lane)
constexpr int kChBwd = 64;           // channels per backward CTA (2 per lane)

__host__ __device__ constexpr uint32_t r16(uint32_t b) { return (b + 15u) & ~15u; }

// dynamic shared-memory layout (byte offsets) of one CTA
struct SmemLayout {
  uint32_t P, rp, col, ea, pos, slot, dm, total;
};
__host__ __device__ inline SmemLayout smem_layout(int ch, int cap_n, int cap_e, int Fe, bool bwd) {
  SmemLayout L;
  L.P = 0;
  L.rp = L.P + (uint32_t)cap_n * ch * 4;
  L.col = L.rp + r16((cap_n + 8) * 4);
  L.ea = L.col + r16((cap_e + 8) * 4);
  L.pos = L.ea + r16(cap_e * Fe * 4 + 32);
  L.slot = L.pos + r16((cap_n + 8) * 4);
  L.dm = L.slot + (bwd ? r16(cap_e + 32) : 0);
  L.total = L.dm + (bwd ? (uint32_t)cap_e * ch * 4 : 0);
  return L;
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// The graph's staged slice: local indices of rowptr (r0), col (c0), pos (p0), slot (s0) --
// each array is copied from a 16-byte aligned start -- and the float offset of edge e0's
// attributes in the ea copy.
struct Slice {
  int n0, n1, e0, e1, r0, c0, p0, s0, ea_skip;
};

// Thread 0: stage rowptr[n0..n1], col/ea/slot[e0..e1), pos[n0..n1) and the graph's P rows
// (channels [ch0, ch0 + CH)) with bulk copies completing on one mbarrier; then every thread
// waits for it. Blob arrays start 16-byte aligned and the copies round up to 16 bytes (the
// overhang stays inside the blob).
template <int CH>
__device__ void stage_graph(const BatchView &b, const float *P, int H, int ch0, const int *pos, bool with_slot,
                            const SmemLayout &L, uint8_t *sm, uint64_t *bar, const Slice &s) {
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
    const uint32_t brp = r16((uint32_t)(s.n1 + 1 - s.r0) * 4);
    const uint32_t bcol = s.e1 > s.e0 ? r16((uint32_t)(s.e1 - s.c0) * 4) : 0;
    const uint32_t ea_a = ((uint32_t)s.e0 * b.Fe * 4) & ~15u;
    const uint32_t bea = s.e1 > s.e0 ? r16((uint32_t)s.e1 * b.Fe * 4 - ea_a) : 0;
    const uint32_t bpos = r16((uint32_t)(s.n1 - s.p0) * 4);
    const uint32_t bsl = with_slot && s.e1 > s.e0 ? r16((uint32_t)(s.e1 - s.s0)) : 0;
    const uint32_t brow = CH * 4, bP = (uint32_t)(s.n1 - s.n0) * brow;
    tc::mbar_expect_tx(bar, bP + brp + bcol + bea + bpos + bsl);
    if (H == CH) {
      bulk_g2s(sm + L.P, P + (size_t)s.n0 * H, bP, bar);
    } else {
      for (int r = 0; r < s.n1 - s.n0; ++r)
        bulk_g2s(sm + L.P + r * brow, P + (size_t)(s.n0 + r) * H + ch0, brow, bar);
    }
    bulk_g2s(sm + L.rp, b.rowptr + s.r0, brp, bar);
    if (bcol) bulk_g2s(sm + L.col, b.col + s.c0, bcol, bar);
    if (bea) bulk_g2s(sm + L.ea, reinterpret_cast<const uint8_t *>(b.ea) + ea_a, bea, bar);
    bulk_g2s(sm + L.pos, pos + s.p0, bpos, bar);
    if (bsl) bulk_g2s(sm + L.slot, b.slot + s.s0, bsl, bar);
  }
  __syncthreads();
  tc::mbar_wait(bar, 0);
}

template <int CPL>
__device__ __forceinline__ void ld_vec(const float *p, float (&v)[CPL]) {
  if constexpr (CPL == 4) {
    const float4 t = *reinterpret_cast<const float4 *>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    const float2 t = *reinterpret_cast<const float2 *>(p);
    v[0] = t.x; v[1] = t.y;
  }
}
template <int CPL>
__device__ __forceinline__ void st_vec(float *p, const float (&v)[CPL]) {
  if constexpr (CPL == 4) *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  else *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
}
template <int FE>
__device__ __forceinline__ void ld_edge(const float *ea, int Fe, float (&ef)[FE]) {
  if constexpr (FE == 4) {
    const float4 t = *reinterpret_cast<const float4 *>(ea);
    ef[0] = t.x; ef[1] = t.y; ef[2] = t.z; ef[3] = t.w;
  } else {
#pragma unroll
    for (int f = 0; f < FE; ++f) ef[f] = f < Fe ? ea[f] : 0.f;
  }
}
// message for CPL channels: m = (P + b_M) + sum_f M_e[:,f] e_f (same order in K2 and K8)
template <int CPL, int FE>
__device__ __forceinline__ void message(const float (&pj)[CPL], const float (&bm)[CPL], const float (&me)[CPL][FE],
                                        const float (&ef)[FE], float (&m)[CPL]) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    float v = pj[c] + bm[c];
#pragma unroll
    for (int f = 0; f < FE; ++f) v = fmaf(me[c][f], ef[f], v);
    m[c] = v;
  }
}

// Graph arrays read either from the staged copy (S) or straight from global memory.
template <bool S, int CH>
struct View {
  const int *rp, *col, *pos;
  const uint8_t *slot;
  const float *ea, *P;
  int r0, c0, p0, s0, e0, n0, Fe, Pstride, ch0;
  __device__ int rowptr(int i) const { return S ? rp[i - r0] : rp[i]; }
  __device__ int colv(int k) const { return S ? col[k - c0] : col[k]; }
  __device__ int posv(int i) const { return S ? pos[i - p0] : pos[i]; }
  __device__ int slotv(int k) const { return S ? slot[k - s0] : slot[k]; }
  __device__ const float *edge(int k) const { return S ? ea + (size_t)(k - e0) * Fe : ea + (size_t)k * Fe; }
  __device__ const float *prow(int j, int lc) const {  // lc = lane's first channel within the chunk
    return S ? P + (j - n0) * CH + lc : P + (size_t)j * Pstride + ch0 + lc;
  }
};
template <bool S, int CH>
__device__ View<S, CH> make_view(const BatchView &b, const float *P, int H, int ch0, const int *pos,
                                 const SmemLayout &L, uint8_t *sm, const Slice &s) {
  View<S, CH> v;
  v.Fe = b.Fe;
  v.ch0 = ch0;
  v.Pstride = H;
  v.n0 = s.n0;
  v.e0 = s.e0;
  if constexpr (S) {
    v.rp = reinterpret_cast<const int *>(sm + L.rp);
    v.col = reinterpret_cast<const int *>(sm + L.col);
    v.pos = reinterpret_cast<const int *>(sm + L.pos);
    v.slot = sm + L.slot;
    v.ea = reinterpret_cast<const float *>(sm + L.ea) + s.ea_skip;
    v.P = reinterpret_cast<const float *>(sm + L.P);
    v.r0 = s.r0; v.c0 = s.c0; v.p0 = s.p0; v.s0 = s.s0;
  } else {
    v.rp = b.rowptr; v.col = b.col; v.pos = pos; v.slot = b.slot; v.ea = b.ea; v.P = P;
    v.r0 = v.c0 = v.p0 = v.s0 = 0;
  }
  return v;
}

__device__ __forceinline__ Slice slice_of(const BatchView &b, int g) {
  Slice s;
  s.n0 = b.gp[g];
  s.n1 = b.gp[g + 1];
  s.e0 = b.rowptr[s.n0];
  s.e1 = b.rowptr[s.n1];
  s.r0 = s.n0 & ~3;
  s.c0 = s.e0 & ~3;
  s.p0 = s.n0 & ~3;
  s.s0 = s.e0 & ~15;
  s.ea_skip = (int)(((uint32_t)s.e0 * b.Fe * 4 - (((uint32_t)s.e0 * b.Fe * 4) & ~15u)) / 4);
  return s;
}

// ---------------------------------------------------------------- K2 forward
// Per destination node i (one warp), lanes over CPL = 4 channels each: messages
// m = P[j] + b_M + M_e e_ji over the CSR row (j ascending) are recomputed, never stored
// (SURVEY §8(a4)); pass 1: sum, min, max with first-position argmin / argmax; pass 2: the
// centred sum of squares (two-pass variance). d = 0 -> all aggregates 0 (C5).
// Writes A at the degree-sorted row pos[i] ([mean | min | max | std], 4H) and arg[i]
// ([argmin | argmax with bit 7 = var > eps_v], 2H bytes).
template <bool S, int FE>
__device__ void fwd_nodes(const View<S, kChFwd> &v, const Slice &s, const float (&me)[4][FE], const float (&bm)[4],
                          float var_floor, float *A, uint8_t *arg, int H, int Hl) {
  constexpr int CPL = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lc = lane * CPL, ch = v.ch0 + lc;
  for (int i = s.n0 + warp; i < s.n1; i += kWarps) {
    const int k0 = v.rowptr(i), k1 = v.rowptr(i + 1), d = k1 - k0;
    const int prow = v.posv(i);
    float sum[CPL], mx[CPL], mn[CPL];
    int amx[CPL], amn[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) { sum[c] = 0.f; mx[c] = -INFINITY; mn[c] = INFINITY; amx[c] = 0; amn[c] = 0; }
    for (int k = k0; k < k1; ++k) {
      const int j = v.colv(k);
      float ef[FE], pj[CPL], m[CPL];
      ld_edge<FE>(v.edge(k), v.Fe, ef);
      ld_vec<CPL>(v.prow(j, lc), pj);
      message<CPL, FE>(pj, bm, me, ef, m);
      const int p = k - k0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        sum[c] += m[c];
        if (m[c] > mx[c]) { mx[c] = m[c]; amx[c] = p; }
        if (m[c] < mn[c]) { mn[c] = m[c]; amn[c] = p; }
      }
    }
    float mean[CPL], sd[CPL];
    int flag[CPL];
    if (d == 0) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) { mean[c] = 0.f; mx[c] = 0.f; mn[c] = 0.f; sd[c] = 0.f; flag[c] = 0; }
    } else {
      const float rd = __frcp_rn((float)d);
      float ss[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) { mean[c] = sum[c] * rd; ss[c] = 0.f; }
      for (int k = k0; k < k1; ++k) {  // pass 2: recompute the messages
        const int j = v.colv(k);
        float ef[FE], pj[CPL], m[CPL];
        ld_edge<FE>(v.edge(k), v.Fe, ef);
        ld_vec<CPL>(v.prow(j, lc), pj);
        message<CPL, FE>(pj, bm, me, ef, m);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const float t = m[c] - mean[c];
          ss[c] = fmaf(t, t, ss[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const float var = ss[c] * rd;
        flag[c] = var > var_floor;
        // channels >= Hl are padding (internal width H > logical Hl): their messages are
        // exactly 0, and their std is forced to 0 instead of sqrt(var_floor) so that no
        // gradient reaches the zero padded parameters (SURVEY §8(d) padding hazard)
        sd[c] = ch + c < Hl ? sqrtf(fmaxf(var, var_floor)) : 0.f;
      }
    }
    float *Ai = A + (size_t)prow * (4 * H) + ch;
    st_vec<CPL>(Ai, mean);
    st_vec<CPL>(Ai + H, mn);
    st_vec<CPL>(Ai + 2 * H, mx);
    st_vec<CPL>(Ai + 3 * H, sd);
    uint8_t *ai = arg + (size_t)i * (2 * H) + ch;
    *reinterpret_cast<uchar4 *>(ai) = make_uchar4(amn[0], amn[1], amn[2], amn[3]);
    *reinterpret_cast<uchar4 *>(ai + H) =
        make_uchar4(amx[0] | (flag[0] << 7), amx[1] | (flag[1] << 7), amx[2] | (flag[2] << 7), amx[3] | (flag[3] << 7));
  }
}

template <int FE>
__global__ void __launch_bounds__(32 * kWarps) k_agg_fwd(const uint8_t *__restrict__ blob, const float *__restrict__ P,
                                                         const float *__restrict__ Me, const float *__restrict__ bM,
                                                         float var_floor, float *__restrict__ A,
                                                         uint8_t *__restrict__ arg, int H, const int *__restrict__ pos,
                                                         int Hl) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  pdl_enter();
  const BatchView b = load_batch(blob);
  const int g = blockIdx.x;
  if (g >= b.B) return;
  constexpr int CPL = 4;
  const int lane = threadIdx.x & 31, ch0 = blockIdx.y * kChFwd, ch = ch0 + lane * CPL;
  const int Fe = b.Fe;
  float me[CPL][FE], bm[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    bm[c] = bM[ch + c];
#pragma unroll
    for (int f = 0; f < FE; ++f) me[c][f] = f < Fe ? Me[(ch + c) * Fe + f] : 0.f;
  }
  const Slice s = slice_of(b, g);
  const SmemLayout L = smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, Fe, false);
  if (s.n1 - s.n0 <= kCapNodes && s.e1 - s.e0 <= kCapEdgesFwd) {  // uniform per CTA
    stage_graph<kChFwd>(b, P, H, ch0, pos, false, L, sm, &bar, s);
    fwd_nodes<true, FE>(make_view<true, kChFwd>(b, P, H, ch0, pos, L, sm, s), s, me, bm, var_floor, A, arg, H, Hl);
  } else {
    fwd_nodes<false, FE>(make_view<false, kChFwd>(b, P, H, ch0, pos, L, sm, s), s, me, bm, var_floor, A, arg, H, Hl);
  }
}

// ---------------------------------------------------------------- K8 backward
// Phase 1, one warp per DESTINATION node i (lanes over CPL = 2 channels): its gradients
// dA_i, mu_i, sigma_i and decisions are read once (coalesced rows), and for each in-edge
// (j -> i) at row position p:
//   dm = dA_mean[i]/d_i + [p = argmax_i] dA_max[i] + [p = argmin_i] dA_min[i]
//        + [var_i > eps_v] dA_std[i] (m - mu_i)/(d_i sigma_i)
// with the message m recomputed; dm goes to the per-edge buffer (destination-major, like the
// CSR), and into this CTA's dM_e = sum dm e^T and db_M = sum dm partials.
// Phase 2, one warp per SOURCE node j: dP_j = sum over its CSR row (edges j -> i, i = col[k])
// of dm at i's row position slot[k] (where phase 1 stored it), in row order.
template <bool S, int FE>
__device__ void bwd_phase1(const View<S, kChBwd> &v, const Slice &s, const float (&me)[2][FE], const float (&bm)[2],
                           const float *A, const uint8_t *arg, const float *dA, int H, float *dmbuf,
                           float (&acc)[2][FE], float (&bsum)[2]) {
  constexpr int CPL = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lc = lane * CPL, ch = v.ch0 + lc;
  for (int i = s.n0 + warp; i < s.n1; i += kWarps) {
    const int k0 = v.rowptr(i), k1 = v.rowptr(i + 1), d = k1 - k0;
    if (d == 0) continue;
    const float *dAi = dA + (size_t)i * (4 * H) + ch;
    const float *Ai = A + (size_t)v.posv(i) * (4 * H) + ch;
    float gmean[CPL], gmin[CPL], gmax[CPL], gstd[CPL], mu[CPL], sg[CPL];
    ld_vec<CPL>(dAi, gmean);
    ld_vec<CPL>(dAi + H, gmin);
    ld_vec<CPL>(dAi + 2 * H, gmax);
    ld_vec<CPL>(dAi + 3 * H, gstd);
    ld_vec<CPL>(Ai, mu);
    ld_vec<CPL>(Ai + 3 * H, sg);
    const uchar2 amn = *reinterpret_cast<const uchar2 *>(arg + (size_t)i * (2 * H) + ch);
    const uchar2 amx = *reinterpret_cast<const uchar2 *>(arg + (size_t)i * (2 * H) + H + ch);
    const int an[CPL] = {amn.x, amn.y}, ax[CPL] = {amx.x, amx.y};
    const float inv_d = __frcp_rn((float)d);
    float gs[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) gs[c] = (ax[c] & 0x80) ? gstd[c] * inv_d * __frcp_rn(sg[c]) : 0.f;
    for (int k = k0; k < k1; ++k) {
      const int j = v.colv(k), p = k - k0;
      float ef[FE], pj[CPL], m[CPL], dm[CPL];
      ld_edge<FE>(v.edge(k), v.Fe, ef);
      ld_vec<CPL>(v.prow(j, lc), pj);
      message<CPL, FE>(pj, bm, me, ef, m);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        float gg = gmean[c] * inv_d;
        if ((ax[c] & 0x7f) == p) gg += gmax[c];
        if (an[c] == p) gg += gmin[c];
        if (ax[c] & 0x80) gg += gs[c] * (m[c] - mu[c]);
        dm[c] = gg;
        bsum[c] += gg;
#pragma unroll
        for (int f = 0; f < FE; ++f) acc[c][f] = fmaf(gg, ef[f], acc[c][f]);
      }
      st_vec<CPL>(dmbuf + (size_t)(k - s.e0) * kChBwd + lc, dm);
    }
  }
}

template <bool S>
__device__ void bwd_phase2(const View<S, kChBwd> &v, const Slice &s, const float *dmbuf, float *dP, int H,
                           const int *dp_pos) {
  constexpr int CPL = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lc = lane * CPL, ch = v.ch0 + lc;
  for (int j = s.n0 + warp; j < s.n1; j += kWarps) {
    const int k0 = v.rowptr(j), k1 = v.rowptr(j + 1);
    float dp[CPL] = {0.f, 0.f};
    for (int k = k0; k < k1; ++k) {
      const int kd = v.rowptr(v.colv(k)) + v.slotv(k);  // edge j -> i in i's row
      float dm[CPL];
      ld_vec<CPL>(dmbuf + (size_t)(kd - s.e0) * kChBwd + lc, dm);
#pragma unroll
      for (int c = 0; c < CPL; ++c) dp[c] += dm[c];
    }
    st_vec<CPL>(dP + (size_t)(dp_pos ? v.posv(j) : j) * H + ch, dp);
  }
}

template <int FE>
__global__ void __launch_bounds__(32 * kWarps) k_agg_bwd(const uint8_t *__restrict__ blob, const float *__restrict__ P,
                                                         const float *__restrict__ Me, const float *__restrict__ bM,
                                                         const float *__restrict__ A, const uint8_t *__restrict__ arg,
                                                         const float *__restrict__ dA, float *__restrict__ dP,
                                                         float *__restrict__ partial, int H,
                                                         const int *__restrict__ pos, const int *__restrict__ dp_pos,
                                                         float *__restrict__ dm_global) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  pdl_enter();
  const BatchView b = load_batch(blob);
  const int g = blockIdx.x;
  constexpr int CPL = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, ch0 = blockIdx.y * kChBwd, ch = ch0 + lane * CPL;
  const int Fe = b.Fe;
  float me[CPL][FE], bm[CPL], acc[CPL][FE], bsum[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    bm[c] = bM[ch + c];
    bsum[c] = 0.f;
#pragma unroll
    for (int f = 0; f < FE; ++f) { me[c][f] = f < Fe ? Me[(ch + c) * Fe + f] : 0.f; acc[c][f] = 0.f; }
  }
  if (g < b.B) {  // (CTAs past the batch write zero partials)
    const Slice s = slice_of(b, g);
    const SmemLayout L = smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, Fe, true);
    if (s.n1 - s.n0 <= kCapNodes && s.e1 - s.e0 <= kCapEdgesBwd) {  // uniform per CTA
      stage_graph<kChBwd>(b, P, H, ch0, pos, true, L, sm, &bar, s);
      const View<true, kChBwd> v = make_view<true, kChBwd>(b, P, H, ch0, pos, L, sm, s);
      float *dmbuf = reinterpret_cast<float *>(sm + L.dm);
      bwd_phase1<true, FE>(v, s, me, bm, A, arg, dA, H, dmbuf, acc, bsum);
      __syncthreads();
      bwd_phase2<true>(v, s, dmbuf, dP, H, dp_pos);
    } else {  // a graph too large to stage: the per-edge buffer lives in global memory
      const View<false, kChBwd> v = make_view<false, kChBwd>(b, P, H, ch0, pos, L, sm, s);
      float *dmbuf = dm_global + (size_t)blockIdx.y * b.E * kChBwd;  // this chunk's [E][64] slice
      Slice sg = s;
      sg.e0 = 0;  // (the global buffer is indexed by the batch edge id)
      bwd_phase1<false, FE>(v, sg, me, bm, A, arg, dA, H, dmbuf, acc, bsum);
      __syncthreads();  // (also orders the block's global writes before phase 2's reads)
      bwd_phase2<false>(v, sg, dmbuf, dP, H, dp_pos);
    }
  }
  // CTA partials of dM_e and db_M, warps combined in fixed order; layout per graph row:
  // [H][Fe] (M_e's layout) then [H] (b_M). The staging area is free again: it holds the
  // per-warp sums red[warp][lane][c * (FE + 1) + f].
  constexpr int RS = CPL * (FE + 1);
  float *red = reinterpret_cast<float *>(sm);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    red[(warp * 32 + lane) * RS + c * (FE + 1) + FE] = bsum[c];
#pragma unroll
    for (int f = 0; f < FE; ++f) red[(warp * 32 + lane) * RS + c * (FE + 1) + f] = acc[c][f];
  }
  __syncthreads();
  float *pb = partial + (size_t)g * H * (Fe + 1);
  for (int t = threadIdx.x; t < kChBwd * (Fe + 1); t += blockDim.x) {
    const bool isb = t >= kChBwd * Fe;
    const int cc = isb ? t - kChBwd * Fe : t / Fe, f = isb ? FE : t - (t / Fe) * Fe;  // channel in chunk, feature
    const int l = cc / CPL, c = cc - l * CPL;
    float sum = 0.f;
    for (int w = 0; w < kWarps; ++w) sum += red[(w * 32 + l) * RS + c * (FE + 1) + f];
    if (isb) pb[(size_t)H * Fe + ch0 + cc] = sum;
    else pb[(size_t)(ch0 + cc) * Fe + f] = sum;
  }
}

}  // namespace

cudaError_t agg_configure() {
  cudaError_t e;
  const uint32_t f4 = smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, 4, false).total;
  const uint32_t f8 = smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, 8, false).total;
  const uint32_t b4 = smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, 4, true).total;
  const uint32_t b8 = smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, 8, true).total;
  if ((e = cudaFuncSetAttribute(k_agg_fwd<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f4)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_agg_fwd<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f8)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_agg_bwd<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b4)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_agg_bwd<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b8)) != cudaSuccess)
    return e;
  return cudaSuccess;
}

void launch_agg_fwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *P, const float *Me,
                    const float *bM, float var_floor, float *A, uint8_t *arg, const int *pos) {
  const dim3 grid(c.maxB, c.H / kChFwd);
  const int Hl = c.Hl > 0 ? c.Hl : c.H;
  if (c.Fe == 4)
    launch_ex(k_agg_fwd<4>, grid, 32 * kWarps, smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, 4, false).total, st, blob,
              P, Me, bM, var_floor, A, arg, c.H, pos, Hl);
  else
    launch_ex(k_agg_fwd<8>, grid, 32 * kWarps, smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, c.Fe, false).total, st,
              blob, P, Me, bM, var_floor, A, arg, c.H, pos, Hl);
  g_launches += 1;
}

size_t agg_bwd_partial_floats(const Caps &c) { return (size_t)c.maxB * c.H * (c.Fe + 1); }
size_t agg_bwd_dm_floats(const Caps &c) { return (size_t)c.maxE * c.H; }

void launch_agg_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *P, const float *Me,
                    const float *bM, const float *A, const uint8_t *arg, const float *dA, float *dP, float *partial,
                    const int *pos, const int *dp_pos, float *dm_scratch) {
  const dim3 grid(c.maxB, c.H / kChBwd);
  if (c.Fe == 4)
    launch_ex(k_agg_bwd<4>, grid, 32 * kWarps, smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, 4, true).total, st, blob,
              P, Me, bM, A, arg, dA, dP, partial, c.H, pos, dp_pos, dm_scratch);
  else
    launch_ex(k_agg_bwd<8>, grid, 32 * kWarps, smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, c.Fe, true).total, st,
              blob, P, Me, bM, A, arg, dA, dP, partial, c.H, pos, dp_pos, dm_scratch);
  g_launches += 1;
}

}  // namespace hg
