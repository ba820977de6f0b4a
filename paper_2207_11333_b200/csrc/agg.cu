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
// (two phases): each edge's message gradient dm_{j->i} is computed once by its destination's
// warp into a per-edge buffer (global, L2-resident), then each source sums its edges' dm in its
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
constexpr int kCapEdgesBwd = 320;    // (backward)
constexpr int kChFwd = 64;           // channels per forward CTA (2 per lane)
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
  L.total = L.dm;  // (the backward's per-edge dm rows live in global memory, L2-resident)
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
__device__ void stage_graph(const BatchView &b, const float *P, int PW, int ch0, const int *pos, bool with_slot,
                            const SmemLayout &L, uint8_t *sm, uint64_t *bar, const Slice &s, uint32_t parity) {
  if (threadIdx.x == 0) {
    const uint32_t brp = r16((uint32_t)(s.n1 + 1 - s.r0) * 4);
    const uint32_t bcol = s.e1 > s.e0 ? r16((uint32_t)(s.e1 - s.c0) * 4) : 0;
    const uint32_t ea_a = ((uint32_t)s.e0 * b.Fe * 4) & ~15u;
    const uint32_t bea = s.e1 > s.e0 ? r16((uint32_t)s.e1 * b.Fe * 4 - ea_a) : 0;
    const uint32_t bpos = r16((uint32_t)(s.n1 - s.p0) * 4);
    const uint32_t bsl = with_slot && s.e1 > s.e0 ? r16((uint32_t)(s.e1 - s.s0)) : 0;
    const uint32_t brow = CH * 4, bP = (uint32_t)(s.n1 - s.n0) * brow;
    tc::mbar_expect_tx(bar, bP + brp + bcol + bea + bpos + bsl);
    if (PW == CH) {
      bulk_g2s(sm + L.P, P + (size_t)s.n0 * PW, bP, bar);
    } else {  // (P rows of PW floats: this chunk's CH columns of each row)
      for (int r = 0; r < s.n1 - s.n0; ++r)
        bulk_g2s(sm + L.P + r * brow, P + (size_t)(s.n0 + r) * PW + ch0, brow, bar);
    }
    bulk_g2s(sm + L.rp, b.rowptr + s.r0, brp, bar);
    if (bcol) bulk_g2s(sm + L.col, b.col + s.c0, bcol, bar);
    if (bea) bulk_g2s(sm + L.ea, reinterpret_cast<const uint8_t *>(b.ea) + ea_a, bea, bar);
    bulk_g2s(sm + L.pos, pos + s.p0, bpos, bar);
    if (bsl) bulk_g2s(sm + L.slot, b.slot + s.s0, bsl, bar);
  }
  tc::mbar_wait(bar, parity);
}

__device__ __forceinline__ void init_bar(uint64_t *bar) {
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
  }
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
__device__ View<S, CH> make_view(const BatchView &b, const float *P, int PW, int ch0, const int *pos,
                                 const SmemLayout &L, uint8_t *sm, const Slice &s) {
  View<S, CH> v;
  v.Fe = b.Fe;
  v.ch0 = ch0;
  v.Pstride = PW;
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

__device__ __forceinline__ Slice slice_of(const BatchView &b, const int4 *gslice, int g) {
  const int4 q = gslice[g];  // (n0, n1, e0, e1), written by the degree sort
  Slice s;
  s.n0 = q.x;
  s.n1 = q.y;
  s.e0 = q.z;
  s.e1 = q.w;
  s.r0 = s.n0 & ~3;
  s.c0 = s.e0 & ~3;
  s.p0 = s.n0 & ~3;
  s.s0 = s.e0 & ~15;
  s.ea_skip = (int)(((uint32_t)s.e0 * b.Fe * 4 - (((uint32_t)s.e0 * b.Fe * 4) & ~15u)) / 4);
  return s;
}

// ---------------------------------------------------------------- K2 forward
// Per destination node i (one warp), lanes over CPL = 4 channels each: messages
// m = P[j] + b_M + M_e e_ji over the CSR row (j ascending) are recomputed, never stored in
// memory; pass 1: sum, min, max with first-position argmin / argmax; pass 2:
// the centred sum of squares (two-pass variance). Rows of degree <= 4 (molecules:
// all but hubs) keep their messages in registers between the passes; larger rows recompute
// them. d = 0 -> all aggregates 0 (C5). Writes A at the degree-sorted row pos[i]
// ([mean | min | max | std], 4H) and arg[i] ([argmin | argmax with bit 7 = var > eps_v], 2H).
template <int CPL>
__device__ __forceinline__ void fold(const float (&m)[CPL], int p, float (&sum)[CPL], float (&mx)[CPL],
                                     float (&mn)[CPL], int (&amx)[CPL], int (&amn)[CPL]) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    sum[c] += m[c];
    if (m[c] > mx[c]) { mx[c] = m[c]; amx[c] = p; }
    if (m[c] < mn[c]) { mn[c] = m[c]; amn[c] = p; }
  }
}

// Self-term variant (Sf): the message also carries Q_i = M_s x_i (the projection's second half,
// P rows [P | Q]), a per-destination constant, so mean, min and max shift by Q_i and std does
// not (d > 0; d = 0 stays all zero, C5); and A's fifth block is the layer input x_i (zero
// padded to H columns) for the update's [.. || x_i] [.. | U_x]^T.
struct SelfIn {
  const float *P;    // the [P | Q] buffer (row stride PW = 2H), null = no self-term
  const float *xin;  // layer input rows, stride Fl (layer 0: the batch's raw x)
  int PW, Fl;
};

template <bool S, bool SELF, int FE>
__device__ void fwd_nodes(const View<S, kChFwd> &v, const Slice &s, const float (&me)[2][FE], const float (&bm)[2],
                          float var_floor, float *A, uint8_t *arg, int H, int Hl, int KA, const SelfIn &si) {
  constexpr int CPL = 2, RM = 4;  // RM: messages held in registers
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lc = lane * CPL, ch = v.ch0 + lc;
  for (int i = s.n0 + warp; i < s.n1; i += kWarps) {
    const int k0 = v.rowptr(i), k1 = v.rowptr(i + 1), d = k1 - k0;
    const int prow = v.posv(i);
    float q[CPL] = {0.f, 0.f}, xi[CPL] = {0.f, 0.f};
    if (SELF) {  // (issued early: hidden behind the edge loop)
      ld_vec<CPL>(si.P + (size_t)i * si.PW + H + ch, q);
#pragma unroll
      for (int c = 0; c < CPL; ++c) xi[c] = ch + c < si.Fl ? si.xin[(size_t)i * si.Fl + ch + c] : 0.f;
    }
    float sum[CPL], mx[CPL], mn[CPL], ss[CPL];
    int amx[CPL], amn[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      sum[c] = 0.f; mx[c] = -INFINITY; mn[c] = INFINITY; amx[c] = 0; amn[c] = 0; ss[c] = 0.f;
    }
    const float rd = d > 0 ? __frcp_rn((float)d) : 0.f;
    if (d <= RM) {  // (warp-uniform) one load pass, messages kept for the variance pass
      float m[RM][CPL];
#pragma unroll
      for (int e = 0; e < RM; ++e) {
        if (e < d) {
          const int j = v.colv(k0 + e);
          float ef[FE], pj[CPL];
          ld_edge<FE>(v.edge(k0 + e), v.Fe, ef);
          ld_vec<CPL>(v.prow(j, lc), pj);
          message<CPL, FE>(pj, bm, me, ef, m[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < RM; ++e)
        if (e < d) fold<CPL>(m[e], e, sum, mx, mn, amx, amn);
#pragma unroll
      for (int e = 0; e < RM; ++e)
        if (e < d) {
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const float t = m[e][c] - sum[c] * rd;
            ss[c] = fmaf(t, t, ss[c]);
          }
        }
    } else {
      for (int k = k0; k < k1; ++k) {
        const int j = v.colv(k);
        float ef[FE], pj[CPL], m[CPL];
        ld_edge<FE>(v.edge(k), v.Fe, ef);
        ld_vec<CPL>(v.prow(j, lc), pj);
        message<CPL, FE>(pj, bm, me, ef, m);
        fold<CPL>(m, k - k0, sum, mx, mn, amx, amn);
      }
      for (int k = k0; k < k1; ++k) {  // pass 2: recompute the messages
        const int j = v.colv(k);
        float ef[FE], pj[CPL], m[CPL];
        ld_edge<FE>(v.edge(k), v.Fe, ef);
        ld_vec<CPL>(v.prow(j, lc), pj);
        message<CPL, FE>(pj, bm, me, ef, m);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const float t = m[c] - sum[c] * rd;
          ss[c] = fmaf(t, t, ss[c]);
        }
      }
    }
    float mean[CPL], sd[CPL];
    int flag[CPL];
    if (d == 0) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) { mean[c] = 0.f; mx[c] = 0.f; mn[c] = 0.f; sd[c] = 0.f; flag[c] = 0; }
    } else {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        mean[c] = sum[c] * rd + q[c];  // (q = 0 without the self-term)
        mx[c] += q[c];
        mn[c] += q[c];
        const float var = ss[c] * rd;
        flag[c] = var > var_floor;
        // channels >= Hl are padding (internal width H > logical Hl): their messages are
        // exactly 0, and their std is forced to 0 instead of sqrt(var_floor) so that no
        // gradient reaches the zero padded parameters (SURVEY §8(d) padding hazard)
        // (sqrt as v * rsqrt(v): two MUFU-based instructions instead of the IEEE sqrt sequence,
        // ~2 ulp -- ncu: the IEEE sqrtf was 14% of this kernel's instructions)
        const float vf = fmaxf(var, var_floor);
        sd[c] = ch + c < Hl ? vf * rsqrtf(vf) : 0.f;
      }
    }
    float *Ai = A + (size_t)prow * KA + ch;
    st_vec<CPL>(Ai, mean);
    st_vec<CPL>(Ai + H, mn);
    st_vec<CPL>(Ai + 2 * H, mx);
    st_vec<CPL>(Ai + 3 * H, sd);
    if (SELF) st_vec<CPL>(Ai + 4 * H, xi);
    uint8_t *ai = arg + (size_t)i * (2 * H) + ch;
    *reinterpret_cast<uchar2 *>(ai) = make_uchar2(amn[0], amn[1]);
    *reinterpret_cast<uchar2 *>(ai + H) = make_uchar2(amx[0] | (flag[0] << 7), amx[1] | (flag[1] << 7));
  }
}

template <bool SELF, int FE>
__global__ void __launch_bounds__(32 * kWarps, 4) k_agg_fwd(const uint8_t *__restrict__ blob,
                                                            const int4 *__restrict__ gslice,
                                                            const float *__restrict__ P, const float *__restrict__ Me,
                                                            const float *__restrict__ bM, float var_floor,
                                                            float *__restrict__ A, uint8_t *__restrict__ arg, int H,
                                                            const int *__restrict__ pos, int Hl, int KA, SelfIn si) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  pdl_enter();
  const BatchView b = load_batch(blob);
  constexpr int CPL = 2;
  const int lane = threadIdx.x & 31, nch = H / kChFwd, PW = si.PW;
  const int Fe = b.Fe;
  const SmemLayout L = smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, Fe, false);
  if (SELF && !si.xin) si.xin = b.x;  // layer 0: the batch's node features
  init_bar(&bar);
  const uint32_t parity = 0;
  {  // one work item (graph, channel chunk) per CTA
    const int item = blockIdx.x;
    if (item >= b.B * nch) return;
    __syncthreads();  // (the barrier's initialisation is visible)
    const int g = item / nch, ch0 = (item - g * nch) * kChFwd, ch = ch0 + lane * CPL;
    const Slice s = slice_of(b, gslice, g);
    const bool staged = s.n1 - s.n0 <= kCapNodes && s.e1 - s.e0 <= kCapEdgesFwd;  // uniform per CTA
    if (staged) stage_graph<kChFwd>(b, P, PW, ch0, pos, false, L, sm, &bar, s, parity);
    float me[CPL][FE], bm[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      bm[c] = bM[ch + c];
#pragma unroll
      for (int f = 0; f < FE; ++f) me[c][f] = f < Fe ? Me[(ch + c) * Fe + f] : 0.f;
    }
    if (staged)
      fwd_nodes<true, SELF, FE>(make_view<true, kChFwd>(b, P, PW, ch0, pos, L, sm, s), s, me, bm, var_floor, A, arg, H,
                                Hl, KA, si);
    else
      fwd_nodes<false, SELF, FE>(make_view<false, kChFwd>(b, P, PW, ch0, pos, L, sm, s), s, me, bm, var_floor, A, arg,
                                 H, Hl, KA, si);
  }
}

// ---------------------------------------------------------------- K8 backward
// Phase 1, one warp per DESTINATION node i (lanes over CPL = 2 channels): its gradients
// dA_i, mu_i, sigma_i and decisions are read once (coalesced rows; the next node's are
// requested before this node is processed), and for each in-edge (j -> i) at row position p
// (SURVEY §8(a10)):
//   dm = dA_mean[i]/d_i + [p = argmax_i] dA_max[i] + [p = argmin_i] dA_min[i]
//        + [var_i > eps_v] dA_std[i] (m - mu_i)/(d_i sigma_i)
// with the message m recomputed from the staged P rows; dm goes to the per-edge buffer
// (destination-major like the CSR, [E][H], L2-resident) and into this CTA's dM_e = sum dm e^T
// and db_M = sum dm partials.
// Phase 2, one warp per SOURCE node j: dP_j = sum over its CSR row (edges j -> i, i = col[k])
// of dm at i's row position slot[k] (where phase 1 stored it), in row order.
struct DstIn {  // one destination's per-channel inputs (CPL = 2)
  float2 gmean, gmin, gmax, gstd, mu, sg, q;
  uchar2 amn, amx;
  int k0, k1;
};
template <bool S, bool SELF>
__device__ __forceinline__ DstIn load_dst(const View<S, kChBwd> &v, int i, const float *A, const uint8_t *arg,
                                          const float *dA, int H, int ch, int KA, const float *Q, int PW) {
  DstIn t;
  t.k0 = v.rowptr(i);
  t.k1 = v.rowptr(i + 1);
  const float *dAi = dA + (size_t)i * KA + ch;
  const float *Ai = A + (size_t)v.posv(i) * KA + ch;
  t.q = SELF ? *reinterpret_cast<const float2 *>(Q + (size_t)i * PW + ch) : make_float2(0.f, 0.f);
  t.gmean = *reinterpret_cast<const float2 *>(dAi);
  t.gmin = *reinterpret_cast<const float2 *>(dAi + H);
  t.gmax = *reinterpret_cast<const float2 *>(dAi + 2 * H);
  t.gstd = *reinterpret_cast<const float2 *>(dAi + 3 * H);
  t.mu = *reinterpret_cast<const float2 *>(Ai);
  t.sg = *reinterpret_cast<const float2 *>(Ai + 3 * H);
  t.amn = *reinterpret_cast<const uchar2 *>(arg + (size_t)i * (2 * H) + ch);
  t.amx = *reinterpret_cast<const uchar2 *>(arg + (size_t)i * (2 * H) + H + ch);
  return t;
}

// (self-term: Qp = the [P | Q] buffer's Q half (stride PW), the messages include Q_i, and the
// destination's dQ_i = dA_mean + dA_min + dA_max (d > 0, else 0) goes to dPQ[i][H + ch])
template <bool S, bool SELF, int FE>
__device__ void bwd_phase1(const View<S, kChBwd> &v, const Slice &s, const float (&me)[2][FE], const float (&bm)[2],
                           const float *A, const uint8_t *arg, const float *dA, int H, float *dmbuf,
                           float (&acc)[2][FE], float (&bsum)[2], int KA, const float *Qp, int PW, float *dPQ) {
  constexpr int CPL = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lc = lane * CPL, ch = v.ch0 + lc;
  int i = s.n0 + warp;
  if (i >= s.n1) return;
  DstIn cur = load_dst<S, SELF>(v, i, A, arg, dA, H, ch, KA, Qp, PW);
  for (; i < s.n1; i += kWarps) {
    DstIn nxt;
    if (i + kWarps < s.n1) nxt = load_dst<S, SELF>(v, i + kWarps, A, arg, dA, H, ch, KA, Qp, PW);  // in flight meanwhile
    const int d = cur.k1 - cur.k0;
    if (SELF)
      *reinterpret_cast<float2 *>(dPQ + (size_t)i * PW + H + ch) =
          d > 0 ? make_float2(cur.gmean.x + cur.gmin.x + cur.gmax.x, cur.gmean.y + cur.gmin.y + cur.gmax.y)
                : make_float2(0.f, 0.f);
    if (d > 0) {
      const float inv_d = __frcp_rn((float)d);
      const float gm[CPL] = {cur.gmean.x * inv_d, cur.gmean.y * inv_d};
      const float gx[CPL] = {cur.gmax.x, cur.gmax.y}, gn[CPL] = {cur.gmin.x, cur.gmin.y};
      const float mu[CPL] = {cur.mu.x - cur.q.x, cur.mu.y - cur.q.y};  // (m below excludes Q_i)
      const int an[CPL] = {cur.amn.x, cur.amn.y}, ax[CPL] = {cur.amx.x, cur.amx.y};
      // (fast division: ~2 ulp, no IEEE reciprocal sequence)
      const float gs[CPL] = {(ax[0] & 0x80) ? __fdividef(cur.gstd.x * inv_d, cur.sg.x) : 0.f,
                             (ax[1] & 0x80) ? __fdividef(cur.gstd.y * inv_d, cur.sg.y) : 0.f};
      for (int k = cur.k0; k < cur.k1; ++k) {
        const int j = v.colv(k), p = k - cur.k0;
        float ef[FE], pj[CPL], m[CPL], dm[CPL];
        ld_edge<FE>(v.edge(k), v.Fe, ef);
        ld_vec<CPL>(v.prow(j, lc), pj);
        message<CPL, FE>(pj, bm, me, ef, m);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          float gg = gm[c];
          if ((ax[c] & 0x7f) == p) gg += gx[c];
          if (an[c] == p) gg += gn[c];
          if (ax[c] & 0x80) gg += gs[c] * (m[c] - mu[c]);
          dm[c] = gg;
          bsum[c] += gg;
#pragma unroll
          for (int f = 0; f < FE; ++f) acc[c][f] = fmaf(gg, ef[f], acc[c][f]);
        }
        st_vec<CPL>(dmbuf + (size_t)k * H + ch, dm);
      }
    }
    cur = nxt;
  }
}

template <bool S>
__device__ void bwd_phase2(const View<S, kChBwd> &v, const Slice &s, const float *dmbuf, float *dP, int H,
                           const int *dp_pos, int PW) {
  constexpr int CPL = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lc = lane * CPL, ch = v.ch0 + lc;
  for (int j = s.n0 + warp; j < s.n1; j += kWarps) {
    const int k0 = v.rowptr(j), k1 = v.rowptr(j + 1);
    float dp[CPL] = {0.f, 0.f};
    for (int k = k0; k < k1; ++k) {
      const int kd = v.rowptr(v.colv(k)) + v.slotv(k);  // edge j -> i in i's row
      float dm[CPL];
      ld_vec<CPL>(dmbuf + (size_t)kd * H + ch, dm);
#pragma unroll
      for (int c = 0; c < CPL; ++c) dp[c] += dm[c];
    }
    st_vec<CPL>(dP + (size_t)(dp_pos ? v.posv(j) : j) * PW + ch, dp);
  }
}

template <bool SELF, int FE>
__global__ void __launch_bounds__(32 * kWarps, 3) k_agg_bwd(const uint8_t *__restrict__ blob,
                                                            const int4 *__restrict__ gslice,
                                                            const float *__restrict__ P, const float *__restrict__ Me,
                                                            const float *__restrict__ bM, const float *__restrict__ A,
                                                            const uint8_t *__restrict__ arg,
                                                            const float *__restrict__ dA, float *__restrict__ dP,
                                                            float *__restrict__ partial, int H,
                                                            const int *__restrict__ pos, const int *__restrict__ dp_pos,
                                                            float *__restrict__ dmbuf, int maxB, int KA, int PW) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  pdl_enter();
  const BatchView b = load_batch(blob);
  constexpr int CPL = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nch = H / kChBwd;
  const int Fe = b.Fe;
  const SmemLayout L = smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, Fe, true);
  init_bar(&bar);
  const uint32_t parity = 0;
  // one item (graph slot, channel chunk) per CTA; slots past the batch write zero partials
  {
    const int item = blockIdx.x;
    __syncthreads();  // (the barrier's initialisation is visible)
    const int g = item / nch, ch0 = (item - g * nch) * kChBwd, ch = ch0 + lane * CPL;
    float me[CPL][FE], bm[CPL], acc[CPL][FE], bsum[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      bsum[c] = 0.f;
#pragma unroll
      for (int f = 0; f < FE; ++f) acc[c][f] = 0.f;
    }
    if (g < b.B) {
      const Slice s = slice_of(b, gslice, g);
      const bool staged = s.n1 - s.n0 <= kCapNodes && s.e1 - s.e0 <= kCapEdgesBwd;  // uniform per CTA
      if (staged) stage_graph<kChBwd>(b, P, PW, ch0, pos, true, L, sm, &bar, s, parity);
      const float *Qp = SELF ? P + H : nullptr;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        bm[c] = bM[ch + c];
#pragma unroll
        for (int f = 0; f < FE; ++f) me[c][f] = f < Fe ? Me[(ch + c) * Fe + f] : 0.f;
      }
      if (staged) {
        const View<true, kChBwd> v = make_view<true, kChBwd>(b, P, PW, ch0, pos, L, sm, s);
        bwd_phase1<true, SELF, FE>(v, s, me, bm, A, arg, dA, H, dmbuf, acc, bsum, KA, Qp, PW, dP);
        __syncthreads();  // (orders the block's dm writes before phase 2's reads)
        bwd_phase2<true>(v, s, dmbuf, dP, H, dp_pos, PW);
      } else {  // a graph too large to stage
        const View<false, kChBwd> v = make_view<false, kChBwd>(b, P, PW, ch0, pos, L, sm, s);
        bwd_phase1<false, SELF, FE>(v, s, me, bm, A, arg, dA, H, dmbuf, acc, bsum, KA, Qp, PW, dP);
        __syncthreads();
        bwd_phase2<false>(v, s, dmbuf, dP, H, dp_pos, PW);
      }
    }
    // this item's partials of dM_e and db_M, warps combined in fixed order; layout per graph
    // row: [H][Fe] (M_e's layout) then [H] (b_M). The staging area is free again: it holds
    // the per-warp sums red[warp][lane][c * (FE + 1) + f].
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
}


}  // namespace

template <class K>
static cudaError_t set_smem(K kern, uint32_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t agg_configure() {
  cudaError_t e;
  const uint32_t f4 = smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, 4, false).total;
  const uint32_t f8 = smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, 8, false).total;
  const uint32_t b4 = smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, 4, true).total;
  const uint32_t b8 = smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, 8, true).total;
  if ((e = set_smem(k_agg_fwd<false, 4>, f4)) || (e = set_smem(k_agg_fwd<false, 8>, f8)) ||
      (e = set_smem(k_agg_fwd<true, 4>, f4)) || (e = set_smem(k_agg_fwd<true, 8>, f8)) ||
      (e = set_smem(k_agg_bwd<false, 4>, b4)) || (e = set_smem(k_agg_bwd<false, 8>, b8)) ||
      (e = set_smem(k_agg_bwd<true, 4>, b4)) || (e = set_smem(k_agg_bwd<true, 8>, b8)))
    return e;
  return cudaSuccess;
}

void launch_agg_fwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const int4 *gslice, const float *P,
                    const float *Me, const float *bM, float var_floor, float *A, uint8_t *arg, const int *pos,
                    const float *xin, int Fl) {
  const int items = c.maxB * (c.H / kChFwd), Hl = c.Hl > 0 ? c.Hl : c.H;
  const SelfIn si{c.self_t ? P : nullptr, xin, c.PW(), Fl};
  const uint32_t smem = smem_layout(kChFwd, kCapNodes, kCapEdgesFwd, c.Fe, false).total;
  auto kern = c.Fe == 4 ? (c.self_t ? k_agg_fwd<true, 4> : k_agg_fwd<false, 4>)
                        : (c.self_t ? k_agg_fwd<true, 8> : k_agg_fwd<false, 8>);
  launch_ex(kern, items, 32 * kWarps, smem, st, blob, gslice, P, Me, bM, var_floor, A, arg, c.H, pos, Hl, c.KA(), si);
  g_launches += 1;
}

size_t agg_bwd_partial_floats(const Caps &c) { return (size_t)c.maxB * c.H * (c.Fe + 1); }
size_t agg_bwd_dm_floats(const Caps &c) { return (size_t)c.maxE * c.H; }

void launch_agg_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const int4 *gslice, const float *P,
                    const float *Me, const float *bM, const float *A, const uint8_t *arg, const float *dA, float *dP,
                    float *partial, const int *pos, const int *dp_pos, float *dm_scratch) {
  const int items = c.maxB * (c.H / kChBwd);
  const uint32_t smem = smem_layout(kChBwd, kCapNodes, kCapEdgesBwd, c.Fe, true).total;
  auto kern = c.Fe == 4 ? (c.self_t ? k_agg_bwd<true, 4> : k_agg_bwd<false, 4>)
                        : (c.self_t ? k_agg_bwd<true, 8> : k_agg_bwd<false, 8>);
  launch_ex(kern, items, 32 * kWarps, smem, st, blob, gslice, P, Me, bM, A, arg, dA, dP, partial, c.H, pos, dp_pos,
            dm_scratch, c.maxB, c.KA(), c.PW());
  g_launches += 1;
}

}  // namespace hg
