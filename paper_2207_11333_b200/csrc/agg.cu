// agg.cu — K2 (edge gather + multi-aggregator segmented reduction) and K8 (its backward +
// scatter to the sources), SURVEY §8(a4), §8(a10).
//
// Paper passages: message passing (§3.1) with the PNA aggregators
// (PAPER.md:148), fixed by SPEC.md:347 (message M [x_j || e_ij] + b_M; aggregators mean, min,
// max, std with variance floor eps_v) and the backward SPEC.md:369-371.
//
// Molecules are graph-local and a batch's graphs are contiguous node ranges, so one CTA owns
// one graph (and one 64-channel chunk): every row it touches -- the CSR slice, the P rows of
// the messages' sources, the per-destination gradients -- belongs to its graph. Warp 0 stages
// the graph's CSR slice and P rows in shared memory with bulk async copies (cp.async.bulk, one
// mbarrier) while the other threads issue their own global loads (weights, the first node's
// rows), so the rowptr -> col -> P dependency chain runs at shared-memory latency and HBM sees
// only large contiguous reads and coalesced row writes. One node per half-warp (16 lanes x 4
// channels): per-node control work is shared by two nodes, channel pairs use the packed
// fp32x2 pipe. A graph larger than the staging capacity runs the same arithmetic straight from
// global memory (L2), so any graph size is supported.
//
// Determinism: no atomics. Forward: one half-warp per destination node, fixed edge order.
// Backward (three phases): each edge's message gradient dm_{j->i} is computed once by its
// destination's half-warp and stored at the same pair's entry of the SOURCE's row (staged
// graphs: rows in shared memory, source-major, so phase 2 reads them contiguously; larger
// graphs: the global [E][H] buffer, destination-major); each source sums its row of dm in row
// order (dP_j); dM_e / db_M are per-CTA partials over the graph's edges, reduced in fixed order
// afterwards.
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

constexpr int kWarpsF = 4;             // forward: 128 threads per CTA (ncu: with 256, the CTA's
                                       // last node round left 30% of the warps idle at EXIT)
constexpr int kHalvesF = 2 * kWarpsF;  // half-warps per CTA: one node per half-warp
constexpr int kWarpsB = 8;             // backward: 256 threads (its smem holds the dm rows too)
constexpr int kHalvesB = 2 * kWarpsB;
constexpr int CPL = 4;                 // channels per lane (16 lanes x 4 = one 64-channel chunk)
constexpr int kCapNodes = 128;         // nodes of one graph staged in shared memory
constexpr int kCapEdgesFwd = 320;      // its directed edges (forward)
constexpr int kCapEdgesBwd = 256;      // (backward: the per-edge dm rows are staged too)
constexpr int kCh = 64;                // channels per CTA

__host__ __device__ constexpr uint32_t r16(uint32_t b) { return (b + 15u) & ~15u; }

// dynamic shared-memory layout (byte offsets) of one CTA
struct SmemLayout {
  uint32_t P, dm, rp, col, ea, pos, slot, total;
};
__host__ __device__ inline SmemLayout smem_layout(int cap_n, int cap_e, int Fe, bool bwd) {
  SmemLayout L;
  L.P = 0;
  L.dm = L.P + (uint32_t)cap_n * kCh * 4;  // (backward: the graph's dm rows, source-major)
  L.rp = L.dm + (bwd ? (uint32_t)cap_e * kCh * 4 : 0);
  L.col = L.rp + r16((cap_n + 8) * 4);
  L.ea = L.col + r16((cap_e + 8) * 4);
  L.pos = L.ea + r16(cap_e * Fe * 4 + 32);
  L.slot = L.pos + r16((cap_n + 8) * 4);
  L.total = L.slot + (bwd ? r16(cap_e + 32) : 0);
  // (the backward's partial reduction reuses the area: kHalvesB x 16 lanes x CPL x (Fe + 1))
  const uint32_t red = (uint32_t)kHalvesB * 16 * CPL * ((Fe <= 4 ? 4 : 8) + 1) * 4;  // (FE template width)
  if (L.total < red) L.total = red;
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

// Warp 0: stage rowptr[n0..n1], col/ea/slot[e0..e1), pos[n0..n1) and the graph's P rows
// (channels [ch0, ch0 + 64)) with bulk copies completing on one mbarrier (lane 0 posts the
// byte count, the lanes issue the row copies in parallel). Blob arrays start 16-byte aligned
// and the copies round up to 16 bytes (the overhang stays inside the blob). The caller issues
// its own global loads (weights, first node's rows) before stage_wait.
__device__ void stage_issue(const BatchView &b, const float *P, int PW, int ch0, const int *pos, bool with_slot,
                            const SmemLayout &L, uint8_t *sm, uint64_t *bar, const Slice &s) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const uint32_t brp = r16((uint32_t)(s.n1 + 1 - s.r0) * 4);
    const uint32_t bcol = s.e1 > s.e0 ? r16((uint32_t)(s.e1 - s.c0) * 4) : 0;
    const uint32_t ea_a = ((uint32_t)s.e0 * b.Fe * 4) & ~15u;
    const uint32_t bea = s.e1 > s.e0 ? r16((uint32_t)s.e1 * b.Fe * 4 - ea_a) : 0;
    const uint32_t bpos = r16((uint32_t)(s.n1 - s.p0) * 4);
    const uint32_t bsl = with_slot && s.e1 > s.e0 ? r16((uint32_t)(s.e1 - s.s0)) : 0;
    const int rows = s.n1 - s.n0;
    const uint32_t brow = kCh * 4, bP = (uint32_t)rows * brow;
    if (lane == 0) tc::mbar_expect_tx(bar, bP + brp + bcol + bea + bpos + bsl);
    __syncwarp();
    if (PW == kCh) {
      if (lane == 0 && bP) bulk_g2s(sm + L.P, P + (size_t)s.n0 * PW, bP, bar);
    } else {  // (P rows of PW floats: this chunk's 64 columns of each row, one copy per row)
      for (int r = lane; r < rows; r += 32) bulk_g2s(sm + L.P + r * brow, P + (size_t)(s.n0 + r) * PW + ch0, brow, bar);
    }
    if (lane == 1) bulk_g2s(sm + L.rp, b.rowptr + s.r0, brp, bar);
    if (lane == 2 && bcol) bulk_g2s(sm + L.col, b.col + s.c0, bcol, bar);
    if (lane == 3 && bea) bulk_g2s(sm + L.ea, reinterpret_cast<const uint8_t *>(b.ea) + ea_a, bea, bar);
    if (lane == 4) bulk_g2s(sm + L.pos, pos + s.p0, bpos, bar);
    if (lane == 5 && bsl) bulk_g2s(sm + L.slot, b.slot + s.s0, bsl, bar);
  }
}
// one thread polls the mbarrier; the others wait at the CTA barrier (no issue slots spent
// spinning: ncu showed the 256-thread poll at 10-14% of the kernels' instructions)
__device__ __forceinline__ void stage_wait(uint64_t *bar, uint32_t parity) {
  if (threadIdx.x == 0) tc::mbar_wait(bar, parity);
  __syncthreads();
}

__device__ __forceinline__ void init_bar(uint64_t *bar) {
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
  }
}

// MUFU approximations without the denormal fix-up (their arguments are normal: the variance
// floor eps_v > 0, degrees >= 1)
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 1/d for d = 0..127 (IEEE-rounded, as __frcp_rn), one table per CTA
__device__ __forceinline__ void fill_rcp(float *t) {
  if (threadIdx.x < 128) t[threadIdx.x] = threadIdx.x ? __frcp_rn((float)threadIdx.x) : 0.f;
}
// (degrees are <= HG_MAX_DEGREE = 127: hg_pack rejects larger ones, HG_E_DEGREE)
__device__ __forceinline__ float rcp_deg(const float *t, int d) { return t[min(d, 127)]; }

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ void st4(float *p, const float (&v)[CPL]) {
  *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
template <int FE>
__device__ __forceinline__ void ld_edge(const float *ea, int Fe, float (&ef)[FE]) {
  if constexpr (FE == 4) {
    const float4 t = ld4(ea);
    ef[0] = t.x; ef[1] = t.y; ef[2] = t.z; ef[3] = t.w;
  } else {
#pragma unroll
    for (int f = 0; f < FE; ++f) ef[f] = f < Fe ? ea[f] : 0.f;
  }
}
// message for the lane's 4 channels: m = (P + b_M) + sum_f M_e[:,f] e_f, f ascending (the same
// order in K2 and K8); channel pairs on the packed fp32x2 pipe (each lane of a pair rounds as
// the scalar fadd / fma)
template <int FE>
__device__ __forceinline__ void message(const float4 pj, const float2 (&bm)[2], const float2 (&me)[2][FE],
                                        const float (&ef)[FE], float (&m)[CPL]) {
  float2 v0 = __fadd2_rn(make_float2(pj.x, pj.y), bm[0]);
  float2 v1 = __fadd2_rn(make_float2(pj.z, pj.w), bm[1]);
#pragma unroll
  for (int f = 0; f < FE; ++f) {
    const float2 e2 = make_float2(ef[f], ef[f]);
    v0 = __ffma2_rn(me[0][f], e2, v0);
    v1 = __ffma2_rn(me[1][f], e2, v1);
  }
  m[0] = v0.x; m[1] = v0.y; m[2] = v1.x; m[3] = v1.y;
}
// the same with M_e read from the CTA's shared copy sme[f][64] (chunk channels; the backward,
// whose registers hold the per-edge gradient sums instead)
template <int FE>
__device__ __forceinline__ void message_sm(const float4 pj, const float2 (&bm)[2], const float *sme, int lc,
                                           const float (&ef)[FE], float (&m)[CPL]) {
  float2 v0 = __fadd2_rn(make_float2(pj.x, pj.y), bm[0]);
  float2 v1 = __fadd2_rn(make_float2(pj.z, pj.w), bm[1]);
#pragma unroll
  for (int f = 0; f < FE; ++f) {
    const float4 w = ld4(sme + f * kCh + lc);
    const float2 e2 = make_float2(ef[f], ef[f]);
    v0 = __ffma2_rn(make_float2(w.x, w.y), e2, v0);
    v1 = __ffma2_rn(make_float2(w.z, w.w), e2, v1);
  }
  m[0] = v0.x; m[1] = v0.y; m[2] = v1.x; m[3] = v1.y;
}

// Graph arrays read either from the staged copy (S) or straight from global memory.
template <bool S>
struct View {
  const int *rp, *col, *pos;
  const uint8_t *slot;
  const float *ea, *P;
  float *dm;
  int r0, c0, p0, s0, e0, n0, Fe, Pstride, ch0, H;
  __device__ int rowptr(int i) const { return S ? rp[i - r0] : rp[i]; }
  __device__ int colv(int k) const { return S ? col[k - c0] : col[k]; }
  __device__ int posv(int i) const { return S ? pos[i - p0] : pos[i]; }
  __device__ int slotv(int k) const { return S ? slot[k - s0] : slot[k]; }
  __device__ const float *edge(int k) const { return S ? ea + (size_t)(k - e0) * Fe : ea + (size_t)k * Fe; }
  __device__ const float *prow(int j, int lc) const {  // lc = lane's first channel within the chunk
    return S ? P + (j - n0) * kCh + lc : P + (size_t)j * Pstride + ch0 + lc;
  }
  // message-gradient row k: staged, the graph's rows in shared memory; else the global [E][H]
  // buffer (L2-resident)
  __device__ float *dmrow(int k, int lc) const {
    return S ? dm + (k - e0) * kCh + lc : dm + (size_t)k * H + ch0 + lc;
  }
  // where phase 1 stores the gradient of in-edge k (j -> i, k in i's row) and where phase 2
  // finds that of row-j entry k: staged graphs use source-major order (the row-j entry of the
  // same pair, so phase 2 reads its rows contiguously); otherwise destination-major
  // (the CSR is symmetric: in-edge k of row i, from j = col[k], is the entry slot[k] of row j)
  __device__ int dm_store(int k) const { return S ? rowptr(colv(k)) + slotv(k) : k; }
  __device__ int dm_load(int k) const { return S ? k : rowptr(colv(k)) + slotv(k); }
};
template <bool S>
__device__ View<S> make_view(const BatchView &b, const float *P, int PW, int ch0, const int *pos, const SmemLayout &L,
                             uint8_t *sm, const Slice &s, float *dmbuf, int H) {
  View<S> v;
  v.Fe = b.Fe;
  v.ch0 = ch0;
  v.Pstride = PW;
  v.n0 = s.n0;
  v.e0 = s.e0;
  v.H = H;
  if constexpr (S) {
    v.rp = reinterpret_cast<const int *>(sm + L.rp);
    v.col = reinterpret_cast<const int *>(sm + L.col);
    v.pos = reinterpret_cast<const int *>(sm + L.pos);
    v.slot = sm + L.slot;
    v.ea = reinterpret_cast<const float *>(sm + L.ea) + s.ea_skip;
    v.P = reinterpret_cast<const float *>(sm + L.P);
    v.dm = reinterpret_cast<float *>(sm + L.dm);
    v.r0 = s.r0; v.c0 = s.c0; v.p0 = s.p0; v.s0 = s.s0;
  } else {
    v.rp = b.rowptr; v.col = b.col; v.pos = pos; v.slot = b.slot; v.ea = b.ea; v.P = P; v.dm = dmbuf;
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

// M_e (this lane's 4 channels as packed pairs) and b_M
template <int FE>
__device__ __forceinline__ void load_edge_weights(const float *Me, const float *bM, int ch, int Fe, float2 (&me)[2][FE],
                                                  float2 (&bm)[2]) {
  bm[0] = make_float2(bM[ch], bM[ch + 1]);
  bm[1] = make_float2(bM[ch + 2], bM[ch + 3]);
#pragma unroll
  for (int f = 0; f < FE; ++f) {
    me[0][f] = f < Fe ? make_float2(Me[ch * Fe + f], Me[(ch + 1) * Fe + f]) : make_float2(0.f, 0.f);
    me[1][f] = f < Fe ? make_float2(Me[(ch + 2) * Fe + f], Me[(ch + 3) * Fe + f]) : make_float2(0.f, 0.f);
  }
}

// ---------------------------------------------------------------- K2 forward
// Per destination node i (one half-warp; 16 lanes x 4 channels), messages
// m = P[j] + b_M + M_e e_ji over the CSR row (j ascending) are recomputed, never stored in
// memory; pass 1: sum, min, max with first-position argmin / argmax; pass 2:
// the centred sum of squares (two-pass variance). When both nodes of a warp have
// degree <= 4 (molecules: all but hubs) the messages stay in registers between the passes;
// otherwise they are recomputed. d = 0 -> all aggregates 0 (C5). Writes A at the
// degree-sorted row pos[i] ([mean | min | max | std], 4H) and arg[i] ([argmin | argmax with
// bit 7 = var > eps_v], 2H bytes).
__device__ __forceinline__ void fold(const float (&m)[CPL], int p, float (&sum)[CPL], float (&mx)[CPL],
                                     float (&mn)[CPL], int (&amx)[CPL], int (&amn)[CPL]) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    sum[c] += m[c];
    if (m[c] > mx[c]) { mx[c] = m[c]; amx[c] = p; }
    if (m[c] < mn[c]) { mn[c] = m[c]; amn[c] = p; }
  }
}
__device__ __forceinline__ void centred(const float (&m)[CPL], const float (&sum)[CPL], float rd, float (&ss)[CPL]) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const float t = m[c] - sum[c] * rd;
    ss[c] = fmaf(t, t, ss[c]);
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
__device__ void fwd_nodes(const View<S> &v, const Slice &s, const float2 (&me)[2][FE], const float2 (&bm)[2],
                          float var_floor, float *A, uint8_t *arg, int H, int Hl, int KA, const SelfIn &si,
                          const float *rcp) {
  constexpr int RM = 4;  // messages held in registers
  const int hl = threadIdx.x & 15, hw = threadIdx.x >> 4, lc = hl * CPL, ch = v.ch0 + lc;
  const int n = s.n1 - s.n0;
  for (int t = 0; t < n; t += kHalvesF) {  // (trip count uniform over the CTA)
    const int i = s.n0 + t + hw;
    const bool valid = t + hw < n;
    int k0 = 0, d = 0, prow = 0;
    if (valid) {
      k0 = v.rowptr(i);
      d = v.rowptr(i + 1) - k0;
      prow = v.posv(i);
    }
    float q[CPL] = {0.f, 0.f, 0.f, 0.f}, xi[CPL] = {0.f, 0.f, 0.f, 0.f};
    if (SELF && valid) {  // (issued early: hidden behind the edge loop)
      const float4 t4 = ld4(si.P + (size_t)i * si.PW + H + ch);
      q[0] = t4.x; q[1] = t4.y; q[2] = t4.z; q[3] = t4.w;
#pragma unroll
      for (int c = 0; c < CPL; ++c) xi[c] = ch + c < si.Fl ? si.xin[(size_t)i * si.Fl + ch + c] : 0.f;
    }
    float sum[CPL], mx[CPL], mn[CPL], ss[CPL];
    int amx[CPL], amn[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      sum[c] = 0.f; mx[c] = -INFINITY; mn[c] = INFINITY; amx[c] = 0; amn[c] = 0; ss[c] = 0.f;
    }
    const float rd = rcp_deg(rcp, d);
    const int dw = __reduce_max_sync(0xffffffffu, d);  // the warp's largest degree (uniform)
    if (dw <= RM) {  // one load pass, messages kept for the variance pass
      float m[RM][CPL];
#pragma unroll
      for (int e = 0; e < RM; ++e) {
        if (e < dw && e < d) {
          const int j = v.colv(k0 + e);
          float ef[FE];
          ld_edge<FE>(v.edge(k0 + e), v.Fe, ef);
          message<FE>(ld4(v.prow(j, lc)), bm, me, ef, m[e]);
        }
      }
      // position 0 initialises (d = 0 rows are overwritten below)
#pragma unroll
      for (int c = 0; c < CPL; ++c) { sum[c] = m[0][c]; mx[c] = m[0][c]; mn[c] = m[0][c]; }
#pragma unroll
      for (int e = 1; e < RM; ++e)
        if (e < dw && e < d) fold(m[e], e, sum, mx, mn, amx, amn);
#pragma unroll
      for (int e = 0; e < RM; ++e)
        if (e < dw && e < d) centred(m[e], sum, rd, ss);
    } else {
      for (int k = k0; k < k0 + d; ++k) {
        const int j = v.colv(k);
        float ef[FE], m[CPL];
        ld_edge<FE>(v.edge(k), v.Fe, ef);
        message<FE>(ld4(v.prow(j, lc)), bm, me, ef, m);
        fold(m, k - k0, sum, mx, mn, amx, amn);
      }
      for (int k = k0; k < k0 + d; ++k) {  // pass 2: recompute the messages
        const int j = v.colv(k);
        float ef[FE], m[CPL];
        ld_edge<FE>(v.edge(k), v.Fe, ef);
        message<FE>(ld4(v.prow(j, lc)), bm, me, ef, m);
        centred(m, sum, rd, ss);
      }
    }
    if (!valid) continue;
    float mean[CPL], sd[CPL];
    uint32_t flags = 0;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      mean[c] = sum[c] * rd + q[c];  // (q = 0 without the self-term)
      mx[c] += q[c];
      mn[c] += q[c];
      const float var = ss[c] * rd;
      flags |= (var > var_floor ? 0x80u : 0u) << (8 * c);
      // channels >= Hl are padding (internal width H > logical Hl): their messages are
      // exactly 0, and their std is forced to 0 instead of sqrt(var_floor) so that no
      // gradient reaches the zero padded parameters (SURVEY §8(d) padding hazard).
      // (sqrt as v * rsqrt(v), ~2 ulp: the IEEE sqrtf sequence was 14% of the instructions)
      const float vf = fmaxf(var, var_floor);
      sd[c] = ch + c < Hl ? vf * rsqrt_ftz(vf) : 0.f;
    }
    // isolated nodes (d = 0, rare): every aggregate 0 (C5) -- a warp-uniform branch, so the
    // common warps skip the per-channel selects
    if (__any_sync(__activemask(), d == 0) && d == 0) {
      flags = 0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) { mean[c] = 0.f; mx[c] = 0.f; mn[c] = 0.f; sd[c] = 0.f; }
    }
    float *Ai = A + (size_t)prow * KA + ch;
    st4(Ai, mean);
    st4(Ai + H, mn);
    st4(Ai + 2 * H, mx);
    st4(Ai + 3 * H, sd);
    if (SELF) st4(Ai + 4 * H, xi);
    uint8_t *ai = arg + (size_t)i * (2 * H) + ch;
    *reinterpret_cast<uint32_t *>(ai) = (uint32_t)amn[0] | (uint32_t)amn[1] << 8 | (uint32_t)amn[2] << 16 |
                                        (uint32_t)amn[3] << 24;
    *reinterpret_cast<uint32_t *>(ai + H) =
        ((uint32_t)amx[0] | (uint32_t)amx[1] << 8 | (uint32_t)amx[2] << 16 | (uint32_t)amx[3] << 24) | flags;
  }
}

template <bool SELF, int FE>
__global__ void __launch_bounds__(32 * kWarpsF, 4) k_agg_fwd(const uint8_t *__restrict__ blob,
                                                            const int4 *__restrict__ gslice,
                                                            const float *__restrict__ P, const float *__restrict__ Me,
                                                            const float *__restrict__ bM, float var_floor,
                                                            float *__restrict__ A, uint8_t *__restrict__ arg, int H,
                                                            const int *__restrict__ pos, int Hl, int KA, SelfIn si) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ float rcp[128];
  pdl_enter();
  const BatchView b = load_batch(blob);
  const int nch = H / kCh, PW = si.PW;
  const SmemLayout L = smem_layout(kCapNodes, kCapEdgesFwd, b.Fe, false);
  if (SELF && !si.xin) si.xin = b.x;  // layer 0: the batch's node features
  init_bar(&bar);
  // one work item (graph, channel chunk) per CTA
  const int item = blockIdx.x;
  if (item >= b.B * nch) return;
  __syncthreads();  // (the barrier's initialisation is visible)
  const int g = item / nch, ch0 = (item - g * nch) * kCh, ch = ch0 + (threadIdx.x & 15) * CPL;
  const Slice s = slice_of(b, gslice, g);
  const bool staged = s.n1 - s.n0 <= kCapNodes && s.e1 - s.e0 <= kCapEdgesFwd;  // uniform per CTA
  if (staged) stage_issue(b, P, PW, ch0, pos, false, L, sm, &bar, s);
  float2 me[2][FE], bm[2];
  load_edge_weights<FE>(Me, bM, ch, b.Fe, me, bm);  // (in flight with the staging copies)
  fill_rcp(rcp);
  if (staged) stage_wait(&bar, 0);
  else __syncthreads();
  if (staged)
    fwd_nodes<true, SELF, FE>(make_view<true>(b, P, PW, ch0, pos, L, sm, s, nullptr, H), s, me, bm, var_floor, A, arg,
                              H, Hl, KA, si, rcp);
  else
    fwd_nodes<false, SELF, FE>(make_view<false>(b, P, PW, ch0, pos, L, sm, s, nullptr, H), s, me, bm, var_floor, A,
                               arg, H, Hl, KA, si, rcp);
}

// ---------------------------------------------------------------- K8 backward
// Phase 1, one half-warp per DESTINATION node i (16 lanes x 4 channels): its gradients dA_i,
// mu_i, sigma_i and decisions are read once (coalesced rows; the next node's are requested
// before this node is processed), and for each in-edge (j -> i) at row position p
// (SURVEY §8(a10)):
//   dm = dA_mean[i]/d_i + [p = argmax_i] dA_max[i] + [p = argmin_i] dA_min[i]
//        + [var_i > eps_v] dA_std[i] (m - mu_i)/(d_i sigma_i)
// with the message m recomputed from the staged P rows; dm goes to the per-edge buffer
// (destination-major like the CSR, [E][H], L2-resident) and into this CTA's dM_e = sum dm e^T
// and db_M = sum dm partials.
// Phase 2, one half-warp per SOURCE node j: dP_j = sum over its CSR row (edges j -> i,
// i = col[k]) of dm at i's row position slot[k] (where phase 1 stored it), in row order.
struct DstIn {  // one destination's per-channel inputs
  float4 gmean, gmin, gmax, gstd, mu, sg, q;
  uint32_t amn, amx;
  int k0, d;
};
// rp / ps: rowptr and pos, either the staged copies (offsets r0 / p0) or global memory (0)
template <bool SELF>
__device__ __forceinline__ DstIn load_dst(const int *rp, int r0, const int *ps, int p0, int i, bool valid,
                                          const float *A, const uint8_t *arg, const float *dA, int H, int ch, int KA,
                                          const float *Q, int PW) {
  DstIn t;
  if (!valid) {
    t.k0 = 0;
    t.d = 0;
    return t;
  }
  const float *dAi = dA + (size_t)i * KA + ch;
  t.gmean = ld4(dAi);
  t.gmin = ld4(dAi + H);
  t.gmax = ld4(dAi + 2 * H);
  t.gstd = ld4(dAi + 3 * H);
  t.amn = *reinterpret_cast<const uint32_t *>(arg + (size_t)i * (2 * H) + ch);
  t.amx = *reinterpret_cast<const uint32_t *>(arg + (size_t)i * (2 * H) + H + ch);
  t.q = SELF ? ld4(Q + (size_t)i * PW + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
  t.k0 = rp[i - r0];
  t.d = rp[i + 1 - r0] - t.k0;
  const float *Ai = A + (size_t)ps[i - p0] * KA + ch;
  t.mu = ld4(Ai);
  t.sg = ld4(Ai + 3 * H);
  return t;
}
__device__ __forceinline__ void f4(const float4 a, float (&v)[CPL]) { v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; }

// one destination's in-edges (self-term: Qp = the [P | Q] buffer's Q half (stride PW), the
// messages include Q_i, and the destination's dQ_i = dA_mean + dA_min + dA_max (d > 0, else 0)
// goes to dPQ[i][H + ch])
template <bool S, bool SELF, int FE>
__device__ __forceinline__ void bwd_dst(const View<S> &v, const DstIn &cur, int i, bool valid, int lc, int ch,
                                        const float *sme, const float2 (&bm)[2], int H, int PW, float *dPQ,
                                        const float *rcp) {
  const int d = cur.d;
  if (SELF && valid)
    *reinterpret_cast<float4 *>(dPQ + (size_t)i * PW + H + ch) =
        d > 0 ? make_float4(cur.gmean.x + cur.gmin.x + cur.gmax.x, cur.gmean.y + cur.gmin.y + cur.gmax.y,
                            cur.gmean.z + cur.gmin.z + cur.gmax.z, cur.gmean.w + cur.gmin.w + cur.gmax.w)
              : make_float4(0.f, 0.f, 0.f, 0.f);
  if (d <= 0) return;
  const float inv_d = rcp_deg(rcp, d);
  float gm[CPL], gx[CPL], gn[CPL], mu[CPL], q[CPL], gstd[CPL], sg[CPL], gs[CPL];
  int an[CPL], ax[CPL];
  f4(cur.gmean, gm); f4(cur.gmax, gx); f4(cur.gmin, gn); f4(cur.mu, mu); f4(cur.q, q); f4(cur.gstd, gstd);
  f4(cur.sg, sg);
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    gm[c] *= inv_d;
    mu[c] -= q[c];  // (m below excludes Q_i)
    an[c] = (cur.amn >> (8 * c)) & 0xff;
    ax[c] = (cur.amx >> (8 * c)) & 0xff;
    // (approximate reciprocal, ~1 ulp: sigma >= sqrt(eps_v) is normal)
    gs[c] = (ax[c] & 0x80) ? gstd[c] * inv_d * rcp_ftz(sg[c]) : 0.f;
    ax[c] &= 0x7f;
  }
  for (int p = 0; p < d; ++p) {
    const int k = cur.k0 + p, j = v.colv(k);
    float ef[FE], m[CPL], dm[CPL];
    ld_edge<FE>(v.edge(k), v.Fe, ef);
    message_sm<FE>(ld4(v.prow(j, lc)), bm, sme, lc, ef, m);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      float gg = gm[c];
      if (ax[c] == p) gg += gx[c];
      if (an[c] == p) gg += gn[c];
      dm[c] = fmaf(gs[c], m[c] - mu[c], gg);  // (gs = 0 when var <= eps_v)
    }
    st4(v.dmrow(v.dm_store(k), lc), dm);
  }
}

// nodes t + hw (t = 0, 16, 32, ...): two register sets alternate (no copies), the next node's
// rows in flight while this one is processed; `first` = the first node's rows, loaded by the
// caller before the staging wait
template <bool S, bool SELF, int FE>
__device__ void bwd_phase1(const View<S> &v, const Slice &s, const float *sme, const float2 (&bm)[2],
                           const float *A, const uint8_t *arg, const float *dA, int H, int KA, const float *Qp,
                           int PW, float *dPQ, const float *rcp,
                           const DstIn &first) {
  const int hl = threadIdx.x & 15, hw = threadIdx.x >> 4, lc = hl * CPL, ch = v.ch0 + lc;
  const int n = s.n1 - s.n0;
  DstIn a = first, b;
  for (int t = 0; t < n; t += 2 * kHalvesB) {
    const int i0 = s.n0 + t + hw, i1 = i0 + kHalvesB, i2 = i1 + kHalvesB;
    b = load_dst<SELF>(v.rp, v.r0, v.pos, v.p0, i1, t + kHalvesB + hw < n, A, arg, dA, H, ch, KA, Qp, PW);
    bwd_dst<S, SELF, FE>(v, a, i0, t + hw < n, lc, ch, sme, bm, H, PW, dPQ, rcp);
    if (t + kHalvesB >= n) break;
    a = load_dst<SELF>(v.rp, v.r0, v.pos, v.p0, i2, t + 2 * kHalvesB + hw < n, A, arg, dA, H, ch, KA, Qp, PW);
    bwd_dst<S, SELF, FE>(v, b, i1, t + kHalvesB + hw < n, lc, ch, sme, bm, H, PW, dPQ, rcp);
  }
}

template <bool S>
__device__ void bwd_phase2(const View<S> &v, const Slice &s, float *dP, int H, const int *dp_pos, int PW) {
  const int hl = threadIdx.x & 15, hw = threadIdx.x >> 4, lc = hl * CPL, ch = v.ch0 + lc;
  for (int j = s.n0 + hw; j < s.n1; j += kHalvesB) {
    const int k0 = v.rowptr(j), k1 = v.rowptr(j + 1);
    float dp[CPL] = {0.f, 0.f, 0.f, 0.f};
    for (int k = k0; k < k1; k += 4) {  // (four edges' loads in flight; sums in row order)
      float4 r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u < k1) r[u] = ld4(v.dmrow(v.dm_load(k + u), lc));
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u < k1) { dp[0] += r[u].x; dp[1] += r[u].y; dp[2] += r[u].z; dp[3] += r[u].w; }
    }
    st4(dP + (size_t)(dp_pos ? v.posv(j) : j) * PW + ch, dp);
  }
}

// Phase 3: this CTA's dM_e = sum_k dm_k e_k^T and db_M = sum_k dm_k partials over the graph's
// edges (half-warp t takes edges e0 + t, e0 + t + 16, ...), from the dm rows phase 1 stored
template <bool S, int FE>
__device__ void bwd_edge_partials(const View<S> &v, const Slice &s, float2 (&acc)[2][FE], float2 (&bsum)[2]) {
  const int hl = threadIdx.x & 15, hw = threadIdx.x >> 4, lc = hl * CPL;
  for (int k = s.e0 + hw; k < s.e1; k += kHalvesB) {
    float ef[FE];
    ld_edge<FE>(v.edge(k), v.Fe, ef);
    const float4 dm = ld4(v.dmrow(v.dm_store(k), lc));
    const float2 d01 = make_float2(dm.x, dm.y), d23 = make_float2(dm.z, dm.w);
    bsum[0] = __fadd2_rn(bsum[0], d01);
    bsum[1] = __fadd2_rn(bsum[1], d23);
#pragma unroll
    for (int f = 0; f < FE; ++f) {
      const float2 e2 = make_float2(ef[f], ef[f]);
      acc[0][f] = __ffma2_rn(d01, e2, acc[0][f]);
      acc[1][f] = __ffma2_rn(d23, e2, acc[1][f]);
    }
  }
}

template <bool SELF, int FE>
__global__ void __launch_bounds__(32 * kWarpsB, 2) k_agg_bwd(const uint8_t *__restrict__ blob,
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
  __shared__ float rcp[128];
  __shared__ __align__(16) float sme[8 * kCh];  // M_e of the chunk, [f][channel]
  pdl_enter();
  const BatchView b = load_batch(blob);
  const int hl = threadIdx.x & 15, hw = threadIdx.x >> 4, nch = H / kCh;
  const int Fe = b.Fe;
  const SmemLayout L = smem_layout(kCapNodes, kCapEdgesBwd, Fe, true);
  init_bar(&bar);
  // one item (graph slot, channel chunk) per CTA; slots past the batch write zero partials
  const int item = blockIdx.x;
  __syncthreads();  // (the barrier's initialisation is visible)
  const int g = item / nch, ch0 = (item - g * nch) * kCh, ch = ch0 + hl * CPL;
  float2 acc[2][FE], bsum[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    bsum[c] = make_float2(0.f, 0.f);
#pragma unroll
    for (int f = 0; f < FE; ++f) acc[c][f] = make_float2(0.f, 0.f);
  }
  if (g < b.B) {
    const Slice s = slice_of(b, gslice, g);
    const bool staged = s.n1 - s.n0 <= kCapNodes && s.e1 - s.e0 <= kCapEdgesBwd;  // uniform per CTA
    if (staged) stage_issue(b, P, PW, ch0, pos, true, L, sm, &bar, s);
    const float *Qp = SELF ? P + H : nullptr;
    // in flight with the staging copies: the weights and the first node's rows (global)
    const float2 bm[2] = {make_float2(bM[ch], bM[ch + 1]), make_float2(bM[ch + 2], bM[ch + 3])};
    for (int t = threadIdx.x; t < FE * kCh; t += blockDim.x) {
      const int f = t / kCh, cc = t - f * kCh;
      sme[t] = f < Fe ? Me[(ch0 + cc) * Fe + f] : 0.f;
    }
    const DstIn first = load_dst<SELF>(b.rowptr, 0, pos, 0, s.n0 + hw, hw < s.n1 - s.n0, A, arg, dA, H, ch, KA, Qp, PW);
    fill_rcp(rcp);
    if (staged) {
      stage_wait(&bar, 0);
      const View<true> v = make_view<true>(b, P, PW, ch0, pos, L, sm, s, dmbuf, H);
      bwd_phase1<true, SELF, FE>(v, s, sme, bm, A, arg, dA, H, KA, Qp, PW, dP, rcp, first);
      __syncthreads();  // (orders the block's dm writes before phase 2's reads)
      bwd_phase2<true>(v, s, dP, H, dp_pos, PW);
      bwd_edge_partials<true, FE>(v, s, acc, bsum);
    } else {  // a graph too large to stage
      __syncthreads();
      const View<false> v = make_view<false>(b, P, PW, ch0, pos, L, sm, s, dmbuf, H);
      bwd_phase1<false, SELF, FE>(v, s, sme, bm, A, arg, dA, H, KA, Qp, PW, dP, rcp, first);
      __syncthreads();
      bwd_phase2<false>(v, s, dP, H, dp_pos, PW);
      bwd_edge_partials<false, FE>(v, s, acc, bsum);
    }
  }
  // this item's partials of dM_e and db_M, half-warps combined in fixed order; layout per
  // graph row: [H][Fe] (M_e's layout) then [H] (b_M). The staging area is free again: it
  // holds the per-half-warp sums red[hw][hl][c * (FE + 1) + f].
  constexpr int RS = CPL * (FE + 1);
  float *red = reinterpret_cast<float *>(sm);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const float2 bs = bsum[c >> 1];
    red[(hw * 16 + hl) * RS + c * (FE + 1) + FE] = (c & 1) ? bs.y : bs.x;
#pragma unroll
    for (int f = 0; f < FE; ++f) {
      const float2 a = acc[c >> 1][f];
      red[(hw * 16 + hl) * RS + c * (FE + 1) + f] = (c & 1) ? a.y : a.x;
    }
  }
  __syncthreads();
  float *pb = partial + (size_t)g * H * (Fe + 1);
  for (int t = threadIdx.x; t < kCh * (Fe + 1); t += blockDim.x) {
    const bool isb = t >= kCh * Fe;
    const int cc = isb ? t - kCh * Fe : t / Fe, f = isb ? FE : t - (t / Fe) * Fe;  // channel in chunk, feature
    const int l = cc / CPL, c = cc - l * CPL;
    float sum = 0.f;
    for (int w = 0; w < kHalvesB; ++w) sum += red[(w * 16 + l) * RS + c * (FE + 1) + f];
    if (isb) pb[(size_t)H * Fe + ch0 + cc] = sum;
    else pb[(size_t)(ch0 + cc) * Fe + f] = sum;
  }
}

}  // namespace

template <class K>
static cudaError_t set_smem(K kern, uint32_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t agg_configure() {
  cudaError_t e;
  const uint32_t f4 = smem_layout(kCapNodes, kCapEdgesFwd, 4, false).total;
  const uint32_t f8 = smem_layout(kCapNodes, kCapEdgesFwd, 8, false).total;
  const uint32_t b4 = smem_layout(kCapNodes, kCapEdgesBwd, 4, true).total;
  const uint32_t b8 = smem_layout(kCapNodes, kCapEdgesBwd, 8, true).total;
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
  const int items = c.maxB * (c.H / kCh), Hl = c.Hl > 0 ? c.Hl : c.H;
  const SelfIn si{c.self_t ? P : nullptr, xin, c.PW(), Fl};
  const uint32_t smem = smem_layout(kCapNodes, kCapEdgesFwd, c.Fe, false).total;
  auto kern = c.Fe == 4 ? (c.self_t ? k_agg_fwd<true, 4> : k_agg_fwd<false, 4>)
                        : (c.self_t ? k_agg_fwd<true, 8> : k_agg_fwd<false, 8>);
  launch_ex(kern, items, 32 * kWarpsF, smem, st, blob, gslice, P, Me, bM, var_floor, A, arg, c.H, pos, Hl, c.KA(),
            si);
  g_launches += 1;
}

size_t agg_bwd_partial_floats(const Caps &c) { return (size_t)c.maxB * c.H * (c.Fe + 1); }
size_t agg_bwd_dm_floats(const Caps &c) { return (size_t)c.maxE * c.H; }

void launch_agg_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const int4 *gslice, const float *P,
                    const float *Me, const float *bM, const float *A, const uint8_t *arg, const float *dA, float *dP,
                    float *partial, const int *pos, const int *dp_pos, float *dm_scratch) {
  const int items = c.maxB * (c.H / kCh);
  const uint32_t smem = smem_layout(kCapNodes, kCapEdgesBwd, c.Fe, true).total;
  auto kern = c.Fe == 4 ? (c.self_t ? k_agg_bwd<true, 4> : k_agg_bwd<false, 4>)
                        : (c.self_t ? k_agg_bwd<true, 8> : k_agg_bwd<false, 8>);
  launch_ex(kern, items, 32 * kWarpsB, smem, st, blob, gslice, P, Me, bM, A, arg, dA, dP, partial, c.H, pos, dp_pos,
            dm_scratch, c.maxB, c.KA(), c.PW());
  g_launches += 1;
}

}  // namespace hg
