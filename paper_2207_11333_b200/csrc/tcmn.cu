// tcmn.cu — TMA-fed 3xTF32 tcgen05 GEMMs with BOTH operands MN-major: the
// weight-gradient Grams that contract over nodes,
//   G_c = dZ_c^T A_c  (per degree class split, SURVEY §8(a9) / reassociation G3)
//   dM_x = dP^T X     (per node split)
// Operands are node-row tensors read as-is: a TMA box {32 features, 32 nodes}
// lands as one MN-major SWIZZLE_128B_BASE32B block (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B),
// so there is no transpose or transform stage. Column sums (db_U, db_M) come from
// an extra N=32 tile whose B operand is a ones matrix: D = sum_k a[k][m] * 1.
// K (node) ranges end inside a 32-row chunk: the MMA skips whole 8-row k-steps
// past the end and the transform warps zero the A operand's trailing rows of the last one.
//   warps 0-3 epilogue (TMEM -> staging -> coalesced partial stores)
//   warp 4    TMA producer (the operands' fp32 tiles)   warp 5  TMEM alloc, MMA issue
//   warps 6-9 per landed stage: zero the A tile's rows past the split, then (3xTF32) the lo
//             terms x - trunc19(x) of the A and B tiles into the stage's lo slots -- the
//             activations are stored once, as fp32, in HBM
// Persistent over (split, m-tile, n-tile) items; double-buffered accumulators.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"
#include "tma.h"

namespace hg {

extern std::atomic<int64_t> g_launches;
int g_mn_grid_override = 0;  // > 0: grid cap for the next MN launches (set by the step builder)

namespace {

constexpr int N_BM = 128;          // output rows (features of the A operand) per tile
constexpr int N_BK = 32;           // nodes per chunk
constexpr int N_BOX = N_BK * 128;  // one MN block: 32 k-rows x 128 bytes
constexpr int N_TMA_WARP = 4, N_MMA_WARP = 5, N_XF_WARP = 6, N_THREADS = 320;
constexpr int N_STG_LD = 36;
constexpr int N_STG_BYTES = 4 * 32 * N_STG_LD * 4;

template <class Op>
constexpr int n_stage_bytes() { return 2 * 4 * N_BOX + 2 * (Op::BN / 32) * N_BOX; }
template <class Op>
constexpr int n_stages() {
  return (224 * 1024 - N_STG_BYTES) / n_stage_bytes<Op>() < 6 ? (224 * 1024 - N_STG_BYTES) / n_stage_bytes<Op>() : 6;
}
template <class Op>
constexpr int n_smem_bytes() {
  return n_stages<Op>() * n_stage_bytes<Op>() + N_STG_BYTES + 1024 + 8 * (4 * n_stages<Op>() + 4) + 16;
}

struct MnItem {
  int m0, n0, k0, len, sp, cs;  // cs: column-sum tile (B = ones, MMA N = 32)
};

}  // namespace

// maps: ah/al = A operand (rows = nodes, cols = M features), bh/bl = B operand
// (cols = N features); ones map rides in a second parameter.
extern int g_gemm_passes;  // tcdirect.cu: 3 = 3xTF32, 1 = plain TF32

template <class Op>
__global__ void __launch_bounds__(N_THREADS, 1) k_tmn(const __grid_constant__ TmaMaps mp,
                                                      const __grid_constant__ CUtensorMap ones, Op op_in,
                                                      int passes) {
  constexpr int BN = Op::BN, ST = n_stages<Op>(), NB = BN / 32;
  constexpr int A_BYTES = 4 * N_BOX, B_BYTES = NB * N_BOX, STAGE = n_stage_bytes<Op>();
  // two buffers of the main accumulator at [0, 2BN), two of the correction accumulator
  // (hi*lo + lo*hi) at [2BN, 4BN) -- see tcdirect.cu k_tma (DESIGN.md F-accumulate)
  constexpr int TCOLS = 4 * BN <= 256 ? 256 : 512;
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256 && ST >= 2, "tile");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  float *stg_all = reinterpret_cast<float *>(smem + ST * STAGE);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + ST * STAGE + N_STG_BYTES);
  uint64_t *empty = full + ST;
  uint64_t *xfull = empty + ST;  // [ST] transform -> MMA
  uint64_t *accf = xfull + ST;
  uint64_t *acce = accf + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(acce + 2);
  const bool p3 = passes == 3;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == N_MMA_WARP) tc::tmem_alloc<TCOLS>(tmem_holder);
  if (threadIdx.x == N_TMA_WARP * 32) {
    tc::tma_prefetch_desc(&mp.ah);
    tc::tma_prefetch_desc(&mp.bh);
    tc::tma_prefetch_desc(&ones);
    for (int s = 0; s < ST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&xfull[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&accf[b], 1);
      tc::mbar_init(&acce[b], 4);
    }
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_holder;
  pdl_enter();

  Op op = op_in;
  const int items = op.items_cap;
  if (warp == N_TMA_WARP) {
    // ---------------- TMA producer
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < items; t += gridDim.x) {
        MnItem w;
        if (!op.item(t, w)) continue;
        const int nch = (w.len + N_BK - 1) / N_BK;
        for (int c = 0; c < nch; ++c, ++it) {
          const int s = it % ST;
          if (it >= ST) tc::mbar_wait(&empty[s], ((it / ST) - 1) & 1);
          uint8_t *sa = smem + s * STAGE;
          const int k = w.k0 + c * N_BK;
          tc::mbar_expect_tx(&full[s], A_BYTES + (w.cs ? N_BOX : B_BYTES));
#pragma unroll
          for (int b = 0; b < 4; ++b) tc::tma_load_2d(sa + b * N_BOX, &mp.ah, w.m0 + 32 * b, k, &full[s]);
          uint8_t *sb = sa + 2 * A_BYTES;
          if (w.cs) {
            tc::tma_load_2d(sb, &ones, 0, k, &full[s]);
          } else {
#pragma unroll
            for (int b = 0; b < NB; ++b) tc::tma_load_2d(sb + b * N_BOX, &mp.bh, w.n0 + 32 * b, k, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= N_XF_WARP) {
    // ---------------- per landed stage: A rows past the split -> 0 (a partial last chunk:
    // rows past ceil8(rem) are skipped as whole k-steps, rows in [rem, ceil8(rem)) must be
    // zero), then the lo terms; generic writes made visible to the tensor core
    const int t = threadIdx.x - N_XF_WARP * 32;
    int it = 0;
    for (int tt = blockIdx.x; tt < items; tt += gridDim.x) {
      MnItem w;
      if (!op.item(tt, w)) continue;
      const int nch = (w.len + N_BK - 1) / N_BK;
      for (int c = 0; c < nch; ++c, ++it) {
        const int s = it % ST;
        const int rem = w.len - c * N_BK;
        tc::mbar_wait(&full[s], (it / ST) & 1);
        uint8_t *sa = smem + s * STAGE;
        if (rem < N_BK) {  // 16-byte chunk i of box i / 256 lies in k-row (i % 256) / 8 (each thread
                           // zeroes exactly the chunks it then splits: no barrier needed)
          for (int i = t; i < 4 * N_BOX / 16; i += 128)
            if (((i & 255) >> 3) >= rem) *reinterpret_cast<float4 *>(sa + 16 * i) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (p3) {
          tc::lo_chunks(sa, sa + A_BYTES, A_BYTES / 16, t, 128);
          if (!w.cs) tc::lo_chunks(sa + 2 * A_BYTES, sa + 2 * A_BYTES + B_BYTES, B_BYTES / 16, t, 128);
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&xfull[s]);
      }
    }
  } else if (warp == N_MMA_WARP) {
    // ---------------- MMA issuer (lane 0)
    constexpr uint32_t idesc = tc::idesc_tf32(N_BM, BN, true, true);
    constexpr uint32_t idesc_cs = tc::idesc_tf32(N_BM, 32, true, true);
    int it = 0, tcount = 0;
    for (int t = blockIdx.x; t < items; t += gridDim.x) {
      MnItem w;
      if (!op.item(t, w)) continue;
      const int buf = tcount & 1;
      if (tcount >= 2) tc::mbar_wait(&acce[buf], ((tcount >> 1) - 1) & 1);
      tc::fence_after_sync();
      const uint32_t d = tmem + (uint32_t)(buf * BN), dc = d + (uint32_t)(2 * BN);
      const int nch = (w.len + N_BK - 1) / N_BK;
      for (int c = 0; c < nch; ++c, ++it) {
        const int s = it % ST;
        const int rem = w.len - c * N_BK;
        const int nks = rem >= N_BK ? N_BK / 8 : (rem + 7) / 8;
        tc::mbar_wait(&full[s], (it / ST) & 1);
        tc::mbar_wait(&xfull[s], (it / ST) & 1);
        uint8_t *sa = smem + s * STAGE;
        __syncwarp();
        tc::fence_after_sync();
        if (lane == 0) {
          const uint32_t aH = tc::smem_u32(sa), aL = aH + A_BYTES;
          const uint32_t bH = aL + A_BYTES, bL = bH + B_BYTES;
          for (int ks = 0; ks < nks; ++ks) {
            const uint32_t off = ks * 1024;  // 8 k-rows = two 4-row groups
            const uint64_t dah = tc::desc_mn32(aH + off, N_BOX, 512), dal = tc::desc_mn32(aL + off, N_BOX, 512);
            const uint64_t dbh = tc::desc_mn32(bH + off, N_BOX, 512);
            const uint32_t acc = (c | ks) != 0;
            if (w.cs) {
              tc::mma_tf32(d, dah, dbh, idesc_cs, acc);
              if (p3) tc::mma_tf32(d, dal, dbh, idesc_cs, 1u);
            } else {
              tc::mma_tf32(d, dah, dbh, idesc, acc);
              if (p3) {
                tc::mma_tf32(dc, dah, tc::desc_mn32(bL + off, N_BOX, 512), idesc, acc);
                tc::mma_tf32(dc, dal, dbh, idesc, 1u);
              }
            }
          }
          tc::mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) tc::mma_commit(&accf[buf]);
      __syncwarp();
      ++tcount;
    }
  } else {
    // ---------------- epilogue
    float *stg = stg_all + warp * 32 * N_STG_LD;
    int tcount = 0;
    for (int t = blockIdx.x; t < items; t += gridDim.x) {
      MnItem w;
      if (!op.item(t, w)) continue;
      const int buf = tcount & 1;
      tc::mbar_wait(&accf[buf], (tcount >> 1) & 1);
      tc::fence_after_sync();
      const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(buf * BN);
      const bool empty_item = w.len <= 0;  // no MMA ran: the partial is zero
      if (w.cs) {  // column sums: every column of the N=32 tile holds the same value
        float acc[32];
        tc::tmem_ld32(trow, acc);
        op.emit_cs(w, w.m0 + warp * 32 + lane, empty_item ? 0.f : acc[0]);
      } else {
#pragma unroll 1
        for (int q = 0; q < BN / 32; ++q) {
          float acc[32], cor[32];
          tc::tmem_ld32(trow + (uint32_t)(q * 32), acc);
          if (p3) {
            tc::tmem_ld32(trow + (uint32_t)(2 * BN + q * 32), cor);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) cor[i] = 0.f;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = empty_item ? 0.f : acc[i] + cor[i];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4 *>(stg + lane * N_STG_LD + 4 * j) =
                make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int r = 4 * j + (lane >> 3), cc = 4 * (lane & 7);
            op.emit(w, w.m0 + warp * 32 + r, w.n0 + q * 32 + cc,
                    *reinterpret_cast<const float4 *>(stg + r * N_STG_LD + cc));
          }
          __syncwarp();
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acce[buf]);
      ++tcount;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == N_MMA_WARP) {
    tc::fence_after_sync();
    tc::tmem_dealloc<TCOLS>(tmem);
  }
}

// ---------------------------------------------------------------- ops
// per-class-split Gram: part[sp][h][n] = sum_{k in split} dZ[k][h] A[k][n] (rows
// degree-sorted, so a split is a contiguous row range), cs[sp][h] = sum_k dZ[k][h]
struct MnGram {
  static constexpr int BN = 128;
  const DegInfo *info; const int4 *splits; float *part, *cs; int H, K; int items_cap;
  __device__ bool item(int t, MnItem &w) const {
    const int NT = K / BN + 1, MT = H / N_BM;
    const int nt = t % NT, mt = (t / NT) % MT, sp = t / (NT * MT);
    if (sp >= info->S) return false;
    const int4 s = splits[sp];
    w = MnItem{mt * N_BM, nt * BN, s.y, s.z, sp, nt == NT - 1};
    return true;
  }
  __device__ void emit(const MnItem &w, int m, int n, float4 v) const {
    *reinterpret_cast<float4 *>(part + ((size_t)w.sp * H + m) * K + n) = v;
  }
  __device__ void emit_cs(const MnItem &w, int m, float v) const { cs[(size_t)w.sp * H + m] = v; }
};

// dM_x partials over node splits: part[sp][h][f] = sum_{k in split} dP[k][h] X[k][f]; cs = sum_k dP[k][h]
// node splits of the dM_x Grams: scaled with the capacity (about 256 nodes per split, 16..148),
// so a large batch fills every SM instead of a fixed 32 CTAs
constexpr int kMaxDMxSplits = 148;
// (512 / 1024 nodes per split measured 1% / 4% slower at config D, round 2)
int dmx_splits(const Caps &c) { return std::max(16, std::min(kMaxDMxSplits, (c.maxN + 255) / 256)); }
struct MnDMx {
  static constexpr int BN = 128;
  const uint8_t *blob; float *part, *cs; int H, F; int items_cap;
  int with_cs;  // 1: a trailing ones tile per (m, split) gives cs = sum_k dP[k][h] (db_M)
  int nsplit;   // node splits (dmx_splits)
  __device__ bool item(int t, MnItem &w) const {
    const int NT = (F + BN - 1) / BN + with_cs, MT = H / N_BM;
    const int nt = t % NT, mt = (t / NT) % MT, sp = t / (NT * MT);
    const int N = batch_N(blob);
    int kc = (N + nsplit - 1) / nsplit;
    kc = (kc + N_BK - 1) / N_BK * N_BK;
    const int k0 = sp * kc, len = max(0, min(N - k0, kc));
    w = MnItem{mt * N_BM, nt * BN, k0, len, sp, with_cs && nt == NT - 1};
    // every split is an item, also an empty one (len 0: its partial is written as zeros),
    // because the fixed-order reduction sums all nsplit partials
    return sp < nsplit;
  }
  __device__ void emit(const MnItem &w, int m, int n, float4 v) const {
    float *o = part + ((size_t)w.sp * H + m) * F + n;
    if ((F & 3) == 0) {
      if (n < F) *reinterpret_cast<float4 *>(o) = v;
    } else {  // narrow layer input (F % 4 != 0): scalar stores, columns >= F dropped
      if (n < F) o[0] = v.x;
      if (n + 1 < F) o[1] = v.y;
      if (n + 2 < F) o[2] = v.z;
      if (n + 3 < F) o[3] = v.w;
    }
  }
  __device__ void emit_cs(const MnItem &w, int m, float v) const { cs[(size_t)w.sp * H + m] = v; }
};

// layer-0 input as a TMA-readable operand: Xp[i][0..Fp) = x_i padded with zeros to a
// 16-byte row pitch
__global__ void __launch_bounds__(256) k_pad_x0(const uint8_t *__restrict__ blob, int Fp, float *__restrict__ Xp,
                                                const int *__restrict__ pos) {
  pdl_enter();
  const BatchView b = load_batch(blob);
  const int F = b.F0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < b.N * Fp; e += gridDim.x * blockDim.x) {
    const int i = e / Fp, f = e - i * Fp;
    const float v = f < F ? b.x[(size_t)i * F + f] : 0.f;
    const size_t o = pos ? (size_t)pos[i] * Fp + f : (size_t)e;  // degree-sorted rows when pos is given
    Xp[o] = v;
  }
}

// ---------------------------------------------------------------- reductions
// Block = RW warps x 32 float4 outputs: lane l of warp w sums parts w, w+RW, ...
// of output float4 (32*block + l) -- coalesced rows -- then warp 0 adds the RW
// warp sums in order (deterministic for a given partial count).
constexpr int RW = 8;
struct RJob {
  const float *part;  // [nparts][stride], the first count of each row summed
  int nparts, count;  // count % 4 == 0
  float *out;
  int stride;         // floats between parts (0 = count)
};
__device__ __forceinline__ void add4(float4 &s, float4 v) {
  s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
}
// up to three independent sums in one launch (dM_x, db_M, dM_e of a layer)
__global__ void __launch_bounds__(32 * RW) k_reduce_jobs(RJob j0, RJob j1, RJob j2) {
  pdl_enter();
  __shared__ float4 red[RW][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = (j0.count / 4 + 31) / 32, b1 = (j1.count / 4 + 31) / 32;
  int blk = blockIdx.x;
  const RJob &j = blk < b0 ? j0 : (blk < b0 + b1 ? j1 : j2);
  blk = blk < b0 ? blk : (blk < b0 + b1 ? blk - b0 : blk - b0 - b1);
  const int e = 4 * (blk * 32 + lane);
  const bool ok = e < j.count;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
    const size_t stride = j.stride > 0 ? j.stride : j.count;
#pragma unroll 4
    for (int p = warp; p < j.nparts; p += RW) add4(s, ldg4(j.part + (size_t)p * stride + e));
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && ok) {
    float4 t = red[0][lane];
#pragma unroll
    for (int w = 1; w < RW; ++w) add4(t, red[w][lane]);
    *reinterpret_cast<float4 *>(j.out + e) = t;
  }
}
static int reduce_blocks(const RJob &j) { return (j.count / 4 + 31) / 32; }

// dU[h][s*4H + n] = sum_sp s(class(sp)) part[sp][h][n] for the S scalers over the 4H aggregate
// columns (blocks over the H x K partial, K = 4H or 5H); the self-term's x block (columns
// [4H, 5H), not scaled): dUx[h][n - 4H] = sum_sp part[sp][h][n] for n - 4H < Fl; db_U[h] =
// sum_sp cs[sp][h] (trailing blocks); info->S splits (device-side). Split order fixed.
__global__ void __launch_bounds__(256) k_reduce_gram(const float *__restrict__ part, const float *__restrict__ cs,
                                                     const DegInfo *__restrict__ info, const int4 *__restrict__ splits,
                                                     int H, int K, int NS, int Fl, float *__restrict__ dU,
                                                     float *__restrict__ dbU, float *__restrict__ dUx) {
  pdl_enter();
  __shared__ float4 red[kMaxScalers][8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = info->S, K4 = 4 * H, bU = H * K / 128;
  const bool gram = (int)blockIdx.x < bU;
  const int e = 4 * (((int)blockIdx.x - (gram ? 0 : bU)) * 32 + lane);
  const bool ok = gram || e < H;
  const int h = gram ? e / K : 0, n = gram ? e - h * K : 0;
  const int ns = gram && n < K4 ? NS : 1;  // sums this thread keeps (uniform per 32-column block)
  float4 acc[kMaxScalers];
#pragma unroll
  for (int q = 0; q < kMaxScalers; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
    for (int sp = warp; sp < S; sp += 8) {
      if (gram) {
        const int c = splits[sp].x;
        const float4 v = ldg4(part + (size_t)sp * H * K + e);
        add4(acc[0], v);
#pragma unroll
        for (int q = 1; q < kMaxScalers; ++q)
          if (q < ns) {
            const float a = info->scal[q][c];
            acc[q].x = fmaf(a, v.x, acc[q].x); acc[q].y = fmaf(a, v.y, acc[q].y);
            acc[q].z = fmaf(a, v.z, acc[q].z); acc[q].w = fmaf(a, v.w, acc[q].w);
          }
      } else {
        add4(acc[0], ldg4(cs + (size_t)sp * H + e));
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kMaxScalers; ++q) red[q][warp][lane] = acc[q];
  __syncthreads();
  if (warp == 0 && ok) {
    float4 t[kMaxScalers];
#pragma unroll
    for (int q = 0; q < kMaxScalers; ++q) {
      t[q] = red[q][0][lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) add4(t[q], red[q][w][lane]);
    }
    if (!gram) {
      *reinterpret_cast<float4 *>(dbU + e) = t[0];
    } else if (n < K4) {
#pragma unroll
      for (int q = 0; q < kMaxScalers; ++q)
        if (q < ns) *reinterpret_cast<float4 *>(dU + (size_t)h * NS * K4 + (size_t)q * K4 + n) = t[q];
    } else {  // self-term block -> U_x [H][Fl] (Fl may be the raw feature width: scalar stores)
      const float v[4] = {t[0].x, t[0].y, t[0].z, t[0].w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (n - K4 + u < Fl) dUx[(size_t)h * Fl + n - K4 + u] = v[u];
    }
  }
}

namespace {
// CTAs of the side-stream Grams (persistent): fewer than the SM count leaves room for
// the critical chain's kernels that run concurrently
// Small steps (config B: ~150 Gram items) run the Grams beside the latency-bound main chain,
// where fewer CTAs interfere less (148 -> 40 measured +2%); large ones (config D/E: thousands
// of items) need every SM. Cap = clamp(items / 2, 40, 148) (items / 4 measured 1% slower at
// B and D, round 2) unless the step builder overrides it (g_mn_grid_override: the Grams that
// end the step use every SM).
int mn_grid_cap(int items) {
  if (g_mn_grid_override > 0) return g_mn_grid_override;
  return std::max(40, std::min(kSMs, items / 2));
}
template <class Op>
void nrun(cudaStream_t st, const TmaMaps &mp, const CUtensorMap &ones, Op op, int items) {
  op.items_cap = items;
  launch_ex(k_tmn<Op>, std::max(1, std::min(items, mn_grid_cap(items))), N_THREADS, n_smem_bytes<Op>(), st, mp, ones,
            op, g_gemm_passes);
  g_launches += 1;
}
}  // namespace

cudaError_t tmn_configure() {
  cudaError_t e = cudaFuncSetAttribute(k_tmn<MnGram>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       n_smem_bytes<MnGram>());
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_tmn<MnDMx>, cudaFuncAttributeMaxDynamicSharedMemorySize, n_smem_bytes<MnDMx>());
}

size_t mn_gram_partial_floats(const Caps &c, int cmax) {
  const size_t S = (size_t)tc_max_splits(c, cmax);
  return S * c.H * c.KA() + S * c.H;
}
size_t mn_dmx_partial_floats(const Caps &c, int F, int R) {
  return (size_t)dmx_splits(c) * (R > 0 ? R : c.PW()) * (F + 1);
}

void launch_mn_dU_cls(cudaStream_t st, const Caps &c, int cmax, const float *dZ, const float *A, const float *ones,
                      const DegInfo *info, const int4 *splits, float *partial, float *dU, float *dbU, float *dUx,
                      int Fl) {
  const int smax = tc_max_splits(c, cmax);
  const int K = c.KA(), total = c.H * K;
  float *cs = partial + (size_t)smax * total;
  const CUtensorMap a = tma_map2d(dZ, c.maxN, c.H, N_BK, true), b = tma_map2d(A, c.maxN, K, N_BK, true);
  const TmaMaps mp{a, a, b, b};  // (lo slots unused: derived in shared memory)
  const CUtensorMap om = tma_map2d(ones, c.maxN, 32, N_BK, true);
  MnGram op{info, splits, partial, cs, c.H, K, 0};
  nrun(st, mp, om, op, smax * (c.H / N_BM) * (K / MnGram::BN + 1));
  launch_ex(k_reduce_gram, total / 128 + cdiv(c.H, 128), 256, 0, st, partial, cs, info, splits, c.H, K, c.S, Fl, dU,
            dbU, dUx);
  g_launches += 1;
}

void launch_mn_dMx(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *X, int F, int Fp,
                   const float *ones, float *partial, float *dMx, float *dbM, int Rr) {
  // rows: dP (H), or [dP | dQ] (2H) -> [dM_x; dM_s], adjacent in the gradient arena (or Rr)
  const int R = Rr > 0 ? Rr : c.PW();
  const int count = R * F;
  const int ns = dmx_splits(c);
  float *cs = partial + (size_t)ns * count;
  const CUtensorMap a = tma_map2d(dP, c.maxN, R, N_BK, true), b = tma_map2d(X, c.maxN, Fp, N_BK, true);
  const TmaMaps mp{a, a, b, b};  // (lo slots unused: derived in shared memory)
  const CUtensorMap om = tma_map2d(ones, c.maxN, 32, N_BK, true);
  const int with_cs = dbM ? 1 : 0;
  MnDMx op{blob, partial, cs, R, F, 0, with_cs, ns};
  nrun(st, mp, om, op, ns * (R / N_BM) * ((F + MnDMx::BN - 1) / MnDMx::BN + with_cs));
  const RJob j0{partial, ns, count, dMx, 0}, j1{cs, ns, with_cs ? R : 0, dbM, 0},
      j2{nullptr, 0, 0, nullptr, 0};
  launch_ex(k_reduce_jobs, reduce_blocks(j0) + (with_cs ? reduce_blocks(j1) : 0), 32 * RW, 0, st, j0, j1, j2);
  g_launches += 1;
}

// fixed-order sums of the aggregation backward's per-graph partials (agg.cu): rows of H*Fe
// dM_e entries then H db_M entries, one row per graph slot (up to thousands of rows). Block =
// 32 warps x 32 lanes over 32 float4 columns: warp w sums rows w, w + 32, ... of its lane's
// column (coalesced 512-byte row segments, four loads in flight), then warp 0 adds the 32
// warp sums in order (deterministic).
__global__ void __launch_bounds__(1024) k_reduce_rows32(const float *__restrict__ part, int nparts, int stride,
                                                         int cnt_e, float *__restrict__ dMe, int cnt_b,
                                                         float *__restrict__ dbM) {
  pdl_enter();
  __shared__ float4 red[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = 4 * (blockIdx.x * 32 + lane);
  const bool ok = e < cnt_e + cnt_b;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
#pragma unroll 4
    for (int p = warp; p < nparts; p += 32) add4(s, ldg4(part + (size_t)p * stride + e));
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && ok) {
    float4 t = red[0][lane];
#pragma unroll
    for (int w = 1; w < 32; ++w) add4(t, red[w][lane]);
    float *o = e < cnt_e ? dMe + e : dbM + (e - cnt_e);
    *reinterpret_cast<float4 *>(o) = t;
  }
}

void launch_reduce_dMe(cudaStream_t st, const Caps &c, const float *partial, float *dMe, float *dbM) {
  const int stride = c.H * (c.Fe + 1), cnt_e = c.H * c.Fe, cnt_b = c.H;  // (both % 4 == 0: H % 128 == 0)
  launch_ex(k_reduce_rows32, (cnt_e + cnt_b + 127) / 128, 1024, 0, st, partial, c.maxB, stride, cnt_e, dMe, cnt_b,
            dbM);
  g_launches += 1;
}

void launch_reduce_cols(cudaStream_t st, const float *part, int parts, int stride, int count, float *out) {
  launch_ex(k_reduce_rows32, (count + 127) / 128, 1024, 0, st, part, parts, stride, count, out, 0, out);
  g_launches += 1;
}

int pad_x0_width(int F0) { return (F0 + 3) / 4 * 4; }  // 16-byte row pitch; TMA zero-fills the rest
void launch_pad_x0(cudaStream_t st, const Caps &c, const uint8_t *blob, float *Xp, const int *pos) {
  const int Fp = pad_x0_width(c.F0);
  launch_ex(k_pad_x0, std::max(1, std::min(cdiv(c.maxN * Fp, 256), kSMs * 2)), 256, 0, st, blob, Fp, Xp, pos);
  g_launches += 1;
}

}  // namespace hg
