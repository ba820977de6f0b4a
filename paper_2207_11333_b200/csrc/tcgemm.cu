// tcgemm.cu — fp32-accurate (3xTF32) tensor-core GEMMs on sm_100a (tcgen05 + TMEM)
// for the three dense contractions of the PNA layer:
//
//   G1 update  Z = sum_s diag(s) A U_s^T + b_U, X' = ReLU(Z)
//   G2 dA      dA = sum_s diag(s) dZ U_s
//   G3 dU      dU_s = (diag(s) dZ)^T A   (split-K partials)
//
// The three degree scalers s in (identity, amplification, attenuation) are
// per-row scalars, so G1/G2 keep THREE accumulators in TMEM (one per scaler,
// stacked along the MMA N dimension: B rows = [U_id; U_amp; U_att] slices) and
// fold amp/att in the epilogue — the 12H-wide concat is never materialised.
// G3 has the scaler on the K (node) dimension, so it scales the B operand.
//
// Kernel structure (one 128-row output tile per CTA, 160 threads):
//   warps 0-3  producers: global fp32 -> registers -> (scale) -> hi/lo split
//              (3xTF32: a*b ~ ah*bh + ah*bl + al*bh) -> SW128 K-major smem stages;
//              then the epilogue: tcgen05.ld of their 32 TMEM lanes -> global.
//   warp 4     TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32,
//              M=128, N = 3*BN), tcgen05.commit -> mbarriers.
// Deterministic: every output element is produced by exactly one CTA (G3's
// split-K partials are reduced in fixed order by k_reduce_parts).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace hg {

extern std::atomic<int64_t> g_launches;

// debug/experiment switch for the tcgen05 pipeline (0 = normal). 1: MMA issues no
// tcgen05.mma (commits only); 2: transform does no LDS/split/STS; 3: loaders issue
// no cp.async (arrive only). Results are wrong in modes 1-3: timing experiments only.
__constant__ int g_tc_mode = 0;

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;            // fp32 elements per 128-byte smem row
constexpr int TC_XF_WARPS = 8;       // transform (+ epilogue) warps
constexpr int TC_LD_WARPS = 4;       // cp.async loader warps
constexpr int TC_MMA_WARP = TC_XF_WARPS + TC_LD_WARPS;
constexpr int TC_THREADS = 32 * (TC_MMA_WARP + 1);

template <int N>
struct TmemCols {
  static constexpr int v = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : N <= 256 ? 256 : 512;
};

// shared memory: RS raw stages (A raw 16 KB + B raw NMMA*128 B, cp.async targets)
// and ST operand stages (A hi, A lo, B hi, B lo in K-major SW128 layout)
template <class Op>
constexpr int tc_raw_bytes() { return TC_BM * 128 + Op::NMMA * 128; }
template <class Op>
constexpr int tc_stage_bytes() { return 2 * TC_BM * 128 + 2 * Op::NMMA * 128; }
template <class Op>
constexpr int tc_smem_bytes() {
  return Op::STAGES * tc_stage_bytes<Op>() + Op::RAW * tc_raw_bytes<Op>() + 1024 + 8 * (2 * Op::STAGES + 2 * Op::RAW + 1) + 16;
}

__device__ __forceinline__ float4 split_hi(float4 v, float4 &lo) {
  float4 hi;
  tc::split_tf32(v.x, hi.x, lo.x);
  tc::split_tf32(v.y, hi.y, lo.y);
  tc::split_tf32(v.z, hi.z, lo.z);
  tc::split_tf32(v.w, hi.w, lo.w);
  return hi;
}

// raw staging layouts: K-major source -> raw[row][32 k] (128-byte rows);
// MN-major source -> raw[k][ROWS] (rows contiguous along MN).
template <bool MN, int ROWS>
__device__ __forceinline__ void load_piece(int p, int &r, int &k, uint32_t &raw_off) {
  if (MN) {  // piece = 4 consecutive rows at one k
    k = p / (ROWS / 4);
    r = (p % (ROWS / 4)) * 4;
    raw_off = (uint32_t)(k * ROWS * 4 + r * 4);
  } else {   // piece = 4 consecutive k of one row
    r = p >> 3;
    k = (p & 7) * 4;
    raw_off = (uint32_t)(r * 128 + k * 4);
  }
}

// transform one 16-byte K-major chunk (row r, k-chunk j) from the raw stage
template <bool MN, int ROWS>
__device__ __forceinline__ float4 read_raw(const uint8_t *raw, int r, int j) {
  if (MN) {
    const float *f = reinterpret_cast<const float *>(raw);
    return make_float4(f[(4 * j + 0) * ROWS + r], f[(4 * j + 1) * ROWS + r], f[(4 * j + 2) * ROWS + r],
                       f[(4 * j + 3) * ROWS + r]);
  }
  return *reinterpret_cast<const float4 *>(raw + r * 128 + j * 16);
}
// task -> (row, k-chunk): lanes over rows for MN sources (conflict-free column reads),
// over k-chunks for K sources (contiguous 128-byte rows)
template <bool MN, int ROWS>
__device__ __forceinline__ void xf_coords(int task, int &r, int &j) {
  if (MN) { r = task % ROWS; j = task / ROWS; }
  else { r = task >> 3; j = task & 7; }
}

template <class Op>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tcgemm(Op op_in) {
  pdl_enter();
  Op op = op_in;
  op.prepare();
  int m0, n0, kb, ke;
  if (!op.tile(blockIdx.x, m0, n0, kb, ke)) return;  // uniform: tile beyond the device-side size

  constexpr int NMMA = Op::NMMA, ST = Op::STAGES, RS = Op::RAW, NACC = Op::NACC, BN = Op::BN;
  constexpr bool AMN = Op::A_MN, BMN = Op::B_MN;
  constexpr int A_BYTES = TC_BM * 128, B_BYTES = NMMA * 128;
  constexpr int STAGE = tc_stage_bytes<Op>(), RAWB = tc_raw_bytes<Op>();
  constexpr int TCOLS = TmemCols<NMMA>::v;
  static_assert(NMMA % 16 == 0 && NMMA <= 256, "MMA N for M=128 must be a multiple of 16 <= 256");
  static_assert(NMMA == NACC * BN && BN % 32 == 0, "accumulator tiling");
  static_assert(B_BYTES % 1024 == 0, "SW128 tiles need 1024-byte alignment");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align within the shared window by indexing smem_raw (keeps the pointer in the
  // shared state space, so the compiler emits LDS/STS rather than generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *raw0 = smem + ST * STAGE;
  uint64_t *full = reinterpret_cast<uint64_t *>(raw0 + RS * RAWB);
  uint64_t *empty = full + ST;
  uint64_t *rfull = empty + ST;
  uint64_t *rempty = rfull + RS;
  uint64_t *accf = rempty + RS;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(accf + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NXF = TC_XF_WARPS * 32, NLD = TC_LD_WARPS * 32;
  if (warp == TC_MMA_WARP) tc::tmem_alloc<TCOLS>(tmem_holder);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      tc::mbar_init(&full[s], NXF);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < RS; ++s) {
      tc::mbar_init(&rfull[s], NLD);
      tc::mbar_init(&rempty[s], NXF);
    }
    tc::mbar_init(accf, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_holder;
  const int nchunks = ke > kb ? (ke - kb + TC_BK - 1) / TC_BK : 0;

  if (warp >= TC_XF_WARPS && warp < TC_MMA_WARP) {
    // ---------------- loaders: cp.async raw fp32 tiles, completion -> rfull[rs].
    // K-major sources: the rows a thread copies are fixed for the whole tile, so
    // their (possibly gathered) base pointers are resolved once, outside the K loop.
    const int t = threadIdx.x - NXF;
    const float *dummy = op.any_src();
    constexpr int NPA = TC_BM * 8 / NLD, NPB = (NMMA * 8 + NLD - 1) / NLD;
    const float *arow[AMN ? 1 : NPA];
    const float *brow[BMN ? 1 : NPB];
    if constexpr (!AMN) {
#pragma unroll
      for (int i = 0; i < NPA; ++i) arow[i] = op.a_src(m0 + ((t + i * NLD) >> 3), kb, ke);
    }
    if constexpr (!BMN) {
#pragma unroll
      for (int i = 0; i < NPB; ++i) {
        const int p = t + i * NLD;
        brow[i] = p < NMMA * 8 ? op.b_src(n0, p >> 3, kb, ke) : nullptr;
      }
    }
    for (int c = 0; c < nchunks; ++c) {
      const int rs = c % RS;
      if (c >= RS) tc::mbar_wait(&rempty[rs], ((c / RS) - 1) & 1);
      uint8_t *rA = raw0 + rs * RAWB;
      uint8_t *rB = rA + A_BYTES;
      const int k0 = kb + c * TC_BK;
#pragma unroll
      for (int i = 0; i < NPA; ++i) {
        const int p = t + i * NLD;
        int r, k;
        uint32_t off;
        load_piece<AMN, TC_BM>(p, r, k, off);
        const float *src;
        if constexpr (AMN) src = op.a_src(m0 + r, k0 + k, ke);
        else src = (arow[i] && k0 + k < ke) ? arow[i] + (k0 - kb) + k : nullptr;
        if (g_tc_mode != 3 && g_tc_mode != 4) tc::cp_async16(rA + off, src ? src : dummy, src ? 16u : 0u);
      }
#pragma unroll
      for (int i = 0; i < NPB; ++i) {
        const int p = t + i * NLD;
        if (p < NMMA * 8) {
          int r, k;
          uint32_t off;
          load_piece<BMN, NMMA>(p, r, k, off);
          const float *src;
          if constexpr (BMN) src = op.b_src(n0, r, k0 + k, ke);
          else src = (brow[i] && k0 + k < ke) ? brow[i] + (k0 - kb) + k : nullptr;
          if (g_tc_mode != 3 && g_tc_mode != 4) tc::cp_async16(rB + off, src ? src : dummy, src ? 16u : 0u);
        }
      }
      tc::cp_async_arrive(&rfull[rs]);
    }
  } else if (warp < TC_XF_WARPS) {
    // ---------------- transform: raw -> (fix-up) -> 3xTF32 hi/lo K-major SW128 tiles
    const int t = threadIdx.x;
    // optional fused column sum of an MN-major A operand (bias gradients): with
    // NXF = 2 * TC_BM each thread always transforms the same row r = t % TC_BM
    float csum = 0.f;
    static_assert(!Op::COLSUM || (AMN && NXF == 2 * TC_BM), "fused column sum layout");
    for (int c = 0; c < nchunks; ++c) {
      const int rs = c % RS, s = c % ST;
      tc::mbar_wait(&rfull[rs], (c / RS) & 1);
      if (c >= ST) tc::mbar_wait(&empty[s], ((c / ST) - 1) & 1);
      const uint8_t *rA = raw0 + rs * RAWB;
      const uint8_t *rB = rA + A_BYTES;
      uint8_t *sAh = smem + s * STAGE;
      uint8_t *sAl = sAh + A_BYTES;
      uint8_t *sBh = sAl + A_BYTES;
      uint8_t *sBl = sBh + B_BYTES;
      const int k0 = kb + c * TC_BK;
      if (g_tc_mode != 2 && g_tc_mode != 4) {
#pragma unroll 4
      for (int task = t; task < TC_BM * 8; task += NXF) {
        int r, j;
        xf_coords<AMN, TC_BM>(task, r, j);
        float4 lo;
        const float4 av = op.a_fix(read_raw<AMN, TC_BM>(rA, r, j), m0 + r, k0 + 4 * j, ke);
        if constexpr (Op::COLSUM) csum += (av.x + av.y) + (av.z + av.w);
        const float4 hi = g_tc_mode == 5 ? (split_hi(av, lo), av) : split_hi(av, lo);
        const uint32_t o = tc::sw128_off(r, j);
        *reinterpret_cast<float4 *>(sAh + o) = hi;
        *reinterpret_cast<float4 *>(sAl + o) = lo;
      }
#pragma unroll 4
      for (int task = t; task < NMMA * 8; task += NXF) {
        int r, j;
        xf_coords<BMN, NMMA>(task, r, j);
        float4 lo;
        const float4 hi = split_hi(op.b_fix(read_raw<BMN, NMMA>(rB, r, j), n0, r, k0 + 4 * j, ke), lo);
        const uint32_t o = tc::sw128_off(r, j);
        *reinterpret_cast<float4 *>(sBh + o) = hi;
        *reinterpret_cast<float4 *>(sBl + o) = lo;
      }
      }
      tc::mbar_arrive(&rempty[rs]);     // raw stage may be refilled
      tc::fence_proxy_async_smem();     // operand tiles -> visible to the tensor core
      tc::mbar_arrive(&full[s]);
    }
    if constexpr (Op::COLSUM) {
      // combine the two half-sums of each row in fixed order (smem reuse of the
      // barrier-free raw region is unsafe, so use a small dedicated array)
      __shared__ float cs[2][TC_BM];
      cs[t / TC_BM][t % TC_BM] = csum;
      asm volatile("bar.sync 1, %0;" ::"n"(NXF));  // transform warps only
      if (t < TC_BM) op.colsum(m0 + t, n0, cs[0][t] + cs[1][t]);
    }
    // ---------------- epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (one row per
    // thread); the two warpgroups split the 32-column chunks of each accumulator
    tc::mbar_wait(accf, 0);
    tc::fence_after_sync();
    const int wq = warp & 3, wg = warp >> 2;
    const int row = wq * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
#pragma unroll 1
    for (int q = wg; q < BN / 32; q += TC_XF_WARPS / 4) {
      float acc[NACC][32];
#pragma unroll
      for (int a = 0; a < NACC; ++a) {
        if (nchunks) {
          tc::tmem_ld32(trow + (uint32_t)(a * BN + q * 32), acc[a]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[a][i] = 0.f;
        }
      }
      op.store(m0 + row, n0, q * 32, acc);
    }
  } else {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(TC_BM, NMMA);
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % ST;
        tc::mbar_wait(&full[s], (c / ST) & 1);
        tc::fence_after_sync();
        const uint32_t aH = tc::smem_u32(smem + s * STAGE);
        const uint32_t aL = aH + A_BYTES, bH = aL + A_BYTES, bL = bH + B_BYTES;
#pragma unroll
        for (int ks = 0; ks < TC_BK / 8; ++ks) {  // K = 8 tf32 (32 bytes) per MMA
          const uint32_t off = ks * 32;
          const uint64_t dah = tc::desc_sw128(aH + off), dal = tc::desc_sw128(aL + off);
          const uint64_t dbh = tc::desc_sw128(bH + off), dbl = tc::desc_sw128(bL + off);
          if (g_tc_mode != 1 && g_tc_mode != 4) {
            tc::mma_tf32(tmem, dah, dbh, idesc, (c | ks) != 0);
            tc::mma_tf32(tmem, dah, dbl, idesc, 1u);
            tc::mma_tf32(tmem, dal, dbh, idesc, 1u);
          }
        }
        tc::mma_commit(&empty[s]);  // frees the stage when these MMAs have read it
      }
      tc::mma_commit(accf);  // accumulators complete
    }
    __syncwarp();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == TC_MMA_WARP) {
    tc::fence_after_sync();
    tc::tmem_dealloc<TCOLS>(tmem);
  }
}

template <class Op>
static cudaError_t configure_tc() {
  return cudaFuncSetAttribute(k_tcgemm<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<Op>());
}

template <class Op>
static void run_tc(cudaStream_t st, const Op &op, int grid) {
  launch_ex(k_tcgemm<Op>, std::max(grid, 1), TC_THREADS, tc_smem_bytes<Op>(), st, op);
  g_launches += 1;
}

__device__ __forceinline__ float scal(const float *amp, const float *att, int m, int s) {
  return s == 0 ? 1.0f : (s == 1 ? amp[m] : att[m]);
}

// ---------------------------------------------------------------- G1 update
struct TcUpdate {
  static constexpr int BN = 32, NACC = 3, NMMA = 96, STAGES = 2, RAW = 3;
  static constexpr bool A_MN = false, B_MN = false;
  static constexpr bool COLSUM = false;
  const uint8_t *blob; const float *A; const float *amp; const float *att; const float *U; const float *bU;
  float *X1; int H; int N;
  __device__ void prepare() { N = batch_N(blob); }
  __device__ bool tile(int t, int &m0, int &n0, int &kb, int &ke) const {
    const int nt = H / BN;
    m0 = (t / nt) * TC_BM;
    n0 = (t % nt) * BN;
    kb = 0;
    ke = 4 * H;
    return m0 < N;
  }
  __device__ const float *any_src() const { return U; }
  __device__ const float *a_src(int m, int k, int) const { return m < N ? A + (size_t)m * 4 * H + k : nullptr; }
  __device__ float4 a_fix(float4 v, int, int, int) const { return v; }
  __device__ const float *b_src(int n0, int r, int k, int) const {
    const int s = r / BN, c = r - s * BN;
    return U + (size_t)(n0 + c) * 12 * H + s * 4 * H + k;
  }
  __device__ float4 b_fix(float4 v, int, int, int, int) const { return v; }
  __device__ void store(int m, int n0, int q0, const float (&acc)[3][32]) const {
    if (m >= N) return;
    const float a1 = amp[m], a2 = att[m];
    float *out = X1 + (size_t)m * H + n0 + q0;
    const float *b = bU + n0 + q0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 z;
      z.x = fmaxf(acc[0][i + 0] + a1 * acc[1][i + 0] + a2 * acc[2][i + 0] + b[i + 0], 0.f);
      z.y = fmaxf(acc[0][i + 1] + a1 * acc[1][i + 1] + a2 * acc[2][i + 1] + b[i + 1], 0.f);
      z.z = fmaxf(acc[0][i + 2] + a1 * acc[1][i + 2] + a2 * acc[2][i + 2] + b[i + 2], 0.f);
      z.w = fmaxf(acc[0][i + 3] + a1 * acc[1][i + 3] + a2 * acc[2][i + 3] + b[i + 3], 0.f);
      *reinterpret_cast<float4 *>(out + i) = z;
    }
  }
};

// ---------------------------------------------------------------- G2 dA
// B_s[n, h] = U[h, s*4H + n] read from the transposed copy UT[s][n][h] (prepared per step)
struct TcDA {
  static constexpr int BN = 32, NACC = 3, NMMA = 96, STAGES = 2, RAW = 3;
  static constexpr bool A_MN = false, B_MN = false;
  static constexpr bool COLSUM = false;
  const uint8_t *blob; const float *dZ; const float *amp; const float *att; const float *UT; float *dA; int H; int N;
  __device__ void prepare() { N = batch_N(blob); }
  __device__ bool tile(int t, int &m0, int &n0, int &kb, int &ke) const {
    const int nt = 4 * H / BN;
    m0 = (t / nt) * TC_BM;
    n0 = (t % nt) * BN;
    kb = 0;
    ke = H;
    return m0 < N;
  }
  __device__ const float *any_src() const { return UT; }
  __device__ const float *a_src(int m, int k, int) const { return m < N ? dZ + (size_t)m * H + k : nullptr; }
  __device__ float4 a_fix(float4 v, int, int, int) const { return v; }
  __device__ const float *b_src(int n0, int r, int k, int) const {
    const int s = r / BN, c = r - s * BN;
    return UT + ((size_t)s * 4 * H + n0 + c) * H + k;
  }
  __device__ float4 b_fix(float4 v, int, int, int, int) const { return v; }
  __device__ void store(int m, int n0, int q0, const float (&acc)[3][32]) const {
    if (m >= N) return;
    const float a1 = amp[m], a2 = att[m];
    float *out = dA + (size_t)m * 4 * H + n0 + q0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 z;
      z.x = acc[0][i + 0] + a1 * acc[1][i + 0] + a2 * acc[2][i + 0];
      z.y = acc[0][i + 1] + a1 * acc[1][i + 1] + a2 * acc[2][i + 1];
      z.z = acc[0][i + 2] + a1 * acc[1][i + 2] + a2 * acc[2][i + 2];
      z.w = acc[0][i + 3] + a1 * acc[1][i + 3] + a2 * acc[2][i + 3];
      *reinterpret_cast<float4 *>(out + i) = z;
    }
  }
};

// ---------------------------------------------------------------- G3 dU (split-K over nodes)
// A(m=h, k=i) = dZ[i, h] (MN-major), B(r=(s,c), k=i) = s_i A_l[i, n0+c]; output
// partial[sp][h][s*4H + n] for the fixed-order reduction.
constexpr int kTcDUSplits = 16;
struct TcDU {
  static constexpr int BN = 32, NACC = 3, NMMA = 96, STAGES = 2, RAW = 3;
  static constexpr bool A_MN = true, B_MN = true;
  static constexpr bool COLSUM = false;
  const uint8_t *blob; const float *dZ; const float *A; const float *amp; const float *att; float *part; int H;
  int N; int sp;
  __device__ void prepare() { N = batch_N(blob); }
  __device__ bool tile(int t, int &m0, int &n0, int &kb, int &ke) {
    const int nt = 4 * H / BN, mt = H / TC_BM;
    sp = t % kTcDUSplits;
    const int t2 = t / kTcDUSplits;
    n0 = (t2 % nt) * BN;
    m0 = (t2 / nt) * TC_BM;
    if (m0 >= mt * TC_BM) return false;
    int kc = (N + kTcDUSplits - 1) / kTcDUSplits;
    kc = (kc + TC_BK - 1) / TC_BK * TC_BK;
    kb = sp * kc;
    ke = min(N, kb + kc);
    return true;  // empty splits still write their (zero) partial
  }
  // MN-major sources: a 16-byte piece = 4 consecutive rows (h, or B rows) at node k;
  // the transform stage transposes them into K-major operand tiles
  __device__ const float *any_src() const { return dZ; }
  __device__ const float *a_src(int m, int k, int ke) const { return k < ke ? dZ + (size_t)k * H + m : nullptr; }
  __device__ float4 a_fix(float4 v, int, int, int) const { return v; }
  __device__ const float *b_src(int n0, int r, int k, int ke) const {
    const int s = r / BN, c = r - s * BN;
    return k < ke ? A + (size_t)k * 4 * H + n0 + c : nullptr;
  }
  // the transformed chunk holds 4 consecutive k (nodes) of B row r: scale each by s_k
  __device__ float4 b_fix(float4 v, int, int r, int k, int ke) const {
    const int s = r / BN;
    if (s == 0) return v;
    const float *sc = s == 1 ? amp : att;
    return make_float4(k + 0 < ke ? v.x * sc[k + 0] : 0.f, k + 1 < ke ? v.y * sc[k + 1] : 0.f,
                       k + 2 < ke ? v.z * sc[k + 2] : 0.f, k + 3 < ke ? v.w * sc[k + 3] : 0.f);
  }
  __device__ void store(int m, int n0, int q0, const float (&acc)[3][32]) const {
    float *base = part + (size_t)sp * H * 12 * H + (size_t)m * 12 * H;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      float *out = base + s * 4 * H + n0 + q0;
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4 *>(out + i) = make_float4(acc[s][i], acc[s][i + 1], acc[s][i + 2], acc[s][i + 3]);
    }
  }
};

// ================================================================ degree classes
// The scalers depend only on a node's degree d, so for the rows of one degree
// class the three scaler blocks collapse into one matrix (exact reassociation
// of SPEC.md:347's U . [A || amp A || att A]):
//   Z_i   = A_i W_d^T + b_U,          W_d = U_id + amp(d) U_amp + att(d) U_att   (G1)
//   dA_i  = dZ_i W_d                                                              (G2)
//   dU_s  = sum_d s(d) G_d,           G_d = dZ_d^T A_d over the class's nodes      (G3)
// so each GEMM runs with ONE accumulator and one B operand (3x fewer MMA FLOPs
// and B bytes). Nodes are gathered through a degree-sorted permutation; tiles
// and K-splits never straddle classes. Used when max_degree + 1 <= kMaxClasses.

// one CTA: stable counting sort of nodes by degree (deterministic), per-node
// scalers, the class table, 128-row tiles and K-splits (DegInfo in kernels.h)
__global__ void __launch_bounds__(1024) k_degsort(const uint8_t *__restrict__ blob, double delta, int cmax,
                                                  int ks, float *__restrict__ amp, float *__restrict__ att,
                                                  int *__restrict__ perm, DegInfo *__restrict__ info,
                                                  int4 *__restrict__ tiles, int4 *__restrict__ splits,
                                                  int *__restrict__ pos) {
  pdl_enter();
  __shared__ int hist[kMaxClasses], bstart[kMaxClasses];
  __shared__ int wcnt[32][kMaxClasses];  // per-warp class counts, then per-warp class bases
  __shared__ float tamp[kMaxClasses], tatt[kMaxClasses];
  const BatchView b = load_batch(blob);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (cmax <= 0) {  // scalers only (no class GEMMs)
    for (int i = tid; i < b.N; i += blockDim.x) {
      const int d = b.rowptr[i + 1] - b.rowptr[i];
      if (d == 0) {
        amp[i] = 1.0f;
        att[i] = 1.0f;
      } else {
        const double ld = log((double)d + 1.0);
        amp[i] = (float)(ld / delta);
        att[i] = (float)(delta / ld);
      }
    }
    return;
  }
  // per-degree scalers once (d < cmax = max_degree + 1), in the same fp64 arithmetic
  if (tid < cmax) {
    if (tid == 0) {
      tamp[0] = 1.0f;
      tatt[0] = 1.0f;
    } else {
      const double ld = log((double)tid + 1.0);
      tamp[tid] = (float)(ld / delta);
      tatt[tid] = (float)(delta / ld);
    }
  }
  for (int e = tid; e < 32 * kMaxClasses; e += blockDim.x) wcnt[e / kMaxClasses][e % kMaxClasses] = 0;
  __syncthreads();
  // stable counting sort: warp w owns the contiguous node range [w*per, (w+1)*per), in
  // rounds of 32 nodes; ranks inside a round come from __match_any_sync
  const int per = (b.N + 31) / 32;
  const int w0 = warp * per, w1 = min(b.N, w0 + per);
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int d = i < w1 ? min(b.rowptr[i + 1] - b.rowptr[i], cmax - 1) : -1;
    if (i < w1) {
      amp[i] = tamp[d];
      att[i] = tatt[d];
    }
    const unsigned mask = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(mask & ((1u << lane) - 1u));
    if (d >= 0 && rank == 0) wcnt[warp][d] += __popc(mask);
    __syncwarp();
  }
  __syncthreads();
  if (tid < cmax) {  // class totals and, per class, exclusive scan over warps in warp order
    int acc = 0;
    for (int w = 0; w < 32; ++w) {
      const int c = wcnt[w][tid];
      wcnt[w][tid] = acc;
      acc += c;
    }
    hist[tid] = acc;
  }
  __syncthreads();
  if (tid < cmax) {
    info->amp[tid] = tamp[tid];  // per degree slot
    info->att[tid] = tatt[tid];
  }
  if (tid == 0) {
    int off = 0, C = 0, T = 0, S = 0;
    for (int d = 0; d < cmax; ++d) {
      bstart[d] = off;
      if (hist[d] > 0) {
        info->deg[C] = d;
        info->start[C] = off;
        info->count[C] = hist[d];
        // tiles and splits carry the degree slot d: weights and scalers are indexed by d
        for (int r = 0; r < hist[d]; r += TC_BM) tiles[T++] = make_int4(d, off + r, min(TC_BM, hist[d] - r), 0);
        for (int r = 0; r < hist[d]; r += ks) splits[S++] = make_int4(d, off + r, min(ks, hist[d] - r), 0);
        ++C;
      }
      off += hist[d];
    }
    info->C = C;
    info->T = T;
    info->S = S;
  }
  __syncthreads();
  // scatter: same rounds again, positions = class start + warp base + running rank
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int d = i < w1 ? min(b.rowptr[i + 1] - b.rowptr[i], cmax - 1) : -1;
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







// ---------------------------------------------------------------- K1 projection (F % 4 == 0)
// P[N, H] = X[N, F] M_x^T : A = X rows (K = F), B = M_x rows
struct TcProj {
  static constexpr int BN = 64, NACC = 1, NMMA = 64, STAGES = 3, RAW = 3;
  static constexpr bool A_MN = false, B_MN = false;
  static constexpr bool COLSUM = false;
  const uint8_t *blob; const float *X; const float *Mx; float *P; int F, H; int N;
  __device__ void prepare() { N = batch_N(blob); }
  __device__ bool tile(int t, int &m0, int &n0, int &kb, int &ke) const {
    const int nt = H / BN;
    m0 = (t / nt) * TC_BM;
    n0 = (t % nt) * BN;
    kb = 0;
    ke = F;
    return m0 < N;
  }
  __device__ const float *any_src() const { return Mx; }
  __device__ const float *a_src(int m, int k, int ke) const {
    return (m < N && k < ke) ? X + (size_t)m * F + k : nullptr;
  }
  __device__ float4 a_fix(float4 v, int, int, int) const { return v; }
  __device__ const float *b_src(int n0, int r, int k, int ke) const {
    return k < ke ? Mx + (size_t)(n0 + r) * F + k : nullptr;
  }
  __device__ float4 b_fix(float4 v, int, int, int, int) const { return v; }
  __device__ void store(int m, int n0, int q0, const float (&acc)[1][32]) const {
    if (m >= N) return;
    float *out = P + (size_t)m * H + n0 + q0;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4 *>(out + i) = make_float4(acc[0][i], acc[0][i + 1], acc[0][i + 2], acc[0][i + 3]);
  }
};

// ---------------------------------------------------------------- K9b dX (l > 0)
// dZprev[N, F] = (dP[N, H] M_x[H, F]) * [X_l > 0] : A = dP rows (K = H), B(f, h) = M_x[h, f] (MN source)
struct TcDX {
  static constexpr int BN = 64, NACC = 1, NMMA = 64, STAGES = 3, RAW = 3;
  static constexpr bool A_MN = false, B_MN = true;
  static constexpr bool COLSUM = false;
  const uint8_t *blob; const float *dP; const float *Mx; const float *Xl; float *dZ; int H, F; int N;
  __device__ void prepare() { N = batch_N(blob); }
  __device__ bool tile(int t, int &m0, int &n0, int &kb, int &ke) const {
    const int nt = F / BN;
    m0 = (t / nt) * TC_BM;
    n0 = (t % nt) * BN;
    kb = 0;
    ke = H;
    return m0 < N;
  }
  __device__ const float *any_src() const { return Mx; }
  __device__ const float *a_src(int m, int k, int) const { return m < N ? dP + (size_t)m * H + k : nullptr; }
  __device__ float4 a_fix(float4 v, int, int, int) const { return v; }
  __device__ const float *b_src(int n0, int r, int k, int) const { return Mx + (size_t)k * F + n0 + r; }
  __device__ float4 b_fix(float4 v, int, int, int, int) const { return v; }
  __device__ void store(int m, int n0, int q0, const float (&acc)[1][32]) const {
    if (m >= N) return;
    const size_t o = (size_t)m * F + n0 + q0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const float4 x = ldg4(Xl + o + i);
      *reinterpret_cast<float4 *>(dZ + o + i) =
          make_float4(x.x > 0.f ? acc[0][i] : 0.f, x.y > 0.f ? acc[0][i + 1] : 0.f, x.z > 0.f ? acc[0][i + 2] : 0.f,
                      x.w > 0.f ? acc[0][i + 3] : 0.f);
    }
  }
};

// ---------------------------------------------------------------- K9a dM_x (split-K over nodes, F % 64 == 0)
// dM_x[h, f] = sum_i dP[i, h] X_l[i, f]: A(h, i) = dP[i, h], B(f, i) = X_l[i, f] (both MN sources)
constexpr int kTcDMxSplits = 16;
struct TcDMx {
  static constexpr int BN = 64, NACC = 1, NMMA = 64, STAGES = 3, RAW = 3;
  static constexpr bool A_MN = true, B_MN = true;
  static constexpr bool COLSUM = true;
  const uint8_t *blob; const float *dP; const float *X; float *part; int H, F; int N; float *cs_part; int sp;
  __device__ void colsum(int m, int n0, float v) const {
    if (n0 == 0) cs_part[(size_t)sp * H + m] = v;
  }
  __device__ void prepare() { N = batch_N(blob); }
  __device__ bool tile(int t, int &m0, int &n0, int &kb, int &ke) {
    const int nt = F / BN, mt = H / TC_BM;
    sp = t % kTcDMxSplits;
    const int t2 = t / kTcDMxSplits;
    n0 = (t2 % nt) * BN;
    m0 = (t2 / nt) * TC_BM;
    if (m0 >= mt * TC_BM) return false;
    int kc = (N + kTcDMxSplits - 1) / kTcDMxSplits;
    kc = (kc + TC_BK - 1) / TC_BK * TC_BK;
    kb = sp * kc;
    ke = min(N, kb + kc);
    return true;
  }
  __device__ const float *any_src() const { return dP; }
  __device__ const float *a_src(int m, int k, int ke) const { return k < ke ? dP + (size_t)k * H + m : nullptr; }
  __device__ float4 a_fix(float4 v, int, int, int) const { return v; }
  __device__ const float *b_src(int n0, int r, int k, int ke) const { return k < ke ? X + (size_t)k * F + n0 + r : nullptr; }
  __device__ float4 b_fix(float4 v, int, int, int, int) const { return v; }
  __device__ void store(int m, int n0, int q0, const float (&acc)[1][32]) const {
    float *out = part + (size_t)sp * H * F + (size_t)m * F + n0 + q0;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4 *>(out + i) = make_float4(acc[0][i], acc[0][i + 1], acc[0][i + 2], acc[0][i + 3]);
  }
};

__global__ void k_reduce_rows(const float *__restrict__ part, int nparts, int count, float *__restrict__ out);

__global__ void k_reduce_parts(const float *__restrict__ part, int nparts, int count, float *__restrict__ out) {
  pdl_enter();
  const int c4 = count / 4;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < c4; e += gridDim.x * blockDim.x) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = 0; p < nparts; ++p) {
      const float4 v = ldg4(part + (size_t)p * count + 4 * (size_t)e);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    reinterpret_cast<float4 *>(out)[e] = s;
  }
}

// column sums (db_U = sum_i dZ[i, :], db_M = sum_i dP[i, :]): fixed 64-row chunks,
// 8 independent loads in flight per thread, then a fixed-order reduction of the
// chunk partials (k_reduce_rows)
constexpr int kColsumRows = 64;
constexpr int kColsumChunks = 128;  // partial slots; chunks beyond ceil(N/64) write zeros
__global__ void __launch_bounds__(256) k_colsum_part(const uint8_t *__restrict__ blob, const float *__restrict__ X,
                                                     int H, float *__restrict__ part) {
  pdl_enter();
  const int N = batch_N(blob);
  const int per = max(kColsumRows, (N + kColsumChunks - 1) / kColsumChunks);
  for (int ch = blockIdx.x; ch < kColsumChunks; ch += gridDim.x) {
    const int i0 = ch * per, i1 = min(N, i0 + per);
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      int i = i0;
      for (; i + 8 <= i1; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] += X[(size_t)(i + u) * H + h];
      }
      float tail = 0.f;
      for (; i < i1; ++i) tail += X[(size_t)i * H + h];
      s[0] += tail;
      part[(size_t)ch * H + h] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    }
  }
}

// UT[l][s][n][h] = U_l[h][s*4H + n] for every layer (32x32 smem-tiled transpose)
__global__ void k_prep_UT(const float *__restrict__ params, const int64_t *__restrict__ u_off, int L, int H,
                          float *__restrict__ UT) {
  pdl_enter();
  __shared__ float tile[32][33];
  const int W = 12 * H;  // U row length
  const int tilesC = W / 32, tilesR = H / 32;
  const int per_layer = tilesC * tilesR;
  for (int t = blockIdx.x; t < L * per_layer; t += gridDim.x) {
    const int l = t / per_layer, tt = t % per_layer;
    const int tr = tt / tilesC, tc = tt % tilesC;  // rows h, cols j = s*4H + n
    const float *U = params + u_off[l];
    for (int r = threadIdx.y; r < 32; r += blockDim.y)
      tile[r][threadIdx.x] = U[(size_t)(tr * 32 + r) * W + tc * 32 + threadIdx.x];
    __syncthreads();
    float *out = UT + (size_t)l * W * H;
    for (int r = threadIdx.y; r < 32; r += blockDim.y)  // out row = j (= s*4H + n), col = h
      out[(size_t)(tc * 32 + r) * H + tr * 32 + threadIdx.x] = tile[threadIdx.x][r];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- launch wrappers
static int mtiles(int n) { return (n + TC_BM - 1) / TC_BM; }

void launch_tc_update(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *A, const float *amp,
                      const float *att, const float *U, const float *bU, float *X1) {
  TcUpdate op{blob, A, amp, att, U, bU, X1, c.H, 0};
  run_tc(st, op, mtiles(c.maxN) * (c.H / TcUpdate::BN));
}

void launch_tc_dA(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dZ, const float *amp,
                  const float *att, const float *UT, float *dA) {
  TcDA op{blob, dZ, amp, att, UT, dA, c.H, 0};
  run_tc(st, op, mtiles(c.maxN) * (4 * c.H / TcDA::BN));
}

size_t tc_dU_partial_floats(const Caps &c) {
  return std::max((size_t)kTcDUSplits * c.H * 12 * c.H, (size_t)kColsumChunks * c.H);
}

void launch_tc_dU(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dZ, const float *A,
                  const float *amp, const float *att, float *partial, float *dU, float *dbU) {
  TcDU op{blob, dZ, A, amp, att, partial, c.H, 0, 0};
  run_tc(st, op, (c.H / TC_BM) * (4 * c.H / TcDU::BN) * kTcDUSplits);
  const int count = c.H * 12 * c.H;
  launch_ex(k_reduce_parts, std::min(cdiv(count / 4, 256), kSMs * 4), 256, 0, st, partial, kTcDUSplits, count, dU);
  launch_ex(k_colsum_part, kColsumChunks, std::min(c.H, 256), 0, st, blob, dZ, c.H, partial);
  launch_ex(k_reduce_rows, cdiv(c.H, 8), 256, 0, st, partial, kColsumChunks, c.H, dbU);
  g_launches += 3;
}

void launch_prep_UT(cudaStream_t st, const Caps &c, const float *params, const int64_t *u_off_dev, int L,
                    float *UT) {
  const int blocks = std::min(L * (12 * c.H / 32) * (c.H / 32), kSMs * 8);
  launch_ex(k_prep_UT, blocks, dim3(32, 8), 0, st, params, u_off_dev, L, c.H, UT);
  g_launches += 1;
}

bool tc_supported(const Caps &c) { return c.H % 128 == 0; }

}  // namespace hg
extern "C" int hg_debug_set_tc_mode(int mode) {  // experiments only (not part of the ABI header)
  return (int)cudaMemcpyToSymbol(hg::g_tc_mode, &mode, sizeof(int));
}
namespace hg {

int tc_num_classes(const Caps &c, int max_degree) {
  const int cm = (max_degree > 0 ? max_degree : HG_MAX_DEGREE_DEV) + 1;
  return (tc_supported(c) && cm <= kMaxClasses) ? cm : 0;
}
int tc_max_tiles(const Caps &c, int cmax) { return mtiles(c.maxN) + cmax; }
int tc_max_splits(const Caps &c, int cmax) { return (c.maxN + gram_ks(c) - 1) / gram_ks(c) + cmax; }

void launch_degsort(cudaStream_t st, const uint8_t *blob, double delta, int cmax, float *amp, float *att, int *perm,
                    DegInfo *info, int4 *tiles, int4 *splits, int *pos, int ks) {
  launch_ex(k_degsort, 1, 1024, 0, st, blob, delta, cmax, ks > 0 ? ks : kGramKS, amp, att, perm, info, tiles, splits,
            pos);
  g_launches += 1;
}






cudaError_t tc_configure() {
  cudaError_t e;
  if ((e = configure_tc<TcUpdate>()) != cudaSuccess) return e;
  if ((e = configure_tc<TcDA>()) != cudaSuccess) return e;
  if ((e = configure_tc<TcProj>()) != cudaSuccess) return e;
  if ((e = configure_tc<TcDX>()) != cudaSuccess) return e;
  if ((e = configure_tc<TcDMx>()) != cudaSuccess) return e;
  return configure_tc<TcDU>();
}

bool tc_proj_ok(const Caps &c, int F) { return c.H % 128 == 0 && F % 4 == 0; }
bool tc_dmx_ok(const Caps &c, int F) { return c.H % 128 == 0 && F % 64 == 0; }

void launch_tc_proj(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *X, int F, const float *Mx,
                    float *P) {
  TcProj op{blob, X, Mx, P, F, c.H, 0};
  run_tc(st, op, mtiles(c.maxN) * (c.H / TcProj::BN));
}

void launch_tc_dX(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *Mx, int F,
                  const float *Xl, float *dZprev) {
  TcDX op{blob, dP, Mx, Xl, dZprev, c.H, F, 0};
  run_tc(st, op, mtiles(c.maxN) * (F / TcDX::BN));
}

size_t tc_dMx_partial_floats(const Caps &c, int F) {
  return (size_t)kTcDMxSplits * (c.H * F + c.H);
}

void launch_tc_dMx(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *dP, const float *X, int F,
                   float *partial, float *dMx, float *dbM) {
  const int count = c.H * F;
  float *cs = partial + (size_t)kTcDMxSplits * count;  // per-split column sums of dP (db_M)
  TcDMx op{blob, dP, X, partial, c.H, F, 0, cs, 0};
  run_tc(st, op, (c.H / TC_BM) * (F / TcDMx::BN) * kTcDMxSplits);
  launch_ex(k_reduce_parts, std::min(cdiv(count / 4, 256), kSMs * 4), 256, 0, st, partial, kTcDMxSplits, count, dMx);
  launch_ex(k_reduce_rows, cdiv(c.H, 8), 256, 0, st, cs, kTcDMxSplits, c.H, dbM);
  g_launches += 2;
}

}  // namespace hg
