// kernels.cu — CUDA kernels of the PNA-GCNN training step for sm_100a.
//
// Paper passages: message passing GC layer (§3.1; PNA,
// PAPER.md:148, 315) with the equations SPEC.md:347 fixes; global mean pool
// (SPEC.md:353); FC head; MSE
// (SPEC.md:365); backward;
// AdamW.
//
// Design: every reduction is deterministic (fixed order,
// no float atomics); sizes come from the device-resident batch header so the
// step is CUDA-graph capturable; segments (CSR rows, degree <= 127) are
// processed one warp per node with lanes over channels (coalesced 16-byte
// feature rows).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "kernels.h"
#include "layout.h"

namespace hg {

std::atomic<int64_t> g_launches{0};
bool g_low_prio = false;
int g_prio_lo = 0, g_prio_hi = 0;
static inline void counted(int n = 1) { g_launches += n; }

// ------------------------------------------------------------------ layer-0 projection (SIMT)
// Layer 0's projection P = x M_x^T contracts over the F0 = |vocab| + 3 raw node features
// (34 for the PCQM vocabulary): 2 N F0 H flops, under 1% of a step's GEMM work, with
// operand rows that are not 16-byte aligned, so it runs on the FP32 pipe (every other
// GEMM of the step is a TMA-fed tcgen05 kernel, tcdirect.cu / tcmn.cu).
// C[M,N] = sum_k a(m,k) b(k,n) with operand transforms supplied by Op; 64x64
// tiles, BK=16, 256 threads, 4x4 outputs per thread, register-prefetched
// double-buffered shared memory. A_KMAJ: a(m,k) contiguous in k (else in m);
// B_KMAJ: b(k,n) contiguous in k (else in n). Persistent over tiles x splits.
constexpr int GBM = 64, GBN = 64, GBK = 16;

template <bool A_KMAJ, bool B_KMAJ, class Op>
__global__ void __launch_bounds__(256) k_gemm(Op op_in) {
  pdl_enter();
  Op op = op_in;
  op.prepare();
  __shared__ __align__(16) float As[2][GBK][GBM + 4];
  __shared__ __align__(16) float Bs[2][GBK][GBN + 4];
  const int M = op.M(), N = op.N(), K = op.K(), S = op.splits();
  const int tilesM = (M + GBM - 1) / GBM, tilesN = (N + GBN - 1) / GBN;
  const int ntiles = tilesM * tilesN * S;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int sp = tile % S;
    const int t2 = tile / S;
    const int tn = t2 % tilesN, tm = t2 / tilesN;
    const int m0 = tm * GBM, n0 = tn * GBN;
    int kc = (K + S - 1) / S;
    kc = (kc + GBK - 1) / GBK * GBK;
    const int kb = sp * kc, ke = min(K, kb + kc);
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    float ra[4], rb[4];
    auto load_regs = [&](int k0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = tid + 256 * r;
        int ml, kl;
        if (A_KMAJ) { ml = e / GBK; kl = e % GBK; } else { ml = e % GBM; kl = e / GBM; }
        const int m = m0 + ml, k = k0 + kl;
        ra[r] = (m < M && k < ke) ? op.a(m, k) : 0.f;
        int nl, kl2;
        if (B_KMAJ) { nl = e / GBK; kl2 = e % GBK; } else { nl = e % GBN; kl2 = e / GBN; }
        const int n = n0 + nl, k2 = k0 + kl2;
        rb[r] = (n < N && k2 < ke) ? op.b(k2, n) : 0.f;
      }
    };
    auto store_smem = [&](int buf) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = tid + 256 * r;
        int ml, kl;
        if (A_KMAJ) { ml = e / GBK; kl = e % GBK; } else { ml = e % GBM; kl = e / GBM; }
        As[buf][kl][ml] = ra[r];
        int nl, kl2;
        if (B_KMAJ) { nl = e / GBK; kl2 = e % GBK; } else { nl = e % GBN; kl2 = e / GBN; }
        Bs[buf][kl2][nl] = rb[r];
      }
    };
    if (kb < ke) {
      load_regs(kb);
      store_smem(0);
      __syncthreads();
      int buf = 0;
      for (int k0 = kb; k0 < ke; k0 += GBK) {
        const bool more = k0 + GBK < ke;
        if (more) load_regs(k0 + GBK);
#pragma unroll
        for (int kk = 0; kk < GBK; ++kk) {
          const float4 a4 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
          const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
          const float av[4] = {a4.x, a4.y, a4.z, a4.w};
          const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if (more) {
          store_smem(buf ^ 1);
          __syncthreads();
          buf ^= 1;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + tx * 4 + j;
        if (n < N) op.store(m, n, acc[i][j], sp);
      }
    }
    __syncthreads();
  }
}

template <bool AK, bool BK_, class Op>
static void run_gemm(cudaStream_t st, const Op &op, int maxM, int N, int splits) {
  const int tiles = cdiv(maxM, GBM) * cdiv(N, GBN) * splits;
  const int grid = std::max(1, std::min(tiles, kSMs * 8));
  launch_ex(k_gemm<AK, BK_, Op>, grid, 256, 0, st, op);
  counted();
}

// P = X Mx^T  (the message M[x_j || e] + b_M is linear, so the
// x-part is projected once per node instead of once per edge)
struct OpProj {
  const uint8_t *blob; const float *X; const float *Mx; float *P; int F, H;
  __device__ void prepare() { if (!X) X = load_batch(blob).x; }  // layer 0 reads the batch's x
  __device__ int M() const { return batch_N(blob); }
  __device__ int N() const { return H; }
  __device__ int K() const { return F; }
  __device__ int splits() const { return 1; }
  __device__ float a(int m, int k) const { return X[(size_t)m * F + k]; }
  __device__ float b(int k, int n) const { return Mx[(size_t)n * F + k]; }
  __device__ void store(int m, int n, float v, int) const { P[(size_t)m * H + n] = v; }
};
void launch_proj(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *X, int F, const float *Mx,
                 float *P) {
  OpProj op{blob, X, Mx, P, F, c.PW()};  // (self-term: the 2H rows [M_x; M_s] -> [P | Q])
  run_gemm<true, true>(st, op, c.maxN, c.PW(), 1);
}

// ------------------------------------------------------------------ head
// Block per graph: G_g = mean of X_L rows, hpre = W1 G + b1,
// yhat = W2 ReLU(hpre) + b2, sqerr = (yhat - y)^2.
__device__ __forceinline__ float block_sum_256(float v, float *red) {
  // deterministic tree over a 256-thread block
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const float r = red[0];
  __syncthreads();
  return r;
}

// Head kernel, block per graph (grid-stride), W1 staged in shared memory when it
// fits. FWD: G_g = mean of X_L rows, hpre = W1 G + b1,
// yhat = W2 ReLU(hpre) + b2, sqerr = (yhat - y)^2.
// BWD: dy = 2(yhat - y)/B, dhid = dy W2 * [hpre > 0],
// dG = W1^T dhid, dZ_L[i] = dG / n_g * [X_L[i] > 0].
// FWD && BWD fuses both when a training step runs them back to back.
template <bool FWD, bool BWD>
__global__ void __launch_bounds__(256) k_head(const uint8_t *__restrict__ blob, const float *__restrict__ XL,
                                              const float *__restrict__ W1, const float *__restrict__ b1,
                                              const float *__restrict__ W2, const float *__restrict__ b2,
                                              float *__restrict__ G, float *__restrict__ hpre,
                                              float *__restrict__ yhat, float *__restrict__ sqerr,
                                              float *__restrict__ dy, float *__restrict__ dhid,
                                              float *__restrict__ dZL, int H, int Hf, int w1_in_smem,
                                              const int *__restrict__ pos) {
  pdl_enter();
  extern __shared__ float sm[];
  float *Gs = sm, *hs = Gs + H, *dh = hs + Hf, *red = dh + Hf, *W1s = red + 256;
  const float *Wr = W1;
  if (w1_in_smem) {
    const int n4 = Hf * H / 4;
    for (int e = threadIdx.x; e < n4; e += blockDim.x)
      reinterpret_cast<float4 *>(W1s)[e] = __ldg(reinterpret_cast<const float4 *>(W1) + e);
    Wr = W1s;
    __syncthreads();
  }
  const BatchView b = load_batch(blob);
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int g = blockIdx.x; g < b.B; g += gridDim.x) {
    const int n0 = b.gp[g], n1 = b.gp[g + 1];
    const float ng = (float)(n1 - n0);
    float yh;
    if (FWD) {
      for (int c = threadIdx.x; c < H; c += blockDim.x) {
        float s = 0.f;
        int i = n0;
        for (; i + 4 <= n1; i += 4) {  // 4 independent loads in flight
          const float a0 = XL[(size_t)i * H + c], a1 = XL[(size_t)(i + 1) * H + c];
          const float a2 = XL[(size_t)(i + 2) * H + c], a3 = XL[(size_t)(i + 3) * H + c];
          s += a0;
          s += a1;
          s += a2;
          s += a3;
        }
        for (; i < n1; ++i) s += XL[(size_t)i * H + c];
        const float v = s / ng;
        Gs[c] = v;
        G[(size_t)g * H + c] = v;
      }
      __syncthreads();
      // hpre[r] = b1[r] + W1[r,:] . G : warp per output row, fixed xor-shuffle order
      for (int r = threadIdx.x >> 5; r < Hf; r += wpb) {
        const float *w = Wr + (size_t)r * H;
        float acc = 0.f;
        for (int c = lane; c < H; c += 32) acc = fmaf(w[c], Gs[c], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
          acc += b1[r];
          hpre[(size_t)g * Hf + r] = acc;
          hs[r] = acc;
        }
      }
      __syncthreads();
      float part = 0.f;
      for (int r = threadIdx.x; r < Hf; r += blockDim.x) part = fmaf(W2[r], fmaxf(hs[r], 0.f), part);
      yh = block_sum_256(part, red) + b2[0];
      if (threadIdx.x == 0) {
        yhat[g] = yh;
        const float e = yh - b.y[g];
        sqerr[g] = e * e;
      }
    } else {
      for (int r = threadIdx.x; r < Hf; r += blockDim.x) hs[r] = hpre[(size_t)g * Hf + r];
      yh = yhat[g];
      __syncthreads();
    }
    if (BWD) {
      const float d = 2.0f * (yh - b.y[g]) / (float)b.B;
      if (threadIdx.x == 0) dy[g] = d;
      for (int r = threadIdx.x; r < Hf; r += blockDim.x) {
        const float v = hs[r] > 0.f ? d * W2[r] : 0.f;
        dh[r] = v;
        dhid[(size_t)g * Hf + r] = v;
      }
      __syncthreads();
      for (int c = threadIdx.x; c < H; c += blockDim.x) {
        float acc = 0.f;
        for (int r = 0; r < Hf; ++r) acc = fmaf(Wr[(size_t)r * H + c], dh[r], acc);
        Gs[c] = acc / ng;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < (n1 - n0) * H; e += blockDim.x) {
        const int i = n0 + e / H, c = e % H;
        const size_t o = (size_t)i * H + c;
        const float v = XL[o] > 0.f ? Gs[c] : 0.f;
        const size_t od = pos ? (size_t)pos[i] * H + c : o;  // degree-sorted row when pos is given
        dZL[od] = v;
      }
    }
    __syncthreads();
  }
}

// Latency-optimised head for H = 128*CH, Hf = 8*RW (one block of 8 warps per
// graph): every global operand of the graph (its X_L rows, the W1 rows a warp
// owns, b1, W2, b2, y) is requested up front, so the whole head costs about one
// memory round trip plus shared-memory reductions. Warp w owns node rows
// n0+w, n0+w+8, ... (kept in registers for the ReLU mask of the backward) and W1
// rows w, w+8, ... (reused by the backward). Reductions are fixed-order
// (per-warp in row order, then warps 0..7; xor-shuffle trees), so deterministic.
template <bool FWD, bool BWD, int CH, int RW>
__global__ void __launch_bounds__(256) k_head_fast(const uint8_t *__restrict__ blob, const float *__restrict__ XL,
                                                   const float *__restrict__ W1, const float *__restrict__ b1,
                                                   const float *__restrict__ W2, const float *__restrict__ b2,
                                                   float *__restrict__ G, float *__restrict__ hpre,
                                                   float *__restrict__ yhat, float *__restrict__ sqerr,
                                                   float *__restrict__ dy, float *__restrict__ dhid,
                                                   float *__restrict__ dZL, const int *__restrict__ pos) {
  constexpr int H = 128 * CH, Hf = 8 * RW, RMAX = 8;
  __shared__ float4 red[8][H / 4];
  __shared__ float Gs[H], hs[Hf], dh[Hf];
  __shared__ float s_yh;
  pdl_enter();
  const BatchView b = load_batch(blob);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this warp's W1 rows (lane owns channels [4*(lane + 32*q), +4) for q < CH)
  float4 w1r[RW][CH];
#pragma unroll
  for (int k = 0; k < RW; ++k)
#pragma unroll
    for (int q = 0; q < CH; ++q) w1r[k][q] = ldg4(W1 + (size_t)(warp + 8 * k) * H + 4 * (lane + 32 * q));
  for (int g = blockIdx.x; g < b.B; g += gridDim.x) {
    const int n0 = b.gp[g], n1 = b.gp[g + 1], n = n1 - n0;
    const float ng = (float)n;
    const bool regs = n <= 8 * RMAX;
    float4 xr[RMAX][CH];
    if (regs) {
#pragma unroll
      for (int j = 0; j < RMAX; ++j) {
        const int i = n0 + warp + 8 * j;
#pragma unroll
        for (int q = 0; q < CH; ++q)
          xr[j][q] = i < n1 ? ldg4(XL + (size_t)i * H + 4 * (lane + 32 * q)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float yh;
    if (FWD) {
      // ---- mean pool
      float4 ps[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) ps[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (regs) {
#pragma unroll
        for (int j = 0; j < RMAX; ++j)
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            ps[q].x += xr[j][q].x; ps[q].y += xr[j][q].y; ps[q].z += xr[j][q].z; ps[q].w += xr[j][q].w;
          }
      } else {
        for (int i = n0 + warp; i < n1; i += 8)
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const float4 v = ldg4(XL + (size_t)i * H + 4 * (lane + 32 * q));
            ps[q].x += v.x; ps[q].y += v.y; ps[q].z += v.z; ps[q].w += v.w;
          }
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) red[warp][lane + 32 * q] = ps[q];
      __syncthreads();
      if (threadIdx.x < H) {
        const float *rf = reinterpret_cast<const float *>(red);
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += rf[w * H + threadIdx.x];
        const float v = s / ng;
        Gs[threadIdx.x] = v;
        G[(size_t)g * H + threadIdx.x] = v;
      }
      __syncthreads();
      // ---- hidden pre-activations: warp-owned W1 rows . G
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const float4 gv = reinterpret_cast<const float4 *>(Gs)[lane + 32 * q];
          acc = fmaf(w1r[k][q].x, gv.x, acc);
          acc = fmaf(w1r[k][q].y, gv.y, acc);
          acc = fmaf(w1r[k][q].z, gv.z, acc);
          acc = fmaf(w1r[k][q].w, gv.w, acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
          const int r = warp + 8 * k;
          acc += b1[r];
          hs[r] = acc;
          hpre[(size_t)g * Hf + r] = acc;
        }
      }
      __syncthreads();
      // ---- output + squared error (warp 0)
      if (warp == 0) {
        float part = 0.f;
        for (int r = lane; r < Hf; r += 32) part = fmaf(W2[r], fmaxf(hs[r], 0.f), part);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) {
          const float y = part + b2[0];
          s_yh = y;
          yhat[g] = y;
          const float e = y - b.y[g];
          sqerr[g] = e * e;
        }
      }
      __syncthreads();
      yh = s_yh;
    } else {
      for (int r = threadIdx.x; r < Hf; r += blockDim.x) hs[r] = hpre[(size_t)g * Hf + r];
      yh = yhat[g];
      __syncthreads();
    }
    if (BWD) {
      const float d = 2.0f * (yh - b.y[g]) / (float)b.B;
      if (threadIdx.x == 0) dy[g] = d;
      for (int r = threadIdx.x; r < Hf; r += blockDim.x) {
        const float v = hs[r] > 0.f ? d * W2[r] : 0.f;
        dh[r] = v;
        dhid[(size_t)g * Hf + r] = v;
      }
      __syncthreads();
      // ---- dG = W1^T dh / n: warp partials over its rows, then warps 0..7
      float4 acc[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const float dv = dh[warp + 8 * k];
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          acc[q].x = fmaf(w1r[k][q].x, dv, acc[q].x);
          acc[q].y = fmaf(w1r[k][q].y, dv, acc[q].y);
          acc[q].z = fmaf(w1r[k][q].z, dv, acc[q].z);
          acc[q].w = fmaf(w1r[k][q].w, dv, acc[q].w);
        }
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) red[warp][lane + 32 * q] = acc[q];
      __syncthreads();
      if (threadIdx.x < H) {
        const float *rf = reinterpret_cast<const float *>(red);
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += rf[w * H + threadIdx.x];
        Gs[threadIdx.x] = s / ng;
      }
      __syncthreads();
      // ---- dZ_L rows = [X_L > 0] * dG (degree-sorted rows when pos is given)
      for (int j = 0; j < (n + 7) / 8; ++j) {
        const int i = n0 + warp + 8 * j;
        if (i >= n1) break;
        const size_t od = (size_t)(pos ? pos[i] : i) * H;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int cc = 4 * (lane + 32 * q);
          float4 x;
          if (regs) {
#pragma unroll
            for (int jj = 0; jj < RMAX; ++jj)
              if (jj == j) x = xr[jj][q];
          } else {
            x = ldg4(XL + (size_t)i * H + cc);
          }
          const float4 gv = reinterpret_cast<const float4 *>(Gs)[cc / 4];
          const float4 v = make_float4(x.x > 0.f ? gv.x : 0.f, x.y > 0.f ? gv.y : 0.f, x.z > 0.f ? gv.z : 0.f,
                                       x.w > 0.f ? gv.w : 0.f);
          *reinterpret_cast<float4 *>(dZL + od + cc) = v;
        }
      }
    }
    __syncthreads();
  }
}

// loss = (1/B) sum_g sqerr_g [+ w (1/N) sum_i sqn_i: node-level head, R-node-head]
__global__ void __launch_bounds__(256) k_loss(const uint8_t *__restrict__ blob, const float *__restrict__ sqerr,
                                              float *__restrict__ loss, const float *__restrict__ sqn, float w) {
  pdl_enter();
  __shared__ float red[256];
  const BatchView b = load_batch(blob);
  float part = 0.f;
  for (int g = threadIdx.x; g < b.B; g += blockDim.x) part += sqerr[g];
  const float s = block_sum_256(part, red);
  float sn = 0.f;
  if (sqn) {
    float pn = 0.f;
    for (int i = threadIdx.x; i < b.N; i += blockDim.x) pn += sqn[i];
    sn = block_sum_256(pn, red);
  }
  if (threadIdx.x == 0) *loss = s / (float)b.B + (sqn ? w * (sn / (float)b.N) : 0.f);
}

// ------------------------------------------------------------------ node-level head
// Model variant (HG_FLAG_NODE_HEAD; reading R-node-head). Per node i:
//   hn_pre = W1n x_i + b1n [Hf],  yn_i = W2n ReLU(hn_pre) + b2n,  sqn_i = (yn_i - y_node,i)^2;
// training (BWD): dyn_i = 2 w (yn_i - y_node,i) / N, dhn = dyn_i W2n * [hn_pre > 0] (-> dhn_out for
// the W1n Gram), dZ_L[pos[i]] += (W1n^T dhn) * [x_i > 0] (after the graph head wrote dZ_L).
// One warp per group of NB nodes (their x rows and dhn staged in shared memory); lanes over
// output rows in chunks of 128 (forward) and over input channels (backward); W1n through L1.
constexpr int kNHNodes = 4;
__global__ void __launch_bounds__(256) k_node_head(const uint8_t *__restrict__ blob, const float *__restrict__ XL,
                                                   const float *__restrict__ W1, const float *__restrict__ b1,
                                                   const float *__restrict__ W2, const float *__restrict__ b2, float w,
                                                   int H, int Hf, float *__restrict__ hpre, float *__restrict__ yn,
                                                   float *__restrict__ sqn, float *__restrict__ dyn,
                                                   float *__restrict__ dhn, float *__restrict__ dZL,
                                                   const int *__restrict__ pos, int bwd) {
  constexpr int NB = kNHNodes;
  extern __shared__ float nsm[];  // per warp: xs[NB][H], dh[NB][Hf]
  pdl_enter();
  const BatchView b = load_batch(blob);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  float *xs = nsm + (size_t)warp * NB * (H + Hf), *dh = xs + NB * H;
  const float invN = 1.0f / (float)b.N;
  for (int i0 = (blockIdx.x * wpb + warp) * NB; i0 < b.N; i0 += gridDim.x * wpb * NB) {
    const int nn = min(NB, b.N - i0);
    for (int e = lane; e < NB * H / 4; e += 32) {  // the group's x rows (zeros past the batch)
      const int n = e / (H / 4), c = 4 * (e - n * (H / 4));
      reinterpret_cast<float4 *>(xs)[e] = n < nn ? ldg4(XL + (size_t)(i0 + n) * H + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    float ydot[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) ydot[n] = 0.f;
    for (int r0 = 0; r0 < Hf; r0 += 128) {  // 4 rows per lane: r = r0 + lane + 32 k
      float acc[NB][4];
#pragma unroll
      for (int n = 0; n < NB; ++n)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[n][k] = 0.f;
      for (int c = 0; c < H; c += 4) {
        float4 wv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = r0 + lane + 32 * k;
          wv[k] = r < Hf ? ldg4(W1 + (size_t)r * H + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const float4 xv = *reinterpret_cast<const float4 *>(xs + n * H + c);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc[n][k] = fmaf(wv[k].x, xv.x, acc[n][k]);
            acc[n][k] = fmaf(wv[k].y, xv.y, acc[n][k]);
            acc[n][k] = fmaf(wv[k].z, xv.z, acc[n][k]);
            acc[n][k] = fmaf(wv[k].w, xv.w, acc[n][k]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = r0 + lane + 32 * k;
        if (r >= Hf) continue;
        const float bb = b1[r], w2 = W2[r];
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const float hp = acc[n][k] + bb;
          if (n < nn) hpre[(size_t)(i0 + n) * Hf + r] = hp;
          ydot[n] = fmaf(w2, fmaxf(hp, 0.f), ydot[n]);
        }
      }
    }
    float dy[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      float v = ydot[n];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // fixed tree
      const float y = v + b2[0];
      const float e = n < nn ? y - b.y_node[i0 + n] : 0.f;
      dy[n] = 2.0f * w * e * invN;
      if (lane == 0 && n < nn) {
        yn[i0 + n] = y;
        sqn[i0 + n] = e * e;
        if (bwd) dyn[i0 + n] = dy[n];
      }
    }
    if (bwd) {
      __syncwarp();  // (hpre rows of the group written by this warp)
      for (int r = lane; r < Hf; r += 32) {
        const float w2 = W2[r];
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const float d = n < nn && hpre[(size_t)(i0 + n) * Hf + r] > 0.f ? dy[n] * w2 : 0.f;
          dh[n * Hf + r] = d;
          if (n < nn) dhn[(size_t)(i0 + n) * Hf + r] = d;
        }
      }
      __syncwarp();
      for (int c = 4 * lane; c < H; c += 128) {  // dX = W1n^T dhn, 4 channels per lane
        float4 dx[NB];
#pragma unroll
        for (int n = 0; n < NB; ++n) dx[n] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < Hf; ++r) {
          const float4 wv = ldg4(W1 + (size_t)r * H + c);
#pragma unroll
          for (int n = 0; n < NB; ++n) {
            const float d = dh[n * Hf + r];
            dx[n].x = fmaf(wv.x, d, dx[n].x); dx[n].y = fmaf(wv.y, d, dx[n].y);
            dx[n].z = fmaf(wv.z, d, dx[n].z); dx[n].w = fmaf(wv.w, d, dx[n].w);
          }
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          if (n >= nn) continue;
          const float4 x = *reinterpret_cast<const float4 *>(xs + n * H + c);
          float4 *o = reinterpret_cast<float4 *>(dZL + (size_t)pos[i0 + n] * H + c);
          float4 z = *o;
          z.x += x.x > 0.f ? dx[n].x : 0.f; z.y += x.y > 0.f ? dx[n].y : 0.f;
          z.z += x.z > 0.f ? dx[n].z : 0.f; z.w += x.w > 0.f ? dx[n].w : 0.f;
          *o = z;
        }
      }
    }
    __syncwarp();
  }
}

// dW2n[r] = sum_i dyn_i ReLU(hpre_i[r]), db2n = sum_i dyn_i: per-block partials over fixed 64-node
// chunks (thread per r), then k_reduce_rows32-style fixed-order sums (tcmn.cu launch_reduce_cols)
constexpr int kNHChunk = 64;
__global__ void __launch_bounds__(256) k_node_head_w2(const uint8_t *__restrict__ blob, const float *__restrict__ hpre,
                                                      const float *__restrict__ dyn, int Hf, int nchunks,
                                                      float *__restrict__ part) {
  pdl_enter();
  const int N = batch_N(blob);
  const int stride = Hf + 4;  // per chunk: Hf weights, db2n, 3 pad (float4 rows)
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int i0 = ch * kNHChunk, i1 = min(N, i0 + kNHChunk);
    for (int r = threadIdx.x; r < stride; r += blockDim.x) {
      float s = 0.f;
      if (r < Hf) {
        for (int i = i0; i < i1; ++i) s = fmaf(dyn[i], fmaxf(hpre[(size_t)i * Hf + r], 0.f), s);
      } else if (r == Hf) {
        for (int i = i0; i < i1; ++i) s += dyn[i];
      }
      part[(size_t)ch * stride + r] = s;
    }
  }
}

template <bool FWD, bool BWD>
static void head_launch(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                        const float *b1, const float *W2, const float *b2, float *G, float *hpre, float *yhat,
                        float *sqerr, float *dy, float *dhid, float *dZL, const int *pos = nullptr) {
  const size_t base = sizeof(float) * (c.H + 2 * c.Hf + 256);
  const size_t w1 = sizeof(float) * (size_t)c.Hf * c.H;
  const int in_smem = base + w1 <= 200 * 1024 ? 1 : 0;  // attribute set once by head_configure
  const size_t smem = base + (in_smem ? w1 : 0);
  if (c.H == 128 && (c.Hf == 128 || c.Hf == 64)) {  // latency-optimised kernel
    // (two blocks per SM: the graphs of one block are processed serially, so at config D's 512
    // graphs one block per SM put ~3.5 graph latencies on the step's critical path)
    const int grid = std::min(c.maxB, 2 * kSMs);
    if (c.Hf == 128)
      launch_ex(k_head_fast<FWD, BWD, 1, 16>, grid, 256, 0, st, blob, XL, W1, b1, W2, b2, G, hpre, yhat, sqerr, dy,
                dhid, dZL, pos);
    else
      launch_ex(k_head_fast<FWD, BWD, 1, 8>, grid, 256, 0, st, blob, XL, W1, b1, W2, b2, G, hpre, yhat, sqerr, dy,
                dhid, dZL, pos);
    return;
  }
  launch_ex(k_head<FWD, BWD>, std::min(c.maxB, kSMs), 256, smem, st, blob, XL, W1, b1, W2, b2, G, hpre, yhat, sqerr, dy,
            dhid, dZL, c.H, c.Hf, in_smem, pos);
}

size_t node_head_smem(const Caps &c);
void head_configure(const Caps &c) {  // outside graph capture: opt into large dynamic smem
  cudaFuncSetAttribute(k_node_head, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)node_head_smem(c));
  const size_t base = sizeof(float) * (c.H + 2 * c.Hf + 256);
  const size_t w1 = sizeof(float) * (size_t)c.Hf * c.H;
  const int v = (int)(base + (base + w1 <= 200 * 1024 ? w1 : 0));
  cudaFuncSetAttribute(k_head<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
  cudaFuncSetAttribute(k_head<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
  cudaFuncSetAttribute(k_head<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
}

void launch_head_fwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                     const float *b1, const float *W2, const float *b2, float *G, float *hpre, float *yhat,
                     float *sqerr, float *loss, const float *sqn, float w) {
  head_launch<true, false>(st, c, blob, XL, W1, b1, W2, b2, G, hpre, yhat, sqerr, nullptr, nullptr, nullptr);
  counted();
  launch_ex(k_loss, 1, 256, 0, st, blob, sqerr, loss, sqn, w);
  counted();
}

size_t node_head_smem(const Caps &c) { return sizeof(float) * 8 * kNHNodes * (c.H + c.Hf); }
int node_head_chunks(const Caps &c) { return (c.maxN + kNHChunk - 1) / kNHChunk; }
size_t node_head_partial_floats(const Caps &c) { return (size_t)node_head_chunks(c) * (c.Hf + 4); }

void launch_node_head(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                      const float *b1, const float *W2, const float *b2, float w, float *hpre, float *yn, float *sqn,
                      float *dyn, float *dhn, float *dZL, const int *pos, bool bwd) {
  const int groups = cdiv(c.maxN, kNHNodes);
  launch_ex(k_node_head, std::max(1, std::min(cdiv(groups, 8), kSMs * 4)), 256, node_head_smem(c), st, blob, XL, W1,
            b1, W2, b2, w, c.H, c.Hf, hpre, yn, sqn, dyn, dhn, dZL, pos, bwd ? 1 : 0);
  counted();
}

void launch_node_head_w2(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *hpre, const float *dyn,
                         float *part) {
  launch_ex(k_node_head_w2, std::min(node_head_chunks(c), kSMs * 4), 256, 0, st, blob, hpre, dyn, c.Hf,
            node_head_chunks(c), part);
  counted();
}

void launch_head_fused(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                       const float *b1, const float *W2, const float *b2, float *G, float *hpre, float *yhat,
                       float *sqerr, float *loss, float *dy, float *dhid, float *dZL, const int *pos) {
  head_launch<true, true>(st, c, blob, XL, W1, b1, W2, b2, G, hpre, yhat, sqerr, dy, dhid, dZL, pos);
  counted();
}

void launch_loss(cudaStream_t st, const uint8_t *blob, const float *sqerr, float *loss, const float *sqn, float w) {
  launch_ex(k_loss, 1, 256, 0, st, blob, sqerr, loss, sqn, w);
  counted();
}

// the loss value into host-mapped pinned memory by a one-thread kernel: a DMA read-back queued
// behind the next batch's H2D copy on the copy engine (measured ~23 us per step in the
// end-to-end loop), a store from the SMs is not
__global__ void k_loss_to_host(const float *__restrict__ loss, float *__restrict__ host) {
  pdl_enter();
  *reinterpret_cast<volatile float *>(host) = loss[0];
  __threadfence_system();
}
void launch_loss_to_host(cudaStream_t st, const float *loss, float *host_mapped) {
  launch_ex(k_loss_to_host, 1, 32, 0, st, loss, host_mapped);
  counted();
}

// evaluation sums: acc[0] += sum (yhat-y)^2, acc[1] += sum |yhat-y|,
// acc[2] += B, in fp64 with a fixed-order block tree (deterministic)
__global__ void __launch_bounds__(256) k_eval_accum(const uint8_t *__restrict__ blob, const float *__restrict__ yhat,
                                                    double *__restrict__ acc) {
  pdl_enter();
  __shared__ double rs[256], ra[256];
  const BatchView b = load_batch(blob);
  double s = 0.0, a = 0.0;
  for (int g = threadIdx.x; g < b.B; g += blockDim.x) {
    const double e = (double)yhat[g] - (double)b.y[g];
    s += e * e;
    a += fabs(e);
  }
  rs[threadIdx.x] = s;
  ra[threadIdx.x] = a;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      rs[threadIdx.x] += rs[threadIdx.x + w];
      ra[threadIdx.x] += ra[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    acc[0] += rs[0];
    acc[1] += ra[0];
    acc[2] += (double)b.B;
  }
}

void launch_eval_accum(cudaStream_t st, const uint8_t *blob, const float *yhat, double *acc) {
  launch_ex(k_eval_accum, 1, 256, 0, st, blob, yhat, acc);
  counted();
}

// head parameter gradients: thread per output element, fixed order over graphs
__global__ void k_head_grads(const uint8_t *__restrict__ blob, const float *__restrict__ G,
                             const float *__restrict__ hpre, const float *__restrict__ dy,
                             const float *__restrict__ dhid, float *__restrict__ gW1, float *__restrict__ gb1,
                             float *__restrict__ gW2, float *__restrict__ gb2, int H, int Hf) {
  pdl_enter();
  const int B = reinterpret_cast<const int *>(blob)[0];
  const int nW1 = Hf * H;
  const int total = nW1 + 2 * Hf + 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    float s = 0.f;
    if (e < nW1) {
      const int r = e / H, c = e - r * H;
      for (int g = 0; g < B; ++g) s = fmaf(dhid[(size_t)g * Hf + r], G[(size_t)g * H + c], s);
      gW1[e] = s;
    } else if (e < nW1 + Hf) {
      const int r = e - nW1;
      for (int g = 0; g < B; ++g) s += dhid[(size_t)g * Hf + r];
      gb1[r] = s;
    } else if (e < nW1 + 2 * Hf) {
      const int r = e - nW1 - Hf;
      for (int g = 0; g < B; ++g) s = fmaf(dy[g], fmaxf(hpre[(size_t)g * Hf + r], 0.f), s);
      gW2[r] = s;
    } else {
      for (int g = 0; g < B; ++g) s += dy[g];
      gb2[0] = s;
    }
  }
}

// H = 128 form: block b < Hf/8 owns W1 rows [8b, 8b + 8) (warp w: row 8b + w, lane: 4 columns),
// the graphs' G rows and dhid entries staged through shared memory in chunks of 32 (the next
// chunk's loads in flight while this one is summed); every output keeps the fixed ascending
// order over graphs of k_head_grads, so the two kernels agree bitwise. The last block does the
// b1 / W2 / b2 gradients. (Thread-per-element with all B graphs from L2 was ~58 us at config D.)
__global__ void __launch_bounds__(256) k_head_grads128(const uint8_t *__restrict__ blob, const float *__restrict__ G,
                                                      const float *__restrict__ hpre, const float *__restrict__ dy,
                                                      const float *__restrict__ dhid, float *__restrict__ gW1,
                                                      float *__restrict__ gb1, float *__restrict__ gW2,
                                                      float *__restrict__ gb2, int Hf) {
  constexpr int H = 128, CG = 32;
  __shared__ float4 sG[2][CG][H / 4];
  __shared__ float sd[2][CG][8];
  pdl_enter();
  const int B = reinterpret_cast<const int *>(blob)[0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((int)blockIdx.x == Hf / 8) {  // b1, W2, b2
    for (int e = threadIdx.x; e < 2 * Hf + 1; e += blockDim.x) {
      float s = 0.f;
      if (e < Hf) {
        for (int g = 0; g < B; ++g) s += dhid[(size_t)g * Hf + e];
        gb1[e] = s;
      } else if (e < 2 * Hf) {
        const int r = e - Hf;
        for (int g = 0; g < B; ++g) s = fmaf(dy[g], fmaxf(hpre[(size_t)g * Hf + r], 0.f), s);
        gW2[r] = s;
      } else {
        for (int g = 0; g < B; ++g) s += dy[g];
        gb2[0] = s;
      }
    }
    return;
  }
  const int r0 = blockIdx.x * 8;
  float4 pg[4];
  float pd = 0.f;
  auto fetch = [&](int g0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // 32 graphs x 32 float4 = 1024 float4, 4 per thread
      const int t = threadIdx.x + 256 * u, gg = t >> 5, q = t & 31;
      pg[u] = g0 + gg < B ? ldg4(G + (size_t)(g0 + gg) * H + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int gg = threadIdx.x >> 3, rr = threadIdx.x & 7;
    pd = g0 + gg < B ? dhid[(size_t)(g0 + gg) * Hf + r0 + rr] : 0.f;
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = threadIdx.x + 256 * u;
      sG[buf][t >> 5][t & 31] = pg[u];
    }
    sd[buf][threadIdx.x >> 3][threadIdx.x & 7] = pd;
  };
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  fetch(0);
  store(0);
  __syncthreads();
  for (int g0 = 0, buf = 0; g0 < B; g0 += CG, buf ^= 1) {
    if (g0 + CG < B) fetch(g0 + CG);
    const int n = min(CG, B - g0);
    for (int gg = 0; gg < n; ++gg) {
      const float d = sd[buf][gg][warp];
      const float4 gv = sG[buf][gg][lane];
      s.x = fmaf(d, gv.x, s.x);
      s.y = fmaf(d, gv.y, s.y);
      s.z = fmaf(d, gv.z, s.z);
      s.w = fmaf(d, gv.w, s.w);
    }
    if (g0 + CG < B) store(buf ^ 1);
    __syncthreads();
  }
  *reinterpret_cast<float4 *>(gW1 + (size_t)(r0 + warp) * H + 4 * lane) = s;
}

void launch_head_bwd(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *XL, const float *W1,
                     const float *W2, const float *G, const float *hpre, const float *yhat, float *dy,
                     float *dhid, float *dZL, float *gW1, float *gb1, float *gW2, float *gb2, bool head_done,
                     const int *pos, bool with_grads) {
  if (!head_done) {
    head_launch<false, true>(st, c, blob, XL, W1, nullptr, W2, nullptr, nullptr, const_cast<float *>(hpre),
                             const_cast<float *>(yhat), nullptr, dy, dhid, dZL, pos);
    counted();
  }
  if (with_grads) launch_head_grads(st, c, blob, G, hpre, dy, dhid, gW1, gb1, gW2, gb2);
}

void launch_head_grads(cudaStream_t st, const Caps &c, const uint8_t *blob, const float *G, const float *hpre,
                       const float *dy, const float *dhid, float *gW1, float *gb1, float *gW2, float *gb2) {
  if (c.H == 128 && c.Hf % 8 == 0) {
    launch_ex(k_head_grads128, c.Hf / 8 + 1, 256, 0, st, blob, G, hpre, dy, dhid, gW1, gb1, gW2, gb2, c.Hf);
    counted();
    return;
  }
  const int total = c.Hf * c.H + 2 * c.Hf + 1;
  launch_ex(k_head_grads, std::min(cdiv(total, 256), kSMs * 4), 256, 0, st, blob, G, hpre, dy, dhid, gW1, gb1, gW2,
            gb2, c.H, c.Hf);
  counted();
}

// ------------------------------------------------------------------ K10 AdamW
// theta <- theta (1 - lr wd); m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2;
// theta <- theta - (lr/bc1) m / (sqrt(v)/sqrt(bc2) + eps)

__global__ void __launch_bounds__(256) k_adamw(float4 *__restrict__ p, const float4 *__restrict__ g,
                                               float4 *__restrict__ m, float4 *__restrict__ v, int64_t n4,
                                               const AdamDev *ad, float lr, float beta1,
                                               float beta2, float eps, float wd, int advance) {
  pdl_enter();
  // bias corrections of step t = ad->step + 1 (fp64 as the oracle), once per block
  __shared__ float s_ss, s_ib;
  const int64_t t = ad->step + 1;
  if (threadIdx.x == 0) {
    const double bc1 = 1.0 - pow((double)beta1, (double)t);
    const double bc2 = 1.0 - pow((double)beta2, (double)t);
    s_ss = (float)((double)lr / bc1);
    s_ib = (float)(1.0 / sqrt(bc2));
  }
  __syncthreads();
  const float ss = s_ss, ib = s_ib;
  const float decay = 1.0f - lr * wd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 P = p[i], Gv = g[i], Mv = m[i], Vv = v[i];
    float *pp = &P.x, *gg = &Gv.x, *mm = &Mv.x, *vv = &Vv.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float gc = gg[c];
      mm[c] = beta1 * mm[c] + (1.0f - beta1) * gc;
      vv[c] = beta2 * vv[c] + (1.0f - beta2) * gc * gc;
      const float den = sqrtf(vv[c]) * ib + eps;
      pp[c] = pp[c] * decay - ss * mm[c] / den;
    }
    p[i] = P; m[i] = Mv; v[i] = Vv;
  }
  // every block has read ad->step above; the last block to finish advances it
  // (only in the launch that updates the last parameter range of the step)
  if (!advance) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    AdamDev *w = const_cast<AdamDev *>(ad);
    if (atomicAdd(&w->ticket, 1) == (int)gridDim.x - 1) {
      w->step = t;
      w->ticket = 0;
    }
  }
}

void launch_adamw(cudaStream_t st, float *p, const float *g, float *m, float *v, int64_t n, AdamDev *ad,
                  float lr, float beta1, float beta2, float eps, float wd, bool advance, int max_blocks) {
  const int64_t n4 = n / 4;
  const int cap = max_blocks > 0 ? max_blocks : kSMs * 8;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, cap));
  launch_ex(k_adamw, blocks, 256, 0, st, reinterpret_cast<float4 *>(p), reinterpret_cast<const float4 *>(g),
            reinterpret_cast<float4 *>(m), reinterpret_cast<float4 *>(v), n4, ad, lr, beta1, beta2, eps, wd,
            advance ? 1 : 0);
  counted();
}

int64_t launches_so_far() { return g_launches.load(); }

}  // namespace hg
