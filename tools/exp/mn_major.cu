// Experiment: tcgen05.mma kind::tf32 with BOTH operands MN-major (SWIZZLE_128B),
// tiles loaded by TMA boxes {32 fp32 along MN, 32 rows along K}. Checks
// D[m][n] = sum_k X[k][m] Y[k][n] (M=128, N=BN, K=64) against a CPU reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mn_major mn_major.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include "../../paper_2207_11333_b200/csrc/tc.cuh"
using namespace hg;

constexpr int M = 128, BN = 64, K = 64, BK = 32;
struct Maps { CUtensorMap x, y; };

__global__ void k(const __grid_constant__ Maps mp, float *D, int lbo_mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = sm + ((1024u - (tc::smem_u32(sm) & 1023u)) & 1023u);
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t holder;
  if (threadIdx.x < 32) tc::tmem_alloc<64>(&holder);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = holder;
  constexpr int XB = M / 32, YB = BN / 32;          // MN blocks of 32 fp32
  constexpr int BLK = BK * 128;                      // one MN block: BK k-rows x 128 B
  if (threadIdx.x == 0) {
    for (int c = 0; c < K / BK; ++c) {
      uint8_t *sx = s, *sy = s + XB * BLK;
      tc::mbar_expect_tx(&bar, (XB + YB) * BLK);
      for (int b = 0; b < XB; ++b) tc::tma_load_2d(sx + b * BLK, &mp.x, b * 32, c * BK, &bar);
      for (int b = 0; b < YB; ++b) tc::tma_load_2d(sy + b * BLK, &mp.y, b * 32, c * BK, &bar);
      tc::mbar_wait(&bar, c & 1);
      tc::fence_after_sync();
      constexpr uint32_t id = tc::idesc_tf32(M, BN, true, true);
      for (int ks = 0; ks < BK / 8; ++ks) {
        // k-group ks (8 rows) starts 1024 B in; MN blocks BLK apart
        const uint32_t ax = tc::smem_u32(sx) + ks * 1024, ay = tc::smem_u32(sy) + ks * 1024;
        uint64_t dx, dy;
        // SWIZZLE_128B_BASE32B (layout type 1): atom = 4 k-rows x 128 B; k-groups 512 B apart
        auto d32 = [](uint32_t a, uint32_t lbo, uint32_t sbo) {
          return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
                 ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1u << 46) | ((uint64_t)1u << 61);
        };
        if (lbo_mode == 0) { dx = d32(ax, BLK, 512); dy = d32(ay, BLK, 512); }
        else { dx = d32(ax, 512, BLK); dy = d32(ay, 512, BLK); }
        tc::mma_tf32(tmem, dx, dy, id, (c | ks) != 0);
      }
      tc::mma_commit(&mbar);
      tc::mbar_wait(&mbar, c & 1);
    }
  }
  __syncthreads();
  tc::fence_after_sync();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, row = w * 32 + l;
  for (int q = 0; q < BN / 32; ++q) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + q * 32, v);
    for (int i = 0; i < 32; ++i) D[row * BN + q * 32 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) { tc::fence_after_sync(); tc::tmem_dealloc<64>(tmem); }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static CUtensorMap mk(float *p, int rows, int cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, BK}, es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", r);
  return m;
}

int main() {
  void *fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  std::vector<float> X(K * M), Y(K * BN), D(M * BN);
  for (int i = 0; i < K * M; ++i) X[i] = (float)((i * 37 % 101) - 50) / 64.f;   // exact in tf32
  for (int i = 0; i < K * BN; ++i) Y[i] = (float)((i * 53 % 97) - 48) / 32.f;
  float *dX, *dY, *dD;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dY, Y.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  Maps mp{mk(dX, K, M), mk(dY, K, BN)};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    k<<<1, 128, 100000>>>(mp, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < BN; ++n) {
        double r = 0;
        for (int kk = 0; kk < K; ++kk) r += (double)X[kk * M + m] * Y[kk * BN + n];
        maxerr = fmax(maxerr, fabs(r - D[m * BN + n]));
        maxref = fmax(maxref, fabs(r));
      }
    printf("mode %d (%s): err=%s maxerr=%g maxref=%g D[0]=%g D[1]=%g\n", mode, mode ? "lbo=512,sbo=BLK" : "lbo=BLK,sbo=512",
           cudaGetErrorString(e), maxerr, maxref, D[0], D[1]);
  }
  return 0;
}
