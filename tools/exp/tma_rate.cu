// Microbenchmark: TMA (cp.async.bulk.tensor 2D, SWIZZLE_128B, 128 x 32 fp32 boxes)
// ingest per SM. grid = G CTAs (1 per SM); each CTA streams `iters` stages of
// 4 boxes (64 KB) through an ST-deep ring from a buffer of `rows` x 512 fp32
// (L2-resident when small). Reports bytes/clk/SM and aggregate TB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2207_11333_b200/csrc/tc.cuh"
using namespace hg;

constexpr int BOX = 128 * 128;  // 16 KB
template <int ST, int NB>
__global__ void k(const __grid_constant__ CUtensorMap m, int iters, int rows, long long *clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = sm + ((1024u - (tc::smem_u32(sm) & 1023u)) & 1023u);
  __shared__ uint64_t full[ST];
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) tc::mbar_init(&full[i], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    const int tiles = rows / 128;
    for (int it = 0; it < iters + ST; ++it) {
      if (it >= ST) tc::mbar_wait(&full[(it - ST) % ST], ((it - ST) / ST) & 1);
      if (it < iters) {
        const int st = it % ST;
        tc::mbar_expect_tx(&full[st], NB * BOX);
        const int tile = (blockIdx.x * 7 + it) % tiles;
        for (int b = 0; b < NB; ++b)
          tc::tma_load_2d(s + (st * NB + b) * BOX, &m, (b % 16) * 32, tile * 128, &full[st]);
      }
    }
    clk[blockIdx.x] = clock64() - t0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
int main() {
  void *fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int rows = 8192;  // 8192 x 512 fp32 = 16 MB (L2 resident)
  float *buf; cudaMalloc(&buf, (size_t)rows * 512 * 4); cudaMemset(buf, 0, (size_t)rows * 512 * 4);
  CUtensorMap m;
  cuuint64_t dims[2] = {512, (cuuint64_t)rows}, str[1] = {512 * 4};
  cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long *clk; cudaMalloc(&clk, 148 * 8);
  const int iters = 400;
  auto run = [&](auto kern, int st, int nb, int G) {
    const int smem = st * nb * BOX + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<G, 32, smem>>>(m, 20, rows, clk);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<G, 32, smem>>>(m, iters, rows, clk);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h[148]; cudaMemcpy(h, clk, G * 8, cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < G; ++i) c += h[i]; c /= G;
    const double bytes = (double)iters * nb * BOX;
    printf("ST=%d boxes/stage=%d (in flight %3d KB) G=%3d: %.1f B/clk/SM, aggregate %.2f TB/s  %s\n", st, nb,
           st * nb * 16, G, bytes / c, bytes * G / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  for (int G : {1, 148}) {
    run(k<4, 3>, 4, 3, G);
    run(k<3, 4>, 3, 4, G);
    run(k<2, 6>, 2, 6, G);
    run(k<2, 4>, 2, 4, G);
    run(k<3, 3>, 3, 3, G);
    run(k<4, 2>, 4, 2, G);
    run(k<8, 1>, 8, 1, G);
  }
  return 0;
}
