// Microbenchmark: tcgen05.mma issue-to-completion rate (cycles per instruction)
// for kind::tf32 and kind::f16 (bf16), M=128, N in {64,128,256}, SS operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2207_11333_b200/csrc/tc.cuh"
using namespace hg;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool TF32>
__global__ void k(int reps, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = sm + ((1024u - (tc::smem_u32(sm) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float *>(s)[i] = 0.001f * (i & 7);
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&holder);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    const uint32_t a = tc::smem_u32(s), b = a + 16384;
    constexpr uint32_t id = TF32 ? tc::idesc_tf32(128, N) : idesc_bf16(128, N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t da = tc::desc_sw128(a + ks * 32), db = tc::desc_sw128(b + ks * 32);
        if (TF32) tc::mma_tf32(tmem, da, db, id, (r | ks) != 0);
        else mma_f16(tmem, da, db, id, (r | ks) != 0);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) { tc::fence_after_sync(); tc::tmem_dealloc<256>(tmem); }
}

template <int N, bool TF32>
void run(long long *d) {
  const int reps = 4096;
  cudaFuncSetAttribute(k<N, TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<N, TF32><<<148, 128, 70000>>>(reps, d);
  k<N, TF32><<<148, 128, 70000>>>(reps, d);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0; for (int i = 0; i < 148; ++i) m += h[i]; m /= 148;
  const double per = m / (reps * 4.0);
  const double macs = 128.0 * N * (TF32 ? 8 : 16);
  printf("%s N=%3d: %.1f cyc/mma  (%.0f MAC/clk/SM)  err=%s\n", TF32 ? "tf32" : "bf16", N, per, macs / per,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long *d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<64, true>(d); run<128, true>(d); run<256, true>(d);
  run<64, false>(d); run<128, false>(d); run<256, false>(d);
  return 0;
}
