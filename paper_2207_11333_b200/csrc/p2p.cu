// p2p.cu — the DDP gradient average fused with the optimizer over NVLink peer memory
// (SURVEY §8(f) row 4 "ReduceScatter -> sharded fused AdamW -> AllGather"
// "gradients are aggregated ... after each backward pass"). One process per GPU; every rank
// maps every other rank's workspace (CUDA IPC, hg_p2p_open). Per step:
//   k_p2p_signal  this rank's gradients are complete: ready[rank] = epoch in every rank's flags
//   k_p2p_wait    wait until every rank's ready flag reached this step's epoch
//   k_p2p_adamw   for the owned shard (1/W of the flat arena) sum the W gradient copies in
//                 rank order over NVLink (deterministic, each shard reduced by exactly one
//                 rank, so all ranks agree bitwise), divide by W, apply AdamW (moments are
//                 sharded: rank r keeps m, v of shard r only) and store the new parameters
//                 into every rank's arena (peer stores); the last block advances the step
//                 counter and raises done[rank] everywhere
//   k_p2p_wait    wait until every rank's shard is written (and so no peer still reads this
//                 rank's gradients) before the next step may touch parameters or gradients.
// No float atomics; flags are monotonic epochs (no resets).
// Fail-stop: every wait is bounded by the ctx's timeout (hg_set_timeout);
// a rank whose peer stops answering records HG_P2P_TIMEOUT in its flag block and traps, so
// the step fails with a CUDA error (sticky in the ctx) instead of hanging the job.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "kernels.h"

namespace hg {
extern std::atomic<int64_t> g_launches;

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// spin until *p >= e (epoch order, wrap-safe); past the deadline: record the timeout and trap
__device__ __forceinline__ void spin_until_geq(const unsigned *p, unsigned e, unsigned long long timeout_ns,
                                               P2PDev *me) {
  const unsigned long long t0 = timeout_ns ? global_ns() : 0ull;
  while ((int)(ld_acquire_sys(p) - e) < 0) {
    __nanosleep(64);
    if (timeout_ns && global_ns() - t0 > timeout_ns) {
      me->error = kP2PTimeout;
      __threadfence_system();
      __trap();
    }
  }
}

// this rank's gradients are complete: ready[rank] = epoch on every rank
__global__ void k_p2p_signal(P2PArgs a) {
  pdl_enter();
  __shared__ unsigned e;
  if (threadIdx.x == 0) {
    e = a.dev[a.rank]->epoch + 1u;
    a.dev[a.rank]->epoch = e;
    __threadfence_system();  // this rank's gradients (earlier kernels) before the flags
  }
  __syncthreads();
  if ((int)threadIdx.x < a.world) st_release_sys(&a.dev[threadIdx.x]->ready[a.rank], e);
}

// one warp waits until every rank's ready (which = 0) or done (which = 1) flag reached this
// step's epoch (a single small CTA spins, so no SM is held by a waiting grid)
__global__ void k_p2p_wait(P2PArgs a, int which) {
  pdl_enter();
  P2PDev *me = a.dev[a.rank];
  const unsigned e = *reinterpret_cast<volatile unsigned *>(&me->epoch);
  if ((int)threadIdx.x < a.world)
    spin_until_geq(which == 0 ? &me->ready[threadIdx.x] : &me->done[threadIdx.x], e, a.timeout_ns, me);
}

// this rank's 1/W shard of the flat arena (float4 range [s0, s1) of [0, n4))
__device__ __forceinline__ void shard_of(int64_t n4, int rank, int world, int64_t &s0, int64_t &s1) {
  s0 = n4 * rank / world;
  s1 = n4 * (rank + 1) / world;
}

__global__ void __launch_bounds__(256) k_p2p_adamw(P2PArgs a) {
  pdl_enter();
  __shared__ float s_ss, s_ib;
  P2PDev *me = a.dev[a.rank];
  const int64_t t = a.ad->step + 1;
  if (threadIdx.x == 0) {  // bias corrections of step t (fp64, as k_adamw and the oracle)
    const double bc1 = 1.0 - pow((double)a.beta1, (double)t);
    const double bc2 = 1.0 - pow((double)a.beta2, (double)t);
    s_ss = (float)((double)a.lr / bc1);
    s_ib = (float)(1.0 / sqrt(bc2));
  }
  __syncthreads();
  const float ss = s_ss, ib = s_ib, decay = 1.0f - a.lr * a.wd, invw = 1.0f / (float)a.world;
  const float b1 = a.beta1, b2 = a.beta2, eps = a.eps;
  int64_t s0, s1;
  shard_of(a.n4, a.rank, a.world, s0, s1);
  float4 *p4 = reinterpret_cast<float4 *>(a.params[a.rank]);
  float4 *m4 = reinterpret_cast<float4 *>(a.m), *v4 = reinterpret_cast<float4 *>(a.v);
  for (int64_t i = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s1; i += (int64_t)gridDim.x * blockDim.x) {
    float4 g = __ldcg(reinterpret_cast<const float4 *>(a.grads[0]) + i);  // peer data: bypass L1
    for (int q = 1; q < a.world; ++q) {
      const float4 h = __ldcg(reinterpret_cast<const float4 *>(a.grads[q]) + i);
      g.x += h.x; g.y += h.y; g.z += h.z; g.w += h.w;
    }
    float4 P = p4[i], M = m4[i], V = v4[i];
    float *pp = &P.x, *mm = &M.x, *vv = &V.x;
    const float gg[4] = {g.x * invw, g.y * invw, g.z * invw, g.w * invw};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      mm[c] = b1 * mm[c] + (1.0f - b1) * gg[c];
      vv[c] = b2 * vv[c] + (1.0f - b2) * gg[c] * gg[c];
      const float den = sqrtf(vv[c]) * ib + eps;
      pp[c] = pp[c] * decay - ss * mm[c] / den;
    }
    m4[i] = M;
    v4[i] = V;
    for (int q = 0; q < a.world; ++q) reinterpret_cast<float4 *>(a.params[q])[i] = P;  // all-gather
  }
  // completion: the last block advances the step and raises done[rank] on every rank
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&me->ticket, 1u) == gridDim.x - 1) {
      me->ticket = 0;
      a.ad->step = t;
      __threadfence_system();
      const unsigned e = *reinterpret_cast<volatile unsigned *>(&me->epoch);
      for (int q = 0; q < a.world; ++q) st_release_sys(&a.dev[q]->done[a.rank], e);
    }
  }
}

// after p2p steps rank q holds valid Adam moments on shard q only: copy every peer's shard
// of m and v into this rank's arrays (peer loads; the peers' last step is complete, which
// the step's final done-wait guarantees), so the moments are whole again
__global__ void __launch_bounds__(256) k_p2p_gather_moments(P2PArgs a) {
  pdl_enter();
  float4 *m4 = reinterpret_cast<float4 *>(a.m), *v4 = reinterpret_cast<float4 *>(a.v);
  for (int q = 0; q < a.world; ++q) {
    if (q == a.rank) continue;
    int64_t s0, s1;
    shard_of(a.n4, q, a.world, s0, s1);
    const float4 *pm = reinterpret_cast<const float4 *>(a.m_all[q]), *pv = reinterpret_cast<const float4 *>(a.v_all[q]);
    for (int64_t i = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s1; i += (int64_t)gridDim.x * blockDim.x) {
      m4[i] = __ldcg(pm + i);
      v4[i] = __ldcg(pv + i);
    }
  }
}

static int p2p_blocks(int64_t n4, int world) {
  const int64_t shard4 = (n4 + world - 1) / world;
  return (int)std::max<int64_t>(1, std::min<int64_t>((shard4 + 255) / 256, kSMs * 8));
}

void launch_p2p_exchange(cudaStream_t st, const P2PArgs &a) {
  launch_ex(k_p2p_signal, 1, 32, 0, st, a);
  launch_ex(k_p2p_wait, 1, 32, 0, st, a, 0);
  launch_ex(k_p2p_adamw, p2p_blocks(a.n4, a.world), 256, 0, st, a);
  launch_ex(k_p2p_wait, 1, 32, 0, st, a, 1);
  g_launches += 4;
}
void launch_p2p_exchange_emulated(cudaStream_t st, const P2PArgs &a) {
  launch_ex(k_p2p_signal, 1, 32, 0, st, a);
  launch_ex(k_p2p_adamw, p2p_blocks(a.n4, a.world), 256, 0, st, a);
  g_launches += 2;
}
void launch_p2p_gather_moments(cudaStream_t st, const P2PArgs &a) {
  launch_ex(k_p2p_gather_moments, p2p_blocks(a.n4, 1), 256, 0, st, a);
  g_launches += 1;
}

}  // namespace hg
