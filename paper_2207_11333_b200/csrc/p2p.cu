// p2p.cu — the DDP gradient average fused with the optimizer over NVLink peer memory
// (SURVEY §8(f) row 4 "ReduceScatter -> sharded fused AdamW -> AllGather"
// "gradients are aggregated ... after each backward pass"). One process per GPU; every rank
// maps every other rank's workspace (CUDA IPC, hg_p2p_open). Per step:
//   k_p2p_signal  this rank's gradients are complete: ready[rank] = epoch in every rank's flags
//   k_p2p_adamw   wait for every ready flag; for the owned shard (1/W of the flat arena) sum
//                 the W gradient copies in rank order over NVLink (deterministic, each shard
//                 reduced by exactly one rank, so all ranks agree bitwise), divide by W, apply
//                 AdamW (moments are sharded: rank r keeps m, v of shard r only) and store the
//                 new parameters into every rank's arena (peer stores); the last block
//                 advances the step counter and raises done[rank] everywhere
//   k_p2p_wait    wait until every rank's shard is written (and so no peer still reads this
//                 rank's gradients) before the next step may touch parameters or gradients.
// No float atomics; flags are monotonic epochs (no resets).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

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
__device__ __forceinline__ void spin_until_geq(const unsigned *p, unsigned e) {
  while ((int)(ld_acquire_sys(p) - e) < 0) __nanosleep(64);
}

// ready / done flags and the finished-block ticket of exchange part `part` (0 = conv0's
// parameters at the step's end, 1 = layers >= 1 and the head, during layer 0's backward)
__device__ __forceinline__ unsigned *flags(P2PDev *d, int part, int which) {
  return which == 0 ? d->ready[part] : d->done[part];
}

// this rank's gradients of `part` are complete: ready[part][rank] = epoch on every rank
// (bump: first exchange of the step, advances the epoch)
__global__ void k_p2p_signal(P2PArgs a, int part, int bump) {
  pdl_enter();
  __shared__ unsigned e;
  if (threadIdx.x == 0) {
    e = a.dev[a.rank]->epoch + (bump ? 1u : 0u);
    a.dev[a.rank]->epoch = e;
    __threadfence_system();  // this rank's gradients (earlier kernels) before the flags
  }
  __syncthreads();
  if ((int)threadIdx.x < a.world) st_release_sys(&flags(a.dev[threadIdx.x], part, 0)[a.rank], e);
}

// one warp waits until every rank's ready (which = 0) or done (which = 1) flag of `part`
// reached this step's epoch (a single small CTA spins, so no SM is held by a waiting grid)
__global__ void k_p2p_wait(P2PArgs a, int part, int which) {
  pdl_enter();
  P2PDev *me = a.dev[a.rank];
  const unsigned e = *reinterpret_cast<volatile unsigned *>(&me->epoch);
  if ((int)threadIdx.x < a.world) spin_until_geq(&flags(me, part, which)[threadIdx.x], e);
}

// float4 range [b4, e4) of the flat arena; this rank owns 1/W of it
__global__ void __launch_bounds__(256) k_p2p_adamw(P2PArgs a, int part, int64_t b4, int64_t e4, int advance) {
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
  const int64_t n = e4 - b4, s0 = b4 + n * a.rank / a.world, s1 = b4 + n * (a.rank + 1) / a.world;
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
  // completion: the last block (advances the step and) raises done[part][rank] on every rank
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&me->ticket[part], 1u) == gridDim.x - 1) {
      me->ticket[part] = 0;
      if (advance) a.ad->step = t;
      __threadfence_system();
      const unsigned e = *reinterpret_cast<volatile unsigned *>(&me->epoch);
      for (int q = 0; q < a.world; ++q) st_release_sys(&flags(a.dev[q], part, 1)[a.rank], e);
    }
  }
}

static int p2p_blocks(int64_t n4, int world) {
  const int64_t shard4 = (n4 + world - 1) / world;
  return (int)std::max<int64_t>(1, std::min<int64_t>((shard4 + 255) / 256, kSMs * 8));
}

void launch_p2p_part(cudaStream_t st, const P2PArgs &a, int part, int64_t b4, int64_t e4, bool bump, bool advance) {
  launch_ex(k_p2p_signal, 1, 32, 0, st, a, part, bump ? 1 : 0);
  launch_ex(k_p2p_wait, 1, 32, 0, st, a, part, 0);
  // part 1 runs beside layer 0's backward: a capped grid leaves it the SMs (HG_P2P1_BLOCKS)
  static const int p1_cap = [] {
    const char *e = getenv("HG_P2P1_BLOCKS");
    return e ? atoi(e) : 0;
  }();
  int blocks = p2p_blocks(e4 - b4, a.world);
  if (part == 1 && p1_cap > 0) blocks = std::min(blocks, p1_cap);
  launch_ex(k_p2p_adamw, blocks, 256, 0, st, a, part, b4, e4, advance ? 1 : 0);
  g_launches += 3;
}
void launch_p2p_wait_done(cudaStream_t st, const P2PArgs &a, int part) {
  launch_ex(k_p2p_wait, 1, 32, 0, st, a, part, 1);
  g_launches += 1;
}

}  // namespace hg
