// tma.h — host-side tensor maps shared by the TMA-fed GEMM translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hg {

// the four operand tensor maps of one launch (kernel parameter, __grid_constant__)
struct TmaMaps {
  CUtensorMap ah, al, bh, bl;
};

// 2-D fp32 map, box = box_rows x 32 fp32; mn_major selects SWIZZLE_128B_ATOM_32B (else SWIZZLE_128B)
CUtensorMap tma_map2d(const float *p, uint64_t rows, uint64_t cols, uint32_t box_rows, bool mn_major);

cudaError_t tmn_configure();  // tcmn.cu: opt-in shared memory of the MN-major kernels

}  // namespace hg
