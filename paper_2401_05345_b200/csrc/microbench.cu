// Roofline microbenchmarks: measured f32 RED throughput of the L2 atomic
// units for the access patterns the policies generate (SURVEY.md §8(d):
// "R_red_distinct, R_red_same, R_red_v4"). There is no published B200
// figure, so bench.py measures these on the box in the same run.
//   0 distinct: each warp instruction = 32 lanes -> 32 consecutive floats
//   1 same:     each warp instruction = 32 lanes -> ONE float (naive pattern)
//   2 v4:       red.global.add.v4.f32, 32 lanes -> 128 consecutive floats
//   3 distwar:  9 lanes -> 9 consecutive floats of a pseudo-random primitive
//               (the SW-B issue pattern of the rasterizer backward)
//   4 same v4:  red.global.add.v4.f32, 32 lanes -> ONE 16-byte address
//   5 fallback, scalar: 4 lanes -> the same pseudo-random primitive row,
//               9 scalar REDs each (SW-B's per-lane path, DW_VEC_RED=0)
//   6 fallback, vector: the same traffic as 5 through red_row9 (3-4 vector
//               REDs per lane, the default per-lane path)
//   7 reduced row, vector: pattern 3's traffic (one 9-float row per warp
//               instruction slot) as red_row9 from ONE lane (3-4 vector REDs)
//   8 / 9 pattern 3 with the rows padded to 16 / 12 floats (64 / 48-byte
//               aligned rows: the line / sector straddles of 36-byte rows gone)
#include <cuda_runtime.h>

#include "distwar.cuh"
#include "dw_internal.h"

namespace dw {

namespace {

constexpr int64_t kRegionFloats = int64_t(1) << 24;  // 64 MB: L2-resident

// Pseudo-random primitive of a warp-iteration: a multiplicative hash to
// 2^20 primitives (36 MB of rows) -- 32-bit math, so the generator costs a
// few instructions and the kernel stays RED-bound, not issue-bound (a u64
// modulo here capped patterns 3 and 5-9 near 22 G warp-iterations/s).
__device__ __forceinline__ uint32_t hash_prim(int64_t w) {
  return (static_cast<uint32_t>(w) * 2654435761u) >> 12;
}

template <int PATTERN>
__global__ void __launch_bounds__(256) k_red(float* __restrict__ buf, int iters) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const float v = 1.0f / 1024.0f;
  for (int k = 0; k < iters; ++k) {
    const int64_t w = warp + static_cast<int64_t>(k) * nwarps;
    if (PATTERN == 0) {
      red_add(buf + ((w * 32) & (kRegionFloats - 1)) + lane, v);
    } else if (PATTERN == 1) {
      red_add(buf + ((w * 32) & (kRegionFloats - 1)), v);
    } else if (PATTERN == 2) {
      float* p = buf + ((w * 128) & (kRegionFloats - 1)) + 4 * lane;
      asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v),
                   "f"(v), "f"(v), "f"(v)
                   : "memory");
    } else if (PATTERN == 4) {
      float* p = buf + ((w * 128) & (kRegionFloats - 1));
      asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v),
                   "f"(v), "f"(v), "f"(v)
                   : "memory");
    } else if (PATTERN == 8 || PATTERN == 9) {
      const uint32_t prim = hash_prim(w);
      const int stride = PATTERN == 8 ? 16 : 12;
      if (lane < 9) red_add(buf + (static_cast<int64_t>(prim) * stride) + lane, v);
    } else if (PATTERN == 7) {
      const uint32_t prim = hash_prim(w);
      if (lane == 0) {
        const float s[9] = {v, v, v, v, v, v, v, v, v};
        red_row9(buf + (static_cast<int64_t>(prim) * 9), s);
      }
    } else if (PATTERN == 5 || PATTERN == 6) {
      const uint32_t prim = hash_prim(w);
      float* row = buf + (static_cast<int64_t>(prim) * 9);
      if (lane < 4) {
        if (PATTERN == 5) {
#pragma unroll
          for (int p = 0; p < 9; ++p) red_add(row + p, v);
        } else {
          const float s[9] = {v, v, v, v, v, v, v, v, v};
          red_row9(row, s);
        }
      }
    } else {
      // multiplicative hash of the warp-iteration -> primitive id
      const uint32_t prim = hash_prim(w);
      if (lane < 9) red_add(buf + (static_cast<int64_t>(prim) * 9) + lane, v);
    }
  }
}

template <int PATTERN>
float run(float* buf, int grid, int iters, cudaStream_t s) {
  cudaEvent_t a, b;
  DW_CUDA(cudaEventCreate(&a));
  DW_CUDA(cudaEventCreate(&b));
  k_red<PATTERN><<<grid, 256, 0, s>>>(buf, 1);  // warm-up
  DW_CUDA(cudaEventRecord(a, s));
  k_red<PATTERN><<<grid, 256, 0, s>>>(buf, iters);
  DW_CUDA(cudaEventRecord(b, s));
  DW_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  DW_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms;
}

}  // namespace

double microbench_red(int pattern, int64_t ops, cudaStream_t s) {
  float* buf = nullptr;
  DW_CUDA(cudaMalloc(&buf, (kRegionFloats + 1024) * sizeof(float)));
  DW_CUDA(cudaMemsetAsync(buf, 0, (kRegionFloats + 1024) * sizeof(float), s));
  const int grid = sm_count() * 8;
  const int64_t warps = static_cast<int64_t>(grid) * 8;
  // floats added per warp-iteration
  const int reds_per_warp_inst = pattern == 2   ? 128
                                 : pattern == 3 ? 9
                                 : pattern >= 7 ? 9
                                 : pattern == 4 ? 128
                                 : pattern >= 5 ? 36
                                                : 32;
  int64_t iters64 = ops / (warps * reds_per_warp_inst);
  if (iters64 < 1) iters64 = 1;
  const int iters = static_cast<int>(iters64 > (1 << 30) ? (1 << 30) : iters64);
  float ms = 0;
  switch (pattern) {
    case 0: ms = run<0>(buf, grid, iters, s); break;
    case 1: ms = run<1>(buf, grid, iters, s); break;
    case 2: ms = run<2>(buf, grid, iters, s); break;
    case 4: ms = run<4>(buf, grid, iters, s); break;
    case 5: ms = run<5>(buf, grid, iters, s); break;
    case 6: ms = run<6>(buf, grid, iters, s); break;
    case 7: ms = run<7>(buf, grid, iters, s); break;
    case 8: ms = run<8>(buf, grid, iters, s); break;
    case 9: ms = run<9>(buf, grid, iters, s); break;
    default: ms = run<3>(buf, grid, iters, s); break;
  }
  DW_CUDA(cudaFree(buf));
  const double reds = static_cast<double>(warps) * iters * reds_per_warp_inst;
  return reds / (ms * 1e-3);
}

}  // namespace dw
