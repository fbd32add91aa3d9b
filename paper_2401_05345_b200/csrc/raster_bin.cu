// Binning: (tile | depth) key duplication and per-tile range extraction.
// The radix sort itself runs between the two (raster.cu, CUB onesweep).
//
// Keys: tile id in bits [32, 32+tile_bits), the IEEE bits of the (positive)
// view depth in [0, 32); duplication order is (Gaussian, tile row, tile
// column), so a stable sort yields exactly the oracle's order
// (oracle/gs_oracle.c gs_forward).
#include <cuda_runtime.h>

#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

__device__ __forceinline__ void rect_of(float2 m, int radius, int tiles_x, int tiles_y, int* r) {
  const float fr = (float)radius;
  int v0 = (int)((m.x - fr) / (float)kTile), v1 = (int)((m.y - fr) / (float)kTile);
  int v2 = (int)((m.x + fr + (float)(kTile - 1)) / (float)kTile);
  int v3 = (int)((m.y + fr + (float)(kTile - 1)) / (float)kTile);
  r[0] = min(tiles_x, max(0, v0));
  r[1] = min(tiles_y, max(0, v1));
  r[2] = min(tiles_x, max(0, v2));
  r[3] = min(tiles_y, max(0, v3));
}

// One lane per Gaussian; rects wider than a warp are written cooperatively
// by the whole warp (C4-style scenes touch thousands of tiles per Gaussian).
__global__ void __launch_bounds__(256)
    k_duplicate(int P, const float2* __restrict__ means2D, const float* __restrict__ depths,
                const int* __restrict__ radii, const uint64_t* __restrict__ offsets,
                int tiles_x, int tiles_y, uint64_t* __restrict__ keys,
                uint32_t* __restrict__ values) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int r[4] = {0, 0, 0, 0};
  uint64_t off = 0;
  uint32_t dbits = 0;
  int area = 0;
  if (i < P && radii[i] > 0) {
    rect_of(means2D[i], radii[i], tiles_x, tiles_y, r);
    off = i == 0 ? 0 : offsets[i - 1];
    dbits = __float_as_uint(depths[i]);
    area = (r[2] - r[0]) * (r[3] - r[1]);
  }
  const bool big = area > 32;
  if (!big) {
    for (int y = r[1]; y < r[3]; ++y)
      for (int x = r[0]; x < r[2]; ++x) {
        keys[off] = (static_cast<uint64_t>(y * tiles_x + x) << 32) | dbits;
        values[off] = static_cast<uint32_t>(i);
        ++off;
      }
  }
  unsigned todo = __ballot_sync(0xffffffffu, big);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1u;
    const int x0 = __shfl_sync(0xffffffffu, r[0], src);
    const int y0 = __shfl_sync(0xffffffffu, r[1], src);
    const int x1 = __shfl_sync(0xffffffffu, r[2], src);
    const int a = __shfl_sync(0xffffffffu, area, src);
    const uint64_t o = __shfl_sync(0xffffffffu, off, src);
    const uint32_t d = __shfl_sync(0xffffffffu, dbits, src);
    const int id = __shfl_sync(0xffffffffu, i, src);
    const int w = x1 - x0;
    for (int k = lane; k < a; k += 32) {
      const int y = y0 + k / w, x = x0 + k % w;
      keys[o + k] = (static_cast<uint64_t>(y * tiles_x + x) << 32) | d;
      values[o + k] = static_cast<uint32_t>(id);
    }
  }
}

__global__ void k_ranges(int64_t L, const uint64_t* __restrict__ keys, uint2* __restrict__ ranges) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= L) return;
  const uint32_t tile = static_cast<uint32_t>(keys[idx] >> 32);
  if (idx == 0) {
    ranges[tile].x = 0;
  } else {
    const uint32_t prev = static_cast<uint32_t>(keys[idx - 1] >> 32);
    if (tile != prev) {
      ranges[prev].y = static_cast<uint32_t>(idx);
      ranges[tile].x = static_cast<uint32_t>(idx);
    }
  }
  if (idx == L - 1) ranges[tile].y = static_cast<uint32_t>(L);
}

}  // namespace

void launch_duplicate(int P, const float2* means2D, const float* depths, const int* radii,
                      const uint64_t* offsets, const CamParams& cam, uint64_t* keys,
                      uint32_t* values, cudaStream_t s) {
  if (P <= 0) return;
  k_duplicate<<<(P + 255) / 256, 256, 0, s>>>(P, means2D, depths, radii, offsets, cam.tiles_x,
                                              cam.tiles_y, keys, values);
  DW_CUDA(cudaGetLastError());
}

void launch_ranges(int64_t L, const uint64_t* keys, uint2* ranges, cudaStream_t s) {
  if (L <= 0) return;
  k_ranges<<<static_cast<unsigned>((L + 255) / 256), 256, 0, s>>>(L, keys, ranges);
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
