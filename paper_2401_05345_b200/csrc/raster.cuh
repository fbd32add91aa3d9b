// Shared declarations of the tile-based Gaussian-splatting rasterizer.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/distwar.h"

namespace dw {

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may
// be scheduled while its predecessor in the stream drains; it must execute
// pdl_wait() before touching global memory the predecessor reads or writes
// (it returns once the predecessor grid has completed and flushed). Each PDL
// kernel then releases its own dependents at once (pdl_trigger), so the
// short, latency-bound binning kernels of the forward do not pay a full
// launch + ramp-up gap each.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

#ifndef DW_PDL
#define DW_PDL 1
#endif

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = DW_PDL ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw std::runtime_error(std::string("launch: ") + cudaGetErrorString(e));
}

constexpr int kTile = 16;         // 16x16-pixel tiles, one 256-thread CTA each
constexpr int kBlock = kTile * kTile;
constexpr int kNParam = 9;        // mean2D.xy, conic.xyz, opacity, rgb
constexpr int kNParam3D = 14;     // means3D xyz, scales xyz, rotation rxyz, opacity, rgb

// Kernel-parameter copy of dw_camera (lives in the constant bank).
struct CamParams {
  float vm[16];
  float pm[16];
  float tan_fovx, tan_fovy;
  float bg[3];
  float scale_modifier;
  int W, H, tiles_x, tiles_y;
  // A frame may stack views vertically (raster_views_host: several views per
  // set of launches): tile rows [v * rows_v, (v + 1) * rows_v) are view v,
  // whose Gaussians carry ids [v * vstride, (v + 1) * vstride) and whose
  // per-pixel buffers (final_T, n_contrib: H*W; image, dL/dpixel: 3*H*W) are
  // the v-th of a [views][...] array. One view: rows_v = tiles_y, vstride = 0.
  int rows_v, vstride;
};

// Tile -> (view slot of a stacked frame, top-left pixel inside that view).
__device__ __forceinline__ int tile_view(const CamParams& cam, int tile, int* tx0, int* ty0) {
  const int ty = tile / cam.tiles_x;
  const int v = ty / cam.rows_v;
  *tx0 = (tile - ty * cam.tiles_x) * kTile;
  *ty0 = (ty - v * cam.rows_v) * kTile;
  return v;
}

// In-tile thread t = warp*32 + lane covers pixel (8*(warp&1) + (lane&7),
// 4*(warp>>1) + (lane>>3)): each warp owns an 8x4 block, the warp tiling of
// the reference's workload model (workload.cpp:107-110), which maximises the
// chance that all 32 lanes of a warp see the same Gaussian.
__device__ __forceinline__ void tile_pixel(int tx0, int ty0, int t, int* px, int* py) {
  const int w = t >> 5, l = t & 31;
  *px = tx0 + (w & 1) * 8 + (l & 7);
  *py = ty0 + (w >> 1) * 4 + (l >> 3);
}

void launch_preprocess(int P, const float* means3D, const float* scales, const float* rotations,
                       const float* opacities, const float* colors, const CamParams& cam,
                       float2* means2D, float* depths, int* radii, float4* conic_opacity,
                       float4* rgb, uint32_t* tiles_touched, uint32_t* dkey, uint32_t* dids,
                       cudaStream_t s, float4* packed = nullptr,
                       uint32_t* rect_out = nullptr,  // dkey/dids (nullable): depth-sort keys and ids;
                                                      // rect_out (nullable): packed tile rectangles
                       int row0 = 0, uint32_t id0 = 0);  // stacked frame: the view's first tile row
                                                         // (added to the rectangles) and first id

// Device buffers of the backward's WarpRecord tap (SoA like dw_device_trace).
struct TapBuf {
  unsigned long long* count = nullptr;
  unsigned long long cap = 0;
  int32_t* warp_id = nullptr;
  int32_t* iteration = nullptr;
  uint32_t* active = nullptr;
  int32_t* prim = nullptr;   // [cap][32]
  float* vals = nullptr;     // [cap][9][32]
};

// SW-B backward that also records its per-warp records (raster_blend.cu).
// tile_order (nullable): CTA i renders tile tile_order[i] (launch_tile_order)
void launch_backward_tap(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                         const float2* means2D, const float4* co, const float4* rgb,
                         const uint32_t* tile_order, const float* final_T,
                         const uint32_t* n_contrib, const float* dL, int thr, float* grad,
                         const TapBuf& tap, cudaStream_t s);

// raster_train.cu: preprocess backward (adds into grad3d[P][14]) and Adam.
void launch_preprocess_backward(int P, const float* means3D, const float* scales,
                                const float* rotations, const int* radii, const CamParams& cam,
                                const float* grad2d, float* grad3d, cudaStream_t s);
void launch_adam(int P, float* means3D, float* scales, float* rotations, float* opacities,
                 float* colors, const float* grad, float* m, float* v, const float lr[5], float b1,
                 float b2, float eps, int step, cudaStream_t s);

// raster_sort.cu: hand-written stable LSD radix sort + scan (no CUB).
size_t radix_sort_temp_bytes(int64_t n);
size_t scan_temp_bytes(int64_t n);
// n_dev (nullable): live element count read on the device (<= n, the
// capacity the grids are sized for) -- the no-host-sync forward.
// gather_src (nullable): the last pass also writes gather_out[i] =
// gather_src[sorted value i] (a payload in sorted order, e.g. tiles touched).
int radix_sort_pairs(uint32_t* k[2], uint32_t* v[2], int64_t n, int bits, void* temp,
                     cudaStream_t s, const unsigned long long* n_dev = nullptr,
                     const uint32_t* gather_src = nullptr, uint32_t* gather_out = nullptr);
void inclusive_scan_gather(const uint32_t* in, const uint32_t* order, int64_t n, uint64_t* out,
                           void* temp, cudaStream_t s, int mode = 0);
// after radix_sort_pairs(..., n, ..., temp): the last pass's 256 digit totals
// (device; live elements only)
const uint32_t* radix_sort_digit_totals(const void* temp, int64_t n);
// per row d of counts[256][tiles]: exclusive scan over the tiles in place and
// the row total to digit_total[d]
void launch_scan_rows(uint32_t* counts, int64_t tiles, uint32_t* digit_total, cudaStream_t s);
// Block binning, fused level 1 (<= 256 coarse blocks): k_bb_hist counts each
// 2,048-Gaussian tile's entries per block into hist[256][tiles] and adds the
// frame's packed total (blocks << 34 | tiles) into *total (zeroed by the
// caller); launch_block_binning_fused then writes the entries straight to
// their block-sorted positions instead of generating and radix-sorting them.
size_t block_binning_hist_words(int64_t P);
void launch_bb_hist(const uint32_t* rect_sorted, int64_t P, const CamParams& cam, uint32_t* hist,
                    uint64_t* total, cudaStream_t s);
void launch_block_binning_fused(const uint32_t* rect_sorted, const uint32_t* order, int64_t P,
                                const CamParams& cam, uint32_t* hist, uint32_t* v[2],
                                uint64_t entry_cap, uint32_t* brect, uint2* branges,
                                uint32_t* cnt, uint2* ranges, uint32_t** values_out,
                                const unsigned long long* n_live,
                                const unsigned long long* n_entries_dev, cudaStream_t s);
// Block binning's level-1 entries in one scan: over the depth-ordered packed
// rectangles (launch_preprocess rect_out, laid out by the depth sort), the
// inclusive (coarse blocks << 32 | tiles touched) -- its total to out[n-1] --
// and, at each Gaussian's block offset, (block id, id) for every coarse
// block it touches (none past cap entries).
void block_entries_scan(const uint32_t* rect_sorted, const uint32_t* order, int64_t n,
                        uint64_t* out, void* temp, int nbx, uint32_t* bkey, uint32_t* bval,
                        uint64_t cap, cudaStream_t s);
void launch_depth_keys(int P, const float* depths, const int* radii, uint32_t* dkey, uint32_t* ids,
                       cudaStream_t s);
void launch_duplicate_sorted(int P, const uint32_t* order, const float2* means2D, const int* radii,
                             const uint64_t* offsets, const CamParams& cam, uint32_t* tile_ids,
                             uint32_t* values, uint64_t cap, cudaStream_t s);
// Dense (tile-major) binning: per-tile lists built directly from the
// depth-ordered Gaussians' tile rectangles (raster_sort.cu).
size_t dense_diff_bytes(int tiles_x, int tiles_y);
size_t dense_scratch_words(int tiles_x, int tiles_y);
bool dense_binning_fits(int tiles_x, int tiles_y);
// n_dev (nullable): live instance count; with it, a count above cap renders empty
void launch_dense_binning(int P, const uint32_t* order, const float2* means2D, const int* radii,
                          const CamParams& cam, uint2* rects, int* scratch, uint2* ranges,
                          uint32_t* values, const unsigned long long* n_dev, uint64_t cap,
                          cudaStream_t s);
void launch_tiles_from_ranges(const uint2* ranges, int ntiles, uint32_t* tiles, cudaStream_t s);
// Per-tile stable depth sort of index-ordered tile lists (tile-first binning);
// scratch: 2 x instances u64 (used by lists longer than the shared-memory cap).
// min_n: only lists of at least min_n elements are sorted (the others are
// left as they are -- already sorted by another kernel).
void launch_segsort_depth(const uint2* ranges, const float* depths, uint32_t* values,
                          unsigned long long* scratch, int64_t capacity, int ntiles,
                          cudaStream_t s, int min_n = 2);
// Scatter binning (raster_scatter.cu): per-(segment, tile) counts, placement,
// per-tile on-chip depth sort. scratch: scatter_scratch_words(P, ntiles) u32;
// seg_scratch = 2 x seg_half u64 for lists longer than scatter_sort_cap().
int scatter_sort_cap();
bool scatter_binning_fits(int ntiles);
size_t scatter_scratch_words(int P, int ntiles);
void launch_scatter_binning(int P, const float2* means2D, const int* radii, const float* depths,
                            const CamParams& cam, uint32_t* scratch, uint2* ranges,
                            uint32_t* values, unsigned long long* seg_scratch, int64_t seg_half,
                            const unsigned long long* n_dev, cudaStream_t s);
// Block binning's packed scan value: (coarse-block entries << kBBTileBits) |
// tile instances -- 34 bits of instances (so a frame past 2^32 instances is
// detected, not wrapped), 30 of entries.
constexpr int kBBTileBits = 34;
constexpr unsigned long long kBBTileMask = (1ull << kBBTileBits) - 1ull;

// Block binning (raster_blockbin.cu): the depth-first lists through coarse
// 8x4-tile blocks (one sorted entry per (Gaussian, block) instead of the
// duplicate + two-pass tile sort of every instance).
bool block_binning_fits(int tiles_x, int tiles_y);
int block_binning_nbx(int tiles_x);  // coarse blocks per row
int block_binning_blocks(int tiles_x, int tiles_y);
size_t block_binning_count_words(int tiles_x, int tiles_y);
void launch_bb_clamp(const uint64_t* offsets, int P, uint64_t cap, uint64_t entry_cap,
                     unsigned long long* n_live,
                     unsigned long long* n_entries, unsigned int* overflow, bool sticky,
                     cudaStream_t s);
// k/v: sort double buffers of >= n_entries (capacity when n_entries_dev is set);
// brect: >= n_entries words; cnt: block_binning_count_words; writes ranges and
// the lists (*values_out: one of v)
// k[0]/v[0]: the entries (block_entries_scan); k/v: sort double buffers of >=
// n_entries (the capacity when n_entries_dev is set); rect_by_id: packed
// rectangles by id (the sort payload); brect: >= n_entries words; cnt:
// block_binning_count_words. Writes ranges and the lists (*values_out: one of v).
void launch_block_binning(const uint32_t* rect_by_id, const CamParams& cam, uint32_t* k[2],
                          uint32_t* v[2], int64_t n_entries, void* sort_tmp, uint32_t* brect,
                          uint2* branges, uint32_t* cnt, uint2* ranges, uint32_t** values_out,
                          const unsigned long long* n_live,
                          const unsigned long long* n_entries_dev, cudaStream_t s);
// order[ntiles]: tiles by descending list length (bucketed), for the blend kernels
void launch_tile_order(const uint2* ranges, int ntiles, uint32_t* order, cudaStream_t s);
// ranges[0, ntiles) of the sorted tile ids (every range written)
void launch_ranges_u32(int64_t L, const uint32_t* tiles, uint2* ranges, int ntiles,
                       cudaStream_t s, const unsigned long long* n_dev = nullptr);
void launch_clamp_total(const uint64_t* offsets, int P, uint64_t cap, unsigned long long* n_live,
                        unsigned int* overflow, bool sticky, cudaStream_t s);
void launch_make_keys(int64_t L, const uint32_t* tiles, const uint32_t* values, const float* depths,
                      uint64_t* keys, cudaStream_t s);

void launch_forward_impl(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                         const float2* means2D, const float4* conic_opacity, const float4* rgb,
                         const uint32_t* tile_order, float* final_T, uint32_t* n_contrib,
                         float* out_color, cudaStream_t s);

// counters (nullable): [0] += contributing (pixel, Gaussian) pairs, [1] += REDs.
void launch_backward_impl(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                          const float2* means2D, const float4* co, const float4* rgb,
                          const uint32_t* tile_order, const float* final_T,
                          const uint32_t* n_contrib,
                          const float* dL, int policy, int thr, float* grad,
                          unsigned long long* counters, cudaStream_t s,
                          const float4* packed = nullptr, bool chained = false,
                          int grad_stride = kNParam);
// grad[P][9] += pad[P][12] (the first 9 floats of each padded row), then pad = 0.
void launch_fold_rows(int64_t P, float* pad, float* grad, cudaStream_t s);

}  // namespace dw
