// Scatter binning: per-tile Gaussian lists without a global sort.
//
// The lists the blend kernels walk are, per tile, the Gaussians whose tile
// rectangle covers the tile, in (depth, index) order -- what a stable sort of
// (tile | depth) 64-bit keys gives (the reference layout).
// The depth-first pipeline builds them with a 4-pass radix sort of all P
// depth keys, a duplication of every instance and a 2-pass radix sort of the
// I instances by tile: ~10 global passes, each a round trip through HBM and
// three to four launches. Here, with the Gaussians cut into segments of 8,192
// (one 1024-thread CTA each):
//   1. k_sc_count    per segment, per tile instance counts (shared atomics);
//   2. k_sc_colscan  per tile, each segment's offset inside the tile's list;
//   3. k_sc_ranges   exclusive scan of the tile totals -> tile ranges;
//   4. k_sc_place    each instance takes the next slot of its segment's share
//                    of its tile's list (shared atomics) -- right set, any order;
//   5. k_tile_sort   one CTA per tile sorts its list on chip into (depth,
//                    index) order (monotone bucket sort + insertion sort of
//                    the buckets, exact); lists longer than the on-chip
//                    capacity go to the chunked sort + merge of k_segsort_depth.
// No global atomics and no global sort: two reads of the Gaussians' rects, a
// per-(segment, tile) count table (~12 MB at 3M Gaussians), one write of the
// lists and one read + write of them by the tile sort.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <stdexcept>

#include "distwar.cuh"
#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

__device__ __forceinline__ void rect_of_s(float2 m, int radius, int tiles_x, int tiles_y, int* r) {
  // identical arithmetic to raster_sort.cu rect_of (and the oracle's rect_of)
  const float fr = (float)radius;
  const int v0 = (int)((m.x - fr) / (float)kTile), v1 = (int)((m.y - fr) / (float)kTile);
  const int v2 = (int)((m.x + fr + (float)(kTile - 1)) / (float)kTile);
  const int v3 = (int)((m.y + fr + (float)(kTile - 1)) / (float)kTile);
  r[0] = min(tiles_x, max(0, v0));
  r[1] = min(tiles_y, max(0, v1));
  r[2] = min(tiles_x, max(0, v2));
  r[3] = min(tiles_y, max(0, v3));
}

// A segment of kScSeg consecutive Gaussians per CTA (1024 threads x 8).
constexpr int kScThreads = 1024;
constexpr int kScPer = 8;
constexpr int kScSeg = kScThreads * kScPer;

// Visit every instance of the CTA's Gaussians: small rectangles by the owning
// lane, rectangles of more than 32 tiles by the whole warp (C4-style scenes
// cover thousands). fn(tile, gaussian) runs once per instance.
template <typename Fn>
__device__ __forceinline__ void for_each_instance(int P, const float2* __restrict__ means2D,
                                                  const int* __restrict__ radii, int tiles_x,
                                                  int tiles_y, Fn fn) {
  const int lane = threadIdx.x & 31;
  // the segment's loads first (independent), then the per-instance work
  float2 m[kScPer];
  int rad[kScPer];
#pragma unroll
  for (int k = 0; k < kScPer; ++k) {
    const int i = blockIdx.x * kScSeg + k * kScThreads + threadIdx.x;
    rad[k] = i < P ? __ldg(radii + i) : 0;
    m[k] = i < P ? __ldg(means2D + i) : make_float2(0.0f, 0.0f);
  }
#pragma unroll
  for (int k = 0; k < kScPer; ++k) {
    const int i = blockIdx.x * kScSeg + k * kScThreads + threadIdx.x;
    int r[4] = {0, 0, 0, 0};
    if (rad[k] > 0) rect_of_s(m[k], rad[k], tiles_x, tiles_y, r);
    const int w = r[2] - r[0], h = r[3] - r[1];
    const int area = (w > 0 && h > 0) ? w * h : 0;
    const bool big = area > 32;
    // small rectangles, expanded by the whole warp: instance e of the warp's
    // run belongs to the lane whose [excl, excl + area) holds it (5-step
    // search over the lanes' exclusive scan), so every lane handles one
    // instance per step instead of walking its own rectangle serially
    const int sa = big ? 0 : area;
    int incl = sa;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - sa;
    const int total = __shfl_sync(kFull, incl, 31);
    for (int e0 = 0; e0 < total; e0 += 32) {  // warp-uniform trips
      const int e = e0 + lane;
      int owner = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int probe = owner + step;
        if (__shfl_sync(kFull, excl, probe) <= e) owner = probe;
      }
      const int q = e - __shfl_sync(kFull, excl, owner);
      const int ww = __shfl_sync(kFull, w, owner);
      const int x0 = __shfl_sync(kFull, r[0], owner), y0 = __shfl_sync(kFull, r[1], owner);
      const int g = __shfl_sync(kFull, i, owner);
      if (e < total) {
        const int row = static_cast<int>((static_cast<float>(q) + 0.5f) / static_cast<float>(ww));
        fn(static_cast<uint32_t>((y0 + row) * tiles_x + x0 + (q - row * ww)), g);
      }
    }
    unsigned todo = __ballot_sync(kFull, big);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1u;
      const int x0 = __shfl_sync(kFull, r[0], src), y0 = __shfl_sync(kFull, r[1], src);
      const int ww = __shfl_sync(kFull, w, src), a = __shfl_sync(kFull, area, src);
      const int g = __shfl_sync(kFull, i, src);
      for (int q = lane; q < a; q += 32)
        fn(static_cast<uint32_t>((y0 + q / ww) * tiles_x + x0 + q % ww), g);
    }
  }
}

// 1. Per segment: how many of its instances fall in each tile (shared-memory
//    atomics -- fast, and no same-address contention at L2), written to
//    seg_cnt[tile][segment] (tile-major: the column scan reads it contiguously).
__global__ void __launch_bounds__(kScThreads)
    k_sc_count(int P, const float2* __restrict__ means2D, const int* __restrict__ radii,
               int tiles_x, int tiles_y, uint32_t* __restrict__ seg_cnt) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  extern __shared__ uint32_t s_cnt[];
  const int ntiles = tiles_x * tiles_y;
  for (int t = threadIdx.x; t < ntiles; t += kScThreads) s_cnt[t] = 0u;
  __syncthreads();
  for_each_instance(P, means2D, radii, tiles_x, tiles_y,
                    [&](uint32_t tile, int) { atomicAdd(s_cnt + tile, 1u); });
  __syncthreads();
  const int nseg = gridDim.x;
  for (int t = threadIdx.x; t < ntiles; t += kScThreads)
    seg_cnt[static_cast<int64_t>(t) * nseg + blockIdx.x] = s_cnt[t];
}

// 2. Per tile (one warp each): exclusive scan of its counts over the
//    segments -- each segment's offset inside the tile's list -- and the
//    tile's total.
__global__ void __launch_bounds__(256)
    k_sc_colscan(uint32_t* __restrict__ seg_cnt, int nseg, int ntiles,
                 uint32_t* __restrict__ tile_total) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int t = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  if (t >= ntiles) return;
  uint32_t* row = seg_cnt + static_cast<int64_t>(t) * nseg;
  uint32_t run = 0;
  for (int c0 = 0; c0 < nseg; c0 += 32) {
    const int c = c0 + lane;
    const uint32_t v = c < nseg ? row[c] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (c < nseg) row[c] = run + incl - v;
    run += __shfl_sync(kFull, incl, 31);
  }
  if (lane == 0) tile_total[t] = run;
}

// 3. One block: exclusive scan of the tile totals -> ranges ((0, 0) when
//    empty, the reference layout). With a live-count bound (no-sync forward,
//    n_dev == 0: the frame exceeded the reserve) every range is empty.
__global__ void __launch_bounds__(1024)
    k_sc_ranges(const uint32_t* __restrict__ tile_total, int ntiles, uint2* __restrict__ ranges,
                const unsigned long long* __restrict__ n_dev) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ uint32_t s_wsum[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int per = (ntiles + 1023) / 1024;
  uint32_t local = 0;
  for (int k = 0; k < per; ++k) {
    const int tile = t * per + k;
    if (tile < ntiles) local += tile_total[tile];
  }
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = s_wsum[lane];
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, vi, o);
      if (lane >= o) vi += y;
    }
    s_wsum[lane] = vi - v;
  }
  __syncthreads();
  const bool over = n_dev && *n_dev == 0ull;
  uint32_t run = s_wsum[w] + incl - local;
  for (int k = 0; k < per; ++k) {
    const int tile = t * per + k;
    if (tile >= ntiles) break;
    const uint32_t c = tile_total[tile];
    ranges[tile] = (c == 0 || over) ? make_uint2(0u, 0u) : make_uint2(run, run + c);
    run += c;
  }
}

// 4. Per segment: every instance takes the next slot of its tile's share
//    (tile start + the segment's offset, advanced by a shared-memory atomic)
//    and writes its Gaussian id there: each list now holds the right SET,
//    in no particular order.
__global__ void __launch_bounds__(kScThreads)
    k_sc_place(int P, const float2* __restrict__ means2D, const int* __restrict__ radii,
               int tiles_x, int tiles_y, const uint32_t* __restrict__ seg_cnt,
               const uint2* __restrict__ ranges, uint32_t* __restrict__ values,
               const unsigned long long* __restrict__ n_dev) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  if (n_dev && *n_dev == 0ull) return;  // over the reserve: nothing to write
  extern __shared__ uint32_t s_pos[];
  const int ntiles = tiles_x * tiles_y, nseg = gridDim.x;
  for (int t = threadIdx.x; t < ntiles; t += kScThreads)
    s_pos[t] = ranges[t].x + seg_cnt[static_cast<int64_t>(t) * nseg + blockIdx.x];
  __syncthreads();
  for_each_instance(P, means2D, radii, tiles_x, tiles_y, [&](uint32_t tile, int g) {
    values[atomicAdd(s_pos + tile, 1u)] = static_cast<uint32_t>(g);
  });
}

// ---------------------------------------------------------------------------
// 5. Per-tile depth sort on chip, by a monotone bucket sort: with lo / hi the
//    tile's smallest / largest depth, element (depth, id) goes to bucket
//    b = min(n - 1, floor((depth - lo) * n / (hi - lo))) -- non-decreasing in
//    depth (every step is a correctly rounded monotone op), so bucket order
//    is depth order -- n buckets for n elements, placed by a counting sort (shared
//    atomics + one block scan); then each bucket (~1 element on average) is
//    insertion-sorted by (key, id). The result is the exact (depth, index)
//    order. A pathological bucket (> kTsRun elements: many equal depths)
//    switches the tile to a bitonic sort of the 64-bit (key << 32 | id).
constexpr int kTsCap = 4096;  // elements sorted on chip; longer lists: k_segsort_depth
constexpr int kTsThreads = 256;
constexpr int kTsPer = kTsCap / kTsThreads;
constexpr int kTsRun = 48;
constexpr size_t kTsSmem = (3 * static_cast<size_t>(kTsCap) + 1) * sizeof(uint32_t);

__global__ void __launch_bounds__(kTsThreads, 4)
    k_tile_sort(const uint2* __restrict__ ranges, const float* __restrict__ depths,
                uint32_t* __restrict__ values, int ntiles) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  extern __shared__ uint32_t sm[];
  uint32_t* sk = sm;                // keys, bucketed
  uint32_t* si = sm + kTsCap;       // ids, bucketed
  uint32_t* sc = sm + 2 * kTsCap;   // bucket counters -> ends (n + 1 words)
  __shared__ uint32_t s_lo, s_hi;
  __shared__ uint32_t s_wsum[kTsThreads / 32];
  __shared__ int s_bad;
  const int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const uint2 rg = ranges[tile];
  const int n = static_cast<int>(rg.y - rg.x);
  if (n <= 1 || n > kTsCap) return;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) {
    s_lo = 0xffffffffu;
    s_hi = 0u;
    s_bad = 0;
  }
  for (int i = t; i <= n; i += kTsThreads) sc[i] = 0u;
  uint32_t key[kTsPer], id[kTsPer];
  uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
  for (int k = 0; k < kTsPer; ++k) {
    const int e = t + k * kTsThreads;
    key[k] = 0u;
    id[k] = 0u;
    if (k * kTsThreads >= n) break;  // block-uniform
    if (e < n) {
      id[k] = values[rg.x + e];
      key[k] = __float_as_uint(__ldg(depths + id[k]));  // depth > 0: bits order like floats
      lo = min(lo, key[k]);
      hi = max(hi, key[k]);
    }
  }
  lo = __reduce_min_sync(kFull, lo);
  hi = __reduce_max_sync(kFull, hi);
  __syncthreads();  // s_lo / s_hi initialised, counters zeroed
  if (lane == 0) {
    atomicMin(&s_lo, lo);
    atomicMax(&s_hi, hi);
  }
  __syncthreads();
  // buckets uniform in depth VALUE (the scenes' depths are spread roughly
  // uniformly; their float bits are not): b = (d - dmin) * n / (dmax - dmin),
  // non-decreasing in d
  const float dmin = __uint_as_float(s_lo), dmax = __uint_as_float(s_hi);
  const float scale = dmax > dmin ? static_cast<float>(n) / (dmax - dmin) : 0.0f;
  uint32_t bk[kTsPer];
#pragma unroll
  for (int k = 0; k < kTsPer; ++k) {
    bk[k] = 0u;
    if (k * kTsThreads >= n) break;  // block-uniform
    if (t + k * kTsThreads < n) {
      bk[k] = min(static_cast<uint32_t>(n - 1),
                  static_cast<uint32_t>((__uint_as_float(key[k]) - dmin) * scale));
      atomicAdd(sc + bk[k], 1u);
    }
  }
  __syncthreads();
  // exclusive scan of sc[0, n): thread t owns a contiguous segment
  const int seg = (n + kTsThreads - 1) / kTsThreads;
  const int b0 = min(n, t * seg), b1 = min(n, b0 + seg);
  uint32_t sum = 0;
  for (int b = b0; b < b1; ++b) sum += sc[b];
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  uint32_t run = incl - sum;
  for (int k = 0; k < w; ++k) run += s_wsum[k];
  for (int b = b0; b < b1; ++b) {
    const uint32_t c = sc[b];
    sc[b] = run;  // bucket start; the scatter below advances it to the bucket's end
    run += c;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTsPer; ++k) {
    if (k * kTsThreads >= n) break;  // block-uniform
    if (t + k * kTsThreads < n) {
      const uint32_t pos = atomicAdd(sc + bk[k], 1u);
      sk[pos] = key[k];
      si[pos] = id[k];
    }
  }
  __syncthreads();
  // bucket b now spans [b ? sc[b - 1] : 0, sc[b]): insertion sort by (key, id)
  bool bad = false;
  for (int b = t; b < n; b += kTsThreads) {
    const int s0 = b ? static_cast<int>(sc[b - 1]) : 0, e0 = static_cast<int>(sc[b]);
    if (e0 - s0 > kTsRun) {
      bad = true;
      continue;
    }
    for (int a = s0 + 1; a < e0; ++a) {
      const uint32_t kk = sk[a], ii = si[a];
      int q = a - 1;
      while (q >= s0 && (sk[q] > kk || (sk[q] == kk && si[q] > ii))) {
        sk[q + 1] = sk[q];
        si[q + 1] = si[q];
        --q;
      }
      sk[q + 1] = kk;
      si[q + 1] = ii;
    }
  }
  if (__syncthreads_or(bad)) {  // rare: fall back to a bitonic sort of (key << 32 | id)
    unsigned long long* s64 = reinterpret_cast<unsigned long long*>(sm);  // sk, si: 2 x kTsCap
    int npad = 32;
    while (npad < n) npad <<= 1;
#pragma unroll
    for (int k = 0; k < kTsPer; ++k) {
      const int e = t + k * kTsThreads;
      if (e < npad) s64[e] = e < n ? (static_cast<unsigned long long>(key[k]) << 32 | id[k]) : ~0ull;
    }
    for (int e = t + kTsPer * kTsThreads; e < npad; e += kTsThreads) s64[e] = ~0ull;
    __syncthreads();
    for (int kk = 2; kk <= npad; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = t; i < npad; i += kTsThreads) {
          const int l = i ^ j;
          if (l > i) {
            const unsigned long long x = s64[i], y = s64[l];
            if ((x > y) == ((i & kk) == 0)) {
              s64[i] = y;
              s64[l] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int i = t; i < n; i += kTsThreads) values[rg.x + i] = static_cast<uint32_t>(s64[i]);
    return;
  }
  for (int i = t; i < n; i += kTsThreads) values[rg.x + i] = si[i];
}

inline unsigned blocks_for_s(int64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

template <typename K>
void smem_optin(K kernel, size_t bytes, std::atomic<bool>* done) {
  int dev = 0;
  DW_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && done[dev].load(std::memory_order_acquire)) return;
  DW_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(bytes)));
  if (dev >= 0 && dev < 64) done[dev].store(true, std::memory_order_release);
}

}  // namespace

int scatter_sort_cap() { return kTsCap; }

bool scatter_binning_fits(int ntiles) { return static_cast<size_t>(ntiles) * 4 <= 160 * 1024; }

size_t scatter_scratch_words(int P, int ntiles) {
  return (static_cast<size_t>(blocks_for_s(std::max(P, 1), kScSeg)) + 1) * ntiles;
}

void launch_scatter_binning(int P, const float2* means2D, const int* radii, const float* depths,
                            const CamParams& cam, uint32_t* scratch, uint2* ranges,
                            uint32_t* values, unsigned long long* seg_scratch, int64_t seg_half,
                            const unsigned long long* n_dev, cudaStream_t s) {
  const int ntiles = cam.tiles_x * cam.tiles_y;
  if (!scatter_binning_fits(ntiles)) throw std::invalid_argument("scatter binning: too many tiles");
  const size_t tbytes = static_cast<size_t>(ntiles) * sizeof(uint32_t);
  static std::atomic<bool> opt_count[64], opt_place[64], opt_sort[64];
  smem_optin(k_sc_count, 160 * 1024, opt_count);
  smem_optin(k_sc_place, 160 * 1024, opt_place);
  smem_optin(k_tile_sort, kTsSmem, opt_sort);
  const int nseg = static_cast<int>(blocks_for_s(std::max(P, 1), kScSeg));
  uint32_t* seg_cnt = scratch;                                   // [ntiles][nseg]
  uint32_t* total = scratch + static_cast<size_t>(nseg) * ntiles;  // [ntiles]
  launch_pdl(k_sc_count, nseg, kScThreads, tbytes, s, P, means2D, radii, cam.tiles_x,
             cam.tiles_y, seg_cnt);
  launch_pdl(k_sc_colscan, blocks_for_s(static_cast<int64_t>(ntiles) * 32, 256), 256, 0, s,
             seg_cnt, nseg, ntiles, total);
  launch_pdl(k_sc_ranges, 1, 1024, 0, s, total, ntiles, ranges, n_dev);
  launch_pdl(k_sc_place, nseg, kScThreads, tbytes, s, P, means2D, radii, cam.tiles_x,
             cam.tiles_y, seg_cnt, ranges, values, n_dev);
  launch_pdl(k_tile_sort, ntiles, kTsThreads, kTsSmem, s, ranges, depths, values, ntiles);
  // lists longer than the on-chip capacity: chunked sort + merge, every
  // shorter tile skipped
  launch_segsort_depth(ranges, depths, values, seg_scratch, seg_half, ntiles, s, kTsCap + 1);
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
