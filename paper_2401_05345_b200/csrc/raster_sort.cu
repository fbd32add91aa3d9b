// Hand-written binning sort for sm_100a (replaces a 64-bit-key library radix
// sort of every (tile, Gaussian) instance).
//
// The reference order is a STABLE sort of the instances by the 64-bit key
// (tile << 32) | float_bits(depth), instances generated in (Gaussian, row,
// column) order: within a tile, ascending depth, ties by Gaussian index. The
// same order is produced here with far fewer bytes moved:
//   1. stable LSD sort of the P Gaussians by their 32-bit depth key
//      (4 passes over P, not over the ~4.5 P instances);
//   2. duplicate the instances in that depth order, writing only a u32 tile
//      id and the Gaussian id;
//   3. stable LSD sort of the instances by tile id (ceil(tile_bits / 8)
//      passes: 2 for 1080p's 8,160 tiles).
// Stability of step 3 keeps step 1's (depth, index) order inside each tile,
// so the result equals the 64-bit-key sort bit for bit (tests compare it with
// the oracle's std-style stable sort).
//
// Each LSD pass is three launches over tiles of 4,096 elements:
//   upsweep    per-tile 8-bit digit histogram (smem atomics) -> counts[d][tile]
//   scan       per-digit exclusive scan over tiles + exclusive scan of the
//              256 digit totals (two small kernels)
//   downsweep  stable in-tile ranking: 16 rounds of 256 elements in
//              element order; __match_any_sync ranks lanes within a warp,
//              an smem per-digit prefix over the 8 warps orders the warps,
//              a running per-digit base orders the rounds; then scatter.
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "distwar.cuh"
#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 elements

constexpr int kWarps = kSortThreads / 32;

// Lanes of this warp whose digit equals mine (warp multi-split by votes: one
// ballot per digit bit instead of a __match_any_sync, which is a multi-cycle
// instruction). Invalid lanes never match valid ones.
#ifndef DW_SORT_MATCH
#define DW_SORT_MATCH 0  // 1: one __match_any_sync instead of `bits` ballots
#endif
// Compile-time digit width and a FULL (every lane valid) fast path.
template <int BITS, bool FULL>
__device__ __forceinline__ unsigned digit_peers_t(uint32_t d, bool valid) {
  if (DW_SORT_MATCH) return __match_any_sync(kFull, FULL || valid ? d : 0xffffffffu);
  unsigned peers = kFull;
  if (!FULL) {
    peers = __ballot_sync(kFull, valid);
    if (!valid) peers = ~peers;
  }
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned m = __ballot_sync(kFull, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

__device__ __forceinline__ unsigned digit_peers(uint32_t d, int bits, bool valid) {
  if (DW_SORT_MATCH) return __match_any_sync(kFull, valid ? d : 0xffffffffu);
  unsigned peers = __ballot_sync(kFull, valid);
  if (!valid) peers = ~peers;
  for (int b = 0; b < bits; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned m = __ballot_sync(kFull, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

// Per-tile digit histogram of ITEMS*256 consecutive elements (the same tiles
// the downsweep ranks).
// n_dev (nullable): element count read on the device, capped by n -- the
// no-host-sync forward sizes the grid for the capacity n.
__device__ __forceinline__ int64_t live_n(int64_t n, const unsigned long long* n_dev) {
  if (!n_dev) return n;
  const int64_t d = static_cast<int64_t>(*n_dev);
  return d < n ? d : n;
}

template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads)
    k_upsweep(const uint32_t* __restrict__ keys, int64_t n, int shift, uint32_t mask,
              int bits, uint32_t* __restrict__ counts, int64_t tiles,
              const unsigned long long* __restrict__ n_dev) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ uint32_t hist[kWarps][256];
  const int t = threadIdx.x, w = t >> 5;
  n = live_n(n, n_dev);
#pragma unroll
  for (int k = 0; k < kWarps; ++k) hist[k][t] = 0;
  __syncthreads();
  (void)bits;
  // Thread-blocked: thread t counts the ITEMS consecutive keys
  // [tile0 + t*ITEMS, +ITEMS) (16-byte loads), run-length aggregated in
  // registers and flushed with one shared atomic per run into its warp's
  // histogram. Sorted-ish inputs (the instance list is generated in
  // (depth, row, column) order: runs of equal high digits) need few atomics;
  // random digits cost one uncontended shared atomic per key.
  const int64_t first = static_cast<int64_t>(blockIdx.x) * (ITEMS * kSortThreads) +
                        static_cast<int64_t>(t) * ITEMS;
  uint32_t key[ITEMS];
  if (first + ITEMS <= n) {
#pragma unroll
    for (int k = 0; k < ITEMS; k += 4) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(keys + first + k));
      key[k] = q.x;
      key[k + 1] = q.y;
      key[k + 2] = q.z;
      key[k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) key[k] = first + k < n ? __ldg(keys + first + k) : 0u;
  }
  uint32_t prev = 0xffffffffu, run = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (first + k < n) {
      const uint32_t d = (key[k] >> shift) & mask;
      if (d != prev) {
        if (run) atomicAdd(&hist[w][prev], run);
        prev = d;
        run = 0;
      }
      ++run;
    }
  }
  if (run) atomicAdd(&hist[w][prev], run);
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) s += hist[k][t];
  counts[static_cast<int64_t>(t) * tiles + blockIdx.x] = s;
}

// One block per digit: exclusive scan of counts[d][0..tiles) in place, total
// to digit_total[d].
__global__ void __launch_bounds__(1024)
    k_scan_rows(uint32_t* __restrict__ counts, int64_t tiles, uint32_t* __restrict__ digit_total) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry;
  uint32_t* row = counts + static_cast<int64_t>(blockIdx.x) * tiles;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < tiles; b += 1024) {
    const int64_t i = b + t;
    const uint32_t v = i < tiles ? row[i] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[w] = incl;
    __syncthreads();
    if (w == 0) {
      uint32_t s = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t before = carry + (w ? warp_sums[w - 1] : 0u) + incl - v;
    if (i < tiles) row[i] = before;
    __syncthreads();
    if (t == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (t == 0) digit_total[blockIdx.x] = carry;
}


// Stable scatter of one tile. Same warp-contiguous chunks as the upsweep:
// each warp ranks its ITEMS*32 elements against a warp-private running
// digit counter (rank = counter + popc(peers below me); the lowest peer
// lane advances the counter), keeping keys / values / ranks in registers;
// then ONE block-wide exclusive prefix per digit over the warps (in warp
// order) turns warp-local ranks into global positions. Element order inside
// the tile is (warp, step, lane) = index order, so the pass is stable.
// Three block barriers per tile.
// (A/B hook: an explicit minimum-blocks bound changes ptxas's register
// heuristic -- 1 gives 95 registers and a slower sort; unset keeps 40)
#ifdef DW_DOWN_MIN_BLOCKS
#define DW_DOWN_BOUNDS __launch_bounds__(kSortThreads, DW_DOWN_MIN_BLOCKS)
#else
#define DW_DOWN_BOUNDS __launch_bounds__(kSortThreads)
#endif
template <int ITEMS, int BITS>
__global__ void DW_DOWN_BOUNDS
    k_downsweep(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                int shift, uint32_t mask, int bits, const uint32_t* __restrict__ counts,
                int64_t tiles, const uint32_t* __restrict__ digit_base,  // digit totals
                uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                const unsigned long long* __restrict__ n_dev,
                const uint32_t* __restrict__ gather_src, uint32_t* __restrict__ gather_out) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  constexpr int TILE = ITEMS * kSortThreads;
  __shared__ uint32_t s_cnt[kWarps][256];  // warp digit counts -> tile-local offsets
  __shared__ uint32_t s_dstart[256];       // tile-local start of each digit's run
  __shared__ uint32_t s_gbase[256];        // global start of this tile's run of each digit
  __shared__ uint32_t s_wsum[kWarps];
  __shared__ uint32_t s_dsum[kWarps];
  __shared__ uint32_t s_key[TILE], s_val[TILE];
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  n = live_n(n, n_dev);
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) s_cnt[k][t] = 0;
  // global start of each digit = exclusive scan of the 256 digit totals
  // (k_scan_rows), done by every CTA instead of a separate launch
  const uint32_t dtot = digit_base[t];
  uint32_t dincl = dtot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, dincl, o);
    if (lane >= o) dincl += y;
  }
  if (lane == 31) s_dsum[w] = dincl;
  const uint32_t my_count = counts[static_cast<int64_t>(t) * tiles + blockIdx.x];
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * TILE;
  const int64_t base = tile0 + static_cast<int64_t>(w) * ITEMS * 32;
  (void)bits;
  uint32_t key[ITEMS], val[ITEMS], rank[ITEMS];
  const bool full = tile0 + TILE <= n;  // block-uniform: every element of the tile is live
  if (full) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      key[k] = __ldg(keys + base + k * 32 + lane);
      val[k] = __ldg(vals + base + k * 32 + lane);
    }
  } else {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int64_t e = base + k * 32 + lane;
      key[k] = e < n ? __ldg(keys + e) : 0u;
      val[k] = e < n ? __ldg(vals + e) : 0u;
    }
  }
  __syncthreads();
  {
    uint32_t before = dincl - dtot;
    for (int k = 0; k < w; ++k) before += s_dsum[k];
    s_gbase[t] = before + my_count;
  }
  // 1. rank inside the warp's contiguous chunk (warp-private counters)
  auto rank_items = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const bool valid = FULL || base + k * 32 + lane < n;
      const uint32_t d = (key[k] >> shift) & mask;
      const unsigned peers = digit_peers_t<BITS, FULL>(d, valid);
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (valid && leader == lane) {
        old = s_cnt[w][d];
        s_cnt[w][d] = old + __popc(peers);
      }
      rank[k] = __shfl_sync(kFull, old, leader) + __popc(peers & lt);
      __syncwarp();
    }
  };
  if (full)
    rank_items(std::true_type{});
  else
    rank_items(std::false_type{});
  __syncthreads();
  // 2. thread t owns digit t: tile total, exclusive scan over digits
  uint32_t tot = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) tot += s_cnt[k][t];
  uint32_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  uint32_t start = incl - tot;
  for (int k = 0; k < w; ++k) start += s_wsum[k];
  s_dstart[t] = start;
  uint32_t run = start;  // warp offsets inside the digit's run, in warp order
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    const uint32_t c = s_cnt[k][t];
    s_cnt[k][t] = run;
    run += c;
  }
  __syncthreads();
  // 3. local sort through shared memory (stable: warp, step, lane order)
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (base + k * 32 + lane < n) {
      const uint32_t local = s_cnt[w][(key[k] >> shift) & mask] + rank[k];
      s_key[local] = key[k];
      s_val[local] = val[k];
    }
  }
  __syncthreads();
  // 4. coalesced write-out: consecutive threads write consecutive elements of
  //    each digit's run
  const int count = static_cast<int>(n - tile0 < TILE ? n - tile0 : TILE);
  for (int i = t; i < count; i += kSortThreads) {
    const uint32_t kk = s_key[i];
    const uint32_t d = (kk >> shift) & mask;
    const uint32_t g = s_gbase[d] + (static_cast<uint32_t>(i) - s_dstart[d]);
    keys_out[g] = kk;
    vals_out[g] = s_val[i];
    if (gather_src) gather_out[g] = __ldg(gather_src + s_val[i]);  // sorted payload
  }
}

constexpr int kScanItems = 8;
constexpr int kScanTile = kSortThreads * kScanItems;  // 2048 elements

// MODE 0: in[] as is; 1: in[] is a packed tile rectangle (x0 | y0 << 8 |
// (x1-1) << 16 | (y1-1) << 24, empty: y0 > y1-1) and the scan runs on
// (coarse 8x4-tile blocks it touches << 34 | tiles it touches) -- both offsets
// of block binning in one pass (raster_blockbin.cu).
template <int MODE>
__device__ __forceinline__ unsigned long long scan_widen(uint32_t x) {
  if (MODE == 1) {
    const int x0 = (int)(x & 0xffu), y0 = (int)((x >> 8) & 0xffu);
    const int x1 = (int)((x >> 16) & 0xffu), y1 = (int)(x >> 24);
    if (y0 > y1) return 0ull;
    const unsigned long long tiles = static_cast<unsigned long long>((x1 - x0 + 1) * (y1 - y0 + 1));
    const unsigned long long blocks =
        static_cast<unsigned long long>((x1 / 8 - x0 / 8 + 1) * (y1 / 4 - y0 / 4 + 1));
    return (blocks << kBBTileBits) | tiles;
  }
  return x;
}

// Inclusive scan u32 -> u64 of widen(in[order[i]]) (order may be null) as
// reduce -> scan of the tile sums -> rescan: three launches and no
// inter-CTA waiting (a decoupled look-back chains the CTAs of a wave that
// start together: 30-40 us for 3M elements against ~10 here).
template <int MODE>
__global__ void __launch_bounds__(kSortThreads)
    k_scan_reduce(const uint32_t* __restrict__ in, const uint32_t* __restrict__ order, int64_t n,
                  unsigned long long* __restrict__ sums) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ unsigned long long s_w[kSortThreads / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * kScanTile;
  unsigned long long x = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t e = tile0 + k * kSortThreads + t;
    if (e < n) x += scan_widen<MODE>(__ldg(in + (order ? __ldg(order + e) : e)));
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  if (lane == 0) s_w[w] = x;
  __syncthreads();
  if (t == 0) {
    unsigned long long a = 0;
#pragma unroll
    for (int k = 0; k < kSortThreads / 32; ++k) a += s_w[k];
    sums[blockIdx.x] = a;
  }
}

// One CTA: exclusive scan of the tile sums, in place.
__global__ void __launch_bounds__(1024) k_scan_top(unsigned long long* __restrict__ sums, int64_t tiles) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long s_w[32];
  __shared__ unsigned long long s_carry;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) s_carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < tiles; b += 1024) {
    const int64_t i = b + t;
    const unsigned long long v = i < tiles ? sums[i] : 0ull;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    if (w == 0) {
      const unsigned long long sv = s_w[lane];
      unsigned long long si = sv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, si, o);
        if (lane >= o) si += y;
      }
      s_w[lane] = si - sv;
    }
    __syncthreads();
    const unsigned long long carry = s_carry;
    if (i < tiles) sums[i] = carry + s_w[w] + incl - v;
    __syncthreads();
    if (t == 1023) s_carry = carry + s_w[w] + incl;
    __syncthreads();
  }
}

// Block binning's level-1 entries (MODE 1): element e (a depth-ordered
// Gaussian, packed rectangle in[e], id ids[e]) writes (block id, id) for every
// coarse 8x4-tile block its rectangle touches at its exclusive block offset;
// only the last element's inclusive (blocks << 34 | tiles) goes to out[n-1].
struct ScanEntries {
  const uint32_t* ids = nullptr;
  uint32_t* bkey = nullptr;
  uint32_t* bval = nullptr;
  uint64_t cap = 0;  // entries the buffers hold (no write past it)
  int nbx = 0;       // coarse blocks per row
};

#ifndef DW_SCAN_MIN_BLOCKS
#define DW_SCAN_MIN_BLOCKS 6  // 40 registers (62 unbounded): C5 entry scan ~4 % faster
#endif
#if DW_SCAN_MIN_BLOCKS > 0
#define DW_SCAN_BOUNDS __launch_bounds__(kSortThreads, DW_SCAN_MIN_BLOCKS)
#else
#define DW_SCAN_BOUNDS __launch_bounds__(kSortThreads)
#endif
template <int MODE>
__global__ void DW_SCAN_BOUNDS
    k_scan_apply(const uint32_t* __restrict__ in, const uint32_t* __restrict__ order, int64_t n,
                 const unsigned long long* __restrict__ sums, uint64_t* __restrict__ out,
                 const ScanEntries ent) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ uint32_t s_in[kScanTile + kScanTile / 32];          // padded: conflict-free transpose
  __shared__ unsigned long long s_out[kScanTile + kScanTile / 16];
  __shared__ unsigned long long s_wsum[kSortThreads / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * kScanTile;
  // coalesced load (element k*256 + t), transposed so thread t scans [8t, 8t+8)
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int i = k * kSortThreads + t;
    const int64_t e = tile0 + i;
    s_in[i + (i >> 5)] = e < n ? __ldg(in + (order ? __ldg(order + e) : e)) : 0u;
  }
  __syncthreads();
  uint32_t v[kScanItems];
  unsigned long long tot = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int i = t * kScanItems + k;
    v[k] = s_in[i + (i >> 5)];
    tot += scan_widen<MODE>(v[k]);
  }
  unsigned long long incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  unsigned long long wbase = 0;
#pragma unroll
  for (int k = 0; k < kSortThreads / 32; ++k) wbase += k < w ? s_wsum[k] : 0ull;
  unsigned long long run = sums[blockIdx.x] + wbase + incl - tot;
  if (MODE == 1) {
    // exclusive block offsets to shared memory (thread-blocked), then each
    // warp expands 32 consecutive Gaussians at a time into their entries with
    // consecutive lanes on consecutive entries (coalesced stores)
    uint32_t* s_bo = reinterpret_cast<uint32_t*>(s_out);
    const int64_t e0 = tile0 + static_cast<int64_t>(t) * kScanItems;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int i = t * kScanItems + k;
      s_bo[i + (i >> 5)] = static_cast<uint32_t>(run >> kBBTileBits);
      run += scan_widen<MODE>(v[k]);
      if (e0 + k == n - 1) out[n - 1] = run;
    }
    uint32_t gids[kScanItems];  // all rounds' ids in flight at once
#pragma unroll
    for (int r = 0; r < kScanItems; ++r) {
      const int64_t e = tile0 + w * (32 * kScanItems) + r * 32 + lane;
      gids[r] = e < n ? __ldg(ent.ids + e) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kScanItems; ++r) {
      const int i = w * (32 * kScanItems) + r * 32 + lane;
      const int64_t e = tile0 + i;
      const uint32_t x = e < n ? s_in[i + (i >> 5)] : 0x0000ff00u;
      const int x0 = (int)(x & 0xffu), y0 = (int)((x >> 8) & 0xffu);
      const int x1 = (int)((x >> 16) & 0xffu), y1 = (int)(x >> 24);
      const int bx0 = x0 / 8, by0 = y0 / 4;
      const int bw = x1 / 8 - bx0 + 1;
      int nb = y0 > y1 ? 0 : bw * (y1 / 4 - by0 + 1);
      const uint32_t o = s_bo[i + (i >> 5)];
      if (static_cast<uint64_t>(o) + static_cast<uint64_t>(nb) > ent.cap) nb = 0;  // host regrows
      const uint32_t gid = gids[r];
      // every Gaussian's first block (its top-left one) is written by its own
      // lane; only the entries beyond the first (~1/3 of them at 1080p) go
      // through the warp-cooperative expansion -- one trip per round instead
      // of two, and none when every rectangle sits inside one block
      if (nb > 0) {
        ent.bkey[o] = static_cast<uint32_t>(by0 * ent.nbx + bx0);
        ent.bval[o] = gid;
      }
      const int extra = nb > 1 ? nb - 1 : 0;
      int incl = extra;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += y;
      }
      const int excl = incl - extra;
      const int total = __shfl_sync(kFull, incl, 31);
      for (int q0 = 0; q0 < total; q0 += 32) {  // warp-uniform trips
        const int q = q0 + lane;
        int owner = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int probe = owner + step;
          if (__shfl_sync(kFull, excl, probe) <= q) owner = probe;
        }
        const int kk = q - __shfl_sync(kFull, excl, owner) + 1;  // entry 1.. of the owner
        const int w_ = __shfl_sync(kFull, bw, owner);
        const int ox = __shfl_sync(kFull, bx0, owner), oy = __shfl_sync(kFull, by0, owner);
        const uint32_t oo = __shfl_sync(kFull, o, owner);
        const uint32_t og = __shfl_sync(kFull, gid, owner);
        if (q < total) {
          const int row = static_cast<int>((static_cast<float>(kk) + 0.5f) / static_cast<float>(w_));
          ent.bkey[oo + kk] = static_cast<uint32_t>((oy + row) * ent.nbx + ox + (kk - row * w_));
          ent.bval[oo + kk] = og;
        }
      }
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    run += scan_widen<MODE>(v[k]);
    const int i = t * kScanItems + k;
    s_out[i + (i >> 4)] = run;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int i = k * kSortThreads + t;
    const int64_t e = tile0 + i;
    if (e < n) out[e] = s_out[i + (i >> 4)];
  }
}

__global__ void k_iota_depthkey(int P, const float* __restrict__ depths, const int* __restrict__ radii,
                                uint32_t* __restrict__ dkey, uint32_t* __restrict__ ids) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  dkey[i] = radii[i] > 0 ? __float_as_uint(depths[i]) : 0xffffffffu;
  ids[i] = static_cast<uint32_t>(i);
}

__device__ __forceinline__ void rect_of(float2 m, int radius, int tiles_x, int tiles_y, int* r) {
  const float fr = (float)radius;
  const int v0 = (int)((m.x - fr) / (float)kTile), v1 = (int)((m.y - fr) / (float)kTile);
  const int v2 = (int)((m.x + fr + (float)(kTile - 1)) / (float)kTile);
  const int v3 = (int)((m.y + fr + (float)(kTile - 1)) / (float)kTile);
  r[0] = min(tiles_x, max(0, v0));
  r[1] = min(tiles_y, max(0, v1));
  r[2] = min(tiles_x, max(0, v2));
  r[3] = min(tiles_y, max(0, v3));
}

// One lane per Gaussian in depth order; rects wider than a warp are written
// by the whole warp (C4-style scenes touch thousands of tiles).
__global__ void __launch_bounds__(256)
    k_duplicate_sorted(int P, const uint32_t* __restrict__ order, const float2* __restrict__ means2D,
                       const int* __restrict__ radii, const uint64_t* __restrict__ offsets,
                       int tiles_x, int tiles_y, uint32_t* __restrict__ tile_ids,
                       uint32_t* __restrict__ values, uint64_t cap) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int r[4] = {0, 0, 0, 0};
  uint64_t off = 0;
  uint32_t gid = 0;
  int area = 0;
  if (i < P) {
    gid = order ? order[i] : static_cast<uint32_t>(i);
    const int rad = radii[gid];
    if (rad > 0) {
      rect_of(means2D[gid], rad, tiles_x, tiles_y, r);
      off = i == 0 ? 0 : offsets[i - 1];
      area = (r[2] - r[0]) * (r[3] - r[1]);
      if (off + static_cast<uint64_t>(area) > cap) area = 0;  // over capacity: write nothing
    }
  }
  if (area == 0) r[0] = r[1] = r[2] = r[3] = 0;
  const bool big = area > 32;
  // Small rectangles, written by the whole warp: element e of the warp's
  // small-rectangle instances belongs to the lane whose [excl, excl + area)
  // holds it (5-step search over the lanes' exclusive scan), so consecutive
  // lanes store consecutive list positions instead of 32 scattered streams.
  {
    const int sa = big ? 0 : area;
    int incl = sa;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - sa;
    const int total = __shfl_sync(kFull, incl, 31);
    const int wdt = r[2] - r[0];
    for (int e0 = 0; e0 < total; e0 += 32) {  // warp-uniform trips: shuffles need every lane
      const int e = e0 + lane;
      int owner = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int probe = owner + step;
        if (__shfl_sync(kFull, excl, probe) <= e) owner = probe;  // probe <= 31
      }
      // lanes of the same owner are contiguous; the shuffles below are per lane
      const int k = e - __shfl_sync(kFull, excl, owner);
      const int w = __shfl_sync(kFull, wdt, owner);
      const int x0 = __shfl_sync(kFull, r[0], owner), y0 = __shfl_sync(kFull, r[1], owner);
      const uint64_t o = __shfl_sync(kFull, off, owner);
      const uint32_t g = __shfl_sync(kFull, gid, owner);
      if (e < total) {
        const int row = static_cast<int>((static_cast<float>(k) + 0.5f) / static_cast<float>(w));
        tile_ids[o + k] = static_cast<uint32_t>((y0 + row) * tiles_x + x0 + (k - row * w));
        values[o + k] = g;
      }
    }
  }
  unsigned todo = __ballot_sync(kFull, big);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1u;
    const int x0 = __shfl_sync(kFull, r[0], src);
    const int y0 = __shfl_sync(kFull, r[1], src);
    const int x1 = __shfl_sync(kFull, r[2], src);
    const int a = __shfl_sync(kFull, area, src);
    const uint64_t o = __shfl_sync(kFull, off, src);
    const uint32_t g = __shfl_sync(kFull, gid, src);
    const int w = x1 - x0;
    for (int k = lane; k < a; k += 32) {
      tile_ids[o + k] = static_cast<uint32_t>((y0 + k / w) * tiles_x + x0 + k % w);
      values[o + k] = g;
    }
  }
}

// ---------------------------------------------------------------------------
// Tile-first binning: duplicate the instances in Gaussian-index order, stable
// radix-sort them by tile (each tile's list then holds its Gaussians in index
// order), then sort every tile's list by depth in shared memory. A stable
// depth order over index order is the (depth, index) order -- the list the
// depth-first pipeline (global depth sort, then duplicate, then tile sort)
// produces -- without four LSD passes over all P Gaussians. The per-tile
// sort is a bitonic network on the 64-bit keys (depth bits << 32 | id), a
// total order equal to that one; lists longer than kSegCap are sorted in
// kSegCap chunks and merged pairwise in global scratch by the same CTA.
constexpr int kSegCap = 2048;

__device__ __forceinline__ void bitonic_smem(unsigned long long* a, int npad) {
  for (int k = 2; k <= npad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npad; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long x = a[i], y = a[l];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(256)
    k_segsort_depth(const uint2* __restrict__ ranges, const float* __restrict__ depths,
                    uint32_t* __restrict__ values, unsigned long long* __restrict__ scratch,
                    int ntiles, int64_t half, int min_n) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ unsigned long long s_k[kSegCap];
  const int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const uint2 r = ranges[tile];
  const int n = static_cast<int>(r.y - r.x);
  if (n <= 1 || n < min_n) return;  // min_n: only the lists another sort left over
  auto key_of = [&](int i) {
    const uint32_t id = values[r.x + i];
    return static_cast<unsigned long long>(__float_as_uint(__ldg(depths + id))) << 32 | id;
  };
  if (n <= kSegCap) {
    int npad = 32;
    while (npad < n) npad <<= 1;
    for (int i = threadIdx.x; i < npad; i += blockDim.x) s_k[i] = i < n ? key_of(i) : ~0ull;
    __syncthreads();
    bitonic_smem(s_k, npad);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      values[r.x + i] = static_cast<uint32_t>(s_k[i]);
    return;
  }
  // long list: sorted chunks into scratch[r.x ..], then pairwise merges
  // per-tile ping-pong halves: [r.x, r.y) of scratch[0, half) and of scratch[half, 2 half)
  unsigned long long* bufs[2] = {scratch + r.x, scratch + half + r.x};
  for (int c0 = 0; c0 < n; c0 += kSegCap) {
    const int m = min(kSegCap, n - c0);
    for (int i = threadIdx.x; i < kSegCap; i += blockDim.x) s_k[i] = i < m ? key_of(c0 + i) : ~0ull;
    __syncthreads();
    bitonic_smem(s_k, kSegCap);
    for (int i = threadIdx.x; i < m; i += blockDim.x) bufs[0][c0 + i] = s_k[i];
    __syncthreads();
  }
  int cur = 0;
  for (int run = kSegCap; run < n; run <<= 1, cur ^= 1) {
    const unsigned long long* in = bufs[cur];
    unsigned long long* out = bufs[cur ^ 1];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int a0 = (i / (2 * run)) * 2 * run;  // pair of runs [a0, a0+run), [a0+run, a0+2run)
      const int b0 = min(a0 + run, n), b1 = min(a0 + 2 * run, n);
      const unsigned long long x = in[i];
      // rank in the other run (keys are distinct): elements of the other run below x
      const bool inA = i < b0;
      int lo = inA ? b0 : a0, hi = inA ? b1 : b0;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (in[mid] < x) lo = mid + 1; else hi = mid;
      }
      const int rank = inA ? (i - a0) + (lo - b0) : (i - b0) + (lo - a0);
      out[a0 + rank] = x;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    values[r.x + i] = static_cast<uint32_t>(bufs[cur][i]);
}

// ---------------------------------------------------------------------------
// Dense binning (tile-major list construction) for scenes whose Gaussians
// cover large tile rectangles (the high-contention C4 scene: ~4,500 tiles per
// Gaussian, 0.9 G instances). Instead of duplicating every instance and
// radix-sorting 0.9 G keys, each tile's list is built directly:
//   1. k_dense_rects: the depth-ordered Gaussians' tile rectangles, packed,
//      plus per SEGMENT of the depth order (kDenseSeg segments) a 2D
//      difference grid of the rectangles (4 shared atomics per Gaussian);
//   2. k_dense_ranges: 2D prefix sums -> per (segment, tile) counts -> tile
//      ranges and each segment's write offset inside each tile's list;
//   3. k_dense_fill: a warp owns (segment, 8 consecutive tiles of a row),
//      turns each rectangle into an 8-bit mask of its tiles and appends the
//      Gaussian to each tile by ballot compaction (order preserved).
// Output is identical to the sort path -- per tile, Gaussians in (depth,
// index) order -- for ~P x tiles / 256 warp steps instead of duplicating and
// sorting I instances; raster.cu picks it when P x tiles <= 4 I.
//
// Packed rectangle: x0 | y0 << 8 | (x1-1) << 16 | (y1-1) << 24 (tile units
// < 256); an empty rectangle packs as y0 = 255 > y1-1 = 0.
constexpr uint32_t kEmptyRect = 0x0000ff00u;
constexpr int kDenseSeg = 16;

__global__ void __launch_bounds__(256)
    k_dense_rects(int P, const uint32_t* __restrict__ order, const float2* __restrict__ means2D,
                  const int* __restrict__ radii, int tiles_x, int tiles_y,
                  uint2* __restrict__ rects, int* __restrict__ diff) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  extern __shared__ int s_diff[];  // (tiles_y + 1) x (tiles_x + 1) corner counts
  const int W1 = tiles_x + 1, cells = W1 * (tiles_y + 1);
  const int per_seg = gridDim.x / kDenseSeg;  // blocks per segment
  const int seg = blockIdx.x / per_seg, sub = blockIdx.x % per_seg;
  const int64_t lo = static_cast<int64_t>(P) * seg / kDenseSeg;
  const int64_t hi = static_cast<int64_t>(P) * (seg + 1) / kDenseSeg;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) s_diff[c] = 0;
  __syncthreads();
  for (int64_t i = lo + static_cast<int64_t>(sub) * blockDim.x + threadIdx.x; i < hi;
       i += static_cast<int64_t>(per_seg) * blockDim.x) {
    const uint32_t gid = order[i];
    uint32_t packed = kEmptyRect;
    const int rad = radii[gid];
    if (rad > 0) {
      int r[4];
      rect_of(means2D[gid], rad, tiles_x, tiles_y, r);
      if (r[2] > r[0] && r[3] > r[1]) {
        packed = (uint32_t)r[0] | (uint32_t)r[1] << 8 | (uint32_t)(r[2] - 1) << 16 |
                 (uint32_t)(r[3] - 1) << 24;
        atomicAdd(&s_diff[r[1] * W1 + r[0]], 1);
        atomicAdd(&s_diff[r[1] * W1 + r[2]], -1);
        atomicAdd(&s_diff[r[3] * W1 + r[0]], -1);
        atomicAdd(&s_diff[r[3] * W1 + r[2]], 1);
      }
    }
    rects[i] = make_uint2(packed, gid);
  }
  __syncthreads();
  int* d = diff + static_cast<int64_t>(seg) * cells;
  int* dt = diff + static_cast<int64_t>(kDenseSeg) * cells;  // all segments
  for (int c = threadIdx.x; c < cells; c += blockDim.x)
    if (s_diff[c]) {
      atomicAdd(&d[c], s_diff[c]);
      atomicAdd(&dt[c], s_diff[c]);
    }
}

// One block per segment and one for all of them: diff[g][cells] -> in place 2D
// inclusive prefix sums in shared memory (the count of the segment's
// rectangles containing each tile; g = kDenseSeg: all segments).
__global__ void __launch_bounds__(1024)
    k_dense_prefix2d(int* __restrict__ diff, int tiles_x, int tiles_y) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  extern __shared__ int s_g[];
  const int W1 = tiles_x + 1, H1 = tiles_y + 1, cells = W1 * H1, t = threadIdx.x;
  int* g = diff + static_cast<int64_t>(blockIdx.x) * cells;
  for (int c = t; c < cells; c += 1024) s_g[c] = g[c];
  __syncthreads();
  for (int y = t; y < H1; y += 1024) {
    int run = 0;
    for (int x = 0; x < W1; ++x) s_g[y * W1 + x] = run += s_g[y * W1 + x];
  }
  __syncthreads();
  for (int x = t; x < W1; x += 1024) {
    int run = 0;
    for (int y = 0; y < H1; ++y) s_g[y * W1 + x] = run += s_g[y * W1 + x];
  }
  __syncthreads();
  for (int c = t; c < cells; c += 1024) g[c] = s_g[c];
}

// One block: tile ranges from the all-segment counts ((0, 0) when empty, the
// reference layout). With a live-count bound (n_dev, no-sync forward) an
// over-capacity frame renders empty.
__global__ void __launch_bounds__(1024)
    k_dense_ranges(const int* __restrict__ counts, int tiles_x, int tiles_y,
                   uint2* __restrict__ ranges, const unsigned long long* __restrict__ n_dev) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ uint32_t s_wsum[32];
  __shared__ unsigned long long s_total;
  const int W1 = tiles_x + 1, cells = W1 * (tiles_y + 1), t = threadIdx.x;
  const int ntiles = tiles_x * tiles_y;
  const int* tot = counts + static_cast<int64_t>(kDenseSeg) * cells;
  const int per = (ntiles + 1023) / 1024;
  const int lane = t & 31, w = t >> 5;
  uint32_t local = 0;
  for (int k = 0; k < per; ++k) {
    const int tile = t * per + k;
    if (tile < ntiles) local += (uint32_t)tot[(tile / tiles_x) * W1 + tile % tiles_x];
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
    if (lane == 31) s_total = vi;
  }
  __syncthreads();
  const bool over = n_dev && *n_dev < s_total;
  uint32_t run = s_wsum[w] + incl - local;
  for (int k = 0; k < per; ++k) {
    const int tile = t * per + k;
    if (tile >= ntiles) break;
    const uint32_t c = (uint32_t)tot[(tile / tiles_x) * W1 + tile % tiles_x];
    ranges[tile] = (c == 0 || over) ? make_uint2(0u, 0u) : make_uint2(run, run + c);
    run += c;
  }
}

// Block = one depth-order segment x 8 warps; warp = 8 consecutive tiles of a
// row. The segment's rectangles are staged 1,024 at a time; each lane turns
// one rectangle into the 8-bit mask of the warp's tiles it covers and the warp
// appends it to each of those tiles' lists by ballot compaction.
#ifndef DW_DENSE_FILL_MIN_BLOCKS
#define DW_DENSE_FILL_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(256, DW_DENSE_FILL_MIN_BLOCKS)
    k_dense_fill(int P, const uint2* __restrict__ rects, const int* __restrict__ counts,
                 const uint2* __restrict__ ranges, int tiles_x, int tiles_y, int groups_x,
                 uint32_t* __restrict__ values,
                 const unsigned long long* __restrict__ n_dev, uint64_t total_cap) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ uint2 s_r[1024];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ngroups = groups_x * tiles_y;
  const int blocks_per_seg = (ngroups + 7) / 8;
  const int seg = blockIdx.x / blocks_per_seg;
  const int grp = (blockIdx.x % blocks_per_seg) * 8 + w;
  const int ntiles = tiles_x * tiles_y;
  // No-sync forward: the clamped live count is 0 when the instances exceed the
  // reserve (the frame renders empty) -- and when there are none to write.
  if (n_dev && *n_dev == 0ull) return;
  (void)total_cap;
  const int ty = grp / groups_x, tx0 = (grp % groups_x) * 8;
  const bool live = grp < ngroups;
  // where this segment starts in each of the warp's 8 tile lists: the tile's
  // range start plus the earlier segments' counts (lanes 0-7, one tile each)
  uint32_t off = 0;
  if (live && lane < 8 && tx0 + lane < tiles_x) {
    const int W1 = tiles_x + 1, cells = W1 * (tiles_y + 1);
    const int cell = ty * W1 + tx0 + lane;
    off = ranges[ty * tiles_x + tx0 + lane].x;
    for (int sg = 0; sg < seg; ++sg) off += (uint32_t)counts[static_cast<int64_t>(sg) * cells + cell];
  }
  uint32_t* dst[8];  // next write position in each of the warp's 8 tile lists
#pragma unroll
  for (int k = 0; k < 8; ++k) dst[k] = values + __shfl_sync(kFull, off, k);
  (void)ntiles;
  const int64_t lo = static_cast<int64_t>(P) * seg / kDenseSeg;
  const int64_t hi = static_cast<int64_t>(P) * (seg + 1) / kDenseSeg;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t last = static_cast<uint32_t>(min(tiles_x - 1 - tx0, 7));  // last tile offset
  for (int64_t c0 = lo; c0 < hi; c0 += 1024) {
    const int nc = static_cast<int>(hi - c0 < 1024 ? hi - c0 : 1024);
    __syncthreads();
    for (int k = threadIdx.x; k < nc; k += 256) s_r[k] = rects[c0 + k];
    __syncthreads();
    if (!live) continue;
    for (int j = 0; j < nc; j += 32) {
      const int k = j + lane;
      const uint2 r = k < nc ? s_r[k] : make_uint2(kEmptyRect, 0u);
      const int x0 = (int)(r.x & 0xffu) - tx0, y0 = (int)((r.x >> 8) & 0xffu);
      const int x1 = (int)((r.x >> 16) & 0xffu) - tx0, y1 = (int)(r.x >> 24);
      const int a = max(x0, 0), b = min(x1, (int)last);
      uint32_t m = 0;
      if (y0 <= ty && ty <= y1 && a <= b) m = (0xffu >> (7 - b)) & (0xffu << a);
      if (__ballot_sync(kFull, m != 0u) == 0u) continue;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool in = (m >> q) & 1u;
        const unsigned bq = __ballot_sync(kFull, in);
        if (in) dst[q][__popc(bq & lt)] = r.y;
        dst[q] += __popc(bq);
      }
    }
  }
}

// Tile id of every list position (debug key materialisation after dense
// binning, which writes no tile-id array): one warp per tile.
__global__ void k_tiles_from_ranges(const uint2* __restrict__ ranges, int ntiles,
                                    uint32_t* __restrict__ tiles) {
  const int lane = threadIdx.x & 31;
  const int tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (tile >= ntiles) return;
  const uint2 r = ranges[tile];
  for (uint32_t i = r.x + lane; i < r.y; i += 32) tiles[i] = (uint32_t)tile;
}

// No-host-sync sizing: the live instance count is the scan total when it fits
// the reserved capacity, else 0 (the frame renders empty) and the overflow
// flag is raised for the host to read later.
__global__ void k_clamp_total(const uint64_t* __restrict__ offsets, int P, uint64_t cap,
                              unsigned long long* __restrict__ n_live,
                              unsigned int* __restrict__ overflow, int sticky) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  const uint64_t total = P > 0 ? offsets[P - 1] : 0;
  const bool fits = total <= cap;
  *n_live = fits ? total : 0ull;
  // sticky: the flag accumulates over a view batch (cleared by the caller)
  if (!fits) *overflow = 1u;
  else if (!sticky) *overflow = 0u;
}

// Tile ranges from the sorted tile ids by search rather than by a pass over
// every instance: warp t finds B(t) and B(t+1), B(x) = #ids < x (lower
// bounds, 32-ary: six rounds of 32 probes for 10^9 instances), and writes
// ranges[t] = [B(t), B(t+1)), or (0, 0) for an empty tile as the reference
// layout has it.
__device__ __forceinline__ int64_t lower_bound_warp(const uint32_t* __restrict__ a, int64_t L,
                                                    uint32_t x, int lane) {
  int64_t lo = 0, hi = L;  // the bound lies in [lo, hi]
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + static_cast<int64_t>(lane) * step;
    const int c = __popc(__ballot_sync(kFull, p < hi && __ldg(a + p) < x));
    const int64_t nlo = c > 0 ? lo + static_cast<int64_t>(c - 1) * step + 1 : lo;
    hi = min(hi, lo + static_cast<int64_t>(c) * step);
    lo = nlo;
  }
  const int64_t p = lo + lane;
  return lo + __popc(__ballot_sync(kFull, p < hi && __ldg(a + p) < x));
}

__global__ void k_ranges_search(int64_t L, const uint32_t* __restrict__ tiles,
                                uint2* __restrict__ ranges, int ntiles,
                                const unsigned long long* __restrict__ n_dev) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int t = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  if (t >= ntiles) return;
  L = live_n(L, n_dev);
  const int64_t b0 = lower_bound_warp(tiles, L, static_cast<uint32_t>(t), lane);
  const int64_t b1 = lower_bound_warp(tiles, L, static_cast<uint32_t>(t) + 1u, lane);
  if (lane == 0)
    ranges[t] = b1 > b0 ? make_uint2(static_cast<uint32_t>(b0), static_cast<uint32_t>(b1))
                        : make_uint2(0u, 0u);
}

__global__ void k_make_keys(int64_t L, const uint32_t* __restrict__ tiles,
                            const uint32_t* __restrict__ values, const float* __restrict__ depths,
                            uint64_t* __restrict__ keys) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < L) keys[i] = (static_cast<uint64_t>(tiles[i]) << 32) | __float_as_uint(depths[values[i]]);
}

// Longest-processing-time-first tile order for the blend kernels: tiles
// bucketed by list length on a 1/8-octave log scale, longest buckets first
// (order within a bucket is arbitrary). The few very long tiles then start in
// the first wave instead of trailing the last one.
__global__ void __launch_bounds__(1024)
    k_tile_order(const uint2* __restrict__ ranges, int ntiles, uint32_t* __restrict__ order) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ uint32_t cnt[256];
  const int t = threadIdx.x;
  if (t < 256) cnt[t] = 0;
  __syncthreads();
  auto bucket = [&](int tile) {
    const uint2 r = ranges[tile];
    const float lg = __log2f(static_cast<float>(r.y - r.x) + 1.0f);
    return 255 - min(255, static_cast<int>(8.0f * lg));
  };
  for (int i = t; i < ntiles; i += 1024) atomicAdd(&cnt[bucket(i)], 1u);
  __syncthreads();
  if (t < 32) {  // exclusive scan of the 256 bucket counts by one warp
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = cnt[t * 8 + k];
      sum += v[k];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (t >= o) incl += y;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cnt[t * 8 + k] = run;
      run += v[k];
    }
  }
  __syncthreads();
  for (int i = t; i < ntiles; i += 1024) order[atomicAdd(&cnt[bucket(i)], 1u)] = static_cast<uint32_t>(i);
}

inline unsigned blocks_for(int64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

}  // namespace

// Tile size per pass: 16 items/thread (4096-element tiles) once there are
// enough tiles to fill every SM a few times over, else 4 (1024-element tiles)
// so small inputs (the P-element depth sort) still spread over 148 SMs.
constexpr int64_t kBigSortN = int64_t(148) * 4 * 4096;
#ifndef DW_SORT_BIG_ITEMS
#define DW_SORT_BIG_ITEMS 8  // A/B on C3: 0.836 vs 0.843 ms forward (16)
#endif
#ifndef DW_SORT_SMALL_MIN
#define DW_SORT_SMALL_MIN kBigSortN
#endif
inline int sort_items(int64_t n) {
  // A/B hook: DW_SORT_ITEMS=4/8/16 forces the items per thread
  static const int forced = [] {
    const char* e = std::getenv("DW_SORT_ITEMS");
    const int v = e ? std::atoi(e) : 0;
    return (v == 4 || v == 8 || v == 16) ? v : 0;
  }();
  if (forced) return forced;
  return n >= DW_SORT_SMALL_MIN ? DW_SORT_BIG_ITEMS : 4;
}

size_t radix_sort_temp_bytes(int64_t n) {
  const int64_t tiles = (n + 1023) / 1024;  // worst case: 4-item tiles
  return (static_cast<size_t>(tiles) * 256 + 256) * sizeof(uint32_t) + 256;
}

size_t scan_temp_bytes(int64_t n) {  // one u64 sum per tile (+ 1)
  return static_cast<size_t>((n + kScanTile - 1) / kScanTile + 1) * sizeof(unsigned long long);
}

// Stable LSD sort of (k[cur], v[cur]) on bits [0, bits); returns the index
// (0/1) of the double buffer holding the result.
template <int ITEMS>
void launch_downsweep(int bits, unsigned grid, cudaStream_t s, const uint32_t* k, const uint32_t* v,
                      int64_t n, int shift, uint32_t mask, const uint32_t* counts, int64_t tiles,
                      const uint32_t* digit, uint32_t* ko, uint32_t* vo,
                      const unsigned long long* n_dev, const uint32_t* gsrc, uint32_t* gout) {
#define DW_DOWN(B)                                                                            \
  case B:                                                                                     \
    launch_pdl(k_downsweep<ITEMS, B>, grid, kSortThreads, 0, s, k, v, n, shift, mask, bits,  \
               counts, tiles, digit, ko, vo, n_dev, gsrc, gout);                              \
    break;
  switch (bits) {
    DW_DOWN(1)
    DW_DOWN(2)
    DW_DOWN(3)
    DW_DOWN(4)
    DW_DOWN(5)
    DW_DOWN(6)
    DW_DOWN(7)
    default:
      launch_pdl(k_downsweep<ITEMS, 8>, grid, kSortThreads, 0, s, k, v, n, shift, mask, bits,
                 counts, tiles, digit, ko, vo, n_dev, gsrc, gout);
  }
#undef DW_DOWN
}

int radix_sort_pairs(uint32_t* k[2], uint32_t* v[2], int64_t n, int bits, void* temp,
                     cudaStream_t s, const unsigned long long* n_dev, const uint32_t* gather_src,
                     uint32_t* gather_out) {
  int cur = 0;
  if (n <= 0 || bits <= 0) return cur;
  const int items = sort_items(n);
  const int64_t tile_n = static_cast<int64_t>(items) * kSortThreads;
  const int64_t tiles = (n + tile_n - 1) / tile_n;
  uint32_t* counts = static_cast<uint32_t*>(temp);
  uint32_t* digit = counts + static_cast<size_t>(tiles) * 256;
  const unsigned grid = static_cast<unsigned>(tiles);
  for (int shift = 0; shift < bits; shift += 8) {
    const int b = bits - shift < 8 ? bits - shift : 8;
    const uint32_t mask = (1u << b) - 1u;
    const bool last = shift + 8 >= bits;
    switch (items) {
      case 16:
        launch_pdl(k_upsweep<16>, grid, kSortThreads, 0, s, k[cur], n, shift, mask, b, counts,
                   tiles, n_dev);
        break;
      case 8:
        launch_pdl(k_upsweep<8>, grid, kSortThreads, 0, s, k[cur], n, shift, mask, b, counts, tiles,
                   n_dev);
        break;
      default:
        launch_pdl(k_upsweep<4>, grid, kSortThreads, 0, s, k[cur], n, shift, mask, b, counts, tiles,
                   n_dev);
    }
    launch_pdl(k_scan_rows, 256, 1024, 0, s, counts, tiles, digit);  // digit totals: scanned per CTA
    switch (items) {
      case 16:
        launch_downsweep<16>(b, grid, s, k[cur], v[cur], n, shift, mask, counts, tiles, digit,
                             k[cur ^ 1], v[cur ^ 1], n_dev, last ? gather_src : nullptr,
                             gather_out);
        break;
      case 8:
        launch_downsweep<8>(b, grid, s, k[cur], v[cur], n, shift, mask, counts, tiles, digit,
                            k[cur ^ 1], v[cur ^ 1], n_dev, last ? gather_src : nullptr,
                            gather_out);
        break;
      default:
        launch_downsweep<4>(b, grid, s, k[cur], v[cur], n, shift, mask, counts, tiles, digit,
                            k[cur ^ 1], v[cur ^ 1], n_dev, last ? gather_src : nullptr,
                            gather_out);
    }
    cur ^= 1;
  }
  DW_CUDA(cudaGetLastError());
  return cur;
}

void launch_scan_rows(uint32_t* counts, int64_t tiles, uint32_t* digit_total, cudaStream_t s) {
  launch_pdl(k_scan_rows, 256, 1024, 0, s, counts, tiles, digit_total);
  DW_CUDA(cudaGetLastError());
}

const uint32_t* radix_sort_digit_totals(const void* temp, int64_t n) {
  const int64_t tile_n = static_cast<int64_t>(sort_items(n)) * kSortThreads;
  const int64_t tiles = (n + tile_n - 1) / tile_n;
  return static_cast<const uint32_t*>(temp) + static_cast<size_t>(tiles) * 256;
}

void inclusive_scan_gather(const uint32_t* in, const uint32_t* order, int64_t n, uint64_t* out,
                           void* temp, cudaStream_t s, int mode) {
  if (n <= 0) return;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  auto* sums = static_cast<unsigned long long*>(temp);
  const unsigned grid = static_cast<unsigned>(tiles);
  if (mode == 1)
    launch_pdl(k_scan_reduce<1>, grid, kSortThreads, 0, s, in, order, n, sums);
  else
    launch_pdl(k_scan_reduce<0>, grid, kSortThreads, 0, s, in, order, n, sums);
  launch_pdl(k_scan_top, 1, 1024, 0, s, sums, tiles);
  if (mode == 1)
    throw std::invalid_argument("scan mode 1 runs through block_entries_scan");
  launch_pdl(k_scan_apply<0>, grid, kSortThreads, 0, s, in, order, n, sums, out, ScanEntries{});
  DW_CUDA(cudaGetLastError());
}

void block_entries_scan(const uint32_t* rect_sorted, const uint32_t* order, int64_t n,
                        uint64_t* out, void* temp, int nbx, uint32_t* bkey, uint32_t* bval,
                        uint64_t cap, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  auto* sums = static_cast<unsigned long long*>(temp);
  const unsigned grid = static_cast<unsigned>(tiles);
  launch_pdl(k_scan_reduce<1>, grid, kSortThreads, 0, s, rect_sorted, nullptr, n, sums);
  launch_pdl(k_scan_top, 1, 1024, 0, s, sums, tiles);
  ScanEntries ent;
  ent.ids = order;
  ent.bkey = bkey;
  ent.bval = bval;
  ent.cap = cap;
  ent.nbx = nbx;
  launch_pdl(k_scan_apply<1>, grid, kSortThreads, 0, s, rect_sorted, nullptr, n, sums, out, ent);
  DW_CUDA(cudaGetLastError());
}

void launch_depth_keys(int P, const float* depths, const int* radii, uint32_t* dkey, uint32_t* ids,
                       cudaStream_t s) {
  if (P <= 0) return;
  launch_pdl(k_iota_depthkey, blocks_for(P, 256), 256, 0, s, P, depths, radii, dkey, ids);
  DW_CUDA(cudaGetLastError());
}

void launch_duplicate_sorted(int P, const uint32_t* order, const float2* means2D, const int* radii,
                             const uint64_t* offsets, const CamParams& cam, uint32_t* tile_ids,
                             uint32_t* values, uint64_t cap, cudaStream_t s) {
  if (P <= 0) return;
  launch_pdl(k_duplicate_sorted, blocks_for(P, 256), 256, 0, s, P, order, means2D, radii, offsets,
             cam.tiles_x, cam.tiles_y, tile_ids, values, cap);
  DW_CUDA(cudaGetLastError());
}

void launch_ranges_u32(int64_t L, const uint32_t* tiles, uint2* ranges, int ntiles,
                       cudaStream_t s, const unsigned long long* n_dev) {
  if (ntiles <= 0) return;
  launch_pdl(k_ranges_search, blocks_for(static_cast<int64_t>(ntiles) * 32, 256), 256, 0, s,
             L, tiles, ranges, ntiles, n_dev);
  DW_CUDA(cudaGetLastError());
}

void launch_clamp_total(const uint64_t* offsets, int P, uint64_t cap, unsigned long long* n_live,
                        unsigned int* overflow, bool sticky, cudaStream_t s) {
  launch_pdl(k_clamp_total, 1, 1, 0, s, offsets, P, cap, n_live, overflow, sticky ? 1 : 0);
  DW_CUDA(cudaGetLastError());
}

void launch_make_keys(int64_t L, const uint32_t* tiles, const uint32_t* values, const float* depths,
                      uint64_t* keys, cudaStream_t s) {
  if (L <= 0) return;
  k_make_keys<<<blocks_for(L, 256), 256, 0, s>>>(L, tiles, values, depths, keys);
  DW_CUDA(cudaGetLastError());
}

void launch_tile_order(const uint2* ranges, int ntiles, uint32_t* order, cudaStream_t s) {
  if (ntiles <= 0) return;
  launch_pdl(k_tile_order, 1, 1024, 0, s, ranges, ntiles, order);
  DW_CUDA(cudaGetLastError());
}

size_t dense_diff_bytes(int tiles_x, int tiles_y) {
  return static_cast<size_t>(tiles_x + 1) * (tiles_y + 1) * sizeof(int);
}

size_t dense_scratch_words(int tiles_x, int tiles_y) {  // per-segment + total count grids
  return static_cast<size_t>(kDenseSeg + 1) * (tiles_x + 1) * (tiles_y + 1);
}

bool dense_binning_fits(int tiles_x, int tiles_y) {
  return tiles_x <= 255 && tiles_y <= 255 && dense_diff_bytes(tiles_x, tiles_y) <= 96 * 1024;
}

void launch_dense_binning(int P, const uint32_t* order, const float2* means2D, const int* radii,
                          const CamParams& cam, uint2* rects, int* scratch, uint2* ranges,
                          uint32_t* values, const unsigned long long* n_dev, uint64_t cap,
                          cudaStream_t s) {
  const size_t dbytes = dense_diff_bytes(cam.tiles_x, cam.tiles_y);
  const int ntiles = cam.tiles_x * cam.tiles_y;
  int* diff = scratch;  // kDenseSeg + 1 grids
  // > 48 KB dynamic smem for 4K-class grids: a per-device, per-kernel
  // attribute, so the opt-in is cached per device (a racing first call just
  // sets it twice)
  static std::atomic<bool> attr_set[64];
  int dev = 0;
  DW_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr_set[dev].load(std::memory_order_acquire)) {
    DW_CUDA(cudaFuncSetAttribute(k_dense_rects, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 96 * 1024));
    DW_CUDA(cudaFuncSetAttribute(k_dense_prefix2d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 96 * 1024));
    if (dev >= 0 && dev < 64) attr_set[dev].store(true, std::memory_order_release);
  }
  DW_CUDA(cudaMemsetAsync(diff, 0, (kDenseSeg + 1) * dbytes, s));
  const int per_seg = std::max(1, std::min<int>(static_cast<int>(blocks_for(P, 256 * kDenseSeg)), 16));
  launch_pdl(k_dense_rects, kDenseSeg * per_seg, 256, dbytes, s, P, order, means2D, radii,
             cam.tiles_x, cam.tiles_y, rects, diff);
  launch_pdl(k_dense_prefix2d, kDenseSeg + 1, 1024, dbytes, s, diff, cam.tiles_x, cam.tiles_y);
  launch_pdl(k_dense_ranges, 1, 1024, 0, s, diff, cam.tiles_x, cam.tiles_y, ranges, n_dev);
  const int groups_x = (cam.tiles_x + 7) / 8;
  const int blocks_per_seg = (groups_x * cam.tiles_y + 7) / 8;
  launch_pdl(k_dense_fill, kDenseSeg * blocks_per_seg, 256, 0, s, P, rects, diff, ranges,
             cam.tiles_x, cam.tiles_y, groups_x, values, n_dev, cap);
  DW_CUDA(cudaGetLastError());
  (void)ntiles;
}

void launch_tiles_from_ranges(const uint2* ranges, int ntiles, uint32_t* tiles, cudaStream_t s) {
  if (ntiles <= 0) return;
  k_tiles_from_ranges<<<blocks_for(static_cast<int64_t>(ntiles) * 32, 256), 256, 0, s>>>(
      ranges, ntiles, tiles);
  DW_CUDA(cudaGetLastError());
}

void launch_segsort_depth(const uint2* ranges, const float* depths, uint32_t* values,
                          unsigned long long* scratch, int64_t capacity, int ntiles,
                          cudaStream_t s, int min_n) {
  if (ntiles <= 0) return;
  launch_pdl(k_segsort_depth, ntiles, 256, 0, s, ranges, depths, values, scratch, ntiles,
             capacity, min_n);
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
