// Block binning: the per-tile lists of the depth-first pipeline built through
// coarse blocks instead of duplicating every (tile, Gaussian) instance and
// radix-sorting the instances by tile id.
//
// The reference's order: a stable sort of the instances
// by (tile << 32 | depth bits), instances generated in Gaussian order -- per
// tile, the Gaussians that touch it in (depth, index) order. Given the
// Gaussians already in (depth, index) order (the depth sort), that list is
// produced here in two levels:
//
//   level 1  every Gaussian is entered once per COARSE BLOCK (8 x 4 tiles,
//            128 x 64 pixels) its tile rectangle touches -- ~1.2 entries per
//            Gaussian on the 1080p scenes instead of ~4.5 instances -- and
//            the entries are stably sorted by block id (one 8-bit LSD pass of
//            raster_sort.cu at 1080p): each block's list holds its Gaussians
//            in depth order;
//   level 2  one CTA per block, each warp a contiguous segment of the block's
//            list; per step of 32 entries every lane forms the 32-bit mask of
//            the block's 32 tiles its rectangle covers and one 32x32 bit
//            transpose (5 xor shuffles) gives, per tile, the lanes covering
//            it: a counting walk yields per-(warp, tile) counts and tile
//            totals, one scan the tile ranges (the reference layout: lists in
//            tile-id order, (0, 0) for an empty tile), and a placing walk
//            appends each Gaussian at (position of its tile) + (lower lanes
//            covering the tile).
//
// Output: ranges and the value array identical, bit for bit, to the
// duplicate + tile-sort path (tests force both). Traffic: ~1.2 P entries
// sorted once instead of ~4.5 P instances sorted twice; the appends are
// ~I scattered 4-byte stores, as the sort's scatter was.
//
// Rectangles use the dense binning's packing (x0 | y0 << 8 | (x1-1) << 16 |
// (y1-1) << 24, tile units < 256), so the path needs tiles_x, tiles_y <= 255.
#include <cuda_runtime.h>

#include "distwar.cuh"
#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

constexpr int kBBW = 8;       // coarse block width in tiles (one warp row)
constexpr int kBBH = 4;       // coarse block height in tiles (one warp per row)
#ifndef DW_BB_WARPS
#define DW_BB_WARPS 16
#endif
#ifndef DW_BB_SPLIT
#define DW_BB_SPLIT 2
#endif
#ifndef DW_BB_STEPS
#define DW_BB_STEPS 4
#endif
constexpr int kBBWarps = DW_BB_WARPS;  // warps per CTA, each a contiguous segment of the list
constexpr int kBBSplit = DW_BB_SPLIT;  // CTAs per block
constexpr int kBBSegs = kBBWarps * kBBSplit;  // segments per block list
constexpr int kBBSteps = DW_BB_STEPS;  // 32-entry steps per warp per round (loaded together)
constexpr uint32_t kEmptyRectBB = 0x0000ff00u;  // y0 = 255 > y1 - 1 = 0

// No-sync sizing for block binning: offsets[P-1] holds (tiles, blocks); the
// live instance count is the tile total when it and the block total fit their
// reserves (else 0 and the overflow flag), the live entry count the block
// total (0 on overflow). The entry reserve sizes the level-1 sort's grid.
__global__ void k_bb_clamp(const uint64_t* __restrict__ offsets, int P, uint64_t cap,
                           uint64_t entry_cap, unsigned long long* __restrict__ n_live,
                           unsigned long long* __restrict__ n_entries,
                           unsigned int* __restrict__ overflow, int sticky) {
  pdl_wait();
  pdl_trigger();
  const uint64_t tot = P > 0 ? offsets[P - 1] : 0;
  const uint64_t tiles = tot & kBBTileMask, blocks = tot >> kBBTileBits;
  const bool fits = tiles <= cap && blocks <= entry_cap;
  *n_live = fits ? tiles : 0ull;
  *n_entries = fits ? blocks : 0ull;
  if (!fits) *overflow = 1u;
  else if (!sticky) *overflow = 0u;
}

// 32 x 32 bit-matrix transpose across the warp: lane l holds row l (bit c =
// column c) on entry, lane c holds column c (bit l = row l) on exit -- five
// xor-shuffle block swaps. At level j a lane keeps its half of the columns
// and takes the other half from its partner rotated by j (left when lane bit
// j is clear, right when set): SHFL + funnel rotate + LOP3 with the per-lane
// amounts and masks of Transpose32.
struct Transpose32 {
  uint32_t rot[5], keep[5];
  __device__ __forceinline__ explicit Transpose32(int lane) {
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int j = 16 >> l;
      const uint32_t M = l == 0 ? 0x0000ffffu
                         : l == 1 ? 0x00ff00ffu
                         : l == 2 ? 0x0f0f0f0fu
                         : l == 3 ? 0x33333333u
                                  : 0x55555555u;
      const bool up = (lane & j) != 0;
      rot[l] = up ? 32u - j : static_cast<uint32_t>(j);
      keep[l] = up ? ~M : M;
    }
  }
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const uint32_t y = __shfl_xor_sync(kFull, x, 16 >> l);
      const uint32_t r = __funnelshift_l(y, y, rot[l]);  // rotate left
      x = (x & keep[l]) | (r & ~keep[l]);
    }
    return x;
  }
};

// The 32-bit mask of block (bx, by)'s tiles (bit r * 8 + c = tile row r,
// column c) that packed rectangle pr covers (branch-free; 0 when disjoint).
__device__ __forceinline__ uint32_t block_cover(uint32_t pr, int bx, int by) {
  const int x0 = (int)(pr & 0xffu) - bx * kBBW, y0 = (int)((pr >> 8) & 0xffu) - by * kBBH;
  const int x1 = (int)((pr >> 16) & 0xffu) - bx * kBBW, y1 = (int)(pr >> 24) - by * kBBH;
  const int c0 = min(max(x0, 0), kBBW), c1 = max(min(x1, kBBW - 1), -1);
  const int r0 = min(max(y0, 0), kBBH), r1 = max(min(y1, kBBH - 1), -1);
  const uint32_t cols = (0xffu << c0) & (0xffu >> (kBBW - 1 - c1));
  const uint32_t rows = (0xfu << r0) & (0xfu >> (kBBH - 1 - r1));
  return cols * ((rows * 0x00204081u) & 0x01010101u);  // row bit r -> byte r
}

// Level 2, pass 1. CTA = (block b, half of its list); warp w walks the w-th
// contiguous segment of that half (entries in depth order, coalesced: the
// sort carried the packed rectangle as payload), 32 entries per step: each
// lane's 32-bit tile mask, transposed, gives lane t the step's count for tile
// t. Per-(half, tile) totals go to tcount (the tile ranges and pass 2's start
// positions).
__global__ void __launch_bounds__(32 * kBBWarps)
    k_bb_count(uint2* __restrict__ branges, const uint32_t* __restrict__ digit_totals,
               const uint32_t* __restrict__ brect, int tiles_x, int tiles_y, int nbx,
               uint32_t* __restrict__ tcount) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_c[kBBWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x / kBBSplit, half = blockIdx.x % kBBSplit, seg = half * kBBWarps + w;
  const int bx = b % nbx, by = b / nbx;
  uint2 br;
  if (digit_totals) {
    // one-pass entry sort (<= 256 blocks): its digit totals are the block
    // sizes, so the block's range is their prefix -- no search over the entries
    const uint32_t x = (threadIdx.x < 256) ? digit_totals[threadIdx.x] : 0u;
    uint32_t below = threadIdx.x < b ? x : 0u;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) below += __shfl_xor_sync(kFull, below, o);
    if (lane == 0) s_c[w][0] = below;
    __syncthreads();
    uint32_t start = 0;
#pragma unroll
    for (int q = 0; q < kBBWarps; ++q) start += s_c[q][0];
    br = make_uint2(start, start + digit_totals[b]);
    __syncthreads();  // s_c is reused below
    if (half == 0 && threadIdx.x == 0) branges[b] = br;  // for k_bb_place
  } else {
    br = branges[b];
  }
  const uint32_t len = br.y - br.x;
  const uint32_t lo = br.x + static_cast<uint32_t>(static_cast<uint64_t>(len) * seg / kBBSegs);
  const uint32_t hi = br.x + static_cast<uint32_t>(static_cast<uint64_t>(len) * (seg + 1) / kBBSegs);
  const Transpose32 tr(lane);
  uint32_t cnt = 0;
  uint32_t pr[kBBSteps];
#pragma unroll
  for (int q = 0; q < kBBSteps; ++q) {
    const uint32_t kq = lo + 32 * q + lane;
    pr[q] = kq < hi ? __ldg(brect + kq) : kEmptyRectBB;
  }
  for (uint32_t k0 = lo; k0 < hi; k0 += 32 * kBBSteps) {
    uint32_t m[kBBSteps];
#pragma unroll
    for (int q = 0; q < kBBSteps; ++q) {
      m[q] = block_cover(pr[q], bx, by);
      const uint32_t kq = k0 + 32 * (kBBSteps + q) + lane;  // next round, in flight
      pr[q] = kq < hi ? __ldg(brect + kq) : kEmptyRectBB;
    }
#pragma unroll
    for (int q = 0; q < kBBSteps; ++q) cnt += __popc(tr(m[q]));
  }
  s_c[w][lane] = cnt;
  __syncthreads();
  if (w == 0) {  // this CTA's share of the block's tile totals
    uint32_t tot = 0;
#pragma unroll
    for (int q = 0; q < kBBWarps; ++q) tot += s_c[q][lane];
    const int tx = bx * kBBW + (lane & (kBBW - 1)), ty = by * kBBH + lane / kBBW;
    if (tx < tiles_x && ty < tiles_y) tcount[(ty * tiles_x + tx) * kBBSplit + half] = tot;
  }
}

__device__ __forceinline__ uint32_t tile_total(const uint32_t* __restrict__ tcount, int tile) {
  uint32_t c = 0;
#pragma unroll
  for (int h = 0; h < kBBSplit; ++h) c += tcount[tile * kBBSplit + h];
  return c;
}

// One CTA: per-tile totals -> exclusive scan in tile order -> ranges ((0, 0)
// when empty or over the no-sync capacity, the reference layout).
__global__ void __launch_bounds__(1024)
    k_bb_tile_ranges(const uint32_t* __restrict__ tcount, int ntiles, uint2* __restrict__ ranges,
                     const unsigned long long* __restrict__ n_live) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_wsum[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const bool over = n_live && *n_live == 0ull;
  uint32_t carry = 0;
  // 1,024 consecutive tiles per round (coalesced), each round's block scan
  // continuing the previous one's total; all rounds' counts loaded up front
  const int rounds = (ntiles + 1023) / 1024;  // <= 64 (255 x 255 tiles)
  uint32_t c[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int tile = r * 1024 + t;
    c[r] = (r < rounds && tile < ntiles) ? tile_total(tcount, tile) : 0u;
  }
  __shared__ uint32_t s_total;
  auto round = [&](int r, uint32_t v) {
    const int tile = r * 1024 + t;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[w] = incl;
    __syncthreads();
    if (w == 0) {  // exclusive scan of the 32 warp totals
      const uint32_t x = s_wsum[lane];
      uint32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, xi, o);
        if (lane >= o) xi += y;
      }
      s_wsum[lane] = xi - x;
      if (lane == 31) s_total = xi;
    }
    __syncthreads();
    const uint32_t before = carry + s_wsum[w] + incl - v;
    if (tile < ntiles)
      ranges[tile] = (v == 0 || over) ? make_uint2(0u, 0u) : make_uint2(before, before + v);
    carry += s_total;
    __syncthreads();
  };
#pragma unroll
  for (int r = 0; r < 8; ++r)
    if (r < rounds) round(r, c[r]);
  for (int r = 8; r < rounds; ++r) {
    const int tile = r * 1024 + t;
    round(r, tile < ntiles ? tile_total(tcount, tile) : 0u);
  }
}

// Level 2, pass 2. CTA = (block, half of its list), walked in rounds of
// kBBSteps x 512 consecutive entries (warp w: the round's entries
// [w * 32 kBBSteps, (w + 1) * 32 kBBSteps), loaded at once, one round ahead).
// Per round: transposed masks -> per-(warp, tile) counts -> in shared memory,
// each tile's run of the round laid out in (tile, warp, step, lane) order =
// the tiles' list order; then each tile's run is copied to its list with
// consecutive lanes on consecutive positions (coalesced), instead of one
// scattered 4-byte store per instance. A round whose output exceeds the
// staging buffer stores directly (same positions).
constexpr int kBBRound = 32 * kBBWarps * kBBSteps;
constexpr int kBBBuf = 11264;  // 44 KB: static shared memory stays under 48 KB

#ifndef DW_BB_PLACE_MIN_BLOCKS
#define DW_BB_PLACE_MIN_BLOCKS 4  // <= 32 registers: the 510 CTAs of a 1080p frame in one wave
#endif
__global__ void __launch_bounds__(32 * kBBWarps, DW_BB_PLACE_MIN_BLOCKS)
    k_bb_place(const uint2* __restrict__ branges, const uint32_t* __restrict__ brect,
               const uint32_t* __restrict__ bgid, const uint32_t* __restrict__ tcount,
               const uint2* __restrict__ ranges, int tiles_x, int tiles_y, int nbx,
               uint32_t* __restrict__ values, const unsigned long long* __restrict__ n_live) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_off[kBBWarps][32];  // per (warp, tile): count -> offset in the tile's run
  __shared__ uint32_t s_tb[33];             // run start of each tile in s_buf (+ total)
  __shared__ uint32_t s_gcur[32];           // next list position of each tile
  __shared__ uint32_t s_buf[kBBBuf];
  if (n_live && *n_live == 0ull) return;  // over the no-sync capacity: empty lists
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x / kBBSplit, half = blockIdx.x % kBBSplit;
  const int bx = b % nbx, by = b / nbx;
  const uint2 br = branges[b];
  const uint32_t len = br.y - br.x;
  const uint32_t lo = br.x + static_cast<uint32_t>(static_cast<uint64_t>(len) * half / kBBSplit);
  const uint32_t hi =
      br.x + static_cast<uint32_t>(static_cast<uint64_t>(len) * (half + 1) / kBBSplit);
  const Transpose32 tr(lane);
  uint32_t tot_prev = 0;  // warp 0, lane t: tile t's count of the previous round
  if (w == 0) {
    const int tx = bx * kBBW + (lane & (kBBW - 1)), ty = by * kBBH + lane / kBBW;
    uint32_t cur = 0;
    if (tx < tiles_x && ty < tiles_y) {
      const int tile = ty * tiles_x + tx;
      cur = ranges[tile].x;
      for (int q = 0; q < half; ++q) cur += tcount[tile * kBBSplit + q];
    }
    s_gcur[lane] = cur;
  }
  uint32_t k = lo + static_cast<uint32_t>(w) * 32 * kBBSteps + lane;
  uint32_t pr[kBBSteps], g[kBBSteps];
#pragma unroll
  for (int q = 0; q < kBBSteps; ++q) {
    const uint32_t kq = k + 32 * q;
    pr[q] = kq < hi ? __ldg(brect + kq) : kEmptyRectBB;
    g[q] = kq < hi ? __ldg(bgid + kq) : 0u;
  }
  for (uint32_t r0 = lo; r0 < hi; r0 += kBBRound) {
    uint32_t col[kBBSteps], c[kBBSteps];
    uint32_t mine = 0;
#pragma unroll
    for (int q = 0; q < kBBSteps; ++q) {
      col[q] = tr(block_cover(pr[q], bx, by));
      c[q] = __popc(col[q]);
      mine += c[q];
    }
    s_off[w][lane] = mine;
    const uint32_t kn = k + kBBRound;  // next round's entries, in flight meanwhile
    uint32_t gq[kBBSteps];
#pragma unroll
    for (int q = 0; q < kBBSteps; ++q) {
      const uint32_t kq = kn + 32 * q;
      gq[q] = g[q];
      pr[q] = kq < hi ? __ldg(brect + kq) : kEmptyRectBB;
      g[q] = kq < hi ? __ldg(bgid + kq) : 0u;
    }
    __syncthreads();
    if (w == 0) {
      s_gcur[lane] += tot_prev;  // the previous round's run (its copy is done)
      uint32_t run = 0;
#pragma unroll
      for (int q = 0; q < kBBWarps; ++q) {
        const uint32_t cq = s_off[q][lane];
        s_off[q][lane] = run;
        run += cq;
      }
      uint32_t incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      s_tb[lane] = incl - run;
      if (lane == 31) s_tb[32] = incl;
      tot_prev = run;
    }
    __syncthreads();
    const bool staged = s_tb[32] <= static_cast<uint32_t>(kBBBuf);
    uint32_t pos = staged ? s_tb[lane] + s_off[w][lane] : s_gcur[lane] + s_off[w][lane];
    uint32_t* out = staged ? s_buf : values;
#pragma unroll
    for (int q = 0; q < kBBSteps; ++q) {
      uint32_t cq = col[q];
      while (__any_sync(kFull, cq != 0u)) {
        const int j = __ffs(cq) - 1;  // -1 when done: the shuffle reads lane 31, unused
        const uint32_t gj = __shfl_sync(kFull, gq[q], j & 31);
        if (cq) {
          out[pos++] = gj;
          cq &= cq - 1u;
        }
      }
    }
    if (staged) {
      __syncthreads();
      for (int t = w; t < 32; t += kBBWarps) {  // tile t's run -> its list, coalesced
        const uint32_t a = s_tb[t], e = s_tb[t + 1];
        uint32_t* dst = values + s_gcur[t] - a;
        for (uint32_t i = a + lane; i < e; i += 32) dst[i] = s_buf[i];
      }
    }
    __syncthreads();
    k = kn;
  }
}

inline unsigned blocks_of(int64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

}  // namespace

bool block_binning_fits(int tiles_x, int tiles_y) { return tiles_x <= 255 && tiles_y <= 255; }

int block_binning_nbx(int tiles_x) { return (tiles_x + kBBW - 1) / kBBW; }

int block_binning_blocks(int tiles_x, int tiles_y) {
  return ((tiles_x + kBBW - 1) / kBBW) * ((tiles_y + kBBH - 1) / kBBH);
}

size_t block_binning_count_words(int tiles_x, int tiles_y) {
  return static_cast<size_t>(tiles_x) * tiles_y * kBBSplit;
}

void launch_bb_clamp(const uint64_t* offsets, int P, uint64_t cap, uint64_t entry_cap,
                     unsigned long long* n_live,
                     unsigned long long* n_entries, unsigned int* overflow, bool sticky,
                     cudaStream_t s) {
  launch_pdl(k_bb_clamp, 1, 1, 0, s, offsets, P, cap, entry_cap, n_live, n_entries, overflow,
             sticky ? 1 : 0);
  DW_CUDA(cudaGetLastError());
}

void launch_block_binning(const uint32_t* rect_by_id, const CamParams& cam, uint32_t* k[2],
                          uint32_t* v[2], int64_t n_entries, void* sort_tmp, uint32_t* brect,
                          uint2* branges, uint32_t* cnt, uint2* ranges, uint32_t** values_out,
                          const unsigned long long* n_live,
                          const unsigned long long* n_entries_dev, cudaStream_t s) {
  const int nbx = (cam.tiles_x + kBBW - 1) / kBBW;
  const int nblocks = block_binning_blocks(cam.tiles_x, cam.tiles_y);
  const int ntiles = cam.tiles_x * cam.tiles_y;
  uint32_t* tcount = cnt;  // [ntiles][split]
  int bits = 1;
  while ((1 << bits) < nblocks) ++bits;
  // level 1: the entries (block_entries_scan) stably sorted by block id
  // (payload: the packed rectangle), block ranges
  const int cur = radix_sort_pairs(k, v, n_entries, bits, sort_tmp, s, n_entries_dev, rect_by_id,
                                   brect);
  // block ranges: from the digit totals of a one-pass sort (<= 256 blocks, in
  // k_bb_count), else by search over the sorted block ids
  const uint32_t* totals = bits <= 8 ? radix_sort_digit_totals(sort_tmp, n_entries) : nullptr;
  if (!totals) launch_ranges_u32(n_entries, k[cur], branges, nblocks, s, n_entries_dev);
  // level 2: counts, tile ranges, appends
  launch_pdl(k_bb_count, static_cast<unsigned>(nblocks * kBBSplit), 32 * kBBWarps, 0, s, branges,
             totals, brect,
             cam.tiles_x, cam.tiles_y, nbx, tcount);
  launch_pdl(k_bb_tile_ranges, 1, 1024, 0, s, tcount, ntiles, ranges, n_live);
  launch_pdl(k_bb_place, static_cast<unsigned>(nblocks * kBBSplit), 32 * kBBWarps, 0, s, branges, brect,
             v[cur], tcount, ranges, cam.tiles_x, cam.tiles_y, nbx, v[cur ^ 1], n_live);
  *values_out = v[cur ^ 1];
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
