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

#include <algorithm>

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

// ---------------------------------------------------------------------------
// Fused level 1 (<= 256 coarse blocks). The entries of a tile of 2,048
// depth-ordered Gaussians go straight to their positions in the block-sorted
// order -- block start (prefix of the block totals) + the earlier tiles'
// entries of that block (hist, scanned over tiles) + the rank inside the tile
// (warp, then entry order: the stable order of the radix pass this replaces).
constexpr int kFuseItems = 8;
constexpr int kFuseTile = 256 * kFuseItems;
constexpr int kFuseCap = 4096;  // staged entries per tile (else direct stores)

__device__ __forceinline__ void rect_blocks(uint32_t x, int* bx0, int* by0, int* bw, int* nb) {
  const int x0 = (int)(x & 0xffu), y0 = (int)((x >> 8) & 0xffu);
  const int x1 = (int)((x >> 16) & 0xffu), y1 = (int)(x >> 24);
  *bx0 = x0 / kBBW;
  *by0 = y0 / kBBH;
  *bw = x1 / kBBW - *bx0 + 1;
  *nb = y0 > y1 ? 0 : *bw * (y1 / kBBH - *by0 + 1);
}

__global__ void __launch_bounds__(256)
    k_bb_hist(const uint32_t* __restrict__ rect_sorted, int64_t n, int nbx, int64_t tiles,
              uint32_t* __restrict__ hist, unsigned long long* __restrict__ total) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_h[256];
  __shared__ unsigned long long s_w[8];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  s_h[t] = 0u;
  __syncthreads();
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * kFuseTile;
  unsigned long long mine = 0;
#pragma unroll
  for (int k = 0; k < kFuseItems; ++k) {
    const int64_t e = tile0 + k * 256 + t;
    if (e >= n) break;
    const uint32_t x = __ldg(rect_sorted + e);
    int bx0, by0, bw, nb;
    rect_blocks(x, &bx0, &by0, &bw, &nb);
    if (nb == 0) continue;
    const int area = ((int)((x >> 16) & 0xffu) - (int)(x & 0xffu) + 1) *
                     ((int)(x >> 24) - (int)((x >> 8) & 0xffu) + 1);
    mine += (static_cast<unsigned long long>(nb) << kBBTileBits) | static_cast<unsigned>(area);
    for (int q = 0; q < nb; ++q)
      atomicAdd(&s_h[(by0 + q / bw) * nbx + bx0 + q % bw], 1u);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mine += __shfl_xor_sync(kFull, mine, o);
  if (lane == 0) s_w[w] = mine;
  __syncthreads();
  if (t == 0) {
    unsigned long long a = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) a += s_w[q];
    if (a) atomicAdd(total, a);
  }
  hist[static_cast<int64_t>(t) * tiles + blockIdx.x] = s_h[t];
}

__global__ void __launch_bounds__(256)
    k_bb_emit(const uint32_t* __restrict__ rect_sorted, const uint32_t* __restrict__ order,
              int64_t n, int nbx, int64_t tiles, const uint32_t* __restrict__ hist,
              const uint32_t* __restrict__ block_totals, uint32_t* __restrict__ bval,
              uint32_t* __restrict__ brect, const unsigned long long* __restrict__ n_entries,
              uint64_t cap) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_cnt[8][256];  // per (warp, block): count -> next staging position
  __shared__ uint32_t s_bstart[256];  // start of each block's run in the staging buffer
  __shared__ uint32_t s_gbase[256];   // global position of that run
  __shared__ uint32_t s_wsum[8], s_dsum[8], s_tot;
  __shared__ uint32_t s_val[kFuseCap], s_rect[kFuseCap];
  __shared__ uint8_t s_blk[kFuseCap];
  if (n_entries && *n_entries == 0ull) return;  // no-sync frame over capacity (or empty)
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * kFuseTile + w * 256;  // warp's chunk
#pragma unroll
  for (int q = 0; q < 8; ++q) s_cnt[q][t] = 0u;
  __syncthreads();
  // sweep 1: this warp's entries per block
#pragma unroll
  for (int r = 0; r < kFuseItems; ++r) {
    const int64_t e = g0 + r * 32 + lane;
    const uint32_t x = e < n ? __ldg(rect_sorted + e) : kEmptyRectBB;
    int bx0, by0, bw, nb;
    rect_blocks(x, &bx0, &by0, &bw, &nb);
    for (int q = 0; q < nb; ++q) atomicAdd(&s_cnt[w][(by0 + q / bw) * nbx + bx0 + q % bw], 1u);
  }
  __syncthreads();
  // thread t = block t: run of the block in this tile (warp order), the
  // tile's staging layout (block order) and the global positions
  uint32_t c[8], tot = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    c[q] = s_cnt[q][t];
    tot += c[q];
  }
  uint32_t incl = tot, dincl = block_totals[t];
  const uint32_t dtot = dincl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o), dy = __shfl_up_sync(kFull, dincl, o);
    if (lane >= o) {
      incl += y;
      dincl += dy;
    }
  }
  if (lane == 31) {
    s_wsum[w] = incl;
    s_dsum[w] = dincl;
  }
  __syncthreads();
  uint32_t bstart = incl - tot, dstart = dincl - dtot;
  for (int q = 0; q < w; ++q) {
    bstart += s_wsum[q];
    dstart += s_dsum[q];
  }
  s_bstart[t] = bstart;
  s_gbase[t] = dstart + hist[static_cast<int64_t>(t) * tiles + blockIdx.x];
  uint32_t run = bstart;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    s_cnt[q][t] = run;
    run += c[q];
  }
  if (t == 255) s_tot = run;
  __syncthreads();
  const uint32_t ntot = s_tot;
  const bool staged = ntot <= static_cast<uint32_t>(kFuseCap);
  // sweep 2: each round's entries, warp-cooperatively in (Gaussian, block)
  // order, ranked per block (ballot multi-split) against the warp's cursor
#pragma unroll 1
  for (int r = 0; r < kFuseItems; ++r) {
    const int64_t e = g0 + r * 32 + lane;
    const uint32_t x = e < n ? __ldg(rect_sorted + e) : kEmptyRectBB;
    int bx0, by0, bw, nb;
    rect_blocks(x, &bx0, &by0, &bw, &nb);
    const uint32_t gid = e < n ? __ldg(order + e) : 0u;
    int inc = nb;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, d);
      if (lane >= d) inc += y;
    }
    const int excl = inc - nb, total = __shfl_sync(kFull, inc, 31);
    for (int q0 = 0; q0 < total; q0 += 32) {
      const int q = q0 + lane;
      int owner = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int probe = owner + step;
        if (__shfl_sync(kFull, excl, probe) <= q) owner = probe;
      }
      const int kk = q - __shfl_sync(kFull, excl, owner);
      const int ow = __shfl_sync(kFull, bw, owner);
      const int ox = __shfl_sync(kFull, bx0, owner), oy = __shfl_sync(kFull, by0, owner);
      const uint32_t og = __shfl_sync(kFull, gid, owner), orc = __shfl_sync(kFull, x, owner);
      const bool valid = q < total;
      const int row = valid ? kk / ow : 0;
      const uint32_t blk = valid ? static_cast<uint32_t>((oy + row) * nbx + ox + (kk - row * ow))
                                 : 0u;
      unsigned peers = __ballot_sync(kFull, valid);
      if (!valid) peers = ~peers;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool bit = (blk >> b) & 1u;
        const unsigned m = __ballot_sync(kFull, bit);
        peers &= bit ? m : ~m;
      }
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (valid && lane == leader) {
        base = s_cnt[w][blk];
        s_cnt[w][blk] = base + __popc(peers);
      }
      base = __shfl_sync(kFull, base, leader);
      if (valid) {
        const uint32_t pos = base + __popc(peers & lt);
        if (staged) {
          s_val[pos] = og;
          s_rect[pos] = orc;
          s_blk[pos] = static_cast<uint8_t>(blk);
        } else {
          const uint64_t g = s_gbase[blk] + (pos - s_bstart[blk]);
          if (g < cap) {
            bval[g] = og;
            brect[g] = orc;
          }
        }
      }
      __syncwarp();
    }
  }
  if (!staged) return;
  __syncthreads();
  for (uint32_t i = t; i < ntot; i += 256) {  // each block's run, coalesced
    const uint32_t b = s_blk[i];
    const uint64_t g = s_gbase[b] + (i - s_bstart[b]);
    if (g < cap) {
      bval[g] = s_val[i];
      brect[g] = s_rect[i];
    }
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

size_t block_binning_hist_words(int64_t P) {
  return static_cast<size_t>((std::max<int64_t>(P, 1) + kFuseTile - 1) / kFuseTile) * 256 + 256;
}

void launch_bb_hist(const uint32_t* rect_sorted, int64_t P, const CamParams& cam, uint32_t* hist,
                    uint64_t* total, cudaStream_t s) {
  if (P <= 0) return;
  const int64_t tiles = (P + kFuseTile - 1) / kFuseTile;
  launch_pdl(k_bb_hist, static_cast<unsigned>(tiles), 256, 0, s, rect_sorted, P,
             block_binning_nbx(cam.tiles_x), tiles, hist,
             reinterpret_cast<unsigned long long*>(total));
  DW_CUDA(cudaGetLastError());
}

void launch_block_binning_fused(const uint32_t* rect_sorted, const uint32_t* order, int64_t P,
                                const CamParams& cam, uint32_t* hist, uint32_t* v[2],
                                uint64_t entry_cap, uint32_t* brect, uint2* branges,
                                uint32_t* cnt, uint2* ranges, uint32_t** values_out,
                                const unsigned long long* n_live,
                                const unsigned long long* n_entries_dev, cudaStream_t s) {
  const int nbx = block_binning_nbx(cam.tiles_x);
  const int nblocks = block_binning_blocks(cam.tiles_x, cam.tiles_y);
  const int ntiles = cam.tiles_x * cam.tiles_y;
  const int64_t tiles = (P + kFuseTile - 1) / kFuseTile;
  uint32_t* totals = hist + static_cast<size_t>(tiles) * 256;
  launch_scan_rows(hist, tiles, totals, s);
  launch_pdl(k_bb_emit, static_cast<unsigned>(tiles), 256, 0, s, rect_sorted, order, P, nbx, tiles,
             hist, totals, v[1], brect, n_entries_dev, entry_cap);
  launch_pdl(k_bb_count, static_cast<unsigned>(nblocks * kBBSplit), 32 * kBBWarps, 0, s, branges,
             static_cast<const uint32_t*>(totals), brect, cam.tiles_x, cam.tiles_y, nbx, cnt);
  launch_pdl(k_bb_tile_ranges, 1, 1024, 0, s, cnt, ntiles, ranges, n_live);
  launch_pdl(k_bb_place, static_cast<unsigned>(nblocks * kBBSplit), 32 * kBBWarps, 0, s, branges,
             brect, v[1], cnt, ranges, cam.tiles_x, cam.tiles_y, nbx, v[0], n_live);
  *values_out = v[0];
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
