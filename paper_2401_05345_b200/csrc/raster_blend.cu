// Front-to-back alpha blending (forward) and its analytic backward with the
// DISTWAR reduction -- the hot path.
//
// One 256-thread CTA per 16x16 tile. The tile's sorted Gaussian list is
// walked in batches of 256 staged in shared memory (48 B per Gaussian:
// xy + id, conic + opacity, rgb). While staging, the thread that loads a
// Gaussian also computes which of the tile's eight 8x4 warp blocks its
// alpha >= 1/255 footprint can reach and stores that as an 8-bit mask; each
// warp then ballots its bits of the 256 masks and walks ONLY the Gaussians
// that can touch its pixels (warp-uniform: ffs over the ballot words), so the
// (warp, Gaussian) pairs that cannot contribute cost no per-lane work.
//
// Footprint bound. alpha = min(0.99, o G) >= 1/255 with G = exp(-q/2),
// q = d^T Q d (Q = conic), needs q <= tau = 2 ln(255 o). The ellipse
// q <= tau lies in |dx| <= sqrt(tau Q^-1_xx), |dy| <= sqrt(tau Q^-1_yy), with
// Q^-1_xx = c / (ac - b^2), Q^-1_yy = a / (ac - b^2). The preprocess computes
// these half-extents once per Gaussian (raster_preprocess.cu
// footprint_extents), inflating tau by 5 % + 0.05 to cover the exp2
// approximation and FMA rounding and rounding up to half precision, so
// culling never drops a pair the per-lane test would keep (o <= 1/255 ->
// never active; a degenerate conic falls back to no culling).
//
// Backward: the GradComputation loop of PAPER.md:1481-1504 -- each pixel
// thread walks its Gaussians back to front, cond1/cond2 are the
// last-contributor and alpha tests, and the 9 atomicAdds are replaced by a
// call of the DISTWAR policy (distwar.cuh) made by all 32 lanes, inactive
// lanes carrying zero gradients. A warp whose 32 lanes
// are all inactive for a Gaussian (ballot == 0) issues nothing, as the
// reference policies emit no request for an empty active mask
// (reducers.cpp:154-156).
#include <cstdlib>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "distwar.cuh"
#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

struct __align__(16) Staged {
  float4 xyi;  // x, y, id (uint bits), - (packed backward: k b, see its mask phase)
  float4 co;   // conic a, b, c, opacity
  float4 col;  // r, g, b, footprint extents (preprocess: half2 bits; packed
               // backward: 1/opacity after its mask phase)
};

// The staged conic is pre-scaled so the exponent of G = exp(-q/2) comes out
// directly in log2 units: (a, b, c) -> (k a, 2 k b, k c), k = -log2(e)/2, and
// log2 G = k a dx^2 + 2 k b dx dy + k c dy^2 = fma(fma(kc, dy, 2kb dx), dy, ka dxx)
// -- two fused multiply-adds where the unscaled form needs four operations
// plus the log2(e) multiply. Every blend kernel evaluates exactly this
// sequence on the same scale_conic() values (the packed backward gathers the
// raw conic with cp.async and scales it in place in its mask phase), so
// forward and backward take identical alpha decisions.
constexpr float kConicScale = -0.5f * 1.4426950408889634f;
__device__ __forceinline__ float4 scale_conic(const float4& co) {
  return make_float4(kConicScale * co.x, 2.0f * kConicScale * co.y, kConicScale * co.z, co.w);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Footprint mask of a Gaussian: the 8x4 bands (8 per 16x16 tile; warp w of
// the one-pixel kernel = band w, warp w of the two-pixel kernels = bands
// 4 (w >> 1) + (w & 1) + {0, 2}) its alpha >= 1/255 ellipse can reach, by
// bounding box. (An exact ellipse-rectangle test per band is slower: C3
// backward 0.835 vs 0.780 ms -- its cost at staging exceeds the walks it
// saves; the remaining empty walks are mostly misses between pixel centres.)
// The half-extents (ex, ey) come precomputed from the preprocess (rgb.w, a
// half2 rounded up: raster_preprocess.cu), so staging does compares only;
// -inf marks a Gaussian that can never reach alpha 1/255, +inf a degenerate
// conic (no culling).
__device__ __forceinline__ uint32_t footprint_mask(float mx, float my, float ext_bits, int tx0,
                                                   int ty0) {
  const uint32_t eb = __float_as_uint(ext_bits);
  const float2 e = __half22float2(*reinterpret_cast<const __half2*>(&eb));
  const float ex = e.x, ey = e.y;
  uint32_t cx = 0, ry = 0;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const float lo = (float)(tx0 + 8 * c), hi = lo + 7.0f;
    if (mx + ex >= lo && mx - ex <= hi) cx |= 1u << c;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float lo = (float)(ty0 + 4 * r), hi = lo + 3.0f;
    if (my + ey >= lo && my - ey <= hi) ry |= 1u << r;
  }
  uint32_t mask = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w)
    if ((cx >> (w & 1) & 1u) && (ry >> (w >> 1) & 1u)) mask |= 1u << w;
  return mask;
}

// Stage Gaussian `id` into slot `slot` (conic pre-scaled, scale_conic) and
// return its 8-bit warp-block mask for the tile whose top-left pixel is
// (tx0, ty0).
// xyi.z = id - vbase: the scene index (vbase = the view slot's first id).
__device__ __forceinline__ uint32_t stage(Staged* s, int slot, uint32_t id, int tx0, int ty0,
                                          const float2* __restrict__ means2D,
                                          const float4* __restrict__ conic_opacity,
                                          const float4* __restrict__ rgb, uint32_t vbase = 0) {
  const float2 m = __ldg(means2D + id);
  const float4 co = __ldg(conic_opacity + id);
  s[slot].xyi = make_float4(m.x, m.y, __uint_as_float(id - vbase), 0.0f);
  s[slot].co = scale_conic(co);
  const float4 c = __ldg(rgb + id);
  s[slot].col = c;
  return footprint_mask(m.x, m.y, c.w, tx0, ty0);
}


// Asynchronous (cp.async, no register staging) gather of Gaussian `id` into
// slot `s`: means2D -> xyi.xy, conic/opacity -> co, rgb (+ extents) -> col.
__device__ __forceinline__ void stage_async(Staged* s, uint32_t id,
                                            const float2* __restrict__ means2D,
                                            const float4* __restrict__ conic_opacity,
                                            const float4* __restrict__ rgb) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(means2D + id) : "memory");
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a + 16u), "l"(conic_opacity + id)
               : "memory");
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a + 32u), "l"(rgb + id)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Bulk-copy staging (the TMA engine's non-tensor cp.async.bulk, completion
// counted in bytes on an mbarrier): one 48-byte copy of a Gaussian's packed
// record (preprocess `packed`: xy, conic + opacity, rgb + extents -- the
// Staged layout) instead of three cp.async. A/B'd against cp.async staging in
// k_backward_x2 (DW_BULK_STAGING=1 selects it at run time).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_stage(Staged* dst, const float4* src, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 48, [%2];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(smem_u32(bar))
      : "memory");
}

#ifndef DW_BWD_MIN_BLOCKS
#define DW_BWD_MIN_BLOCKS 5  // 5 x 256 threads/SM: <= 51 registers, no spills (ptxas -v)
#endif

// One pixel per thread -- the paper's GradComputation layout ("thread corr.
// to pixel"): the native (naive-atomic) baseline, whose
// fastest layout this is (7.8 vs 8.2 ms two-pixel on C3). The reduction
// policies run k_backward_x2 below.
template <int POL, bool COUNT>
__global__ void __launch_bounds__(kBlock, DW_BWD_MIN_BLOCKS)
    k_backward(const CamParams cam, const uint2* __restrict__ ranges,
               const uint32_t* __restrict__ values, const float2* __restrict__ means2D,
               const float4* __restrict__ conic_opacity, const float4* __restrict__ rgb,
               const float* __restrict__ final_Ts, const uint32_t* __restrict__ n_contrib,
               const float* __restrict__ dL_dpixels, int thr, float* __restrict__ grad,
               unsigned long long* __restrict__ counters) {
  __shared__ Staged sm[kBlock];
  __shared__ uint8_t s_mask[kBlock];
  __shared__ uint32_t s_wmax[kBlock / 32];
  const int tile = blockIdx.x, t = threadIdx.x, w = t >> 5, lane = t & 31;
  int tx0, ty0;
  const int view = tile_view(cam, tile, &tx0, &ty0);
  int px, py;
  tile_pixel(tx0, ty0, t, &px, &py);
  const bool inside = px < cam.W && py < cam.H;
  const int pix = py * cam.W + px;
  const int HW = cam.H * cam.W;
  final_Ts += static_cast<int64_t>(view) * HW;  // the view's per-pixel buffers
  n_contrib += static_cast<int64_t>(view) * HW;
  dL_dpixels += static_cast<int64_t>(view) * 3 * HW;
  const uint32_t vbase = static_cast<uint32_t>(view * cam.vstride);
  const float pfx = (float)px, pfy = (float)py;
  const uint2 range = ranges[tile];

  const float T_final = inside ? final_Ts[pix] : 0.0f;
  float T = T_final;
  const uint32_t last_contributor = inside ? n_contrib[pix] : 0u;
  float dLp0 = 0.0f, dLp1 = 0.0f, dLp2 = 0.0f;
  if (inside) {
    dLp0 = dL_dpixels[pix];
    dLp1 = dL_dpixels[HW + pix];
    dLp2 = dL_dpixels[2 * HW + pix];
  }
  const float bg_dot = cam.bg[0] * dLp0 + cam.bg[1] * dLp1 + cam.bg[2] * dLp2;
  const float ddelx_dx = 0.5f * (float)cam.W, ddely_dy = 0.5f * (float)cam.H;

  // List positions >= max(last_contributor) over the tile cannot contribute
  // to any of its pixels: start the back-to-front walk there.
  const uint32_t wmax = __reduce_max_sync(kFull, last_contributor);
  if (lane == 0) s_wmax[w] = wmax;
  __syncthreads();
  uint32_t bmax = 0;
#pragma unroll
  for (int k = 0; k < kBlock / 32; ++k) bmax = max(bmax, s_wmax[k]);

  float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
  float lc0 = 0.0f, lc1 = 0.0f, lc2 = 0.0f, last_alpha = 0.0f;
  uint32_t nred = 0, npairs = 0;
  bool issuer;
  const int slot = bfly_slot<kNParam>(lane, &issuer);
  const int rounds = (int)((bmax + kBlock - 1) / kBlock);
  int todo = (int)bmax;
  const uint32_t top = range.x + bmax;  // exclusive end of the live list
  for (int i = 0; i < rounds; ++i, todo -= kBlock) {
    __syncthreads();
    uint32_t mask = 0;
    if (t < todo)
      mask = stage(sm, t, values[top - 1 - (i * kBlock + t)], tx0, ty0, means2D, conic_opacity,
                   rgb, vbase);
    s_mask[t] = (uint8_t)mask;
    __syncthreads();
    const int n = min(kBlock, todo);
    // slot j holds list position c_j = bmax - 1 - (i*256 + j)
    const uint32_t base = bmax - 1 - (uint32_t)(i * kBlock);
    for (int k = 0; k * 32 < n; ++k) {
      const int jl = k * 32 + lane;
      unsigned bits = __ballot_sync(
          kFull, jl < n && ((s_mask[jl] >> w) & 1u) && (base - (uint32_t)jl) < wmax);
      while (bits) {
        const int j = k * 32 + __ffs(bits) - 1;
        bits &= bits - 1u;
        const uint32_t contributor = base - (uint32_t)j;
        const float4 g = sm[j].xyi;
        const float4 co = sm[j].co;
        const float dx = g.x - pfx, dy = g.y - pfy;
        const float dxx = dx * dx, dxy = dx * dy, dyy = dy * dy;
        // the packed forward's exact operation sequence (eval2), so this
        // kernel walks exactly the forward's contributors
        const float power = __fmaf_rn(__fmaf_rn(co.z, dy, co.y * dx), dy, co.x * dxx);  // log2 G
        const float G = ex2_approx(power);
        const float alpha = fminf(0.99f, G * co.w);
        const bool act = inside && contributor < last_contributor && power <= 0.0f &&
                         alpha >= 1.0f / 255.0f;
        const unsigned ballot = __ballot_sync(kFull, act);
        if (ballot == 0u) continue;
        float v[kNParam];
        if (act) {
          const float4 c = sm[j].col;
          const float inv = __fdividef(1.0f, 1.0f - alpha);
          T = T * inv;
          const float dchannel_dcolor = alpha * T;
          acc0 += last_alpha * (lc0 - acc0);  // = la*lc + (1-la)*acc
          acc1 += last_alpha * (lc1 - acc1);
          acc2 += last_alpha * (lc2 - acc2);
          lc0 = c.x;
          lc1 = c.y;
          lc2 = c.z;
          float dL_dalpha = (c.x - acc0) * dLp0;
          dL_dalpha += (c.y - acc1) * dLp1;
          dL_dalpha += (c.z - acc2) * dLp2;
          v[6] = dchannel_dcolor * dLp0;
          v[7] = dchannel_dcolor * dLp1;
          v[8] = dchannel_dcolor * dLp2;
          dL_dalpha *= T;
          last_alpha = alpha;
          dL_dalpha += (-T_final * inv) * bg_dot;
          // dL/dG = o dL/dalpha; with q = G dL/dG the 3DGS terms
          // dL_dG * dG/d(delta) and -0.5 G d d^T dL_dG reuse power's products
          const float q = G * (co.w * dL_dalpha);
          const float qh = -0.5f * q;
          // unscaled conic (a, b, c) = (A, B/2, C) / k (scale_conic)
          const float ca = co.x * (1.0f / kConicScale), cb = co.y * (0.5f / kConicScale),
                      cc = co.z * (1.0f / kConicScale);
          v[0] = -q * (ca * dx + cb * dy) * ddelx_dx;
          v[1] = -q * (cc * dy + cb * dx) * ddely_dy;
          v[2] = qh * dxx;
          v[3] = qh * dxy;
          v[4] = qh * dyy;
          v[5] = G * dL_dalpha;
        } else {
#pragma unroll
          for (int p = 0; p < kNParam; ++p) v[p] = 0.0f;
        }
        const int id = (int)__float_as_uint(g.z);
        if (COUNT && lane == 0) npairs += __popc(ballot);
        if (POL == kNative) {
          native_atomics<kNParam, COUNT>(grad + static_cast<int64_t>(id) * kNParam, v, act, nred);
        } else if (POL == kSwB) {
          reduce_bfly<kNParam, COUNT, true>(id, grad, v, thr, act, lane, nred, ballot, slot, issuer);
        } else if (POL == kSwS) {
          reduce_serial<kNParam, COUNT>(id, grad, v, thr, act, lane, nred, ballot, slot, issuer);
        } else {
          reduce_cccl<kNParam, COUNT>(id, grad, v, act, lane, nred, ballot);
        }
      }
    }
  }
  if (COUNT) {
    flush_count(counters, npairs, lane);
    flush_count(counters + 1, nred, lane);
  }
}

// CTAs per SM the register allocator must allow for the packed kernels (ptxas -v: no spills).
#ifndef DW_MULTI_MIN_BLOCKS
#define DW_MULTI_MIN_BLOCKS 8
#endif
// The timed SW-B instantiation is bounded for 7 CTAs/SM: ptxas then takes 64
// registers, still 8 CTAs/SM resident (C3 0.711 vs 0.717 ms bounded for 8,
// 0.750 for 6); the others stay bounded for 8 (SW-S would take 72 registers)
#ifndef DW_SWB_MIN_BLOCKS
#define DW_SWB_MIN_BLOCKS 7
#endif

// ---------------------------------------------------------------------------
// Packed-FP32 two-pixel kernels (sm_100 FFMA2 / FMUL2 / FADD2).
//
// A lane's two pixels (px, py) and (px, py + 4) run the same blend / gradient
// arithmetic on different data, which is exactly the shape of Blackwell's
// packed f32x2 instructions: one issue slot computes both pixels. The backward
// is issue-bound (ncu: issue slots ~80 % busy, FMA pipe ~42 %), so halving the
// FP instruction count of the per-pixel math is the lever. To keep the packed
// path branch-free, a pixel's per-Gaussian activity enters as a multiplier
// m in {0, 1}: the effective alpha am = m * alpha leaves T and the colour
// accumulator unchanged when m = 0, and zeroes its nine gradients. The
// accumulator is folded eagerly (acc += am (c - acc) after the gradient, the
// same value the paper's loop folds lazily at the next contributor), which
// removes the last_alpha / last_color state. dx is shared by both pixels.
// The mean2D / conic factors (-W/2, -H/2, -1/2) are linear in the sums and
// are applied after the warp reduction (reduce_bfly_scaled).
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Offsets, quadratic form and Gaussian of one staged Gaussian at the lane's two
// pixels -- shared by the forward and the backward so both take identical
// alpha decisions.
struct Eval2 {
  float dx, dxx;
  float2 dy, power, G;
};
// co is the staged scale_conic() conic (every blend kernel stages or
// rewrites it so), g.xy the mean.
__device__ __forceinline__ void eval2(const float4& g, const float4& co, float pfx, float2 npfy,
                                      Eval2& e) {
  e.dx = g.x - pfx;
  e.dy = add2(bc2(g.y), npfy);
  e.dxx = e.dx * e.dx;
  // power = log2 G (its sign is the unscaled power's), in Horner form over dy -- the lane's two pixels share
  // dx: power = (k a dx^2) + dy (2 k b dx + k c dy)
  e.power = fma2(fma2(bc2(co.z), e.dy, bc2(co.y * e.dx)), e.dy, bc2(co.x * e.dxx));
  e.G = make_float2(ex2_approx(e.power.x), ex2_approx(e.power.y));
}

// The forward keeps synchronous staging: with the backward's cp.async double
// buffer it is slower on C3 (0.869 vs 0.833 ms: early-terminating tiles waste
// the prefetched batch) and on C4 too (3.49 vs 3.29 ms: the doubled shared
// memory costs occupancy the latency hiding does not repay).
#ifdef DW_FWD_MIN_BLOCKS  // A/B hook; by default ptxas picks 48 registers (10 CTAs/SM)
#define DW_FWD_BOUNDS __launch_bounds__(128, DW_FWD_MIN_BLOCKS)
#else
#define DW_FWD_BOUNDS __launch_bounds__(128)
#endif
__global__ void DW_FWD_BOUNDS
    k_forward_x2(const CamParams cam, const uint2* __restrict__ ranges,
                 const uint32_t* __restrict__ values, const float2* __restrict__ means2D,
                 const float4* __restrict__ conic_opacity, const float4* __restrict__ rgb,
                 float* __restrict__ final_T, uint32_t* __restrict__ n_contrib,
                 float* __restrict__ out_color, const uint32_t* __restrict__ tile_order) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ Staged sm[kBlock];
  __shared__ uint8_t s_mask[kBlock];
  const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  int tx0, ty0;
  const int view = tile_view(cam, tile, &tx0, &ty0);
  {  // the view's per-pixel outputs (stacked frame)
    const int64_t HWv = static_cast<int64_t>(cam.H) * cam.W;
    final_T += view * HWv;
    n_contrib += view * HWv;
    out_color += view * 3 * HWv;
  }
  const int px = tx0 + (w & 1) * 8 + (lane & 7);
  const int py = ty0 + (w >> 1) * 8 + (lane >> 3);
  const float pfx = (float)px;
  const float2 npfy = make_float2(-(float)py, -(float)(py + 4));
  // A pixel is live while T > 0; termination stores -T (the transmittance
  // at termination, which final_T reports) so no separate done flag is kept.
  // Pixels outside the image start terminated.
  float2 T = make_float2(px < cam.W && py < cam.H ? 1.0f : -1.0f,
                         px < cam.W && py + 4 < cam.H ? 1.0f : -1.0f);
  float2 C0 = bc2(0.0f), C1 = bc2(0.0f), C2 = bc2(0.0f);
  uint32_t last0 = 0, last1 = 0;
  const uint32_t wbits = (1u << (4 * (w >> 1) + (w & 1))) | (1u << (4 * (w >> 1) + (w & 1) + 2));
  const uint2 range = ranges[tile];
  const int rounds = (int)((range.y - range.x + kBlock - 1) / kBlock);
  int todo = (int)(range.y - range.x);
  for (int i = 0; i < rounds; ++i, todo -= kBlock) {
    if (__syncthreads_count(T.x < 0.0f && T.y < 0.0f) == 128) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int st = t + h * 128;
      const uint32_t progress = range.x + i * kBlock + st;
      uint32_t mask = 0;
      if (progress < range.y)
        mask = stage(sm, st, values[progress], tx0, ty0, means2D, conic_opacity, rgb);
      s_mask[st] = (uint8_t)mask;
    }
    __syncthreads();
    const int n = min(kBlock, todo);
    for (int k = 0; k * 32 < n; ++k) {
      if (__all_sync(kFull, T.x < 0.0f && T.y < 0.0f)) break;
      const int jl = k * 32 + lane;
      const uint32_t m = jl < n ? s_mask[jl] : 0u;
      unsigned bits = __ballot_sync(kFull, (m & wbits) != 0u);
      while (bits) {
        const int j = k * 32 + __ffs(bits) - 1;
        bits &= bits - 1u;
        const float4 g = sm[j].xyi;
        const float4 co = sm[j].co;
        Eval2 e;
        eval2(g, co, pfx, npfy, e);
        const float2 Go = mul2(e.G, bc2(co.w));
        const float2 alpha = make_float2(fminf(0.99f, Go.x), fminf(0.99f, Go.y));
        const float2 test_T = mul2(T, add2(bc2(1.0f), make_float2(-alpha.x, -alpha.y)));
        // a terminated pixel (T < 0) has test_T < 0, so the T > 0 check is
        // folded into test_T >= 1e-4 and the termination store into -|T|
        const bool a0 = e.power.x <= 0.0f && alpha.x >= 1.0f / 255.0f;
        const bool a1 = e.power.y <= 0.0f && alpha.y >= 1.0f / 255.0f;
        const bool b0 = a0 && test_T.x >= 0.0001f;  // blends; a0 && !b0 terminates
        const bool b1 = a1 && test_T.y >= 0.0001f;
        const float2 am = make_float2(b0 ? alpha.x : 0.0f, b1 ? alpha.y : 0.0f);
        const float4 c = sm[j].col;
        const float2 aT = mul2(am, T);
        C0 = fma2(bc2(c.x), aT, C0);
        C1 = fma2(bc2(c.y), aT, C1);
        C2 = fma2(bc2(c.z), aT, C2);
        T = make_float2(b0 ? test_T.x : (a0 ? -fabsf(T.x) : T.x),
                        b1 ? test_T.y : (a1 ? -fabsf(T.y) : T.y));
        const uint32_t pos = (uint32_t)(i * kBlock + j + 1);  // 1-based list position
        last0 = b0 ? pos : last0;
        last1 = b1 ? pos : last1;
      }
    }
  }
  const int HW = cam.H * cam.W;
  const float Ts[2] = {fabsf(T.x), fabsf(T.y)}, c0[2] = {C0.x, C0.y}, c1[2] = {C1.x, C1.y},
              c2[2] = {C2.x, C2.y};
  const uint32_t ls[2] = {last0, last1};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int y = py + 4 * k;
    if (px < cam.W && y < cam.H) {
      const int pix = y * cam.W + px;
      final_T[pix] = Ts[k];
      n_contrib[pix] = ls[k];
      out_color[pix] = c0[k] + Ts[k] * cam.bg[0];
      out_color[HW + pix] = c1[k] + Ts[k] * cam.bg[1];
      out_color[2 * HW + pix] = c2[k] + Ts[k] * cam.bg[2];
    }
  }
}

// Backward with two pixels per lane for the reduction policies: warp w owns
// the 8x8 block (column w & 1, row band w >> 1), lane l the pixels
// (l & 7, l >> 3) and 4 rows below; per Gaussian a lane sums its two pixels'
// gradients before the warp runs the DISTWAR policy on the lane sums, so the
// mask / ballot / staging overhead and the warp reduction are paid once per
// 64 pixels.
// GS: floats per gradient row, kNParam ([P][9], Address order) or 12 (the
// padded batch accumulation buffer, reduce_bfly_scaled), SW-B / SW-S only.
template <int POL, bool COUNT, bool TAP = false, bool BULK = false, bool VEC = DW_VEC_RED != 0,
          int GS = kNParam>
__global__ void __launch_bounds__(128, (POL == kSwB && !COUNT && !TAP) ? DW_SWB_MIN_BLOCKS
                                                                      : DW_MULTI_MIN_BLOCKS)
    k_backward_x2(const CamParams cam, const uint2* __restrict__ ranges,
                  const uint32_t* __restrict__ values, const float2* __restrict__ means2D,
                  const float4* __restrict__ conic_opacity, const float4* __restrict__ rgb,
                  const float* __restrict__ final_Ts, const uint32_t* __restrict__ n_contrib,
                  const float* __restrict__ dL_dpixels, int thr, float* __restrict__ grad,
                  unsigned long long* __restrict__ counters, const TapBuf tap,
                  const uint32_t* __restrict__ tile_order, const float4* __restrict__ packed,
                  bool chained) {
  // chained: the caller guarantees nothing this launch reads is written by
  // the previous kernel on the stream (a chain of backwards of independent,
  // already-rendered views adding into one gradient): no grid-completion
  // wait before the work, so this launch's CTAs fill the SMs the previous
  // launch's last wave leaves idle. The wait moves to the end of the last
  // CTA (the last dispatched, so it rarely waits), so this grid still
  // completes only after its predecessor: whatever follows a chain (a PDL
  // kernel waits for its immediate predecessor only) sees every backward of
  // the chain done.
  if (!chained) pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  static_assert(POL != kNative, "native runs the thread-per-pixel kernel");
  static_assert(GS == kNParam || (GS == 12 && !COUNT && !TAP && (POL == kSwB || POL == kSwS)),
                "padded rows: the SW-B reduction path only");
  constexpr int NW = 4;
  __shared__ Staged sm[2][kBlock];  // double buffer: batch i+1 lands while batch i is walked
  __shared__ uint8_t s_mask[kBlock];
  __shared__ uint32_t s_wmax[NW];
  const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  int tx0, ty0;
  const int view = tile_view(cam, tile, &tx0, &ty0);
  const int px = tx0 + (w & 1) * 8 + (lane & 7);
  const int py = ty0 + (w >> 1) * 8 + (lane >> 3);
  const float pfx = (float)px;
  const float2 npfy = make_float2(-(float)py, -(float)(py + 4));
  const int HW = cam.H * cam.W;
  final_Ts += static_cast<int64_t>(view) * HW;  // the view's per-pixel buffers
  n_contrib += static_cast<int64_t>(view) * HW;
  dL_dpixels += static_cast<int64_t>(view) * 3 * HW;
  const uint32_t vbase = static_cast<uint32_t>(view * cam.vstride);  // scene id = id - vbase
  // per-pixel constants and state, packed (pixel 0 in .x, pixel 1 in .y)
  float2 T, nTb, dL0, dL1, dL2;
  uint32_t last0 = 0, last1 = 0;
  {
    float Tf[2] = {0.0f, 0.0f}, d0[2] = {0.0f, 0.0f}, d1[2] = {0.0f, 0.0f}, d2[2] = {0.0f, 0.0f};
    uint32_t ls[2] = {0u, 0u};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int y = py + 4 * k;
      if (px < cam.W && y < cam.H) {
        const int pix = y * cam.W + px;
        Tf[k] = final_Ts[pix];
        ls[k] = n_contrib[pix];
        d0[k] = dL_dpixels[pix];
        d1[k] = dL_dpixels[HW + pix];
        d2[k] = dL_dpixels[2 * HW + pix];
      }
    }
    T = make_float2(Tf[0], Tf[1]);
    dL0 = make_float2(d0[0], d0[1]);
    dL1 = make_float2(d1[0], d1[1]);
    dL2 = make_float2(d2[0], d2[1]);
    const float2 bg_dot = fma2(bc2(cam.bg[2]), dL2,
                               fma2(bc2(cam.bg[1]), dL1, mul2(bc2(cam.bg[0]), dL0)));
    nTb = mul2(mul2(T, bc2(-1.0f)), bg_dot);  // -T_final * (bg . dL/dpixel)
    last0 = ls[0];
    last1 = ls[1];
  }
  float2 accd = bc2(0.0f);  // per pixel: (accumulated colour behind) . dL/dpixel
  const float hw = 0.5f * (float)cam.W, hh = 0.5f * (float)cam.H;
  // mean2D lane values carry the staged conic's factor k (below): 1/k here
  const float scale[kNParam] = {-hw / kConicScale, -hh / kConicScale, -0.5f, -0.5f, -0.5f,
                                1.0f, 1.0f, 1.0f, 1.0f};
  const uint2 range = ranges[tile];
  const uint32_t wmax = __reduce_max_sync(kFull, max(last0, last1));
  if (lane == 0) s_wmax[w] = wmax;
  __syncthreads();
  uint32_t bmax = 0;
#pragma unroll
  for (int k = 0; k < NW; ++k) bmax = max(bmax, s_wmax[k]);
  const uint32_t wbits = (1u << (4 * (w >> 1) + (w & 1))) | (1u << (4 * (w >> 1) + (w & 1) + 2));
  uint32_t nred = 0, npairs = 0;
  bool issuer;
  const int slot = bfly_slot<kNParam>(lane, &issuer);
  float lane_scale = 1.0f;
#pragma unroll
  for (int p = 0; p < kNParam; ++p)
    if (slot == p) lane_scale = scale[p];
  // keep it in a register: ptxas otherwise re-derives it in every reducing iteration
  asm volatile("" : "+f"(lane_scale));
  const int rounds = (int)((bmax + kBlock - 1) / kBlock);
  int todo = (int)bmax;
  const uint32_t top = range.x + bmax;
  // Staging pipeline: ids of batch i+2 are loaded while batch i is walked, the
  // cp.async gather of batch i+1 is in flight meanwhile, so neither global
  // latency is exposed at the batch barrier. Slot st of batch r holds list
  // position top - 1 - (r * 256 + st) (back to front).
  uint32_t cur_id[2], nxt_id[2];
  bool cur_v[2], nxt_v[2];
  __shared__ uint64_t s_bar[BULK ? 2 : 1];  // bulk staging: one mbarrier per buffer
  if (BULK) {
    if (t == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0 && rounds > 0) mbar_expect_tx(&s_bar[0], 48u * min(kBlock, (int)bmax));
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int st = t + h * 128;
    cur_v[h] = st < (int)bmax;
    cur_id[h] = cur_v[h] ? values[top - 1 - st] : 0u;
    if (cur_v[h]) {
      if (BULK) bulk_stage(&sm[0][st], packed + 3 * static_cast<size_t>(cur_id[h]), &s_bar[0]);
      else stage_async(&sm[0][st], cur_id[h], means2D, conic_opacity, rgb);
    }
    nxt_v[h] = kBlock + st < (int)bmax;
    nxt_id[h] = nxt_v[h] ? values[top - 1 - (kBlock + st)] : 0u;
  }
  if (!BULK) cp_async_commit();
  for (int i = 0; i < rounds; ++i, todo -= kBlock) {
    if (BULK) mbar_wait(&s_bar[i & 1], (i >> 1) & 1);
    else cp_async_wait_all();
    __syncthreads();  // batch i landed; every warp is done with batch i-1's buffer
    Staged* cur = sm[i & 1];
    if (BULK) {
      // the async proxy is about to overwrite a buffer the walk wrote through
      // the generic proxy (the mask phase's slot rewrites)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int nn = min(kBlock, (int)bmax - (i + 1) * kBlock);
      if (t == 0 && nn > 0) mbar_expect_tx(&s_bar[(i + 1) & 1], 48u * nn);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int st = t + h * 128;
      if (nxt_v[h]) {
        if (BULK)
          bulk_stage(&sm[(i + 1) & 1][st], packed + 3 * static_cast<size_t>(nxt_id[h]),
                     &s_bar[(i + 1) & 1]);
        else
          stage_async(&sm[(i + 1) & 1][st], nxt_id[h], means2D, conic_opacity, rgb);
      }
    }
    if (!BULK) cp_async_commit();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int st = t + h * 128;
      uint32_t mask = 0;
      if (cur_v[h]) {
        const float4 xy = cur[st].xyi;
        const float4 co = cur[st].co;
        mask = footprint_mask(xy.x, xy.y, cur[st].col.w, tx0, ty0);
        // xyi.zw = (id, k b): RED address, mean2D gradient; co = the walk's
        // exponent coefficients (scale_conic); col.w = 1/opacity
        *reinterpret_cast<float2*>(&cur[st].xyi.z) =
            make_float2(__uint_as_float(cur_id[h] - vbase), kConicScale * co.y);
        cur[st].co = scale_conic(co);
        cur[st].col.w = rcp_approx(co.w);
      }
      s_mask[st] = (uint8_t)mask;
      cur_id[h] = nxt_id[h];
      cur_v[h] = nxt_v[h];
      const int st2 = (i + 2) * kBlock + st;
      nxt_v[h] = st2 < (int)bmax;
      nxt_id[h] = nxt_v[h] ? values[top - 1 - st2] : 0u;
    }
    __syncthreads();
    const int n = min(kBlock, todo);
    const uint32_t base = bmax - 1 - (uint32_t)(i * kBlock);
    for (int k = 0; k * 32 < n; ++k) {
      const int jl = k * 32 + lane;
      const uint32_t m = jl < n ? s_mask[jl] : 0u;
      unsigned bits = __ballot_sync(kFull, (m & wbits) != 0u && (base - (uint32_t)jl) < wmax);
      while (bits) {
        const int j = k * 32 + __ffs(bits) - 1;
        bits &= bits - 1u;
        const uint32_t contributor = base - (uint32_t)j;
        const float4 g = cur[j].xyi;
        const float4 co = cur[j].co;
        Eval2 e;
        eval2(g, co, pfx, npfy, e);
        const float2 Go = mul2(e.G, bc2(co.w));
        // min(0.99, Go) >= 1/255 <=> Go >= 1/255: the clamp waits for the active path
        const bool a0 = contributor < last0 && e.power.x <= 0.0f && Go.x >= 1.0f / 255.0f;
        const bool a1 = contributor < last1 && e.power.y <= 0.0f && Go.y >= 1.0f / 255.0f;
        const bool act = a0 || a1;
        const unsigned ballot = __ballot_sync(kFull, act);
        if (ballot == 0u) continue;
        const float2 alpha = make_float2(fminf(0.99f, Go.x), fminf(0.99f, Go.y));
        const float2 msk = make_float2(a0 ? 1.0f : 0.0f, a1 ? 1.0f : 0.0f);
        const float4 c = cur[j].col;
        const float2 am = mul2(alpha, msk);
        const float2 om = add2(bc2(1.0f), make_float2(-am.x, -am.y));
        const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
        T = mul2(T, inv);
        const float2 dcd = mul2(am, T);
        // dL/dalpha's colour term sum_ch (c_ch - acc_ch) dL_ch = CD - S with
        // CD = c . dL and S = acc . dL carried instead of the three colour
        // accumulators: acc += am (c - acc) gives S += am (CD - S)
        const float2 CD = fma2(bc2(c.z), dL2, fma2(bc2(c.y), dL1, mul2(bc2(c.x), dL0)));
        const float2 dcol = add2(CD, make_float2(-accd.x, -accd.y));
        accd = fma2(am, dcol, accd);
        const float2 dLa = fma2(dcol, T, mul2(nTb, inv));
        // Lane sums of the nine gradients with the factors -W/2, -H/2 (mean2D)
        // and -1/2 (conic) left for after the warp sum. With q = o G dL/dalpha
        // per pixel and dx shared by the lane's two pixels:
        //   mean2D = (a dx Q + b Qy, c Qy + b dx Q),  conic = (dx^2 Q, dx Qy, Qyy),
        //   opacity = Q / o,  colour = sum_pix alpha T dL/dpixel,
        // Q = sum q, Qy = sum q dy, Qyy = sum q dy^2 -- the pixel sum folds into
        // the products instead of nine separate adds.
        const float2 q = mul2(mul2(Go, msk), dLa);
        const float2 qdy = mul2(q, e.dy);
        const float Q = q.x + q.y, Qy = qdy.x + qdy.y;
        const float Qyy = fmaf(qdy.y, e.dy.y, qdy.x * e.dy.x);
        const float tq = e.dx * Q;
        // co = (k a, 2 k b, k c), g.w = k b: mean2D = k (a dx Q + b Qy, c Qy + b dx Q)
        float v[kNParam] = {fmaf(co.x, tq, g.w * Qy),
                            fmaf(co.z, Qy, g.w * tq),
                            e.dxx * Q,
                            e.dx * Qy,
                            Qyy,
                            Q * c.w,
                            fmaf(dcd.y, dL0.y, dcd.x * dL0.x),
                            fmaf(dcd.y, dL1.y, dcd.x * dL1.x),
                            fmaf(dcd.y, dL2.y, dcd.x * dL2.x)};
        const int id = (int)__float_as_uint(g.z);
        if (COUNT) {
          const uint32_t cnt = __popc(__ballot_sync(kFull, a0)) + __popc(__ballot_sync(kFull, a1));
          if (lane == 0) npairs += cnt;
        }
        // SW-S here takes SW-B's path: every lane of the warp walks the same
        // Gaussian, so SW-S's __match_any_sync grouping (reducers.cpp:95-136)
        // is provably one group -- all active lanes, reduced iff popc >= t --
        // which is SW-B's decision and request count (reducers.cpp:138-175);
        // the counting instantiation keeps reduce_serial and checks exactly that
        constexpr bool kBflyPath = POL == kSwB || (POL == kSwS && !COUNT);
        if (TAP || !kBflyPath) {
#pragma unroll
          for (int p = 0; p < kNParam; ++p) v[p] *= scale[p];
        }
        if (TAP) {  // the record the policy reduces: lane value = its pixels' sum
          unsigned long long rec = 0;
          if (lane == 0) rec = atomicAdd(tap.count, 1ull);
          rec = __shfl_sync(kFull, rec, 0);
          if (rec < tap.cap) {
            if (lane == 0) {
              tap.warp_id[rec] = tile * NW + w;
              tap.iteration[rec] = (int32_t)contributor;
              tap.active[rec] = ballot;
            }
            tap.prim[rec * 32 + lane] = id;
#pragma unroll
            for (int p = 0; p < kNParam; ++p) tap.vals[(rec * kNParam + p) * 32 + lane] = v[p];
          }
          reduce_bfly<kNParam, COUNT, true>(id, grad, v, thr, act, lane, nred, ballot, slot,
                                            issuer);
        } else if (kBflyPath) {
          reduce_bfly_scaled<kNParam, COUNT, VEC, GS>(id, grad, v, thr, act, lane, nred, ballot,
                                                      slot, issuer, lane_scale, scale);
        } else if (POL == kSwS) {
          reduce_serial<kNParam, COUNT>(id, grad, v, thr, act, lane, nred, ballot, slot, issuer);
        } else {
          reduce_cccl<kNParam, COUNT>(id, grad, v, act, lane, nred, ballot);
        }
      }
    }
  }
  if (COUNT) {
    flush_count(counters, npairs, lane);
    flush_count(counters + 1, nred, lane);
  }
#ifndef DW_CHAIN_ENDWAIT  // A/B hook: 0 none (unsafe), 1 the last CTA, 2 every CTA
#define DW_CHAIN_ENDWAIT 1
#endif
  if (chained && (DW_CHAIN_ENDWAIT == 2 || (DW_CHAIN_ENDWAIT == 1 && blockIdx.x == gridDim.x - 1)))
    pdl_wait();  // complete after the predecessor
}

// DW_VEC_RED=0 in the environment (read per launch): the SW-B per-lane
// fallback as one scalar RED per param -- bench.py's decomposition arm
bool scalar_fallback() {
  const char* e = std::getenv("DW_VEC_RED");
  return e && *e == '0';
}

template <int POL>
void launch_bwd(bool count, const CamParams& cam, const uint2* ranges, const uint32_t* values,
                const float2* means2D, const float4* co, const float4* rgb,
                const uint32_t* tile_order, const float* fT,
                const uint32_t* nc, const float* dL, int thr, float* grad,
                unsigned long long* ctr, cudaStream_t s, const float4* packed, bool chained,
                int gs) {
  const int grid = cam.tiles_x * cam.tiles_y;
  if constexpr (POL == kSwB || POL == kSwS) {
    if (gs == 12) {  // padded accumulation rows (the batch paths; padded_rows_ok)
      launch_pdl(k_backward_x2<POL, false, false, false, true, 12>, grid, 128, 0, s, cam, ranges,
                 values, means2D, co, rgb, fT, nc, dL, thr, grad, nullptr, TapBuf{}, tile_order,
                 nullptr, chained);
      return;
    }
  }
  // The reduction policies run two pixels per lane; native keeps the paper's
  // thread-per-pixel kernel (profiles/r01/ab_ppt.jsonl).
  if constexpr (POL != kNative) {
    if (count)
      launch_pdl(k_backward_x2<POL, true>, grid, 128, 0, s, cam, ranges, values, means2D, co, rgb,
                 fT, nc, dL, thr, grad, ctr, TapBuf{}, tile_order, nullptr, chained);
    else if (packed)
      launch_pdl(k_backward_x2<POL, false, false, true>, grid, 128, 0, s, cam, ranges, values,
                 means2D, co, rgb, fT, nc, dL, thr, grad, nullptr, TapBuf{}, tile_order, packed,
                 chained);
    else if (POL == kSwB && scalar_fallback())  // DW_VEC_RED=0: scalar per-lane REDs
      launch_pdl(k_backward_x2<POL, false, false, false, false>, grid, 128, 0, s, cam, ranges,
                 values, means2D, co, rgb, fT, nc, dL, thr, grad, nullptr, TapBuf{}, tile_order,
                 nullptr, chained);
    else
      launch_pdl(k_backward_x2<POL, false>, grid, 128, 0, s, cam, ranges, values, means2D, co,
                 rgb, fT, nc, dL, thr, grad, nullptr, TapBuf{}, tile_order, nullptr, chained);
    return;
  }
  if (count)
    k_backward<POL, true><<<grid, kBlock, 0, s>>>(cam, ranges, values, means2D, co, rgb, fT, nc,
                                                  dL, thr, grad, ctr);
  else
    k_backward<POL, false><<<grid, kBlock, 0, s>>>(cam, ranges, values, means2D, co, rgb, fT,
                                                   nc, dL, thr, grad, nullptr);
}

// grad[p][0..9) += pad[p][0..9); pad[p] = 0 (ready for the next batch). One
// thread per primitive: three 16-byte loads and stores of the padded row,
// nine adds into the Address-order row (consecutive threads, consecutive rows).
__global__ void __launch_bounds__(256) k_fold_rows(int64_t P, float4* __restrict__ pad,
                                                   float* __restrict__ grad) {
  pdl_wait();
  pdl_trigger();
  const int64_t p = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  if (p >= P) return;
  const float4 a = pad[3 * p], b = pad[3 * p + 1], c = pad[3 * p + 2];
  float* g = grad + 9 * p;
  const float v[9] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x};
#pragma unroll
  for (int k = 0; k < 9; ++k) g[k] += v[k];
  const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  pad[3 * p] = z;
  pad[3 * p + 1] = z;
  pad[3 * p + 2] = z;
}

}  // namespace

void launch_fold_rows(int64_t P, float* pad, float* grad, cudaStream_t s) {
  if (P <= 0) return;
  launch_pdl(k_fold_rows, static_cast<unsigned>((P + 255) / 256), 256, 0, s, P,
             reinterpret_cast<float4*>(pad), grad);
  DW_CUDA(cudaGetLastError());
}

void launch_backward_tap(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                         const float2* means2D, const float4* co, const float4* rgb,
                         const uint32_t* tile_order, const float* final_T,
                         const uint32_t* n_contrib, const float* dL, int thr, float* grad,
                         const TapBuf& tap, cudaStream_t s) {
  const int grid = cam.tiles_x * cam.tiles_y;
  launch_pdl(k_backward_x2<kSwB, false, true>, grid, 128, 0, s, cam, ranges, values, means2D, co,
             rgb, final_T, n_contrib, dL, thr, grad, nullptr, tap, tile_order, nullptr, false);
  DW_CUDA(cudaGetLastError());
}

void launch_forward_impl(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                         const float2* means2D, const float4* conic_opacity, const float4* rgb,
                         const uint32_t* tile_order, float* final_T, uint32_t* n_contrib,
                         float* out_color, cudaStream_t s) {
  const int grid = cam.tiles_x * cam.tiles_y;
  launch_pdl(k_forward_x2, grid, 128, 0, s, cam, ranges, values, means2D, conic_opacity, rgb,
             final_T, n_contrib, out_color, tile_order);
  DW_CUDA(cudaGetLastError());
}

void launch_backward_impl(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                          const float2* means2D, const float4* co, const float4* rgb,
                          const uint32_t* tile_order, const float* final_T,
                          const uint32_t* n_contrib, const float* dL, int policy, int thr,
                          float* grad, unsigned long long* counters, cudaStream_t s,
                          const float4* packed, bool chained, int grad_stride) {
  const bool count = counters != nullptr;
  if (grad_stride != kNParam &&
      !(grad_stride == 12 && !count && !packed && (policy == kSwB || policy == kSwS)))
    throw std::invalid_argument("padded gradient rows: SW-B / SW-S, uncounted, cp.async staging");
  switch (policy) {
    case kNative:
      launch_bwd<kNative>(count, cam, ranges, values, means2D, co, rgb, tile_order, final_T,
                          n_contrib, dL, thr, grad, counters, s, packed, chained, grad_stride);
      break;
    case kSwS:
      launch_bwd<kSwS>(count, cam, ranges, values, means2D, co, rgb, tile_order, final_T, n_contrib,
                       dL, thr, grad, counters, s, packed, chained, grad_stride);
      break;
    case kSwB:
      launch_bwd<kSwB>(count, cam, ranges, values, means2D, co, rgb, tile_order, final_T, n_contrib,
                       dL, thr, grad, counters, s, packed, chained, grad_stride);
      break;
    default:
      launch_bwd<kCccl>(count, cam, ranges, values, means2D, co, rgb, tile_order, final_T,
                        n_contrib, dL, thr, grad, counters, s, packed, chained, grad_stride);
  }
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
