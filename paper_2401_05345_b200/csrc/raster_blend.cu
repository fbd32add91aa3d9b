// Front-to-back alpha blending (forward) and its analytic backward with the
// DISTWAR reduction -- the hot path.
//
// One 256-thread CTA per 16x16 tile. The tile's sorted Gaussian list is
// walked in batches of 256 staged in shared memory (48 B per Gaussian:
// xy + radius + id, conic + opacity, rgb). Each warp owns an 8x4 pixel block
// and, per Gaussian, first tests that block against the Gaussian's
// conservative alpha footprint (warp-uniform branch): a Gaussian whose
// alpha is below 1/255 over the whole block is skipped without any per-lane
// exp. The footprint bound: alpha >= 1/255 needs d^T Sigma^-1 d <=
// 2 ln(255 o) <= 2 ln 255, i.e. |d| <= sqrt(2 ln 255) sigma_max < 1.11 *
// radius (radius = ceil(3 sigma_max)), so culling at 1.11 * radius + 1 px
// never drops a pair the oracle keeps.
//
// Backward: the GradComputation loop of PAPER.md:1481-1504 -- each pixel
// thread walks its Gaussians back to front, cond1/cond2 are the
// last-contributor and alpha tests, and the 9 atomicAdds are replaced by a
// call of the DISTWAR policy (distwar.cuh) made by all 32 lanes, inactive
// lanes carrying zero gradients. A warp whose 32 lanes
// are all inactive for a Gaussian (ballot == 0) issues nothing, as the
// reference policies emit no request for an empty active mask
// (reducers.cpp:154-156).
#include <cuda_runtime.h>

#include "distwar.cuh"
#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

struct __align__(16) Staged {
  float4 xyri;  // x, y, radius (int bits), id (uint bits)
  float4 co;    // conic a, b, c, opacity
  float4 col;   // r, g, b, -
};

__device__ __forceinline__ bool warp_culled(float gx, float gy, int radius, float opacity,
                                            int wx0, int wy0) {
  if (opacity > 1.0f) return false;  // the footprint bound assumes o <= 1
  const float rc = 1.11f * (float)radius + 1.0f;
  const float dx = fmaxf(0.0f, fmaxf((float)wx0 - gx, gx - (float)(wx0 + 7)));
  const float dy = fmaxf(0.0f, fmaxf((float)wy0 - gy, gy - (float)(wy0 + 3)));
  return dx > rc || dy > rc;
}

__device__ __forceinline__ void stage(Staged* s, int slot, uint32_t id,
                                      const float2* __restrict__ means2D,
                                      const float4* __restrict__ conic_opacity,
                                      const float4* __restrict__ rgb, const int* __restrict__ radii) {
  const float2 m = __ldg(means2D + id);
  s[slot].xyri = make_float4(m.x, m.y, __int_as_float(__ldg(radii + id)), __uint_as_float(id));
  s[slot].co = __ldg(conic_opacity + id);
  s[slot].col = __ldg(rgb + id);
}

__global__ void __launch_bounds__(kBlock)
    k_forward(const CamParams cam, const uint2* __restrict__ ranges,
              const uint32_t* __restrict__ values, const float2* __restrict__ means2D,
              const float4* __restrict__ conic_opacity, const float4* __restrict__ rgb,
              const int* __restrict__ radii, float* __restrict__ final_T,
              uint32_t* __restrict__ n_contrib, float* __restrict__ out_color) {
  __shared__ Staged sm[kBlock];
  const int tile = blockIdx.x, t = threadIdx.x, w = t >> 5;
  int px, py;
  tile_pixel(tile, t, cam.tiles_x, &px, &py);
  const int wx0 = (tile % cam.tiles_x) * kTile + (w & 1) * 8;
  const int wy0 = (tile / cam.tiles_x) * kTile + (w >> 1) * 4;
  const bool inside = px < cam.W && py < cam.H;
  const float pfx = (float)px, pfy = (float)py;
  const uint2 range = ranges[tile];
  const int rounds = (int)((range.y - range.x + kBlock - 1) / kBlock);
  int todo = (int)(range.y - range.x);
  bool done = !inside;
  float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  uint32_t contributor = 0, last = 0;
  for (int i = 0; i < rounds; ++i, todo -= kBlock) {
    if (__syncthreads_count(done) == kBlock) break;
    const uint32_t progress = range.x + i * kBlock + t;
    if (progress < range.y) stage(sm, t, values[progress], means2D, conic_opacity, rgb, radii);
    __syncthreads();
    const int n = min(kBlock, todo);
    for (int j = 0; j < n && !done; ++j) {
      contributor++;
      const float4 g = sm[j].xyri;
      const float4 co = sm[j].co;
      if (warp_culled(g.x, g.y, __float_as_int(g.z), co.w, wx0, wy0)) continue;
      const float dx = g.x - pfx, dy = g.y - pfy;
      const float power = -0.5f * (co.x * dx * dx + co.z * dy * dy) - co.y * dx * dy;
      if (power > 0.0f) continue;
      const float alpha = fminf(0.99f, co.w * __expf(power));
      if (alpha < 1.0f / 255.0f) continue;
      const float test_T = T * (1.0f - alpha);
      if (test_T < 0.0001f) {
        done = true;
        continue;
      }
      const float4 c = sm[j].col;
      const float aT = alpha * T;
      C0 += c.x * aT;
      C1 += c.y * aT;
      C2 += c.z * aT;
      T = test_T;
      last = contributor;
    }
  }
  if (inside) {
    const int pix = py * cam.W + px;
    const int HW = cam.H * cam.W;
    final_T[pix] = T;
    n_contrib[pix] = last;
    out_color[pix] = C0 + T * cam.bg[0];
    out_color[HW + pix] = C1 + T * cam.bg[1];
    out_color[2 * HW + pix] = C2 + T * cam.bg[2];
  }
}

template <int POL, bool COUNT>
__global__ void __launch_bounds__(kBlock)
    k_backward(const CamParams cam, const uint2* __restrict__ ranges,
               const uint32_t* __restrict__ values, const float2* __restrict__ means2D,
               const float4* __restrict__ conic_opacity, const float4* __restrict__ rgb,
               const int* __restrict__ radii, const float* __restrict__ final_Ts,
               const uint32_t* __restrict__ n_contrib, const float* __restrict__ dL_dpixels,
               int thr, float* __restrict__ grad, unsigned long long* __restrict__ counters) {
  __shared__ Staged sm[kBlock];
  __shared__ uint32_t s_wmax[kBlock / 32];
  const int tile = blockIdx.x, t = threadIdx.x, w = t >> 5, lane = t & 31;
  int px, py;
  tile_pixel(tile, t, cam.tiles_x, &px, &py);
  const int wx0 = (tile % cam.tiles_x) * kTile + (w & 1) * 8;
  const int wy0 = (tile / cam.tiles_x) * kTile + (w >> 1) * 4;
  const bool inside = px < cam.W && py < cam.H;
  const int pix = py * cam.W + px;
  const int HW = cam.H * cam.W;
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

  // Gaussians at list index >= max(last_contributor) over the tile cannot
  // contribute to any of its pixels: start the back-to-front walk there.
  const uint32_t wmax = __reduce_max_sync(kFull, last_contributor);
  if (lane == 0) s_wmax[w] = wmax;
  __syncthreads();
  uint32_t bmax = 0;
#pragma unroll
  for (int k = 0; k < kBlock / 32; ++k) bmax = max(bmax, s_wmax[k]);

  float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
  float lc0 = 0.0f, lc1 = 0.0f, lc2 = 0.0f, last_alpha = 0.0f;
  uint32_t contributor = bmax;
  uint32_t nred = 0, npairs = 0;
  const int rounds = (int)((bmax + kBlock - 1) / kBlock);
  int todo = (int)bmax;
  const uint32_t top = range.x + bmax;  // exclusive end of the live list
  for (int i = 0; i < rounds; ++i, todo -= kBlock) {
    __syncthreads();
    if (t < todo) stage(sm, t, values[top - 1 - (i * kBlock + t)], means2D, conic_opacity, rgb, radii);
    __syncthreads();
    const int n = min(kBlock, todo);
    for (int j = 0; j < n; ++j) {
      contributor--;
      if (contributor >= wmax) continue;  // warp-uniform: no lane can be active
      const float4 g = sm[j].xyri;
      const float4 co = sm[j].co;
      if (warp_culled(g.x, g.y, __float_as_int(g.z), co.w, wx0, wy0)) continue;
      const float dx = g.x - pfx, dy = g.y - pfy;
      const float power = -0.5f * (co.x * dx * dx + co.z * dy * dy) - co.y * dx * dy;
      const float G = __expf(power);
      const float alpha = fminf(0.99f, co.w * G);
      const bool act = inside && contributor < last_contributor && power <= 0.0f &&
                       alpha >= 1.0f / 255.0f;
      const unsigned ballot = __ballot_sync(kFull, act);
      if (ballot == 0u) continue;
      float v[kNParam];
      if (act) {
        const float4 c = sm[j].col;
        const float one_m = 1.0f - alpha;
        T = T / one_m;
        const float dchannel_dcolor = alpha * T;
        acc0 = last_alpha * lc0 + (1.0f - last_alpha) * acc0;
        acc1 = last_alpha * lc1 + (1.0f - last_alpha) * acc1;
        acc2 = last_alpha * lc2 + (1.0f - last_alpha) * acc2;
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
        dL_dalpha += (-T_final / one_m) * bg_dot;
        const float dL_dG = co.w * dL_dalpha;
        const float gdx = G * dx, gdy = G * dy;
        const float dG_ddelx = -gdx * co.x - gdy * co.y;
        const float dG_ddely = -gdy * co.z - gdx * co.y;
        v[0] = dL_dG * dG_ddelx * ddelx_dx;
        v[1] = dL_dG * dG_ddely * ddely_dy;
        v[2] = -0.5f * gdx * dx * dL_dG;
        v[3] = -0.5f * gdx * dy * dL_dG;
        v[4] = -0.5f * gdy * dy * dL_dG;
        v[5] = G * dL_dalpha;
      } else {
#pragma unroll
        for (int p = 0; p < kNParam; ++p) v[p] = 0.0f;
      }
      const int id = (int)__float_as_uint(g.w);
      if (COUNT && lane == 0) npairs += __popc(ballot);
      if (POL == kNative) {
        native_atomics<kNParam, COUNT>(grad + static_cast<int64_t>(id) * kNParam, v, act, nred);
      } else if (POL == kSwB) {
        reduce_bfly<kNParam, COUNT, true>(id, grad, v, thr, act, lane, nred, ballot);
      } else if (POL == kSwS) {
        reduce_serial<kNParam, COUNT>(id, grad, v, thr, act, lane, nred, ballot);
      } else {
        reduce_cccl<kNParam, COUNT>(id, grad, v, act, lane, nred, ballot);
      }
    }
  }
  if (COUNT) {
    flush_count(counters, npairs, lane);
    flush_count(counters + 1, nred, lane);
  }
}

template <int POL>
void launch_bwd(bool count, const CamParams& cam, const uint2* ranges, const uint32_t* values,
                const float2* means2D, const float4* co, const float4* rgb, const int* radii,
                const float* fT, const uint32_t* nc, const float* dL, int thr, float* grad,
                unsigned long long* ctr, cudaStream_t s) {
  const int grid = cam.tiles_x * cam.tiles_y;
  if (count)
    k_backward<POL, true><<<grid, kBlock, 0, s>>>(cam, ranges, values, means2D, co, rgb, radii,
                                                  fT, nc, dL, thr, grad, ctr);
  else
    k_backward<POL, false><<<grid, kBlock, 0, s>>>(cam, ranges, values, means2D, co, rgb, radii,
                                                   fT, nc, dL, thr, grad, nullptr);
}

}  // namespace

void launch_forward_impl(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                         const float2* means2D, const float4* conic_opacity, const float4* rgb,
                         const int* radii, float* final_T, uint32_t* n_contrib, float* out_color,
                         cudaStream_t s) {
  const int grid = cam.tiles_x * cam.tiles_y;
  k_forward<<<grid, kBlock, 0, s>>>(cam, ranges, values, means2D, conic_opacity, rgb, radii,
                                    final_T, n_contrib, out_color);
  DW_CUDA(cudaGetLastError());
}

void launch_backward_impl(const CamParams& cam, const uint2* ranges, const uint32_t* values,
                          const float2* means2D, const float4* co, const float4* rgb,
                          const int* radii, const float* final_T, const uint32_t* n_contrib,
                          const float* dL, int policy, int thr, float* grad,
                          unsigned long long* counters, cudaStream_t s) {
  const bool count = counters != nullptr;
  switch (policy) {
    case kNative:
      launch_bwd<kNative>(count, cam, ranges, values, means2D, co, rgb, radii, final_T,
                          n_contrib, dL, thr, grad, counters, s);
      break;
    case kSwS:
      launch_bwd<kSwS>(count, cam, ranges, values, means2D, co, rgb, radii, final_T, n_contrib,
                       dL, thr, grad, counters, s);
      break;
    case kSwB:
      launch_bwd<kSwB>(count, cam, ranges, values, means2D, co, rgb, radii, final_T, n_contrib,
                       dL, thr, grad, counters, s);
      break;
    default:
      launch_bwd<kCccl>(count, cam, ranges, values, means2D, co, rgb, radii, final_T, n_contrib,
                        dL, thr, grad, counters, s);
  }
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
