// Preprocess / projection: one thread per Gaussian, coalesced float4 staging.
//
// COMPILED WITH -fmad=false: every product and sum rounds separately, in the
// exact operation order of the CPU oracle (oracle/gs_oracle.c
// preprocess_one, built with -ffp-contract=off). That makes means2D,
// depths, radii and tiles_touched -- and therefore the (tile|depth) keys,
// the sorted instance order and the tile ranges -- bit-exact between GPU and
// oracle. The kernel is HBM-bound (~64 B in, ~60 B out per Gaussian), so the
// lost FMA contraction costs nothing measurable.
//
// The P x 3 inputs (means3D, scales, colors) are not 16 B aligned per
// Gaussian, so each CTA stages its 256 Gaussians' 768 floats through shared
// memory with 192 coalesced float4 loads, then each thread reads its triple.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

// Half-extents of the alpha >= 1/255 ellipse: alpha = min(0.99, o G) with
// G = exp(-q/2), q = d^T Q d (Q = conic) needs q <= tau = 2 ln(255 o); the
// ellipse q <= tau lies in |dx| <= sqrt(tau Q^-1_xx), |dy| <= sqrt(tau Q^-1_yy)
// with Q^-1_xx = c / (ac - b^2), Q^-1_yy = a / (ac - b^2). tau is inflated by
// 5 % + 0.05 (the blend's exp2 approximation and FMA rounding) and the half2
// is rounded up: -inf = never visible (o <= 1/255), +inf = degenerate conic.
__device__ __forceinline__ uint32_t footprint_extents(const float4& co) {
  float ex, ey;
  if (!(co.w * 255.0f > 1.0f)) {
    ex = ey = -INFINITY;
  } else {
    const float det = co.x * co.z - co.y * co.y;
    if (!(det > 0.0f) || !(co.x > 0.0f)) {
      ex = ey = INFINITY;
    } else {
      // fast-math reciprocal / rsqrt: the 0.2 % margin covers their few-ulp error
      const float tau = 1.05f * 2.0f * __logf(255.0f * co.w) + 0.05f;
      const float rdet = __fdividef(1.0f, det);
      const float x = tau * co.z * rdet, y = tau * co.x * rdet;
      ex = x * rsqrtf(x) * 1.002f;
      ey = y * rsqrtf(y) * 1.002f;
    }
  }
  const __half2 h = __halves2half2(__float2half_ru(ex), __float2half_ru(ey));
  return *reinterpret_cast<const uint32_t*>(&h);
}

template <bool VEC>
__device__ __forceinline__ void stage3(const float* __restrict__ src, float* sm, int64_t first,
                                       int64_t total) {
  if (VEC) {
    for (int i = threadIdx.x; i < 3 * kBlock / 4; i += blockDim.x) {
      const int64_t f = first + 4 * i;
      if (f + 4 <= total) {
        *reinterpret_cast<float4*>(sm + 4 * i) = __ldg(reinterpret_cast<const float4*>(src + f));
      } else {
        for (int k = 0; k < 4; ++k)
          if (f + k < total) sm[4 * i + k] = __ldg(src + f + k);
      }
    }
  } else {
    for (int i = threadIdx.x; i < 3 * kBlock; i += blockDim.x)
      if (first + i < total) sm[i] = __ldg(src + first + i);
  }
}

__device__ __forceinline__ float ndc2pix(float v, int S) {
  return ((v + 1.0f) * (float)S - 1.0f) * 0.5f;
}

#ifndef DW_PRE_MIN_BLOCKS
#define DW_PRE_MIN_BLOCKS 8  // 32 registers, 8 CTAs/SM: C5 preprocess 0.103 -> 0.084 ms (latency-bound loads)
#endif
template <bool VEC>
__global__ void __launch_bounds__(kBlock, DW_PRE_MIN_BLOCKS)
    k_preprocess(int P, const float* __restrict__ means3D, const float* __restrict__ scales,
                 const float* __restrict__ rotations, const float* __restrict__ opacities,
                 const float* __restrict__ colors, const CamParams cam,
                 float2* __restrict__ means2D, float* __restrict__ depths,
                 int* __restrict__ radii, float4* __restrict__ conic_opacity,
                 float4* __restrict__ rgb, uint32_t* __restrict__ tiles_touched,
                 uint32_t* __restrict__ dkey, uint32_t* __restrict__ dids,
                 float4* __restrict__ packed, uint32_t* __restrict__ rect_out, int row0,
                 uint32_t id0) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  __shared__ __align__(16) float s_mean[3 * kBlock];
  __shared__ __align__(16) float s_scale[3 * kBlock];
  __shared__ __align__(16) float s_col[3 * kBlock];
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kBlock;
  stage3<VEC>(means3D, s_mean, 3 * b0, 3 * static_cast<int64_t>(P));
  stage3<VEC>(scales, s_scale, 3 * b0, 3 * static_cast<int64_t>(P));
  stage3<VEC>(colors, s_col, 3 * b0, 3 * static_cast<int64_t>(P));
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t i = b0 + t;
  if (i >= P) return;
  radii[i] = 0;
  tiles_touched[i] = 0;
  // block binning (nullable): the tile rectangle packed x0 | y0 << 8 |
  // (x1-1) << 16 | (y1-1) << 24 (tile units < 256), empty = 0x0000ff00
  if (rect_out) rect_out[i] = 0x0000ff00u;
  // depth-sort input (nullable): (depth bits, id), culled Gaussians last
  if (dkey) {
    dkey[i] = 0xffffffffu;
    dids[i] = id0 + static_cast<uint32_t>(i);  // id0: the view's first id in a stacked frame
  }

  const float px = s_mean[3 * t], py = s_mean[3 * t + 1], pz = s_mean[3 * t + 2];
  const float* vm = cam.vm;
  const float* pm = cam.pm;
  float tv0 = vm[0] * px + vm[4] * py + vm[8] * pz + vm[12];
  float tv1 = vm[1] * px + vm[5] * py + vm[9] * pz + vm[13];
  const float tv2 = vm[2] * px + vm[6] * py + vm[10] * pz + vm[14];
  if (tv2 <= 0.2f) return;  // near-plane cull
  const float hx = pm[0] * px + pm[4] * py + pm[8] * pz + pm[12];
  const float hy = pm[1] * px + pm[5] * py + pm[9] * pz + pm[13];
  const float hw = pm[3] * px + pm[7] * py + pm[11] * pz + pm[15];
  const float pw = 1.0f / (hw + 0.0000001f);
  const float nx = hx * pw, ny = hy * pw;

  // Sigma = R diag(s^2) R^T from the normalised (r, x, y, z) quaternion.
  float4 q;
  if (VEC) q = __ldg(reinterpret_cast<const float4*>(rotations) + i);
  else q = make_float4(rotations[4 * i], rotations[4 * i + 1], rotations[4 * i + 2],
                       rotations[4 * i + 3]);
  const float inv = 1.0f / sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
  const float r = q.x * inv, x = q.y * inv, y = q.z * inv, z = q.w * inv;
  float R[3][3];
  R[0][0] = 1.0f - 2.0f * (y * y + z * z);
  R[0][1] = 2.0f * (x * y - r * z);
  R[0][2] = 2.0f * (x * z + r * y);
  R[1][0] = 2.0f * (x * y + r * z);
  R[1][1] = 1.0f - 2.0f * (x * x + z * z);
  R[1][2] = 2.0f * (y * z - r * x);
  R[2][0] = 2.0f * (x * z - r * y);
  R[2][1] = 2.0f * (y * z + r * x);
  R[2][2] = 1.0f - 2.0f * (x * x + y * y);
  const float mod = cam.scale_modifier;
  const float s0 = mod * s_scale[3 * t], s1 = mod * s_scale[3 * t + 1],
              s2 = mod * s_scale[3 * t + 2];
  const float v0 = s0 * s0, v1 = s1 * s1, v2 = s2 * s2;
#define SIG(i, j) (R[i][0] * v0 * R[j][0] + R[i][1] * v1 * R[j][1] + R[i][2] * v2 * R[j][2])
  const float c00 = SIG(0, 0), c01 = SIG(0, 1), c02 = SIG(0, 2);
  const float c11 = SIG(1, 1), c12 = SIG(1, 2), c22 = SIG(2, 2);
#undef SIG

  // EWA: cov2D = T Sigma T^T + 0.3 I with T = J W.
  const float fx = (float)cam.W / (2.0f * cam.tan_fovx);
  const float fy = (float)cam.H / (2.0f * cam.tan_fovy);
  const float limx = 1.3f * cam.tan_fovx, limy = 1.3f * cam.tan_fovy;
  const float txtz = tv0 / tv2, tytz = tv1 / tv2;
  tv0 = fminf(limx, fmaxf(-limx, txtz)) * tv2;
  tv1 = fminf(limy, fmaxf(-limy, tytz)) * tv2;
  const float j00 = fx / tv2, j02 = -(fx * tv0) / (tv2 * tv2);
  const float j11 = fy / tv2, j12 = -(fy * tv1) / (tv2 * tv2);
  float T0[3], T1[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    T0[j] = j00 * vm[j * 4 + 0] + j02 * vm[j * 4 + 2];
    T1[j] = j11 * vm[j * 4 + 1] + j12 * vm[j * 4 + 2];
  }
  const float S[3][3] = {{c00, c01, c02}, {c01, c11, c12}, {c02, c12, c22}};
  float A0[3], A1[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    A0[j] = T0[0] * S[0][j] + T0[1] * S[1][j] + T0[2] * S[2][j];
    A1[j] = T1[0] * S[0][j] + T1[1] * S[1][j] + T1[2] * S[2][j];
  }
  const float ca = A0[0] * T0[0] + A0[1] * T0[1] + A0[2] * T0[2];
  const float cb = A0[0] * T1[0] + A0[1] * T1[1] + A0[2] * T1[2];
  const float cc = A1[0] * T1[0] + A1[1] * T1[1] + A1[2] * T1[2];
  const float cv0 = ca + 0.3f, cv1 = cb, cv2 = cc + 0.3f;

  const float det = cv0 * cv2 - cv1 * cv1;
  if (det == 0.0f) return;
  const float det_inv = 1.0f / det;
  const float mid = 0.5f * (cv0 + cv2);
  const float disc = sqrtf(fmaxf(0.1f, mid * mid - det));
  const float l1 = mid + disc, l2 = mid - disc;
  const int radius = (int)ceilf(3.0f * sqrtf(fmaxf(l1, l2)));
  const float ix = ndc2pix(nx, cam.W), iy = ndc2pix(ny, cam.H);
  const float fr = (float)radius;
  int rminx = (int)((ix - fr) / (float)kTile), rminy = (int)((iy - fr) / (float)kTile);
  int rmaxx = (int)((ix + fr + (float)(kTile - 1)) / (float)kTile);
  int rmaxy = (int)((iy + fr + (float)(kTile - 1)) / (float)kTile);
  rminx = min(cam.tiles_x, max(0, rminx));
  rmaxx = min(cam.tiles_x, max(0, rmaxx));
  rminy = min(cam.tiles_y, max(0, rminy));
  rmaxy = min(cam.tiles_y, max(0, rmaxy));
  const int area = (rmaxx - rminx) * (rmaxy - rminy);
  if (area == 0) return;
  depths[i] = tv2;
  if (dkey && radius > 0) dkey[i] = __float_as_uint(tv2);
  radii[i] = radius;
  means2D[i] = make_float2(ix, iy);
  const float op = __ldg(opacities + i);
  const float4 co = make_float4(cv2 * det_inv, -cv1 * det_inv, cv0 * det_inv, op);
  conic_opacity[i] = co;
  // w: the blend kernels' footprint half-extents (raster_blend.cu
  // footprint_mask) as a half2, rounded up with a margin so the mask stays a
  // superset of the alpha >= 1/255 ellipse's pixel bands
  const float4 c4 = make_float4(s_col[3 * t], s_col[3 * t + 1], s_col[3 * t + 2],
                                __uint_as_float(footprint_extents(co)));
  rgb[i] = c4;
  if (packed) {  // the blend kernels' 48-byte staged record (bulk-copy staging)
    packed[3 * i] = make_float4(ix, iy, 0.0f, 0.0f);
    packed[3 * i + 1] = co;
    packed[3 * i + 2] = c4;
  }
  tiles_touched[i] = static_cast<uint32_t>(area);
  if (rect_out)  // rows in the (stacked) frame: row0 = the view's first tile row
    rect_out[i] = (uint32_t)rminx | (uint32_t)(rminy + row0) << 8 | (uint32_t)(rmaxx - 1) << 16 |
                  (uint32_t)(rmaxy - 1 + row0) << 24;
}

}  // namespace

void launch_preprocess(int P, const float* means3D, const float* scales, const float* rotations,
                       const float* opacities, const float* colors, const CamParams& cam,
                       float2* means2D, float* depths, int* radii, float4* conic_opacity,
                       float4* rgb, uint32_t* tiles_touched, uint32_t* dkey, uint32_t* dids,
                       cudaStream_t s, float4* packed, uint32_t* rect_out, int row0,
                       uint32_t id0) {
  if (P <= 0) return;
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool vec = aligned(means3D) && aligned(scales) && aligned(colors) && aligned(rotations);
  const int grid = (P + kBlock - 1) / kBlock;
  if (vec)
    launch_pdl(k_preprocess<true>, grid, kBlock, 0, s, P, means3D, scales, rotations, opacities,
               colors, cam, means2D, depths, radii, conic_opacity, rgb, tiles_touched, dkey, dids,
               packed, rect_out, row0, id0);
  else
    launch_pdl(k_preprocess<false>, grid, kBlock, 0, s, P, means3D, scales, rotations, opacities,
               colors, cam, means2D, depths, radii, conic_opacity, rgb, tiles_touched, dkey, dids,
               packed, rect_out, row0, id0);
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
