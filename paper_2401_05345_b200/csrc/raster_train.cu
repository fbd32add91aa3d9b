// The steps either side of the hot path: preprocess-backward
// turns one view's screen-space gradients grad2d[P][9] into 3D gradients
// grad3d[P][14] (means3D xyz, scales xyz, rotation r x y z, opacity, rgb),
// accumulated over views so the per-rank buffer is a real training gradient
// before the all-reduce; a fused Adam step consumes it.
//
// Math: the public 3DGS preprocess backward, restated (oracle/gs_oracle.c
// gs_preprocess_backward is the float64 reference, pinned by finite
// differences in tests/test_gs_oracle.py):
//   conic -> cov2D (A, B, C):  d/dA = (-C^2 ga + B C gb - B^2 gc) / D^2, ...
//                              with gb = 2 * grad2d.conic_y (half convention)
//   cov2D = T Sigma T^T + 0.3 I, T = J W:  dSigma = T^T G T, dT = 2 G T Sigma
//   J(t) with the 1.3 tan(fov) clamp zeroing the x/y terms, t = W m + t0
//   ndc = (P m)_xy / ((P m)_w + 1e-7)
//   Sigma = R diag((mod s)^2) R^T from the normalised quaternion (its
//   normalisation differentiated).
// One thread per Gaussian, HBM-bound: ~116 B read + 56 B read-modify-write.
#include <cuda_runtime.h>

#include "dw_internal.h"
#include "raster.cuh"

namespace dw {

namespace {

__global__ void __launch_bounds__(256)
    k_preprocess_backward(int P, const float* __restrict__ means3D, const float* __restrict__ scales,
                          const float* __restrict__ rotations, const int* __restrict__ radii,
                          const CamParams cam, const float* __restrict__ grad2d,
                          float* __restrict__ grad3d) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P || radii[i] <= 0) return;
  const float* g2 = grad2d + static_cast<int64_t>(i) * kNParam;
  float* g3 = grad3d + static_cast<int64_t>(i) * kNParam3D;
  const float* vm = cam.vm;
  const float* pm = cam.pm;
  const float mx = means3D[3 * i], my = means3D[3 * i + 1], mz = means3D[3 * i + 2];
  const float4 q0 = make_float4(rotations[4 * i], rotations[4 * i + 1], rotations[4 * i + 2],
                                rotations[4 * i + 3]);
  const float qn = sqrtf(q0.x * q0.x + q0.y * q0.y + q0.z * q0.z + q0.w * q0.w);
  const float r = q0.x / qn, x = q0.y / qn, y = q0.z / qn, z = q0.w / qn;
  const float R[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - r * z), 2.f * (x * z + r * y)},
                         {2.f * (x * y + r * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - r * x)},
                         {2.f * (x * z - r * y), 2.f * (y * z + r * x), 1.f - 2.f * (x * x + y * y)}};
  const float mod = cam.scale_modifier;
  float sv[3], var[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    sv[k] = mod * scales[3 * i + k];
    var[k] = sv[k] * sv[k];
  }
  float Sig[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      Sig[a][b] = R[a][0] * var[0] * R[b][0] + R[a][1] * var[1] * R[b][1] + R[a][2] * var[2] * R[b][2];
  float t[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) t[a] = vm[a] * mx + vm[4 + a] * my + vm[8 + a] * mz + vm[12 + a];
  const float fx = (float)cam.W / (2.0f * cam.tan_fovx), fy = (float)cam.H / (2.0f * cam.tan_fovy);
  const float limx = 1.3f * cam.tan_fovx, limy = 1.3f * cam.tan_fovy;
  const float txtz = t[0] / t[2], tytz = t[1] / t[2];
  const float xmul = (txtz < -limx || txtz > limx) ? 0.f : 1.f;
  const float ymul = (tytz < -limy || tytz > limy) ? 0.f : 1.f;
  const float tz = t[2];
  const float tx = fminf(limx, fmaxf(-limx, txtz)) * tz, ty = fminf(limy, fmaxf(-limy, tytz)) * tz;
  const float J[2][3] = {{fx / tz, 0.f, -fx * tx / (tz * tz)}, {0.f, fy / tz, -fy * ty / (tz * tz)}};
  float Wm[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) Wm[a][b] = vm[b * 4 + a];
  float T[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) T[a][b] = J[a][0] * Wm[0][b] + J[a][1] * Wm[1][b] + J[a][2] * Wm[2][b];
  float TS[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) TS[a][b] = T[a][0] * Sig[0][b] + T[a][1] * Sig[1][b] + T[a][2] * Sig[2][b];
  const float A = TS[0][0] * T[0][0] + TS[0][1] * T[0][1] + TS[0][2] * T[0][2] + 0.3f;
  const float B = TS[0][0] * T[1][0] + TS[0][1] * T[1][1] + TS[0][2] * T[1][2];
  const float Cc = TS[1][0] * T[1][0] + TS[1][1] * T[1][1] + TS[1][2] * T[1][2] + 0.3f;
  const float D = A * Cc - B * B;
  const float iD2 = 1.0f / (D * D);
  const float ga = g2[2], gb = 2.0f * g2[3], gc = g2[4];
  const float dA = (-Cc * Cc * ga + B * Cc * gb - B * B * gc) * iD2;
  const float dC = (-B * B * ga + A * B * gb - A * A * gc) * iD2;
  const float dB = (2.f * B * Cc * ga - (D + 2.f * B * B) * gb + 2.f * A * B * gc) * iD2;
  const float G[2][2] = {{dA, 0.5f * dB}, {0.5f * dB, dC}};
  float dSig[3][3], dT[2][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      dSig[a][b] = T[0][a] * (G[0][0] * T[0][b] + G[0][1] * T[1][b]) +
                   T[1][a] * (G[1][0] * T[0][b] + G[1][1] * T[1][b]);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) dT[a][b] = 2.f * (G[a][0] * TS[0][b] + G[a][1] * TS[1][b]);
  float dJ[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) dJ[a][b] = dT[a][0] * Wm[b][0] + dT[a][1] * Wm[b][1] + dT[a][2] * Wm[b][2];
  const float tz2 = tz * tz, tz3 = tz2 * tz;
  const float dt0 = xmul * (-fx / tz2) * dJ[0][2];
  const float dt1 = ymul * (-fy / tz2) * dJ[1][2];
  const float dt2 = -fx / tz2 * dJ[0][0] - fy / tz2 * dJ[1][1] + 2.f * fx * tx / tz3 * dJ[0][2] +
                    2.f * fy * ty / tz3 * dJ[1][2];
  float dm[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) dm[b] = Wm[0][b] * dt0 + Wm[1][b] * dt1 + Wm[2][b] * dt2;
  const float hx = pm[0] * mx + pm[4] * my + pm[8] * mz + pm[12];
  const float hy = pm[1] * mx + pm[5] * my + pm[9] * mz + pm[13];
  const float hw = pm[3] * mx + pm[7] * my + pm[11] * mz + pm[15] + 0.0000001f;
  const float ihw2 = 1.0f / (hw * hw);
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const float dnx = (pm[4 * b] * hw - hx * pm[4 * b + 3]) * ihw2;
    const float dny = (pm[4 * b + 1] * hw - hy * pm[4 * b + 3]) * ihw2;
    dm[b] += g2[0] * dnx + g2[1] * dny;
  }
  float dscale[3], dR[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) acc += R[a][k] * dSig[a][b] * R[b][k];
    dscale[k] = acc * 2.f * mod * sv[k];
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dR[a][k] = 2.f * (dSig[a][0] * R[0][k] + dSig[a][1] * R[1][k] + dSig[a][2] * R[2][k]) * var[k];
  // d R / d (r, x, y, z), contracted with dR
  const float dqr = 2.f * (-z * dR[0][1] + y * dR[0][2] + z * dR[1][0] - x * dR[1][2] - y * dR[2][0] +
                           x * dR[2][1]);
  const float dqx = 2.f * (y * dR[0][1] + z * dR[0][2] + y * dR[1][0] - 2.f * x * dR[1][1] -
                           r * dR[1][2] + z * dR[2][0] + r * dR[2][1] - 2.f * x * dR[2][2]);
  const float dqy = 2.f * (-2.f * y * dR[0][0] + x * dR[0][1] + r * dR[0][2] + x * dR[1][0] +
                           z * dR[1][2] - r * dR[2][0] + z * dR[2][1] - 2.f * y * dR[2][2]);
  const float dqz = 2.f * (-2.f * z * dR[0][0] - r * dR[0][1] + x * dR[0][2] + r * dR[1][0] -
                           2.f * z * dR[1][1] + y * dR[1][2] + x * dR[2][0] + y * dR[2][1]);
  const float dot = r * dqr + x * dqx + y * dqy + z * dqz;
  g3[0] += dm[0];
  g3[1] += dm[1];
  g3[2] += dm[2];
  g3[3] += dscale[0];
  g3[4] += dscale[1];
  g3[5] += dscale[2];
  g3[6] += (dqr - r * dot) / qn;
  g3[7] += (dqx - x * dot) / qn;
  g3[8] += (dqy - y * dot) / qn;
  g3[9] += (dqz - z * dot) / qn;
  g3[10] += g2[5];
  g3[11] += g2[6];
  g3[12] += g2[7];
  g3[13] += g2[8];
}

// Adam over the 14 parameters of every Gaussian: element k of the flat
// [P][14] gradient / moment buffers maps to its parameter array; lr per
// group (means, scales, rotations, opacity, colours).
__global__ void __launch_bounds__(256)
    k_adam(int64_t n, float* __restrict__ means3D, float* __restrict__ scales,
           float* __restrict__ rotations, float* __restrict__ opacities, float* __restrict__ colors,
           const float* __restrict__ grad, float* __restrict__ m, float* __restrict__ v,
           float lr0, float lr1, float lr2, float lr3, float lr4, float b1, float b2, float eps,
           float bc1, float bc2) {
  pdl_wait();  // predecessor grid complete (programmatic dependent launch)
  pdl_trigger();
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t i = k / kNParam3D;
  const int s = static_cast<int>(k - i * kNParam3D);
  float* p;
  float lr;
  if (s < 3) { p = means3D + 3 * i + s; lr = lr0; }
  else if (s < 6) { p = scales + 3 * i + (s - 3); lr = lr1; }
  else if (s < 10) { p = rotations + 4 * i + (s - 6); lr = lr2; }
  else if (s == 10) { p = opacities + i; lr = lr3; }
  else { p = colors + 3 * i + (s - 11); lr = lr4; }
  const float g = grad[k];
  const float mk = b1 * m[k] + (1.f - b1) * g;
  const float vk = b2 * v[k] + (1.f - b2) * g * g;
  m[k] = mk;
  v[k] = vk;
  *p -= lr * (mk / bc1) / (sqrtf(vk / bc2) + eps);
}

}  // namespace

void launch_preprocess_backward(int P, const float* means3D, const float* scales,
                                const float* rotations, const int* radii, const CamParams& cam,
                                const float* grad2d, float* grad3d, cudaStream_t s) {
  if (P <= 0) return;
  launch_pdl(k_preprocess_backward, (P + 255) / 256, 256, 0, s, P, means3D, scales, rotations,
             radii, cam, grad2d, grad3d);
  DW_CUDA(cudaGetLastError());
}

void launch_adam(int P, float* means3D, float* scales, float* rotations, float* opacities,
                 float* colors, const float* grad, float* m, float* v, const float lr[5], float b1,
                 float b2, float eps, int step, cudaStream_t s) {
  if (P <= 0) return;
  const int64_t n = static_cast<int64_t>(P) * kNParam3D;
  const float bc1 = 1.f - powf(b1, (float)step), bc2 = 1.f - powf(b2, (float)step);
  launch_pdl(k_adam, static_cast<unsigned>((n + 255) / 256), 256, 0, s, n, means3D, scales,
             rotations, opacities, colors, grad, m, v, lr[0], lr[1], lr[2], lr[3], lr[4], b1, b2,
             eps, bc1, bc2);
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
