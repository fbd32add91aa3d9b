// Host orchestration of one view: render_forward / render_backward.
//
// Per-view device state lives in grow-only HBM buffers owned by the
// dw_rasterizer handle, so a training loop re-renders without reallocating:
//   per Gaussian: means2D f32x2, depth, radius, conic+opacity f32x4,
//                 rgb f32x4, tiles_touched u32, inclusive offsets u64
//   per instance: keys u64 x2, values u32 x2 (double-buffered radix sort)
//   per tile:     ranges u32x2;  per pixel: final_T f32, n_contrib u32
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "distwar.cuh"
#include "dw_internal.h"
#include "raster.cuh"

namespace {

template <typename T>
void grow(T*& p, size_t& cap, size_t want) {
  if (want <= cap && p) return;
  if (p) DW_CUDA(cudaFree(p));
  p = nullptr;
  const size_t n = std::max<size_t>(want, 1) + std::max<size_t>(want, 1) / 8;
  DW_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(T)));
  cap = n;
}

}  // namespace

struct dw_rasterizer {
  int P = 0, W = 0, H = 0;
  int64_t num_rendered = 0;
  dw::CamParams cam{};
  int tile_bits = 0;
  bool forward_done = false;

  size_t cap_p = 0, cap_p2 = 0, cap_p3 = 0, cap_p4 = 0, cap_p5 = 0, cap_p6 = 0, cap_p7 = 0;
  float2* means2D = nullptr;
  float* depths = nullptr;
  int* radii = nullptr;
  float4* conic_opacity = nullptr;
  float4* rgb = nullptr;
  uint32_t* tiles_touched = nullptr;
  uint64_t* offsets = nullptr;

  size_t cap_i = 0, cap_i2 = 0, cap_i3 = 0, cap_i4 = 0;
  uint64_t* keys_in = nullptr;
  uint64_t* keys = nullptr;
  uint32_t* vals_in = nullptr;
  uint32_t* vals = nullptr;

  size_t cap_t = 0, cap_px = 0, cap_px2 = 0;
  uint2* ranges = nullptr;
  float* final_T = nullptr;
  uint32_t* n_contrib = nullptr;

  size_t cap_tmp = 0;
  unsigned char* tmp = nullptr;
  unsigned long long* counters = nullptr;  // [pairs, reds]
  uint64_t* h_total = nullptr;             // pinned

  // host-entry scratch (dw_render_host)
  size_t cap_h[8] = {0};
  float* h_bufs[8] = {nullptr};

  ~dw_rasterizer() {
    void* ps[] = {means2D, depths, radii, conic_opacity, rgb, tiles_touched, offsets, keys_in,
                  keys, vals_in, vals, ranges, final_T, n_contrib, tmp, counters};
    for (void* p : ps)
      if (p) cudaFree(p);
    for (float* p : h_bufs)
      if (p) cudaFree(p);
    if (h_total) cudaFreeHost(h_total);
  }

  void forward(int32_t P_, const float* means3D, const float* scales, const float* rotations,
               const float* opacities, const float* colors, const dw_camera& c, float* out_color,
               int32_t* radii_out, cudaStream_t s) {
    if (P_ < 0) throw std::invalid_argument("P must be >= 0");
    if (c.width < 1 || c.height < 1) throw std::invalid_argument("camera size must be >= 1");
    if (!(c.tan_fovx > 0.0f) || !(c.tan_fovy > 0.0f))
      throw std::invalid_argument("tan_fov must be > 0");
    P = P_;
    W = c.width;
    H = c.height;
    std::memcpy(cam.vm, c.viewmatrix, sizeof(cam.vm));
    std::memcpy(cam.pm, c.projmatrix, sizeof(cam.pm));
    cam.tan_fovx = c.tan_fovx;
    cam.tan_fovy = c.tan_fovy;
    std::memcpy(cam.bg, c.bg, sizeof(cam.bg));
    cam.scale_modifier = c.scale_modifier;
    cam.W = W;
    cam.H = H;
    cam.tiles_x = (W + dw::kTile - 1) / dw::kTile;
    cam.tiles_y = (H + dw::kTile - 1) / dw::kTile;
    const int ntiles = cam.tiles_x * cam.tiles_y;
    tile_bits = 0;
    while ((1 << tile_bits) < ntiles) ++tile_bits;

    const size_t np = static_cast<size_t>(std::max(P, 1));
    grow(means2D, cap_p, np);
    grow(depths, cap_p2, np);
    grow(radii, cap_p3, np);
    grow(conic_opacity, cap_p4, np);
    grow(rgb, cap_p5, np);
    grow(tiles_touched, cap_p6, np);
    grow(offsets, cap_p7, np);
    grow(ranges, cap_t, static_cast<size_t>(ntiles));
    grow(final_T, cap_px, static_cast<size_t>(W) * H);
    grow(n_contrib, cap_px2, static_cast<size_t>(W) * H);
    if (!counters) DW_CUDA(cudaMalloc(&counters, 2 * sizeof(unsigned long long)));
    if (!h_total) DW_CUDA(cudaMallocHost(&h_total, sizeof(uint64_t)));

    dw::launch_preprocess(P, means3D, scales, rotations, opacities, colors, cam, means2D, depths,
                          radii, conic_opacity, rgb, tiles_touched, s);
    num_rendered = 0;
    if (P > 0) {
      size_t scan_bytes = 0;
      DW_CUDA(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, tiles_touched, offsets, P, s));
      ensure_tmp(scan_bytes);
      DW_CUDA(cub::DeviceScan::InclusiveSum(tmp, scan_bytes, tiles_touched, offsets, P, s));
      DW_CUDA(cudaMemcpyAsync(h_total, offsets + P - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      DW_CUDA(cudaStreamSynchronize(s));
      num_rendered = static_cast<int64_t>(*h_total);
    }
    if (num_rendered >= (int64_t(1) << 32))
      throw std::runtime_error("more than 2^32 tile instances");
    const size_t ni = static_cast<size_t>(std::max<int64_t>(num_rendered, 1));
    grow(keys_in, cap_i, ni);
    grow(keys, cap_i2, ni);
    grow(vals_in, cap_i3, ni);
    grow(vals, cap_i4, ni);
    dw::launch_duplicate(P, means2D, depths, radii, offsets, cam, keys_in, vals_in, s);
    if (num_rendered > 0) {
      size_t sort_bytes = 0;
      DW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys_in, keys, vals_in, vals,
                                              num_rendered, 0, 32 + tile_bits, s));
      ensure_tmp(sort_bytes);
      DW_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, keys_in, keys, vals_in, vals,
                                              num_rendered, 0, 32 + tile_bits, s));
    }
    DW_CUDA(cudaMemsetAsync(ranges, 0, sizeof(uint2) * ntiles, s));
    dw::launch_ranges(num_rendered, keys, ranges, s);
    dw::launch_forward_impl(cam, ranges, vals, means2D, conic_opacity, rgb, radii, final_T,
                            n_contrib, out_color, s);
    if (radii_out && P > 0)
      DW_CUDA(cudaMemcpyAsync(radii_out, radii, sizeof(int) * P, cudaMemcpyDeviceToDevice, s));
    forward_done = true;
  }

  void backward(const float* dL_dpixels, int policy, int thr, float* grad, uint64_t* pairs_out,
                cudaStream_t s) {
    if (!forward_done) throw std::invalid_argument("render_backward before render_forward");
    if (policy == DW_POLICY_HW_ATOMRED || policy < 0 || policy > 4)
      throw std::invalid_argument("policy has no B200 kernel (hw_atomred is simulated hardware)");
    if (thr < 0 || thr > 33) throw std::invalid_argument("balance threshold out of range 0..33");
    if (P == 0) {
      if (pairs_out) *pairs_out = 0;
      return;
    }
    unsigned long long* ctr = nullptr;
    if (pairs_out) {
      DW_CUDA(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), s));
      ctr = counters;
    }
    dw::launch_backward_impl(cam, ranges, vals, means2D, conic_opacity, rgb, radii, final_T,
                             n_contrib, dL_dpixels, policy, thr, grad, ctr, s);
    if (pairs_out) {
      unsigned long long h[2];
      DW_CUDA(cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, s));
      DW_CUDA(cudaStreamSynchronize(s));
      *pairs_out = h[0];
      last_reds = h[1];
    }
  }

  uint64_t last_reds = 0;

  void ensure_tmp(size_t bytes) { grow(tmp, cap_tmp, bytes); }

  float* host_scratch(int slot, size_t n) {
    grow(h_bufs[slot], cap_h[slot], n);
    return h_bufs[slot];
  }
};

namespace dw {

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    DW_CUDA(cudaGetDevice(&dev));
    DW_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

}  // namespace dw

// Entry points used by capi.cpp.
namespace dw {

void raster_forward(dw_rasterizer* r, int32_t P, const float* m, const float* sc, const float* rot,
                    const float* op, const float* col, const dw_camera* cam, float* out,
                    int32_t* radii, int64_t* nr, cudaStream_t s) {
  r->forward(P, m, sc, rot, op, col, *cam, out, radii, s);
  if (nr) *nr = r->num_rendered;
}

void raster_backward(dw_rasterizer* r, const float* dL, int policy, int thr, float* grad,
                     uint64_t* pairs, cudaStream_t s) {
  r->backward(dL, policy, thr, grad, pairs, s);
}

uint64_t raster_last_reds(const dw_rasterizer* r) { return r->last_reds; }

void raster_buffer(const dw_rasterizer* r, int which, const void** p, int64_t* count) {
  const int64_t P = r->P, I = r->num_rendered, npx = int64_t(r->W) * r->H;
  const int64_t nt = int64_t(r->cam.tiles_x) * r->cam.tiles_y;
  switch (which) {
    case 0: *p = r->means2D; *count = 2 * P; break;
    case 1: *p = r->depths; *count = P; break;
    case 2: *p = r->radii; *count = P; break;
    case 3: *p = r->conic_opacity; *count = 4 * P; break;
    case 4: *p = r->tiles_touched; *count = P; break;
    case 5: *p = r->keys; *count = I; break;
    case 6: *p = r->vals; *count = I; break;
    case 7: *p = r->ranges; *count = 2 * nt; break;
    case 8: *p = r->final_T; *count = npx; break;
    case 9: *p = r->n_contrib; *count = npx; break;
    default: throw std::invalid_argument("unknown rasterizer buffer");
  }
}

void raster_host(dw_rasterizer* r, int32_t P, const float* m, const float* sc, const float* rot,
                 const float* op, const float* col, const dw_camera* cam, const float* dL,
                 int policy, int thr, float* out_color, float* grad, cudaStream_t s) {
  const size_t np = static_cast<size_t>(std::max(P, 1));
  const size_t npx = static_cast<size_t>(cam->width) * cam->height;
  float* d_m = r->host_scratch(0, 3 * np);
  float* d_sc = r->host_scratch(1, 3 * np);
  float* d_rot = r->host_scratch(2, 4 * np);
  float* d_op = r->host_scratch(3, np);
  float* d_col = r->host_scratch(4, 3 * np);
  float* d_dl = r->host_scratch(5, 3 * npx);
  float* d_img = r->host_scratch(6, 3 * npx);
  float* d_g = r->host_scratch(7, kNParam * np);
  auto h2d = [&](float* d, const float* h, size_t n) {
    if (n) DW_CUDA(cudaMemcpyAsync(d, h, n * sizeof(float), cudaMemcpyHostToDevice, s));
  };
  h2d(d_m, m, 3 * size_t(P));
  h2d(d_sc, sc, 3 * size_t(P));
  h2d(d_rot, rot, 4 * size_t(P));
  h2d(d_op, op, size_t(P));
  h2d(d_col, col, 3 * size_t(P));
  h2d(d_dl, dL, 3 * npx);
  r->forward(P, d_m, d_sc, d_rot, d_op, d_col, *cam, d_img, nullptr, s);
  DW_CUDA(cudaMemsetAsync(d_g, 0, kNParam * np * sizeof(float), s));
  r->backward(d_dl, policy, thr, d_g, nullptr, s);
  DW_CUDA(cudaMemcpyAsync(out_color, d_img, 3 * npx * sizeof(float), cudaMemcpyDeviceToHost, s));
  if (P > 0)
    DW_CUDA(cudaMemcpyAsync(grad, d_g, kNParam * size_t(P) * sizeof(float),
                            cudaMemcpyDeviceToHost, s));
  DW_CUDA(cudaStreamSynchronize(s));
}

}  // namespace dw

namespace dw {
dw_rasterizer* raster_new() { return new dw_rasterizer(); }
void raster_delete(dw_rasterizer* r) { delete r; }
}  // namespace dw
