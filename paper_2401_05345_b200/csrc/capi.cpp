// extern "C" boundary of libdistwar.so (include/distwar.h). Error handling
// mirrors the reference's capi.cpp:16-44: a thread-local last-error string
// and an exception -> status mapping in guarded().
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and enum values only: the symbols are resolved at run time

#include <algorithm>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "dw_internal.h"

struct dw_rasterizer;

namespace dw {
void raster_forward(dw_rasterizer* r, int32_t P, const float* m, const float* sc, const float* rot,
                    const float* op, const float* col, const dw_camera* cam, float* out,
                    int32_t* radii, int64_t* nr, cudaStream_t s, bool nosync);
void raster_forward_views(dw_rasterizer* r, int32_t P, const float* m, const float* sc,
                          const float* rot, const float* op, const float* col,
                          const dw_camera* cams, int32_t nv, float* out, int64_t* nr,
                          cudaStream_t s);
int raster_max_stacked_views(int32_t W, int32_t H);
void raster_backward_views(dw_rasterizer* const* rs, const float* const* dLs, int32_t n,
                           int policy, int thr, float* grad, cudaStream_t s);
void raster_reserve(dw_rasterizer* r, int32_t P, int32_t W, int32_t H, int64_t max_instances);
int64_t raster_resolve(dw_rasterizer* r, bool* overflowed);
void raster_backward(dw_rasterizer* r, const float* dL, int policy, int thr, float* grad,
                     uint64_t* pairs, cudaStream_t s, bool chained = false);
uint64_t raster_last_reds(const dw_rasterizer* r);
void raster_stage_timing(dw_rasterizer* r, bool on);
int raster_stage_ms(dw_rasterizer* r, double* out, int cap);
void raster_buffer(const dw_rasterizer* r, int which, const void** p, int64_t* count);
void raster_host(dw_rasterizer* r, int32_t P, const float* m, const float* sc, const float* rot,
                 const float* op, const float* col, const dw_camera* cam, const float* dL,
                 int policy, int thr, float* out_color, float* grad, cudaStream_t s);
void raster_views_host(dw_rasterizer* r, int32_t P, const float* m, const float* sc,
                       const float* rot, const float* op, const float* col, const dw_camera* cams,
                       int32_t V, const float* dL, int policy, int thr, float* out_images,
                       float* grad, cudaStream_t s, bool grad_on_device);
float* raster_scratch_grad(dw_rasterizer* r, int32_t P);
void raster_preprocess_backward(dw_rasterizer* r, const float* means3D, const float* scales,
                                const float* rotations, const float* grad2d, float* grad3d,
                                cudaStream_t s);
dw::HostTrace raster_backward_tap(dw_rasterizer* r, const float* dL, int thr, float* grad,
                                  int64_t max_records, int64_t* total, cudaStream_t s);
void launch_adam(int P, float* means3D, float* scales, float* rotations, float* opacities,
                 float* colors, const float* grad, float* m, float* v, const float lr[5], float b1,
                 float b2, float eps, int step, cudaStream_t s);
dw_rasterizer* raster_new();
void raster_delete(dw_rasterizer* r);
}  // namespace dw

namespace {

thread_local std::string last_error = "ok";

dw_status fail(dw_status code, const std::string& message) {
  last_error = message;
  return code;
}

dw_status fail_invalid(const std::string& m) { return fail(DW_ERR_INVALID_ARGUMENT, m); }

template <typename Fn>
dw_status guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const std::invalid_argument& e) {
    return fail(DW_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::ios_base::failure& e) {
    return fail(DW_ERR_IO, e.what());
  } catch (const std::exception& e) {
    return fail(DW_ERR_RUNTIME, e.what());
  }
}

void check_policy(dw_policy_kind kind, int threshold) {
  if (kind == DW_POLICY_HW_ATOMRED)
    throw std::invalid_argument("apply_policy: hw_atomred has no per-record core policy");
  if (kind < DW_POLICY_NATIVE || kind > DW_POLICY_HW_ATOMRED)
    throw std::invalid_argument("unknown policy kind");
  if ((kind == DW_POLICY_SW_S || kind == DW_POLICY_SW_B) && (threshold < 0 || threshold > 33))
    throw std::invalid_argument("balance threshold out of range 0..33");
}

struct Events {
  cudaEvent_t a{}, b{};
  Events() {
    DW_CUDA(cudaEventCreate(&a));
    DW_CUDA(cudaEventCreate(&b));
  }
  ~Events() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  float ms() const {
    float m = 0;
    DW_CUDA(cudaEventElapsedTime(&m, a, b));
    return m;
  }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { DW_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T))); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

dw_device_trace* upload(const dw::HostTrace& t, cudaStream_t s) {
  const int64_t R = t.records();
  const int n = t.scene.params_per_primitive;
  auto d = std::make_unique<dw_device_trace>();
  d->records = R;
  d->params = n;
  d->num_primitives = t.scene.num_primitives;
  for (int64_t r = 0; r < R; ++r) {
    for (int l = 0; l < 32; ++l) {
      const int32_t id = t.prim[r * 32 + l];
      if ((t.active[r] >> l & 1u) && (id < 0 || id >= d->num_primitives))
        throw std::invalid_argument("active lane references a primitive out of range");
    }
    d->contributions += static_cast<uint64_t>(__builtin_popcount(t.active[r])) * n;
  }
  std::vector<float> vals(static_cast<size_t>(R) * 32 * n);
  for (int64_t r = 0; r < R; ++r)
    for (int l = 0; l < 32; ++l)
      for (int p = 0; p < n; ++p)
        vals[(static_cast<size_t>(r) * n + p) * 32 + l] =
            static_cast<float>(t.grads[(static_cast<size_t>(r) * 32 + l) * n + p]);
  DW_CUDA(cudaMalloc(&d->active, std::max<int64_t>(R, 1) * sizeof(uint32_t)));
  DW_CUDA(cudaMalloc(&d->prim, std::max<int64_t>(R, 1) * 32 * sizeof(int32_t)));
  DW_CUDA(cudaMalloc(&d->vals, std::max<size_t>(vals.size(), 1) * sizeof(float)));
  if (R) {
    DW_CUDA(cudaMemcpyAsync(d->active, t.active.data(), R * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    DW_CUDA(cudaMemcpyAsync(d->prim, t.prim.data(), R * 32 * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    DW_CUDA(cudaMemcpyAsync(d->vals, vals.data(), vals.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  }
  DW_CUDA(cudaStreamSynchronize(s));
  return d.release();
}

void free_device_trace(dw_device_trace* d) {
  if (!d) return;
  cudaFree(d->active);
  cudaFree(d->prim);
  cudaFree(d->vals);
  delete d;
}

}  // namespace

extern "C" {

const char* dw_version(void) { return "distwar-b200 0.1.0"; }

const char* dw_last_error(void) { return last_error.c_str(); }

int dw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

int dw_device_clock_khz(void) {
  int dev = 0, khz = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev) != cudaSuccess) {
    last_error = cudaGetErrorString(cudaGetLastError());
    return -1;
  }
  return khz;
}

void dw_scene_spec_init(dw_scene_spec* scene) {
  if (scene) dw::scene_defaults(scene);
}

dw_status dw_trace_generate(const dw_scene_spec* scene, dw_trace** out) {
  if (!scene || !out) return fail_invalid("null argument");
  return guarded([&] {
    auto t = std::make_unique<dw_trace>();
    t->t = dw::generate(*scene);
    *out = t.release();
    return DW_OK;
  });
}

void dw_trace_free(dw_trace* trace) { delete trace; }

int64_t dw_trace_record_count(const dw_trace* trace) { return trace ? trace->t.records() : -1; }

dw_status dw_trace_save(const dw_trace* trace, const char* path, int binary) {
  if (!trace || !path) return fail_invalid("null argument");
  return guarded([&] {
    if (!binary) throw std::invalid_argument("only the WRTRACEB binary container is supported");
    dw::save_binary(trace->t, path);
    return DW_OK;
  });
}

dw_status dw_trace_load(const char* path, int binary, dw_trace** out) {
  if (!path || !out) return fail_invalid("null argument");
  return guarded([&] {
    if (!binary) throw std::invalid_argument("only the WRTRACEB binary container is supported");
    auto t = std::make_unique<dw_trace>();
    t->t = dw::load_binary(path);
    *out = t.release();
    return DW_OK;
  });
}

dw_status dw_trace_histogram_distinct(const dw_trace* trace, uint64_t out_counts[33]) {
  if (!trace || !out_counts) return fail_invalid("null argument");
  return guarded([&] {
    uint64_t act[33];
    dw::histograms(trace->t, out_counts, act);
    return DW_OK;
  });
}

dw_status dw_trace_histogram_active(const dw_trace* trace, uint64_t out_counts[33]) {
  if (!trace || !out_counts) return fail_invalid("null argument");
  return guarded([&] {
    uint64_t distinct[33];
    dw::histograms(trace->t, distinct, out_counts);
    return DW_OK;
  });
}

dw_status dw_trace_from_arrays(int64_t num_records, int32_t params, int32_t num_primitives,
                               const int32_t* warp_id, const int32_t* iteration,
                               const uint32_t* active, const int32_t* prim, const double* grads,
                               dw_trace** out) {
  if (!out || (num_records > 0 && (!active || !prim || !grads))) return fail_invalid("null argument");
  return guarded([&] {
    if (num_records < 0 || params < 1 || num_primitives < 1)
      throw std::invalid_argument("invalid trace dimensions");
    auto t = std::make_unique<dw_trace>();
    dw::scene_defaults(&t->t.scene);
    t->t.scene.params_per_primitive = params;
    t->t.scene.num_primitives = num_primitives;
    const size_t R = static_cast<size_t>(num_records);
    t->t.warp_id.assign(R, 0);
    t->t.iteration.assign(R, 0);
    if (warp_id) t->t.warp_id.assign(warp_id, warp_id + R);
    if (iteration) t->t.iteration.assign(iteration, iteration + R);
    t->t.active.assign(active, active + R);
    t->t.prim.assign(prim, prim + R * 32);
    t->t.grads.assign(grads, grads + R * 32 * params);
    *out = t.release();
    return DW_OK;
  });
}

dw_status dw_trace_arrays(const dw_trace* trace, const uint32_t** active, const int32_t** prim,
                          const double** grads, dw_scene_spec* scene) {
  if (!trace) return fail_invalid("null argument");
  if (active) *active = trace->t.active.data();
  if (prim) *prim = trace->t.prim.data();
  if (grads) *grads = trace->t.grads.data();
  if (scene) *scene = trace->t.scene;
  return DW_OK;
}

dw_status dw_trace_ids(const dw_trace* trace, const int32_t** warp_id, const int32_t** iteration) {
  if (!trace) return fail_invalid("null argument");
  if (warp_id) *warp_id = trace->t.warp_id.data();
  if (iteration) *iteration = trace->t.iteration.data();
  return DW_OK;
}

dw_status dw_trace_set_scene(dw_trace* trace, const dw_scene_spec* scene) {
  if (!trace || !scene) return fail_invalid("null argument");
  return guarded([&] {
    if (scene->params_per_primitive != trace->t.scene.params_per_primitive)
      throw std::invalid_argument("params_per_primitive must match the trace's records");
    trace->t.scene = *scene;
    return DW_OK;
  });
}

dw_status dw_trace_upload(const dw_trace* trace, void* stream, dw_device_trace** out) {
  if (!trace || !out) return fail_invalid("null argument");
  return guarded([&] {
    *out = upload(trace->t, dw::as_stream(stream));
    return DW_OK;
  });
}

void dw_device_trace_free(dw_device_trace* d) { free_device_trace(d); }

dw_status dw_device_trace_view(const dw_device_trace* d, const uint32_t** a, const int32_t** p,
                               const float** v, int64_t* R, int32_t* n, int32_t* P) {
  if (!d) return fail_invalid("null argument");
  if (a) *a = d->active;
  if (p) *p = d->prim;
  if (v) *v = d->vals;
  if (R) *R = d->records;
  if (n) *n = d->params;
  if (P) *P = d->num_primitives;
  return DW_OK;
}

dw_status dw_reduce_records(const uint32_t* d_active, const int32_t* d_prim, const float* d_vals,
                            int64_t num_records, int32_t params, int32_t num_primitives,
                            dw_policy_kind policy, int32_t threshold, float* d_grad,
                            unsigned long long* d_red_count, void* stream) {
  if (num_records > 0 && (!d_active || !d_prim || !d_vals || !d_grad))
    return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    if (num_records < 0 || params < 1 || num_primitives < 1)
      throw std::invalid_argument("invalid trace dimensions");
    dw::launch_reduce_records(d_active, d_prim, d_vals, num_records, params, policy, threshold,
                              d_grad, d_red_count, dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_gpu_run(const dw_device_trace* d, dw_policy_kind policy, int32_t threshold,
                     float* host_grad_out, dw_gpu_metrics* out) {
  if (!d || !out) return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    const size_t words = static_cast<size_t>(d->num_primitives) * d->params;
    DevBuf<float> grad(words);
    DevBuf<unsigned long long> ctr(1);
    cudaStream_t s = nullptr;
    // counting pass (its own instantiation, so the timed pass carries no counter)
    DW_CUDA(cudaMemsetAsync(grad.p, 0, words * sizeof(float), s));
    DW_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned long long), s));
    dw::launch_reduce_records(d->active, d->prim, d->vals, d->records, d->params, policy,
                              threshold, grad.p, ctr.p, s);
    unsigned long long reds = 0;
    DW_CUDA(cudaMemcpy(&reds, ctr.p, sizeof(reds), cudaMemcpyDeviceToHost));
    // timed pass
    Events ev;
    DW_CUDA(cudaMemsetAsync(grad.p, 0, words * sizeof(float), s));
    DW_CUDA(cudaEventRecord(ev.a, s));
    dw::launch_reduce_records(d->active, d->prim, d->vals, d->records, d->params, policy,
                              threshold, grad.p, nullptr, s);
    DW_CUDA(cudaEventRecord(ev.b, s));
    DW_CUDA(cudaEventSynchronize(ev.b));
    out->kernel_ms = ev.ms();
    out->atomic_requests_to_l2 = reds;
    out->contributions = d->contributions;
    out->records = static_cast<uint64_t>(d->records);
    if (host_grad_out)
      DW_CUDA(cudaMemcpy(host_grad_out, grad.p, words * sizeof(float), cudaMemcpyDeviceToHost));
    return DW_OK;
  });
}

dw_status dw_model_costs(const dw_device_trace* d, dw_policy_kind policy, int32_t threshold,
                         uint64_t out[2]) {
  if (!d || !out) return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    DevBuf<unsigned long long> ctr(2);
    DW_CUDA(cudaMemsetAsync(ctr.p, 0, 2 * sizeof(unsigned long long), nullptr));
    dw::launch_model_costs(d->active, d->prim, d->records, d->params, policy, threshold, ctr.p,
                           nullptr);
    unsigned long long h[2] = {0, 0};
    DW_CUDA(cudaMemcpy(h, ctr.p, sizeof h, cudaMemcpyDeviceToHost));
    out[0] = h[0];
    out[1] = h[1];
    return DW_OK;
  });
}

dw_status dw_tune(const dw_trace* trace, dw_policy_family family, int32_t iteration,
                  int32_t reps, dw_tune_report* out) {
  if (!trace || !out) return fail_invalid("null argument");
  return guarded([&] {
    // tuner::extract_iteration (tuner.cpp:14-22)
    dw::HostTrace seg;
    seg.scene = trace->t.scene;
    const int n = seg.scene.params_per_primitive;
    for (int64_t r = 0; r < trace->t.records(); ++r) {
      if (iteration >= 0 && trace->t.iteration[r] != iteration) continue;
      seg.warp_id.push_back(trace->t.warp_id[r]);
      seg.iteration.push_back(trace->t.iteration[r]);
      seg.active.push_back(trace->t.active[r]);
      seg.prim.insert(seg.prim.end(), trace->t.prim.begin() + r * 32,
                      trace->t.prim.begin() + (r + 1) * 32);
      seg.grads.insert(seg.grads.end(), trace->t.grads.begin() + r * 32 * n,
                       trace->t.grads.begin() + (r + 1) * 32 * n);
    }
    if (seg.records() == 0) throw std::invalid_argument("tune: empty trace segment");
    std::unique_ptr<dw_device_trace, void (*)(dw_device_trace*)> d(upload(seg, nullptr),
                                                                   free_device_trace);
    const size_t words = static_cast<size_t>(d->num_primitives) * d->params;
    DevBuf<float> grad(words);
    const int kind = family == DW_FAMILY_SW_S ? DW_POLICY_SW_S : DW_POLICY_SW_B;
    if (reps < 1) reps = 5;
    Events ev;
    out->profile_iteration = *std::min_element(seg.iteration.begin(), seg.iteration.end());
    out->reprofile_period = 2000;
    double best = 0;
    for (int t = 0; t <= 32; ++t) {
      dw::launch_reduce_records(d->active, d->prim, d->vals, d->records, n, kind, t, grad.p,
                                nullptr, nullptr);  // warm-up
      double total = 0;
      for (int k = 0; k < reps; ++k) {
        DW_CUDA(cudaMemsetAsync(grad.p, 0, words * sizeof(float), nullptr));
        DW_CUDA(cudaEventRecord(ev.a, nullptr));
        dw::launch_reduce_records(d->active, d->prim, d->vals, d->records, n, kind, t, grad.p,
                                  nullptr, nullptr);
        DW_CUDA(cudaEventRecord(ev.b, nullptr));
        DW_CUDA(cudaEventSynchronize(ev.b));
        total += ev.ms();
      }
      const double us = 1000.0 * total / reps;
      out->us_by_threshold[t] = us;
      if (t == 0 || us < best) {  // strict <: ties break toward the lowest t
        best = us;
        out->chosen = t;
      }
    }
    return DW_OK;
  });
}

dw_status dw_tune_report_save_csv(const dw_tune_report* report, const char* path) {
  if (!report || !path) return fail_invalid("null argument");
  return guarded([&] {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::ios_base::failure(std::string("cannot write: ") + path);
    f << "threshold,us\n";  // tuner.cpp:54-62 layout, cycles -> measured us
    for (int t = 0; t <= 32; ++t) f << t << ',' << report->us_by_threshold[t] << '\n';
    f << "# chosen=" << report->chosen << " profile_iteration=" << report->profile_iteration
      << " reprofile_period=" << report->reprofile_period << '\n';
    return DW_OK;
  });
}

dw_status dw_rasterizer_create(dw_rasterizer** out) {
  if (!out) return fail_invalid("null argument");
  return guarded([&] {
    *out = dw::raster_new();
    return DW_OK;
  });
}

void dw_rasterizer_free(dw_rasterizer* r) { dw::raster_delete(r); }

dw_status dw_render_forward(dw_rasterizer* r, int32_t P, const float* means3D, const float* scales,
                            const float* rotations, const float* opacities, const float* colors,
                            const dw_camera* cam, float* out_color, int32_t* radii,
                            int64_t* num_rendered, void* stream) {
  if (!r || !cam || !out_color || (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors)))
    return fail_invalid("null argument");
  return guarded([&] {
    dw::raster_forward(r, P, means3D, scales, rotations, opacities, colors, cam, out_color, radii,
                       num_rendered, dw::as_stream(stream), false);
    return DW_OK;
  });
}

dw_status dw_render_forward_async(dw_rasterizer* r, int32_t P, const float* means3D,
                                  const float* scales, const float* rotations,
                                  const float* opacities, const float* colors, const dw_camera* cam,
                                  float* out_color, int32_t* radii, void* stream) {
  if (!r || !cam || !out_color || (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors)))
    return fail_invalid("null argument");
  return guarded([&] {
    dw::raster_forward(r, P, means3D, scales, rotations, opacities, colors, cam, out_color, radii,
                       nullptr, dw::as_stream(stream), true);
    return DW_OK;
  });
}

dw_status dw_render_forward_views(dw_rasterizer* r, int32_t P, const float* means3D,
                                  const float* scales, const float* rotations,
                                  const float* opacities, const float* colors,
                                  const dw_camera* cams, int32_t num_views, float* out_images,
                                  int64_t* num_rendered, void* stream) {
  if (!r || !cams || !out_images ||
      (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors)))
    return fail_invalid("null argument");
  return guarded([&] {
    dw::raster_forward_views(r, P, means3D, scales, rotations, opacities, colors, cams, num_views,
                             out_images, num_rendered, dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_rasterizer_max_stacked_views(int32_t width, int32_t height, int32_t* out) {
  if (!out) return fail_invalid("null argument");
  if (width < 1 || height < 1) return fail_invalid("image size must be >= 1");
  return guarded([&] {
    *out = dw::raster_max_stacked_views(width, height);
    return DW_OK;
  });
}

dw_status dw_rasterizer_reserve(dw_rasterizer* r, int32_t P, int32_t width, int32_t height,
                                int64_t max_instances) {
  if (!r) return fail_invalid("null argument");
  return guarded([&] {
    dw::raster_reserve(r, P, width, height, max_instances);
    return DW_OK;
  });
}

dw_status dw_rasterizer_num_rendered(dw_rasterizer* r, int64_t* num_rendered, int* overflowed) {
  if (!r || !num_rendered) return fail_invalid("null argument");
  return guarded([&] {
    bool ovf = false;
    *num_rendered = dw::raster_resolve(r, &ovf);
    if (overflowed) *overflowed = ovf ? 1 : 0;
    return DW_OK;
  });
}

dw_status dw_render_backward(dw_rasterizer* r, const float* dL_dpixels, dw_policy_kind policy,
                             int32_t threshold, float* grad, uint64_t* pairs_out, void* stream) {
  if (!r || !dL_dpixels || !grad) return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    dw::raster_backward(r, dL_dpixels, policy, threshold, grad, pairs_out, dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_render_backward_chained(dw_rasterizer* r, const float* dL_dpixels,
                                     dw_policy_kind policy, int32_t threshold, float* grad,
                                     void* stream) {
  if (!r || !dL_dpixels || !grad) return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    dw::raster_backward(r, dL_dpixels, policy, threshold, grad, nullptr, dw::as_stream(stream),
                        true);
    return DW_OK;
  });
}

dw_status dw_render_backward_views(dw_rasterizer* const* rasterizers,
                                   const float* const* dL_dpixels, int32_t num_views,
                                   dw_policy_kind policy, int32_t threshold, float* grad,
                                   void* stream) {
  if (!rasterizers || !dL_dpixels || !grad) return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    dw::raster_backward_views(rasterizers, dL_dpixels, num_views, policy, threshold, grad,
                              dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_render_backward_tap(dw_rasterizer* r, const float* dL_dpixels, int32_t threshold,
                                 float* grad, int64_t max_records, dw_trace** out,
                                 int64_t* total_records, void* stream) {
  if (!r || !dL_dpixels || !grad || !out) return fail_invalid("null argument");
  return guarded([&] {
    check_policy(DW_POLICY_SW_B, threshold);
    int64_t total = 0;
    auto t = std::make_unique<dw_trace>();
    t->t = dw::raster_backward_tap(r, dL_dpixels, threshold, grad, max_records, &total,
                                   dw::as_stream(stream));
    if (total_records) *total_records = total;
    *out = t.release();
    return DW_OK;
  });
}

dw_status dw_preprocess_backward(dw_rasterizer* r, const float* means3D, const float* scales,
                                 const float* rotations, const float* grad2d, float* grad3d,
                                 void* stream) {
  if (!r || !means3D || !scales || !rotations || !grad2d || !grad3d)
    return fail_invalid("null argument");
  return guarded([&] {
    dw::raster_preprocess_backward(r, means3D, scales, rotations, grad2d, grad3d,
                                   dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_adam_step(int32_t P, float* means3D, float* scales, float* rotations,
                       float* opacities, float* colors, const float* grad3d, float* exp_avg,
                       float* exp_avg_sq, const dw_adam_config* cfg, int32_t step, void* stream) {
  if (!cfg || (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors || !grad3d ||
                         !exp_avg || !exp_avg_sq)))
    return fail_invalid("null argument");
  return guarded([&] {
    if (P < 0) throw std::invalid_argument("P must be >= 0");
    if (step < 1) throw std::invalid_argument("adam step must be >= 1");
    if (!(cfg->beta1 >= 0.f && cfg->beta1 < 1.f) || !(cfg->beta2 >= 0.f && cfg->beta2 < 1.f))
      throw std::invalid_argument("adam betas must be in [0, 1)");
    dw::launch_adam(P, means3D, scales, rotations, opacities, colors, grad3d, exp_avg, exp_avg_sq,
                    cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, step, dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_rasterizer_last_reds(const dw_rasterizer* r, uint64_t* out) {
  if (!r || !out) return fail_invalid("null argument");
  *out = dw::raster_last_reds(r);
  return DW_OK;
}

dw_status dw_rasterizer_stage_timing(dw_rasterizer* r, int32_t enable) {
  if (!r) return fail_invalid("null argument");
  dw::raster_stage_timing(r, enable != 0);
  return DW_OK;
}

dw_status dw_rasterizer_stage_ms(dw_rasterizer* r, double out_ms[6], int32_t* count) {
  if (!r || !out_ms || !count) return fail_invalid("null argument");
  return guarded([&] {
    *count = dw::raster_stage_ms(r, out_ms, 6);
    return DW_OK;
  });
}

dw_status dw_rasterizer_buffer(const dw_rasterizer* r, int32_t which, const void** dptr,
                               int64_t* count) {
  if (!r || !dptr || !count) return fail_invalid("null argument");
  return guarded([&] {
    dw::raster_buffer(r, which, dptr, count);
    return DW_OK;
  });
}

dw_status dw_render_host(dw_rasterizer* r, int32_t P, const float* means3D, const float* scales,
                         const float* rotations, const float* opacities, const float* colors,
                         const dw_camera* cam, const float* dL_dpixels, dw_policy_kind policy,
                         int32_t threshold, float* out_color, float* grad, void* stream) {
  if (!r || !cam || !dL_dpixels || !out_color || !grad ||
      (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors)))
    return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    dw::raster_host(r, P, means3D, scales, rotations, opacities, colors, cam, dL_dpixels, policy,
                    threshold, out_color, grad, dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_render_views_host(dw_rasterizer* r, int32_t P, const float* means3D,
                               const float* scales, const float* rotations,
                               const float* opacities, const float* colors,
                               const dw_camera* cams, int32_t num_views,
                               const float* dL_dpixels, dw_policy_kind policy, int32_t threshold,
                               float* out_images, float* grad, void* stream) {
  if (!r || !cams || !dL_dpixels || !grad ||
      (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors)))
    return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    dw::raster_views_host(r, P, means3D, scales, rotations, opacities, colors, cams, num_views,
                          dL_dpixels, policy, threshold, out_images, grad,
                          dw::as_stream(stream), false);
    return DW_OK;
  });
}

dw_status dw_render_views(dw_rasterizer* r, int32_t P, const float* means3D, const float* scales,
                          const float* rotations, const float* opacities, const float* colors,
                          const dw_camera* cams, int32_t num_views, const float* dL_dpixels,
                          dw_policy_kind policy, int32_t threshold, float* out_images,
                          float* d_grad, void* stream) {
  if (!r || !cams || !dL_dpixels || (P > 0 && !d_grad) ||
      (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors)))
    return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    dw::raster_views_host(r, P, means3D, scales, rotations, opacities, colors, cams, num_views,
                          dL_dpixels, policy, threshold, out_images, d_grad,
                          dw::as_stream(stream), true);
    return DW_OK;
  });
}

}  // extern "C"

namespace {

// ncclAllReduce of the NCCL library already loaded in the process (the one
// that made the caller's communicator: torch bundles its own), else the
// system's libnccl.so.2.
using AllReduceFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                     ncclComm_t, cudaStream_t);
using ErrStrFn = const char* (*)(ncclResult_t);

struct Nccl {
  AllReduceFn all_reduce = nullptr;
  ErrStrFn err = nullptr;
  Nccl() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return;
    all_reduce = reinterpret_cast<AllReduceFn>(dlsym(h, "ncclAllReduce"));
    err = reinterpret_cast<ErrStrFn>(dlsym(h, "ncclGetErrorString"));
  }
};

void nccl_allreduce(void* comm, float* grad, int64_t count, cudaStream_t s) {
  static Nccl nccl;
  if (!nccl.all_reduce) throw std::runtime_error("NCCL (libnccl.so.2) is not available");
  if (count <= 0) return;
  const ncclResult_t rc = nccl.all_reduce(grad, grad, static_cast<size_t>(count), ncclFloat32,
                                          ncclSum, static_cast<ncclComm_t>(comm), s);
  if (rc != ncclSuccess)
    throw std::runtime_error(std::string("ncclAllReduce: ") +
                             (nccl.err ? nccl.err(rc) : std::to_string(static_cast<int>(rc))));
}

}  // namespace

extern "C" {

dw_status dw_allreduce_grads(void* nccl_comm, float* grad, int64_t count, void* stream) {
  if (!nccl_comm || (count > 0 && !grad)) return fail_invalid("null argument");
  return guarded([&] {
    if (count < 0) throw std::invalid_argument("count must be >= 0");
    nccl_allreduce(nccl_comm, grad, count, dw::as_stream(stream));
    return DW_OK;
  });
}

dw_status dw_render_views_allreduce(dw_rasterizer* r, int32_t P, const float* means3D,
                                    const float* scales, const float* rotations,
                                    const float* opacities, const float* colors,
                                    const dw_camera* cams, int32_t num_views,
                                    const float* dL_dpixels, dw_policy_kind policy,
                                    int32_t threshold, float* out_images, float* d_grad,
                                    float* grad, void* nccl_comm, void* stream) {
  if (!r || !cams || !dL_dpixels || !nccl_comm || (P > 0 && !grad) ||
      (P > 0 && (!means3D || !scales || !rotations || !opacities || !colors)))
    return fail_invalid("null argument");
  return guarded([&] {
    check_policy(policy, threshold);
    const cudaStream_t s = dw::as_stream(stream);
    const int64_t n = static_cast<int64_t>(P) * 9;
    float* dg = d_grad ? d_grad : dw::raster_scratch_grad(r, P);
    dw::raster_views_host(r, P, means3D, scales, rotations, opacities, colors, cams, num_views,
                          dL_dpixels, policy, threshold, out_images, dg, s, true);
    nccl_allreduce(nccl_comm, dg, n, s);
    if (n > 0) DW_CUDA(cudaMemcpyAsync(grad, dg, n * sizeof(float), cudaMemcpyDeviceToHost, s));
    DW_CUDA(cudaStreamSynchronize(s));
    return DW_OK;
  });
}

dw_status dw_copy_to_host(void* host_dst, const void* device_src, size_t bytes) {
  if (bytes && (!host_dst || !device_src)) return fail_invalid("null argument");
  return guarded([&] {
    if (bytes) DW_CUDA(cudaMemcpy(host_dst, device_src, bytes, cudaMemcpyDeviceToHost));
    return DW_OK;
  });
}

dw_status dw_microbench_red(int32_t pattern, int64_t ops, double* reds_per_s, void* stream) {
  if (!reds_per_s) return fail_invalid("null argument");
  return guarded([&] {
    if (pattern < 0 || pattern > 9) throw std::invalid_argument("unknown RED pattern");
    if (ops < 1) throw std::invalid_argument("ops must be >= 1");
    *reds_per_s = dw::microbench_red(pattern, ops, dw::as_stream(stream));
    return DW_OK;
  });
}

}  // extern "C"
