#ifndef DISTWAR_H
#define DISTWAR_H

/* distwar -- B200-native (sm_100a) DISTWAR hot path: warp-level reduction of
 * per-primitive gradient contributions, both trace-driven (the reference's
 * WarpRecord model) and inside a tile-based Gaussian-splatting backward pass.
 *
 * Conventions are those of the reference C ABI (warpred.h:4-11, 20-33,
 * capi.cpp:16-44), unchanged:
 *   - every fallible call returns dw_status; DW_OK = 0;
 *   - on failure the message is read with dw_last_error() (thread-local,
 *     never NULL);
 *   - a NULL required argument returns DW_ERR_INVALID_ARGUMENT with
 *     "null argument";
 *   - std::invalid_argument -> 1, std::ios_base::failure -> 2, any other
 *     exception (including CUDA errors) -> 3;
 *   - opaque handles are released with the matching _free;
 *   - out-structs are caller-owned PODs; returned strings are library-owned.
 * Device pointers are plain CUDA device addresses; `stream` is a
 * cudaStream_t (NULL = legacy default stream). No torch types cross this
 * boundary. Gradient buffers are [primitive][param] fp32, i.e. the reference's
 * Address order (reducers.hpp:19-23): index = primitive * N + param.
 */

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* warpred.h:20-25 */
typedef enum dw_status {
  DW_OK = 0,
  DW_ERR_INVALID_ARGUMENT = 1,
  DW_ERR_IO = 2,
  DW_ERR_RUNTIME = 3
} dw_status;

/* warpred.h:27-33 (same values). DW_POLICY_HW_ATOMRED is the reference's
 * simulated hardware unit; B200 has no such instruction, so it is rejected
 * with DW_ERR_INVALID_ARGUMENT, as reducers::apply_policy rejects it
 * (reducers.cpp:232-236). */
typedef enum dw_policy_kind {
  DW_POLICY_NATIVE = 0,
  DW_POLICY_SW_S = 1,
  DW_POLICY_SW_B = 2,
  DW_POLICY_CCCL = 3,
  DW_POLICY_HW_ATOMRED = 4
} dw_policy_kind;

/* warpred.h:35-38 */
typedef enum dw_policy_family { DW_FAMILY_SW_S = 0, DW_FAMILY_SW_B = 1 } dw_policy_family;

/* warpred.h:42-53 (same layout; replaces workload::SceneSpec). */
typedef struct dw_scene_spec {
  int32_t num_primitives;
  int32_t params_per_primitive;
  int32_t image_width;
  int32_t image_height;
  double mean_fragment_span;
  double fragments_per_pixel_mean;
  double activity_prob;
  double locality;
  uint64_t seed;
  int32_t quantized_values;
} dw_scene_spec;

typedef struct dw_trace dw_trace;               /* host WarpRecord trace    */
typedef struct dw_device_trace dw_device_trace; /* SoA fp32 copy in HBM     */
typedef struct dw_rasterizer dw_rasterizer;     /* per-view device state    */

/* Measured replacement of wr_run_metrics (warpred.h:68-77): cycles become
 * device milliseconds; request counts are counted on the device. */
typedef struct dw_gpu_metrics {
  double kernel_ms;                 /* CUDA-event time of the reduce kernel */
  uint64_t atomic_requests_to_l2;   /* global REDs issued (== reference
                                       PolicyOutput.requests summed)        */
  uint64_t contributions;           /* sum over records popc(active) * N    */
  uint64_t records;
} dw_gpu_metrics;

/* warpred.h:79-84, cycles -> measured microseconds per threshold. */
typedef struct dw_tune_report {
  double us_by_threshold[33];
  int32_t chosen;              /* argmin; ties -> lowest threshold (tuner.cpp:46-49) */
  int32_t profile_iteration;
  int32_t reprofile_period;    /* 2000, tuner.hpp:15 */
} dw_tune_report;

/* Camera for the Gaussian rasterizer: column-major 4x4 matrices
 * (p' = M p, M[col*4+row]); projmatrix is the full proj*view transform. */
typedef struct dw_camera {
  int32_t width, height;
  float viewmatrix[16];
  float projmatrix[16];
  float tan_fovx, tan_fovy;
  float bg[3];
  float scale_modifier;
} dw_camera;

/* ------------------------------------------------------------- library */
const char* dw_version(void);          /* wr_version, warpred.h:86        */
const char* dw_last_error(void);       /* wr_last_error, warpred.h:88-89  */
int dw_device_count(void);             /* -1 when the CUDA runtime fails  */
int dw_device_clock_khz(void);         /* max SM clock of the current device; -1 on failure */

/* --------------------------------------------------- host traces (input) */
void dw_scene_spec_init(dw_scene_spec* scene);                 /* warpred.h:91  */
dw_status dw_trace_generate(const dw_scene_spec* scene, dw_trace** out); /* :98 */
void dw_trace_free(dw_trace* trace);                            /* :99  */
int64_t dw_trace_record_count(const dw_trace* trace);           /* :100, -1 on NULL */
/* WRTRACEB binary container (trace_io.cpp:209-276); binary must be nonzero. */
dw_status dw_trace_save(const dw_trace* trace, const char* path, int binary); /* :101 */
dw_status dw_trace_load(const char* path, int binary, dw_trace** out);       /* :102 */
dw_status dw_trace_histogram_distinct(const dw_trace* trace, uint64_t out_counts[33]); /* :106 */
dw_status dw_trace_histogram_active(const dw_trace* trace, uint64_t out_counts[33]);   /* :108 */
/* Builds a trace from flat caller arrays (prim[R*32], grads[R*32*N] lane-major). */
dw_status dw_trace_from_arrays(int64_t num_records, int32_t params, int32_t num_primitives,
                               const int32_t* warp_id, const int32_t* iteration,
                               const uint32_t* active, const int32_t* prim,
                               const double* grads, dw_trace** out);
/* Borrowed views into a trace (valid until dw_trace_free). */
dw_status dw_trace_arrays(const dw_trace* trace, const uint32_t** active,
                          const int32_t** prim, const double** grads,
                          dw_scene_spec* scene);

/* Borrowed views of the records' warp ids and iteration indices. */
dw_status dw_trace_ids(const dw_trace* trace, const int32_t** warp_id, const int32_t** iteration);
/* Replaces the trace's scene spec (e.g. the seed of a text-format trace);
 * params_per_primitive must match the records. */
dw_status dw_trace_set_scene(dw_trace* trace, const dw_scene_spec* scene);

/* ------------------------------------- trace-driven DISTWAR reduction (GPU) */
/* Uploads a trace to HBM as SoA fp32: active u32[R], prim i32[R][32],
 * vals f32[R][N][32] (param-major per record, so each param is one 128 B
 * coalesced warp load). */
dw_status dw_trace_upload(const dw_trace* trace, void* stream, dw_device_trace** out);
void dw_device_trace_free(dw_device_trace* dtrace);
dw_status dw_device_trace_view(const dw_device_trace* dtrace, const uint32_t** d_active,
                               const int32_t** d_prim, const float** d_vals,
                               int64_t* num_records, int32_t* params, int32_t* num_primitives);

/* The hot path over raw device arrays: each warp applies `policy` (threshold
 * in 0..33, used by SW_S / SW_B; warpred.h:113) to each record and issues the
 * resulting RED.ADD.F32 into d_grad[prim * params + param] (accumulates; the
 * caller zeroes). d_red_count (nullable) receives the number of global REDs
 * issued -- the counting variant is a separate instantiation. */
dw_status dw_reduce_records(const uint32_t* d_active, const int32_t* d_prim,
                            const float* d_vals, int64_t num_records, int32_t params,
                            int32_t num_primitives, dw_policy_kind policy,
                            int32_t threshold, float* d_grad,
                            unsigned long long* d_red_count, void* stream);

/* Replaces wr_simulate (warpred.h:114-116): runs the policy on the real
 * machine; host_grad_out (nullable, P*N floats) receives the sums. */
dw_status dw_gpu_run(const dw_device_trace* dtrace, dw_policy_kind policy, int32_t threshold,
                     float* host_grad_out, dw_gpu_metrics* out);

/* The reference's per-record cost model (reducers.cpp:84-206, InstructionCosts
 * all 1) evaluated on the device over the uploaded records: out[0] =
 * core_instructions, out[1] = core_fp_adds of wr_run_metrics (warpred.h:68-77)
 * for (policy, threshold). */
dw_status dw_model_costs(const dw_device_trace* dtrace, dw_policy_kind policy, int32_t threshold,
                         uint64_t out[2]);

/* Replaces wr_tune (warpred.h:120-122): measured sweep t = 0..32 on the
 * records of `iteration` (< 0: the whole trace), argmin with ties to the
 * lowest threshold (tuner.cpp:29-52). reps = timed repetitions per t. */
dw_status dw_tune(const dw_trace* trace, dw_policy_family family, int32_t iteration,
                  int32_t reps, dw_tune_report* out);
dw_status dw_tune_report_save_csv(const dw_tune_report* report, const char* path); /* :123 */

/* ------------------------------------------- Gaussian-splatting rasterizer */
dw_status dw_rasterizer_create(dw_rasterizer** out);
void dw_rasterizer_free(dw_rasterizer* r);

/* render_forward: preprocess -> tile keys -> radix sort -> tile ranges ->
 * front-to-back blend. All pointers are device pointers: means3D/scales P*3,
 * rotations P*4 (r,x,y,z), opacities P, colors P*3 (RGB), out_color 3*H*W
 * (channel-major), radii P (nullable). num_rendered (host, nullable) receives
 * the number of (tile, Gaussian) instances. Synchronises `stream` once to
 * size the sort. */
dw_status dw_render_forward(dw_rasterizer* r, int32_t P, const float* means3D,
                            const float* scales, const float* rotations,
                            const float* opacities, const float* colors,
                            const dw_camera* cam, float* out_color, int32_t* radii,
                            int64_t* num_rendered, void* stream);

/* render_forward without any host synchronisation (CUDA-graph capturable):
 * the instance count stays on the device and the binning kernels run over the
 * capacity set by dw_rasterizer_reserve (required first; no allocation
 * happens). If the view needs more instances than reserved, nothing is binned
 * (the image is the background) and the overflow flag is raised -- read it,
 * with the count, through dw_rasterizer_num_rendered (which synchronises). */
dw_status dw_render_forward_async(dw_rasterizer* r, int32_t P, const float* means3D,
                                  const float* scales, const float* rotations,
                                  const float* opacities, const float* colors,
                                  const dw_camera* cam, float* out_color, int32_t* radii,
                                  void* stream);

/* render_forward of num_views views of one scene stacked into one frame
 * (1 <= num_views <= dw_rasterizer_max_stacked_views): every launch of the
 * forward -- projection per view, then one depth sort, one binning, one blend
 * -- covers all of them, and the next dw_render_backward takes dL_dpixels as
 * num_views*3*H*W and adds every view's gradients into grad[P*9]. Per-tile
 * lists equal the single-view lists bit for bit (ids of view v offset by
 * v*P in the frame). cams: num_views cameras of one image size and one
 * background; out_images: num_views*3*H*W (device). num_rendered (host,
 * nullable): instances of the whole frame. Synchronises `stream` once. */
dw_status dw_render_forward_views(dw_rasterizer* r, int32_t P, const float* means3D,
                                  const float* scales, const float* rotations,
                                  const float* opacities, const float* colors,
                                  const dw_camera* cams, int32_t num_views, float* out_images,
                                  int64_t* num_rendered, void* stream);
/* How many views of a width x height image fit one stacked frame. */
dw_status dw_rasterizer_max_stacked_views(int32_t width, int32_t height, int32_t* out);

/* Pre-size every per-view buffer for up to P Gaussians, a width x height
 * image and max_instances (tile, Gaussian) instances. */
dw_status dw_rasterizer_reserve(dw_rasterizer* r, int32_t P, int32_t width, int32_t height,
                                int64_t max_instances);

/* Instance count of the last forward (synchronises after a no-sync forward);
 * overflowed (nullable) = 1 if that no-sync forward exceeded the reserve. */
dw_status dw_rasterizer_num_rendered(dw_rasterizer* r, int64_t* num_rendered, int* overflowed);

/* render_backward: the DISTWAR hot path. dL_dpixels 3*H*W (device). Adds the
 * 9 screen-space gradients per Gaussian into grad[P*9] in Address order
 * (mean2D.x, mean2D.y, conic.x, conic.y, conic.z, opacity, r, g, b).
 * pairs_out (host, nullable): number of (pixel, Gaussian) pairs that
 * contributed, counted by a separate counting instantiation (so the timed
 * path carries no counter). */
dw_status dw_render_backward(dw_rasterizer* r, const float* dL_dpixels,
                             dw_policy_kind policy, int32_t threshold, float* grad,
                             uint64_t* pairs_out, void* stream);

/* render_backward for a chain of independent views adding into one gradient
 * (a rank's batch: one rasterizer per view, each already rendered): the
 * caller guarantees that nothing this backward reads -- its forward state,
 * dL_dpixels, the zeroing of grad -- is written by the PREVIOUS kernel on
 * `stream` (that kernel may be another chained backward). The launch then
 * does not wait for the previous grid to finish: its CTAs start on the SMs
 * the previous backward's last wave leaves idle. The first backward after
 * the data it reads was produced must be a plain dw_render_backward. */
dw_status dw_render_backward_chained(dw_rasterizer* r, const float* dL_dpixels,
                                     dw_policy_kind policy, int32_t threshold, float* grad,
                                     void* stream);

/* The backwards of a batch of rendered views of one scene (one rasterizer
 * per view, each already rendered; dL_dpixels[k] belongs to rasterizers[k])
 * added into grad[P*9] (device, Address order) as ONE chain on `stream`:
 * the first launch waits for the stream, the others start on the SMs their
 * predecessor's last wave leaves idle. SW-B / SW-S accumulate into a
 * padded [P][12] buffer (16-byte aligned rows) held by rasterizers[0] and
 * folded into grad at the end -- one batch per rasterizers[0] in flight at a
 * time (like every call on one handle). Returns once everything is enqueued. */
dw_status dw_render_backward_views(dw_rasterizer* const* rasterizers,
                                   const float* const* dL_dpixels, int32_t num_views,
                                   dw_policy_kind policy, int32_t threshold, float* grad,
                                   void* stream);

/* SW-B render_backward that also taps the rasterizer's per-warp WarpRecords
 * (SURVEY §8(f2)): every (warp, Gaussian) with >= 1 active lane becomes one
 * record (prim = the Gaussian in all 32 lanes, 9 grads per lane, zeros in
 * inactive lanes), returned as a host trace that dw_trace_save writes as
 * WRTRACEB -- the reference's simulator / tuner / reducers read it directly.
 * At most max_records are kept; total_records (nullable) gets the count. */
dw_status dw_render_backward_tap(dw_rasterizer* r, const float* dL_dpixels, int32_t threshold,
                                 float* grad, int64_t max_records, dw_trace** out,
                                 int64_t* total_records, void* stream);

/* Preprocess backward (the step before the all-reduce): turns
 * this view's screen-space grad2d[P*9] (dw_render_backward output) into 3D
 * gradients, ADDED into grad3d[P*14] = (means3D xyz, scales xyz, rotation
 * r x y z, opacity, r g b). means3D/scales/rotations are the forward's inputs
 * (device). Accumulating over views yields the training gradient. */
dw_status dw_preprocess_backward(dw_rasterizer* r, const float* means3D, const float* scales,
                                 const float* rotations, const float* grad2d, float* grad3d,
                                 void* stream);

/* Adam step over the scene's parameters (device, updated in place) from
 * grad3d[P*14]; exp_avg / exp_avg_sq are caller-owned [P*14] moment buffers
 * (zero-initialised); step >= 1 (bias correction); lr per group: means,
 * scales, rotations, opacities, colors. */
typedef struct dw_adam_config {
  float lr[5];
  float beta1, beta2, eps;
} dw_adam_config;
dw_status dw_adam_step(int32_t P, float* means3D, float* scales, float* rotations,
                       float* opacities, float* colors, const float* grad3d, float* exp_avg,
                       float* exp_avg_sq, const dw_adam_config* cfg, int32_t step, void* stream);

/* Number of global REDs issued by the last render_backward called with a
 * non-NULL pairs_out (the counting instantiation). */
/* Per-stage timing of later forwards (diagnostic: CUDA events between the
 * stages serialise the programmatic-dependent launches): after a forward,
 * dw_rasterizer_stage_ms returns *count (6) stage times in ms -- preprocess,
 * depth sort, instance offsets (+ count read-back), binning (duplicate + tile
 * sort, or dense), tile ranges (+ per-tile sort), blend. */
dw_status dw_rasterizer_stage_timing(dw_rasterizer* r, int32_t enable);
dw_status dw_rasterizer_stage_ms(dw_rasterizer* r, double out_ms[6], int32_t* count);
dw_status dw_rasterizer_last_reds(const dw_rasterizer* r, uint64_t* out);

/* Device views of the rasterizer's intermediate buffers (parity tests):
 * 0 means2D f32[P*2], 1 depths f32[P], 2 radii i32[P], 3 conic_opacity
 * f32[P*4], 4 tiles_touched u32[P], 5 keys u64[I] (sorted), 6 values u32[I]
 * (sorted), 7 ranges u32[tiles*2], 8 final_T f32[H*W], 9 n_contrib u32[H*W].
 * count = number of elements. */
dw_status dw_rasterizer_buffer(const dw_rasterizer* r, int32_t which, const void** dptr,
                               int64_t* count);

/* Host-buffer end-to-end call (copies inside): forward + backward for one
 * view, H2D of the scene and dL/dpixels, D2H of image and grad. */
dw_status dw_render_host(dw_rasterizer* r, int32_t P, const float* means3D,
                         const float* scales, const float* rotations, const float* opacities,
                         const float* colors, const dw_camera* cam, const float* dL_dpixels,
                         dw_policy_kind policy, int32_t threshold, float* out_color,
                         float* grad, void* stream);

/* Synchronous device->host copy of `bytes` (reads back dw_rasterizer_buffer
 * views without the caller linking the CUDA runtime). */
dw_status dw_copy_to_host(void* host_dst, const void* device_src, size_t bytes);

/* One training step's rasterization from host buffers: the scene is uploaded
 * once, then `num_views` cameras (same image size) are rendered and
 * back-propagated into ONE gradient buffer (grad[P*9], host, overwritten).
 * dL_dpixels is num_views*3*H*W (host); out_images (host, nullable) receives
 * num_views*3*H*W. Per-view uploads/downloads run on two internal copy
 * streams double-buffered against `stream` (overlap needs pinned memory). */
dw_status dw_render_views_host(dw_rasterizer* r, int32_t P, const float* means3D,
                               const float* scales, const float* rotations,
                               const float* opacities, const float* colors,
                               const dw_camera* cams, int32_t num_views,
                               const float* dL_dpixels, dw_policy_kind policy, int32_t threshold,
                               float* out_images, float* grad, void* stream);
/* dw_render_views_host with the gradient left in HBM: d_grad is a device
 * buffer of P*9 floats (overwritten, complete when the call returns), so a
 * multi-GPU caller all-reduces it over NVLink before ONE device-to-host copy
 * (dw_allreduce_grads, or dw_render_views_allreduce for the whole step). */
dw_status dw_render_views(dw_rasterizer* r, int32_t P, const float* means3D, const float* scales,
                          const float* rotations, const float* opacities, const float* colors,
                          const dw_camera* cams, int32_t num_views, const float* dL_dpixels,
                          dw_policy_kind policy, int32_t threshold, float* out_images,
                          float* d_grad, void* stream);

/* ----------------------------------------------- multi-GPU exchange (NCCL) */
/* SURVEY §8(b) wr_gs_allreduce_grads: sum a gradient buffer (count floats,
 * device, in place) across the ranks of an NCCL communicator on `stream` --
 * the one exchange of view-parallel training. nccl_comm is a
 * caller-owned ncclComm_t (e.g. torch's ProcessGroupNCCL._comm_ptr()); the
 * NCCL library the process already loaded is used (resolved at run time, so
 * the communicator and the call agree on the library). Returns when the
 * reduction is enqueued. */
dw_status dw_allreduce_grads(void* nccl_comm, float* grad, int64_t count, void* stream);
/* The whole view-parallel step of one rank from host buffers: its views
 * rendered and back-propagated into d_grad (device, P*9, overwritten), the
 * buffer summed across nccl_comm, then ONE device-to-host copy into grad
 * (host, P*9). d_grad may be NULL (an internal buffer is used). */
dw_status dw_render_views_allreduce(dw_rasterizer* r, int32_t P, const float* means3D,
                                    const float* scales, const float* rotations,
                                    const float* opacities, const float* colors,
                                    const dw_camera* cams, int32_t num_views,
                                    const float* dL_dpixels, dw_policy_kind policy,
                                    int32_t threshold, float* out_images, float* d_grad,
                                    float* grad, void* nccl_comm, void* stream);

/* --------------------------------------------------- roofline microbenchmarks */
/* Measured f32 RED throughput (REDs/s) for `pattern`: 0 distinct addresses,
 * 1 all 32 lanes of a warp on one address (the naive pattern), 2 distinct
 * addresses with red.global.add.v4.f32 (counted as 4 REDs), 3 nine lanes on
 * one pseudo-random primitive row (SW-B's issue pattern), 4 all lanes on one
 * 16-byte address with v4, 5 / 6 four lanes on one primitive row with 9
 * scalar REDs each / the same floats as 3-4 vector REDs (SW-B's per-lane
 * path without / with DW_VEC_RED), 7 pattern 3's rows as 3-4 vector REDs
 * from one lane. Every float added counts as one RED. */
dw_status dw_microbench_red(int32_t pattern, int64_t ops, double* reds_per_s, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif
#endif /* DISTWAR_H */
