/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the DISTWAR reduction stage.
 * See warpred_oracle.c for the reference file:line each function restates. */
#ifndef WARPRED_ORACLE_H
#define WARPRED_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field order as wr_scene_spec (reference include/warpred.h:42-53). */
typedef struct or_scene_spec {
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
} or_scene_spec;

/* Flat WarpRecord arrays (reference workload.hpp:41-65): prim[R*32],
 * grads[R*32*N] lane-major (param fastest), f64. */
typedef struct or_trace {
  or_scene_spec scene;
  int64_t num_records;
  int64_t capacity;
  int32_t* warp_id;
  int32_t* iteration;
  uint32_t* active;
  int32_t* prim;
  double* grads;
} or_trace;

enum { OR_NATIVE = 0, OR_SW_S = 1, OR_SW_B = 2, OR_CCCL = 3, OR_HW_ATOMRED = 4 };

const char* or_last_error(void);
void or_scene_spec_init(or_scene_spec* s);
or_trace* or_trace_new(const or_scene_spec* s);
void or_trace_free(or_trace* t);
int or_generate(const or_scene_spec* s, or_trace** out);
int or_record_policy(uint32_t active, const int32_t* prim, const double* grads,
                     int32_t n, int kind, int threshold, int32_t* out_prim,
                     int32_t* out_param, double* out_val, int64_t* out_count,
                     uint64_t* instr, uint64_t* fp_adds);
int or_apply_policy(const or_trace* t, int kind, int threshold,
                    int32_t num_prims, double* sums, uint64_t counts3[3]);
int or_oracle_sum(const or_trace* t, int32_t num_prims, double* sums,
                  uint8_t* touched);
int or_histograms(const or_trace* t, uint64_t distinct[33], uint64_t act[33]);
int or_save_binary(const or_trace* t, const char* path);
int or_load_binary(const char* path, or_trace** out);

#ifdef __cplusplus
}
#endif
#endif
