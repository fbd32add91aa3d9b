/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the tile-based Gaussian-splatting
 * rasterizer that feeds the DISTWAR reduction (see gs_oracle.c).
 * PARITY UNPINNED by the reference: /root/reference contains no rasterizer
 * (SPEC.md:16 puts it out of scope); this restates the public 3DGS algorithm. */
#ifndef GS_ORACLE_H
#define GS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_TILE 16
#define GS_NPARAM 9 /* mean2D.xy, conic.xyz, opacity, rgb */

/* Column-major 4x4 matrices (p' = M p with M[col*4+row]), the convention of
 * the public 3DGS rasterizer; projmatrix is the full proj*view transform. */
typedef struct gs_camera {
  int32_t width, height;
  float viewmatrix[16];
  float projmatrix[16];
  float tan_fovx, tan_fovy;
  float bg[3];
  float scale_modifier;
} gs_camera;

typedef struct gs_state {
  int32_t P, W, H, tiles_x, tiles_y;
  float* means2D;        /* P*2 */
  float* depths;         /* P */
  int32_t* radii;        /* P */
  float* conic_opacity;  /* P*4 */
  float* rgb;            /* P*3 */
  uint32_t* tiles_touched;
  int64_t num_rendered;
  uint64_t* keys;        /* sorted (tile<<32 | depth bits) */
  uint32_t* values;      /* sorted Gaussian ids */
  uint32_t* ranges;      /* tiles*2 (start, end) */
  float* out_color;      /* 3*H*W, channel-major */
  float* final_T;        /* H*W */
  uint32_t* n_contrib;   /* H*W */
  /* backward tap: one record per (warp, Gaussian) with >=1 active lane */
  int64_t tap_count, tap_cap;
  int32_t* tap_warp;
  int32_t* tap_iter;
  uint32_t* tap_active;
  int32_t* tap_prim;     /* 32 per record (warp-uniform) */
  double* tap_grads;     /* 32*9 per record, lane-major */
  int32_t tap_ppt;       /* record layout: 1 (8x4 px per warp) or 2 (8x8, 2 px per lane) */
} gs_state;

const char* gs_last_error(void);
gs_state* gs_state_new(void);
void gs_state_free(gs_state* s);

/* preprocess + duplicate keys + stable sort + tile ranges + forward blend */
int gs_forward(gs_state* s, int32_t P, const float* means3D, const float* scales,
               const float* rotations, const float* opacities,
               const float* colors, const gs_camera* cam, int threads);

/* backward blend; grad/grad_abs are P*9 f64 (grad_abs = sum of |terms|, for
 * the tolerance bound). tile_stride>1 processes every k-th tile only (bounded
 * CPU-baseline sample). tap: 0 accumulate only; 1 accumulate and record the
 * per-warp WarpRecords (per-thread buffers, appended in thread order); 2
 * record only (grad untouched). pairs_out = number of (pixel, Gaussian) pairs that contributed. */
int gs_backward(gs_state* s, const gs_camera* cam, const float* dL_dpixels,
                double* grad, double* grad_abs, int threads, int tile_stride,
                int tap, int64_t* pairs_out);

#define GS_NPARAM3D 14 /* means3D xyz, scales xyz, rotation rxyz, opacity, rgb */

/* Preprocess backward, float64: screen-space gradients
 * grad2d[P*9] of one view (gs_backward's output for the SAME camera and
 * scene as the last gs_forward) -> 3D gradients grad3d[P*14], ADDED. */
int gs_preprocess_backward(const gs_state* s, int32_t P, const float* means3D,
                           const float* scales, const float* rotations,
                           const gs_camera* cam, const double* grad2d, double* grad3d);

/* One Adam step (float64 reference) over n parameters. */
void gs_adam(int64_t n, double* param, const double* grad, double* m, double* v, double lr,
             double beta1, double beta2, double eps, int step);

#ifdef __cplusplus
}
#endif
#endif
