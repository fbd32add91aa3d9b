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


/* ---- decision-matched verification (gs_verify.c) -------------------------- */

/* Projection + per-tile lists by (depth, index) bucketing: the lists of
 * gs_forward without its blend (out_color / final_T / n_contrib stay zero);
 * keys only when with_keys (C4 has 0.9 G instances). */
int gs_forward_lists(gs_state* s, int32_t P, const float* means3D, const float* scales,
                     const float* rotations, const float* opacities, const float* colors,
                     const gs_camera* cam, int threads, int with_keys);

typedef struct gs_flip {
  int32_t pixel;      /* y * W + x */
  uint32_t position;  /* tile-list position of the decision */
  int32_t gaussian;   /* Gaussian id */
  int32_t kind;       /* 0 alpha >= 1/255 test, 1 T >= 1e-4 termination test */
} gs_flip;

typedef struct gs_verify_report {
  int64_t pairs;          /* blended (pixel, Gaussian) pairs in the matched worlds */
  int64_t pairs_default;  /* ... in the oracle's own world (no flips) */
  int64_t amb_alpha;      /* ambiguous alpha decisions met (default world) */
  int64_t amb_term;       /* ambiguous termination decisions met (default world) */
  int64_t pix_ambiguous;  /* pixels with >= 2 worlds */
  int64_t pix_flipped;    /* pixels whose matched world is not the default */
  int64_t flips;          /* flipped decisions in the matched worlds */
  int64_t pix_unresolved; /* the GPU outputs fit >1 world (grad_slack covers) */
  int64_t pix_nomatch;    /* no world fits the GPU outputs: FAILURE */
  int64_t pix_world_cap;  /* world enumeration truncated: FAILURE */
  int32_t max_worlds;
  int32_t nflip_rec;
} gs_verify_report;

typedef struct gs_verify_out {
  double* grad;        /* P*9 gradients of the matched worlds (float64 arithmetic) */
  double* grad_bound;  /* P*9 sum of E_pix * |term| magnitude, units of u = 2^-24 */
  double* grad_abs;    /* P*9 sum of |term| */
  double* grad_slack;  /* P*9 world spread of unresolved pixels (normally 0) */
  int32_t* npix;       /* P contributing pixels per Gaussian */
  double* image;       /* 3*H*W */
  double* image_mag;   /* 3*H*W sum |c alpha T| + T |bg| */
  double* image_slack; /* 3*H*W without GPU outputs: spread over the worlds (else 0) */
  double* final_T;     /* H*W */
  double* epix;        /* H*W E_pix, units of u */
  uint32_t* n_contrib; /* H*W */
  uint8_t* status;     /* H*W 0 unambiguous, 1 ambiguous-default, 2 flipped, 3 unresolved,
                          4 no match, 5 world cap */
  gs_flip* flips;
  int32_t flip_cap;
  int32_t nflip_rec;
} gs_verify_out;

/* Needs the lists of gs_forward or gs_forward_lists. Any output pointer may
 * be NULL. gpu_* (all three or none): the GPU's per-pixel n_contrib, final_T
 * and image [3][H][W]; without them every pixel takes the default world and
 * the spread of the other worlds goes to grad_slack / image_slack.
 * kappa scales the per-pixel tolerance used to match worlds. */
int gs_verify(const gs_state* s, const gs_camera* cam, const float* dL_dpixels,
              const uint32_t* gpu_n_contrib, const float* gpu_final_T, const float* gpu_image,
              double kappa, gs_verify_out* out, gs_verify_report* rep, int threads);
const char* gs_verify_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
