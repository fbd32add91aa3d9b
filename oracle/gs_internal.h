/* TEST INFRASTRUCTURE ONLY -- helpers shared by gs_oracle.c and gs_verify.c. */
#ifndef GS_INTERNAL_H
#define GS_INTERNAL_H
#include "gs_oracle.h"

/* Projection of Gaussian i (gs_oracle.c preprocess_one): fills means2D,
 * depths, radii, conic_opacity, rgb and tiles_touched of state s. */
void gs_i_preprocess_one(int i, const float* means3D, const float* scales,
                         const float* rotations, const float* opacities,
                         const float* colors, const gs_camera* cam, gs_state* s);
/* Clamped tile rectangle [x0, y0, x1, y1) of a projected Gaussian. */
void gs_i_rect_of(const gs_state* s, int i, int* r);

#endif
