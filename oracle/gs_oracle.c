/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the tile-based Gaussian-
 * splatting rasterizer around the DISTWAR hot path.
 *
 * PARITY UNPINNED BY THE REFERENCE: /root/reference has no rasterizer
 * ("OUT OF SCOPE ... forward-pass rendering"); the only pinned
 * pieces are the abstract loop shape of the gradient step (PAPER.md:1481-1504:
 * each pixel-thread iterates its primitives, skips on cond1/cond2, and issues
 * N atomicAdds) and the SW-B integration (inactive
 * threads carry zero gradients and a was_active flag). Everything else
 * restates the public 3DGS algorithm (Kerbl et al. 2023): EWA projection,
 * (tile|depth) keys, stable sort, per-tile ranges, front-to-back blending and
 * its analytic backward.
 *
 * Floating-point contract: compiled with -ffp-contract=off and written in the
 * same operation order as the CUDA kernels (which are compiled -fmad=false
 * for preprocess), so means2D / depths / radii / tiles_touched -- and hence
 * keys, the sorted order and tile ranges -- are BIT-EXACT between the two.
 * Blending uses expf here and __expf on the GPU, so images and gradients are
 * compared under a stated tolerance (tests/test_gpu_raster.py).
 */
#include "gs_oracle.h"
#include "gs_internal.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256] = "ok";
const char* gs_last_error(void) { return g_err; }
static int fail(const char* m) {
  snprintf(g_err, sizeof g_err, "%s", m);
  return 1;
}

gs_state* gs_state_new(void) { return calloc(1, sizeof(gs_state)); }

static void free_fwd(gs_state* s) {
  free(s->means2D); free(s->depths); free(s->radii); free(s->conic_opacity);
  free(s->rgb); free(s->tiles_touched); free(s->keys); free(s->values);
  free(s->ranges); free(s->out_color); free(s->final_T); free(s->n_contrib);
  s->means2D = s->depths = s->conic_opacity = s->rgb = s->out_color = s->final_T = NULL;
  s->radii = NULL; s->tiles_touched = s->values = s->ranges = s->n_contrib = NULL;
  s->keys = NULL;
}

static void free_tap(gs_state* s) {
  free(s->tap_warp); free(s->tap_iter); free(s->tap_active); free(s->tap_prim);
  free(s->tap_grads);
  s->tap_warp = s->tap_iter = s->tap_prim = NULL;
  s->tap_active = NULL;
  s->tap_grads = NULL;
  s->tap_count = s->tap_cap = 0;
}

void gs_state_free(gs_state* s) {
  if (!s) return;
  free_fwd(s);
  free_tap(s);
  free(s);
}

/* ------------------------------------------------------------ preprocess */
static float ndc2pix(float v, int S) { return ((v + 1.0f) * (float)S - 1.0f) * 0.5f; }

/* Sigma = R diag(s^2) R^T from a normalised (r, x, y, z) quaternion. */
static void cov3d(const float* sc, float mod, const float* rot, float* c6) {
  const float qr = rot[0], qx = rot[1], qy = rot[2], qz = rot[3];
  const float inv = 1.0f / sqrtf(qr * qr + qx * qx + qy * qy + qz * qz);
  const float r = qr * inv, x = qx * inv, y = qy * inv, z = qz * inv;
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
  const float s0 = mod * sc[0], s1 = mod * sc[1], s2 = mod * sc[2];
  const float v0 = s0 * s0, v1 = s1 * s1, v2 = s2 * s2;
  /* Sigma_ij = R_i0 v0 R_j0 + R_i1 v1 R_j1 + R_i2 v2 R_j2 */
#define SIG(i, j) (R[i][0] * v0 * R[j][0] + R[i][1] * v1 * R[j][1] + R[i][2] * v2 * R[j][2])
  c6[0] = SIG(0, 0); c6[1] = SIG(0, 1); c6[2] = SIG(0, 2);
  c6[3] = SIG(1, 1); c6[4] = SIG(1, 2); c6[5] = SIG(2, 2);
#undef SIG
}

/* EWA: cov2D = T Sigma T^T + 0.3 I, T = J W (J: perspective Jacobian at the
 * clamped view-space point, W: rotation block of the view matrix). */
static void cov2d(const float* tv, float fx, float fy, float tfx, float tfy,
                  const float* c6, const float* vm, float* out3) {
  const float limx = 1.3f * tfx, limy = 1.3f * tfy;
  const float tz = tv[2];
  const float txtz = tv[0] / tz, tytz = tv[1] / tz;
  const float tx = fminf(limx, fmaxf(-limx, txtz)) * tz;
  const float ty = fminf(limy, fmaxf(-limy, tytz)) * tz;
  const float j00 = fx / tz, j02 = -(fx * tx) / (tz * tz);
  const float j11 = fy / tz, j12 = -(fy * ty) / (tz * tz);
  float T[2][3];
  for (int j = 0; j < 3; ++j) {
    T[0][j] = j00 * vm[j * 4 + 0] + j02 * vm[j * 4 + 2];
    T[1][j] = j11 * vm[j * 4 + 1] + j12 * vm[j * 4 + 2];
  }
  const float S[3][3] = {{c6[0], c6[1], c6[2]}, {c6[1], c6[3], c6[4]}, {c6[2], c6[4], c6[5]}};
  float A[2][3];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      A[i][j] = T[i][0] * S[0][j] + T[i][1] * S[1][j] + T[i][2] * S[2][j];
  const float a = A[0][0] * T[0][0] + A[0][1] * T[0][1] + A[0][2] * T[0][2];
  const float b = A[0][0] * T[1][0] + A[0][1] * T[1][1] + A[0][2] * T[1][2];
  const float c = A[1][0] * T[1][0] + A[1][1] * T[1][1] + A[1][2] * T[1][2];
  out3[0] = a + 0.3f;
  out3[1] = b;
  out3[2] = c + 0.3f;
}

void gs_i_preprocess_one(int i, const float* means3D, const float* scales,
                           const float* rotations, const float* opacities,
                           const float* colors, const gs_camera* cam, gs_state* s) {
  s->radii[i] = 0;
  s->tiles_touched[i] = 0;
  const float* m = means3D + 3 * i;
  const float* vm = cam->viewmatrix;
  const float* pm = cam->projmatrix;
  const float px = m[0], py = m[1], pz = m[2];
  float tv[3];
  tv[0] = vm[0] * px + vm[4] * py + vm[8] * pz + vm[12];
  tv[1] = vm[1] * px + vm[5] * py + vm[9] * pz + vm[13];
  tv[2] = vm[2] * px + vm[6] * py + vm[10] * pz + vm[14];
  if (tv[2] <= 0.2f) return;
  const float hx = pm[0] * px + pm[4] * py + pm[8] * pz + pm[12];
  const float hy = pm[1] * px + pm[5] * py + pm[9] * pz + pm[13];
  const float hw = pm[3] * px + pm[7] * py + pm[11] * pz + pm[15];
  const float pw = 1.0f / (hw + 0.0000001f);
  const float nx = hx * pw, ny = hy * pw;
  float c6[6], cv[3];
  cov3d(scales + 3 * i, cam->scale_modifier, rotations + 4 * i, c6);
  const float fx = (float)cam->width / (2.0f * cam->tan_fovx);
  const float fy = (float)cam->height / (2.0f * cam->tan_fovy);
  cov2d(tv, fx, fy, cam->tan_fovx, cam->tan_fovy, c6, vm, cv);
  const float det = cv[0] * cv[2] - cv[1] * cv[1];
  if (det == 0.0f) return;
  const float det_inv = 1.0f / det;
  const float mid = 0.5f * (cv[0] + cv[2]);
  const float disc = sqrtf(fmaxf(0.1f, mid * mid - det));
  const float l1 = mid + disc, l2 = mid - disc;
  const int radius = (int)ceilf(3.0f * sqrtf(fmaxf(l1, l2)));
  const float ix = ndc2pix(nx, cam->width), iy = ndc2pix(ny, cam->height);
  const float fr = (float)radius;
  int rminx = (int)((ix - fr) / (float)GS_TILE), rminy = (int)((iy - fr) / (float)GS_TILE);
  int rmaxx = (int)((ix + fr + (float)(GS_TILE - 1)) / (float)GS_TILE);
  int rmaxy = (int)((iy + fr + (float)(GS_TILE - 1)) / (float)GS_TILE);
#define CLAMP(v, hi) ((v) < 0 ? 0 : ((v) > (hi) ? (hi) : (v)))
  rminx = CLAMP(rminx, s->tiles_x); rmaxx = CLAMP(rmaxx, s->tiles_x);
  rminy = CLAMP(rminy, s->tiles_y); rmaxy = CLAMP(rmaxy, s->tiles_y);
#undef CLAMP
  const int area = (rmaxx - rminx) * (rmaxy - rminy);
  if (area == 0) return;
  s->depths[i] = tv[2];
  s->radii[i] = radius;
  s->means2D[2 * i] = ix;
  s->means2D[2 * i + 1] = iy;
  s->conic_opacity[4 * i + 0] = cv[2] * det_inv;
  s->conic_opacity[4 * i + 1] = -cv[1] * det_inv;
  s->conic_opacity[4 * i + 2] = cv[0] * det_inv;
  s->conic_opacity[4 * i + 3] = opacities[i];
  s->rgb[3 * i + 0] = colors[3 * i + 0];
  s->rgb[3 * i + 1] = colors[3 * i + 1];
  s->rgb[3 * i + 2] = colors[3 * i + 2];
  s->tiles_touched[i] = (uint32_t)area;
}

void gs_i_rect_of(const gs_state* s, int i, int* r) {
  const float ix = s->means2D[2 * i], iy = s->means2D[2 * i + 1];
  const float fr = (float)s->radii[i];
  int v[4] = {(int)((ix - fr) / (float)GS_TILE), (int)((iy - fr) / (float)GS_TILE),
              (int)((ix + fr + (float)(GS_TILE - 1)) / (float)GS_TILE),
              (int)((iy + fr + (float)(GS_TILE - 1)) / (float)GS_TILE)};
  const int hi[4] = {s->tiles_x, s->tiles_y, s->tiles_x, s->tiles_y};
  for (int k = 0; k < 4; ++k) r[k] = v[k] < 0 ? 0 : (v[k] > hi[k] ? hi[k] : v[k]);
}

/* Stable LSD radix sort of (key, value) pairs on the low `bits` key bits. */
static int radix_sort(uint64_t* k, uint32_t* v, int64_t n, int bits) {
  uint64_t* k2 = malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
  uint32_t* v2 = malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
  if (!k2 || !v2) { free(k2); free(v2); return fail("out of memory"); }
  for (int shift = 0; shift < bits; shift += 8) {
    int64_t cnt[257] = {0};
    for (int64_t i = 0; i < n; ++i) cnt[((k[i] >> shift) & 255) + 1]++;
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t d = cnt[(k[i] >> shift) & 255]++;
      k2[d] = k[i];
      v2[d] = v[i];
    }
    memcpy(k, k2, sizeof(uint64_t) * (size_t)n);
    memcpy(v, v2, sizeof(uint32_t) * (size_t)n);
  }
  free(k2);
  free(v2);
  return 0;
}

/* -------------------------------------------------------------- blending */
/* Pixel (px, py) of in-tile thread t = warp*32 + lane: each warp owns an 8x4
 * block (the warp tiling of the reference workload model, workload.cpp:107). */
static void pixel_of(int tile, int t, int tiles_x, int* px, int* py) {
  const int w = t >> 5, l = t & 31;
  *px = (tile % tiles_x) * GS_TILE + (w & 1) * 8 + (l & 7);
  *py = (tile / tiles_x) * GS_TILE + (w >> 1) * 4 + (l >> 3);
}

typedef struct {
  gs_state* s;
  const gs_camera* cam;
  const float* dL;
  double* grad;
  double* gabs;
  int tid, nthreads, stride, tap;
  int64_t pairs;
  gs_state tapbuf; /* per-thread tap records, merged after join */
} job;

static void forward_tile(gs_state* s, const gs_camera* cam, int tile) {
  const uint32_t rs = s->ranges[2 * tile], re = s->ranges[2 * tile + 1];
  for (int t = 0; t < GS_TILE * GS_TILE; ++t) {
    int px, py;
    pixel_of(tile, t, s->tiles_x, &px, &py);
    if (px >= s->W || py >= s->H) continue;
    const float pfx = (float)px, pfy = (float)py;
    float T = 1.0f, C[3] = {0.0f, 0.0f, 0.0f};
    uint32_t contributor = 0, last = 0;
    for (uint32_t j = rs; j < re; ++j) {
      const uint32_t id = s->values[j];
      contributor++;
      const float* co = s->conic_opacity + 4 * id;
      const float dx = s->means2D[2 * id] - pfx, dy = s->means2D[2 * id + 1] - pfy;
      const float power = -0.5f * (co[0] * dx * dx + co[2] * dy * dy) - co[1] * dx * dy;
      if (power > 0.0f) continue;
      const float alpha = fminf(0.99f, co[3] * expf(power));
      if (alpha < 1.0f / 255.0f) continue;
      const float test_T = T * (1.0f - alpha);
      if (test_T < 0.0001f) break;
      for (int ch = 0; ch < 3; ++ch) C[ch] += s->rgb[3 * id + ch] * alpha * T;
      T = test_T;
      last = contributor;
    }
    const int pix = py * s->W + px;
    s->final_T[pix] = T;
    s->n_contrib[pix] = last;
    for (int ch = 0; ch < 3; ++ch)
      s->out_color[ch * s->H * s->W + pix] = C[ch] + T * cam->bg[ch];
  }
}

static void* forward_worker(void* arg) {
  job* jb = arg;
  const int ntiles = jb->s->tiles_x * jb->s->tiles_y;
  for (int tile = jb->tid; tile < ntiles; tile += jb->nthreads)
    forward_tile(jb->s, jb->cam, tile);
  return NULL;
}

int gs_forward(gs_state* s, int32_t P, const float* means3D, const float* scales,
               const float* rotations, const float* opacities, const float* colors,
               const gs_camera* cam, int threads) {
  if (!s || !means3D || !scales || !rotations || !opacities || !colors || !cam)
    return fail("null argument");
  if (P < 0 || cam->width < 1 || cam->height < 1) return fail("invalid size");
  free_fwd(s);
  s->P = P;
  s->W = cam->width;
  s->H = cam->height;
  s->tiles_x = (cam->width + GS_TILE - 1) / GS_TILE;
  s->tiles_y = (cam->height + GS_TILE - 1) / GS_TILE;
  const size_t np = (size_t)(P ? P : 1), npix = (size_t)s->W * s->H;
  const int ntiles = s->tiles_x * s->tiles_y;
  s->means2D = calloc(np * 2, sizeof(float));
  s->depths = calloc(np, sizeof(float));
  s->radii = calloc(np, sizeof(int32_t));
  s->conic_opacity = calloc(np * 4, sizeof(float));
  s->rgb = calloc(np * 3, sizeof(float));
  s->tiles_touched = calloc(np, sizeof(uint32_t));
  s->ranges = calloc((size_t)ntiles * 2, sizeof(uint32_t));
  s->out_color = calloc(npix * 3, sizeof(float));
  s->final_T = calloc(npix, sizeof(float));
  s->n_contrib = calloc(npix, sizeof(uint32_t));
  for (int i = 0; i < P; ++i)
    gs_i_preprocess_one(i, means3D, scales, rotations, opacities, colors, cam, s);
  /* duplicate keys in (Gaussian, row, column) order */
  int64_t total = 0;
  for (int i = 0; i < P; ++i) total += s->tiles_touched[i];
  s->num_rendered = total;
  s->keys = malloc(sizeof(uint64_t) * (size_t)(total ? total : 1));
  s->values = malloc(sizeof(uint32_t) * (size_t)(total ? total : 1));
  int64_t off = 0;
  for (int i = 0; i < P; ++i) {
    if (s->radii[i] <= 0) continue;
    int r[4];
    gs_i_rect_of(s, i, r);
    uint32_t dbits;
    memcpy(&dbits, &s->depths[i], 4);
    for (int y = r[1]; y < r[3]; ++y)
      for (int x = r[0]; x < r[2]; ++x) {
        s->keys[off] = ((uint64_t)(uint32_t)(y * s->tiles_x + x) << 32) | dbits;
        s->values[off] = (uint32_t)i;
        ++off;
      }
  }
  int tile_bits = 0;
  while ((1 << tile_bits) < ntiles) ++tile_bits;
  if (radix_sort(s->keys, s->values, total, 32 + tile_bits)) return 1;
  for (int64_t j = 0; j < total; ++j) {
    const uint32_t tile = (uint32_t)(s->keys[j] >> 32);
    if (j == 0 || (uint32_t)(s->keys[j - 1] >> 32) != tile) s->ranges[2 * tile] = (uint32_t)j;
    if (j == total - 1 || (uint32_t)(s->keys[j + 1] >> 32) != tile)
      s->ranges[2 * tile + 1] = (uint32_t)(j + 1);
  }
  if (threads < 1) threads = 1;
  pthread_t th[64];
  job jobs[64];
  if (threads > 64) threads = 64;
  for (int t = 0; t < threads; ++t) {
    memset(&jobs[t], 0, sizeof(job));
    jobs[t].s = s;
    jobs[t].cam = cam;
    jobs[t].tid = t;
    jobs[t].nthreads = threads;
    pthread_create(&th[t], NULL, forward_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}

static int tap_push(gs_state* s, int32_t warp, int32_t iter, uint32_t active,
                    int32_t prim, const double* g) {
  if (s->tap_count == s->tap_cap) {
    const int64_t cap = s->tap_cap ? s->tap_cap * 2 : 4096;
    s->tap_warp = realloc(s->tap_warp, sizeof(int32_t) * (size_t)cap);
    s->tap_iter = realloc(s->tap_iter, sizeof(int32_t) * (size_t)cap);
    s->tap_active = realloc(s->tap_active, sizeof(uint32_t) * (size_t)cap);
    s->tap_prim = realloc(s->tap_prim, sizeof(int32_t) * 32 * (size_t)cap);
    s->tap_grads = realloc(s->tap_grads, sizeof(double) * 32 * GS_NPARAM * (size_t)cap);
    if (!s->tap_warp || !s->tap_iter || !s->tap_active || !s->tap_prim || !s->tap_grads)
      return fail("out of memory");
    s->tap_cap = cap;
  }
  const int64_t r = s->tap_count++;
  s->tap_warp[r] = warp;
  s->tap_iter[r] = iter;
  s->tap_active[r] = active;
  for (int l = 0; l < 32; ++l) s->tap_prim[r * 32 + l] = prim;
  memcpy(s->tap_grads + r * 32 * GS_NPARAM, g, sizeof(double) * 32 * GS_NPARAM);
  return 0;
}

/* Backward of one warp (8x4 pixels) over its tile's list, back to front: the
 * GradComputation loop of PAPER.md:1481-1504 with the 3DGS analytic
 * gradients as the "..." and 9 atomicAdds per participating pixel. */
/* ppt = pixels per lane of the record layout: 1 = one 8x4 pixel block per
 * warp (warp w of 8); 2 = the GPU's reduction-policy kernel layout
 * (k_backward_ppt2): warp w of 4 owns an 8x8 block and lane l holds pixels
 * (l & 7, l >> 3) and (l & 7, (l >> 3) + 4); the lane's record value is the
 * sum of its pixels' gradients and it is active if either pixel is. */
static void backward_warp(job* jb, int tile, int w, int ppt) {
  gs_state* s = jb->s;
  const gs_camera* cam = jb->cam;
  const uint32_t rs = s->ranges[2 * tile], re = s->ranges[2 * tile + 1];
  const int HW = s->H * s->W;
  const int npix = 32 * ppt;
  float T[64], Tfin[64], dLp[64][3], acc[64][3], lastc[64][3], lasta[64], bgdot[64];
  uint32_t contrib[64], lastcontrib[64];
  int inside[64], pxs[64], pys[64];
  for (int l = 0; l < npix; ++l) {
    int px, py;
    if (ppt == 1) {
      pixel_of(tile, w * 32 + l, s->tiles_x, &px, &py);
    } else {
      px = (tile % s->tiles_x) * GS_TILE + (w & 1) * 8 + (l & 7);
      py = (tile / s->tiles_x) * GS_TILE + (w >> 1) * 8 + (l >> 3);
    }
    pxs[l] = px;
    pys[l] = py;
    inside[l] = px < s->W && py < s->H;
    const int pix = py * s->W + px;
    Tfin[l] = inside[l] ? s->final_T[pix] : 0.0f;
    T[l] = Tfin[l];
    contrib[l] = re - rs;
    lastcontrib[l] = inside[l] ? s->n_contrib[pix] : 0;
    lasta[l] = 0.0f;
    bgdot[l] = 0.0f;
    for (int ch = 0; ch < 3; ++ch) {
      dLp[l][ch] = inside[l] ? jb->dL[ch * HW + pix] : 0.0f;
      acc[l][ch] = 0.0f;
      lastc[l][ch] = 0.0f;
      bgdot[l] += cam->bg[ch] * dLp[l][ch];
    }
  }
  const float ddelx_dx = 0.5f * (float)s->W, ddely_dy = 0.5f * (float)s->H;
  double g[64 * GS_NPARAM], rec[32 * GS_NPARAM];
  int32_t iter = 0;
  for (uint32_t jj = re; jj > rs; --jj, ++iter) {
    const uint32_t id = s->values[jj - 1];
    const float* co = s->conic_opacity + 4 * id;
    const float* col = s->rgb + 3 * id;
    uint64_t active = 0;
    memset(g, 0, sizeof g);
    for (int l = 0; l < npix; ++l) {
      if (!inside[l]) continue;
      contrib[l]--;
      if (contrib[l] >= lastcontrib[l]) continue;
      const float dx = s->means2D[2 * id] - (float)pxs[l];
      const float dy = s->means2D[2 * id + 1] - (float)pys[l];
      const float power = -0.5f * (co[0] * dx * dx + co[2] * dy * dy) - co[1] * dx * dy;
      if (power > 0.0f) continue;
      const float G = expf(power);
      const float alpha = fminf(0.99f, co[3] * G);
      if (alpha < 1.0f / 255.0f) continue;
      T[l] = T[l] / (1.0f - alpha);
      const float dchannel_dcolor = alpha * T[l];
      float dL_dalpha = 0.0f;
      double* gl = g + l * GS_NPARAM;
      for (int ch = 0; ch < 3; ++ch) {
        const float c = col[ch];
        acc[l][ch] = lasta[l] * lastc[l][ch] + (1.0f - lasta[l]) * acc[l][ch];
        lastc[l][ch] = c;
        dL_dalpha += (c - acc[l][ch]) * dLp[l][ch];
        gl[6 + ch] = dchannel_dcolor * dLp[l][ch];
      }
      dL_dalpha *= T[l];
      lasta[l] = alpha;
      dL_dalpha += (-Tfin[l] / (1.0f - alpha)) * bgdot[l];
      const float dL_dG = co[3] * dL_dalpha;
      const float gdx = G * dx, gdy = G * dy;
      const float dG_ddelx = -gdx * co[0] - gdy * co[1];
      const float dG_ddely = -gdy * co[2] - gdx * co[1];
      gl[0] = dL_dG * dG_ddelx * ddelx_dx;
      gl[1] = dL_dG * dG_ddely * ddely_dy;
      gl[2] = -0.5f * gdx * dx * dL_dG;
      gl[3] = -0.5f * gdx * dy * dL_dG;
      gl[4] = -0.5f * gdy * dy * dL_dG;
      gl[5] = G * dL_dalpha;
      active |= 1ull << l;
    }
    if (!active) continue;
    for (int l = 0; l < npix; ++l) {
      if (!(active >> l & 1ull)) continue;
      jb->pairs++;
      if (jb->tap == 2) continue; /* records only */
      for (int p = 0; p < GS_NPARAM; ++p) {
        const double v = g[l * GS_NPARAM + p];
        jb->grad[(size_t)id * GS_NPARAM + p] += v;
        if (jb->gabs) jb->gabs[(size_t)id * GS_NPARAM + p] += fabs(v);
      }
    }
    if (jb->tap) {
      uint32_t lanes = 0;
      for (int l = 0; l < 32; ++l) {
        const int hit = (int)(active >> l & 1ull) | (ppt == 2 ? (int)(active >> (l + 32) & 1ull) : 0);
        if (hit) lanes |= 1u << l;
        for (int p = 0; p < GS_NPARAM; ++p)
          rec[l * GS_NPARAM + p] = g[l * GS_NPARAM + p] +
                                   (ppt == 2 ? g[(l + 32) * GS_NPARAM + p] : 0.0);
      }
      tap_push(&jb->tapbuf, tile * (8 / ppt) + w, iter, lanes, (int32_t)id, rec);
    }
  }
}

static void* backward_worker(void* arg) {
  job* jb = arg;
  const int ntiles = jb->s->tiles_x * jb->s->tiles_y;
  const int ppt = jb->s->tap_ppt == 2 ? 2 : 1;
  for (int tile = jb->tid * jb->stride; tile < ntiles; tile += jb->nthreads * jb->stride)
    for (int w = 0; w < 8 / ppt; ++w) backward_warp(jb, tile, w, ppt);
  return NULL;
}

int gs_backward(gs_state* s, const gs_camera* cam, const float* dL_dpixels,
                double* grad, double* grad_abs, int threads, int tile_stride,
                int tap, int64_t* pairs_out) {
  if (!s || !cam || !dL_dpixels || !grad) return fail("null argument");
  if (!s->ranges) return fail("gs_backward before gs_forward");
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  if (tile_stride < 1) tile_stride = 1;
  free_tap(s);
  const size_t words = (size_t)s->P * GS_NPARAM;
  memset(grad, 0, words * sizeof(double));
  if (grad_abs) memset(grad_abs, 0, words * sizeof(double));
  pthread_t th[64];
  job jobs[64];
  for (int t = 0; t < threads; ++t) {
    memset(&jobs[t], 0, sizeof(job));
    jobs[t].s = s;
    jobs[t].cam = cam;
    jobs[t].dL = dL_dpixels;
    jobs[t].tid = t;
    jobs[t].nthreads = threads;
    jobs[t].stride = tile_stride;
    jobs[t].tap = tap;
    jobs[t].grad = t == 0 ? grad : calloc(words ? words : 1, sizeof(double));
    jobs[t].gabs = t == 0 ? grad_abs
                          : (grad_abs ? calloc(words ? words : 1, sizeof(double)) : NULL);
    if (threads == 1) backward_worker(&jobs[0]);
    else pthread_create(&th[t], NULL, backward_worker, &jobs[t]);
  }
  int64_t pairs = 0;
  for (int t = 0; t < threads; ++t) {
    if (threads > 1) pthread_join(th[t], NULL);
    pairs += jobs[t].pairs;
    if (tap) {
      gs_state* b = &jobs[t].tapbuf;
      for (int64_t r = 0; r < b->tap_count; ++r)
        tap_push(s, b->tap_warp[r], b->tap_iter[r], b->tap_active[r], b->tap_prim[r * 32],
                 b->tap_grads + r * 32 * GS_NPARAM);
      free_tap(b);
    }
    if (t == 0) continue;
    for (size_t i = 0; i < words; ++i) grad[i] += jobs[t].grad[i];
    if (grad_abs)
      for (size_t i = 0; i < words; ++i) grad_abs[i] += jobs[t].gabs[i];
    free(jobs[t].grad);
    free(jobs[t].gabs);
  }
  if (pairs_out) *pairs_out = pairs;
  return 0;
}

/* ------------------------------------------------- preprocess backward (f1)
 * Restates the public 3DGS preprocess backward (Kerbl et al. 2023, their
 * computeCov2D / computeCov3D / preprocess backward) in float64, for
 * Sigma = R diag(s^2) R^T from a normalised (r, x, y, z) quaternion (the
 * normalisation is differentiated too), cov2D = T Sigma T^T + 0.3 I with
 * T = J W, and ndc = (P m)_xy / (P m)_w. Conventions of the screen-space
 * gradients (gs_backward): mean2D is d/d ndc (pixel gradient x 0.5 W), the
 * conic off-diagonal is HALF of d/d b. The clamp of the view-space x/y in J
 * zeroes the x/y gradient (as 3DGS); mean gradients flow through both the
 * projection and the covariance. Invisible Gaussians (radius 0) get none. */
int gs_preprocess_backward(const gs_state* s, int32_t P, const float* means3D,
                           const float* scales, const float* rotations,
                           const gs_camera* cam, const double* grad2d, double* grad3d) {
  if (!s || !means3D || !scales || !rotations || !cam || !grad2d || !grad3d)
    return fail("null argument");
  if (s->P != P || !s->radii) return fail("gs_preprocess_backward: forward state mismatch");
  const float* vm = cam->viewmatrix;
  const float* pm = cam->projmatrix;
  const double fx = (double)cam->width / (2.0 * cam->tan_fovx);
  const double fy = (double)cam->height / (2.0 * cam->tan_fovy);
  for (int i = 0; i < P; ++i) {
    if (s->radii[i] <= 0) continue;
    const double* g2 = grad2d + (size_t)i * GS_NPARAM;
    double* g3 = grad3d + (size_t)i * GS_NPARAM3D;
    const double mx = means3D[3 * i], my = means3D[3 * i + 1], mz = means3D[3 * i + 2];
    /* covariance chain */
    const double qr0 = rotations[4 * i], qx0 = rotations[4 * i + 1], qy0 = rotations[4 * i + 2],
                 qz0 = rotations[4 * i + 3];
    const double qn = sqrt(qr0 * qr0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0);
    const double r = qr0 / qn, x = qx0 / qn, y = qy0 / qn, z = qz0 / qn;
    double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - r * z), 2 * (x * z + r * y)},
                      {2 * (x * y + r * z), 1 - 2 * (x * x + z * z), 2 * (y * z - r * x)},
                      {2 * (x * z - r * y), 2 * (y * z + r * x), 1 - 2 * (x * x + y * y)}};
    const double mod = cam->scale_modifier;
    double sv[3], var[3];
    for (int k = 0; k < 3; ++k) {
      sv[k] = mod * scales[3 * i + k];
      var[k] = sv[k] * sv[k];
    }
    double Sig[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        Sig[a][b] = R[a][0] * var[0] * R[b][0] + R[a][1] * var[1] * R[b][1] + R[a][2] * var[2] * R[b][2];
    double t[3];
    for (int a = 0; a < 3; ++a) t[a] = vm[a] * mx + vm[4 + a] * my + vm[8 + a] * mz + vm[12 + a];
    const double limx = 1.3 * cam->tan_fovx, limy = 1.3 * cam->tan_fovy;
    const double txtz = t[0] / t[2], tytz = t[1] / t[2];
    const double xmul = (txtz < -limx || txtz > limx) ? 0.0 : 1.0;
    const double ymul = (tytz < -limy || tytz > limy) ? 0.0 : 1.0;
    const double tx = fmin(limx, fmax(-limx, txtz)) * t[2];
    const double ty = fmin(limy, fmax(-limy, tytz)) * t[2];
    const double tz = t[2];
    double J[2][3] = {{fx / tz, 0, -fx * tx / (tz * tz)}, {0, fy / tz, -fy * ty / (tz * tz)}};
    double Wm[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) Wm[a][b] = vm[b * 4 + a];
    double T[2][3];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) T[a][b] = J[a][0] * Wm[0][b] + J[a][1] * Wm[1][b] + J[a][2] * Wm[2][b];
    double cov[2][2];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double acc = 0;
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) acc += T[a][k] * Sig[k][l] * T[b][l];
        cov[a][b] = acc;
      }
    const double A = cov[0][0] + 0.3, B = cov[0][1], Cc = cov[1][1] + 0.3;
    const double D = A * Cc - B * B, D2 = D * D;
    const double ga = g2[2], gb = 2.0 * g2[3], gc = g2[4];
    const double dA = (-Cc * Cc * ga + B * Cc * gb - B * B * gc) / D2;
    const double dC = (-B * B * ga + A * B * gb - A * A * gc) / D2;
    const double dB = (2 * B * Cc * ga - (D + 2 * B * B) * gb + 2 * A * B * gc) / D2;
    const double G[2][2] = {{dA, 0.5 * dB}, {0.5 * dB, dC}};
    /* dL/dSigma = T^T G T ; dL/dT = 2 G T Sigma */
    double dSig[3][3], dT[2][3], TS[2][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0;
        for (int k = 0; k < 2; ++k)
          for (int l = 0; l < 2; ++l) acc += T[k][a] * G[k][l] * T[l][b];
        dSig[a][b] = acc;
      }
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) TS[a][b] = T[a][0] * Sig[0][b] + T[a][1] * Sig[1][b] + T[a][2] * Sig[2][b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) dT[a][b] = 2 * (G[a][0] * TS[0][b] + G[a][1] * TS[1][b]);
    /* dL/dJ = dT W^T */
    double dJ[2][3];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) dJ[a][b] = dT[a][0] * Wm[b][0] + dT[a][1] * Wm[b][1] + dT[a][2] * Wm[b][2];
    const double tz2 = tz * tz, tz3 = tz2 * tz;
    double dt[3];
    dt[0] = xmul * (-fx / tz2) * dJ[0][2];
    dt[1] = ymul * (-fy / tz2) * dJ[1][2];
    dt[2] = -fx / tz2 * dJ[0][0] - fy / tz2 * dJ[1][1] + 2 * fx * tx / tz3 * dJ[0][2] +
            2 * fy * ty / tz3 * dJ[1][2];
    double dm[3];
    for (int b = 0; b < 3; ++b) dm[b] = Wm[0][b] * dt[0] + Wm[1][b] * dt[1] + Wm[2][b] * dt[2];
    /* projection path: ndc = (P m)_xy / ((P m)_w + 1e-7) */
    const double hx = pm[0] * mx + pm[4] * my + pm[8] * mz + pm[12];
    const double hy = pm[1] * mx + pm[5] * my + pm[9] * mz + pm[13];
    const double hw = pm[3] * mx + pm[7] * my + pm[11] * mz + pm[15] + 1e-7;
    for (int b = 0; b < 3; ++b) {
      const double dnx = (pm[4 * b] * hw - hx * pm[4 * b + 3]) / (hw * hw);
      const double dny = (pm[4 * b + 1] * hw - hy * pm[4 * b + 3]) / (hw * hw);
      dm[b] += g2[0] * dnx + g2[1] * dny;
    }
    /* Sigma = R diag(var) R^T: dvar_k = (R^T dSig R)_kk; dR = 2 dSig R diag(var) */
    double dR[3][3];
    for (int k = 0; k < 3; ++k) {
      double acc = 0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) acc += R[a][k] * dSig[a][b] * R[b][k];
      g3[3 + k] += acc * 2.0 * mod * sv[k];
    }
    for (int a = 0; a < 3; ++a)
      for (int k = 0; k < 3; ++k)
        dR[a][k] = 2 * (dSig[a][0] * R[0][k] + dSig[a][1] * R[1][k] + dSig[a][2] * R[2][k]) * var[k];
    const double dRr[3][3] = {{0, -2 * z, 2 * y}, {2 * z, 0, -2 * x}, {-2 * y, 2 * x, 0}};
    const double dRx[3][3] = {{0, 2 * y, 2 * z}, {2 * y, -4 * x, -2 * r}, {2 * z, 2 * r, -4 * x}};
    const double dRy[3][3] = {{-4 * y, 2 * x, 2 * r}, {2 * x, 0, 2 * z}, {-2 * r, 2 * z, -4 * y}};
    const double dRz[3][3] = {{-4 * z, -2 * r, 2 * x}, {2 * r, -4 * z, 2 * y}, {2 * x, 2 * y, 0}};
    double dqn[4] = {0, 0, 0, 0};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        dqn[0] += dR[a][b] * dRr[a][b];
        dqn[1] += dR[a][b] * dRx[a][b];
        dqn[2] += dR[a][b] * dRy[a][b];
        dqn[3] += dR[a][b] * dRz[a][b];
      }
    const double qv[4] = {r, x, y, z};
    const double dot = qv[0] * dqn[0] + qv[1] * dqn[1] + qv[2] * dqn[2] + qv[3] * dqn[3];
    for (int k = 0; k < 4; ++k) g3[6 + k] += (dqn[k] - qv[k] * dot) / qn;
    for (int b = 0; b < 3; ++b) g3[b] += dm[b];
    g3[10] += g2[5];
    g3[11] += g2[6];
    g3[12] += g2[7];
    g3[13] += g2[8];
  }
  return 0;
}

void gs_adam(int64_t n, double* param, const double* grad, double* m, double* v, double lr,
             double beta1, double beta2, double eps, int step) {
  const double bc1 = 1.0 - pow(beta1, step), bc2 = 1.0 - pow(beta2, step);
  for (int64_t i = 0; i < n; ++i) {
    m[i] = beta1 * m[i] + (1.0 - beta1) * grad[i];
    v[i] = beta2 * v[i] + (1.0 - beta2) * grad[i] * grad[i];
    param[i] -= lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
  }
}
