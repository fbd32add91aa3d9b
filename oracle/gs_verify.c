/*
 * TEST INFRASTRUCTURE ONLY -- decision-matched verification oracle for the
 * Gaussian-splatting blend at full size (BASELINE configs[2..4]).
 *
 * PARITY UNPINNED BY THE REFERENCE (no rasterizer under /root/reference, see
 * gs_oracle.c); the pinned pieces are the loop shape of the gradient step
 * and the reduction semantics checked elsewhere.
 *
 * What it does, per view:
 *
 * 1. Lists (gs_forward_lists): projection (gs_oracle.c, bit-exact with the
 *    GPU preprocess) and per-tile lists built by bucketing the Gaussians in
 *    (depth, index) order into the tiles of their rectangles -- the same
 *    lists as the stable (tile | depth) sort of gs_forward, in O(P log P + I)
 *    and without materialising 64-bit keys (C4 has 0.9 G instances).
 *
 * 2. Decisions. Which (pixel, Gaussian) pairs blend is decided by fp32
 *    arithmetic: the log2-scaled quadratic form in the blend kernels' Horner
 *    order (raster_blend.cu eval2: power = fma(fma(k c, dy, 2 k b dx), dy,
 *    k a dx^2)), then o * 2^power >= 1/255 and the transmittance test
 *    T (1 - alpha) >= 1e-4. The oracle evaluates power bit-exactly (fmaf) and
 *    2^power with the C library's exp2f, where the GPU uses ex2.approx. A
 *    decision therefore agrees with the GPU's unless its operand lies inside
 *    the error band of that approximation: |o G - 1/255| <= 2^-18 / 255 for
 *    the alpha test, |T (1 - alpha) - 1e-4| <= 2 e_T u 1e-4 for termination
 *    (e_T: running relative-error bound of the GPU's T in units of
 *    u = 2^-24, below). Such decisions are AMBIGUOUS: the oracle enumerates
 *    every "world" (each combination of taken / not-taken ambiguous
 *    decisions, depth-first, capped) and, given the GPU's per-pixel outputs
 *    (n_contrib, final_T, image), identifies which world the GPU took.
 *    Every flipped decision is reported (gs_flip); a pixel no world explains
 *    is reported as a mismatch.
 *
 * 3. Values in exact-ish arithmetic. For the matched world the blend and
 *    its analytic backward (3DGS, Kerbl et al. 2023; same conventions as
 *    gs_oracle.c backward_warp: mean2D in pixel units x W/2, H/2; conic
 *    terms -1/2 G d d^T dL/dG; colour alpha T dL/dpixel; the 0.99 clamp
 *    not differentiated) are computed in float64 with G = 2^power, so the
 *    oracle's own rounding is negligible against the GPU's fp32.
 *
 * 4. Error bounds. Per pixel E = 2 e_T + 64 (units of u), with
 *    e_T = sum over blended Gaussians of 12 alpha / (1 - alpha) + 3: the
 *    relative error the GPU's fp32 transmittance can accumulate (ex2.approx
 *    <= 2^-21 relative in G, one rounding per product / difference, T
 *    reconstructed back to front by rcp.approx in the backward: twice the
 *    forward's), plus a constant for the dozen roundings inside one term.
 *    Per pair and parameter the term MAGNITUDE is the term with every
 *    subexpression replaced by its absolute value (so cancellation inside
 *    dL/dalpha is not hidden). Outputs: grad_bound = sum E * magnitude,
 *    grad_abs = sum |term|, npix = contributing pixels. A GPU gradient
 *    element g satisfies |g - grad| <= kappa u grad_bound
 *    + (npix + 16) u grad_abs (the second term: fp32 summation of npix
 *    terms in any order), with kappa stated by the test.
 */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gs_internal.h"
#include "gs_oracle.h"

#define U_F32 (1.0 / 16777216.0)
#define MAX_WORLDS 64
#define MAX_AMB 32

static __thread char v_err[256] = "ok";
static int vfail(const char* m) {
  snprintf(v_err, sizeof v_err, "%s", m);
  return 1;
}
const char* gs_verify_last_error(void) { return v_err; }

/* ----------------------------------------------------------------- lists */

/* Stable LSD radix sort of 32-bit keys carrying 32-bit values. */
static int radix32(uint32_t* k, uint32_t* v, int64_t n) {
  uint32_t* k2 = malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
  uint32_t* v2 = malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
  if (!k2 || !v2) { free(k2); free(v2); return vfail("out of memory"); }
  for (int shift = 0; shift < 32; shift += 8) {
    int64_t cnt[257] = {0};
    for (int64_t i = 0; i < n; ++i) cnt[((k[i] >> shift) & 255u) + 1]++;
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t d = cnt[(k[i] >> shift) & 255u]++;
      k2[d] = k[i];
      v2[d] = v[i];
    }
    memcpy(k, k2, sizeof(uint32_t) * (size_t)n);
    memcpy(v, v2, sizeof(uint32_t) * (size_t)n);
  }
  free(k2);
  free(v2);
  return 0;
}

typedef struct {
  const gs_state* s;
  const uint32_t* order;  /* visible Gaussians in (depth, index) order */
  const int32_t* rects;   /* 4 per Gaussian */
  int64_t norder;
  uint64_t* cursor;       /* per tile: next write position */
  uint32_t* values;
  uint64_t* keys;         /* optional */
  int y0, y1;             /* tile rows owned by this thread */
} fill_job;

static void* fill_worker(void* arg) {
  fill_job* jb = arg;
  const gs_state* s = jb->s;
  for (int64_t k = 0; k < jb->norder; ++k) {
    const uint32_t id = jb->order[k];
    const int32_t* r = jb->rects + 4 * (size_t)id;
    const int ya = r[1] > jb->y0 ? r[1] : jb->y0, yb = r[3] < jb->y1 ? r[3] : jb->y1;
    if (ya >= yb) continue;
    uint32_t dbits;
    memcpy(&dbits, &s->depths[id], 4);
    for (int y = ya; y < yb; ++y)
      for (int x = r[0]; x < r[2]; ++x) {
        const uint32_t tile = (uint32_t)(y * s->tiles_x + x);
        const uint64_t at = jb->cursor[tile]++;
        jb->values[at] = id;
        if (jb->keys) jb->keys[at] = ((uint64_t)tile << 32) | dbits;
      }
  }
  return NULL;
}

int gs_forward_lists(gs_state* s, int32_t P, const float* means3D, const float* scales,
                     const float* rotations, const float* opacities, const float* colors,
                     const gs_camera* cam, int threads, int with_keys) {
  if (!s || !means3D || !scales || !rotations || !opacities || !colors || !cam)
    return vfail("null argument");
  if (P < 0 || cam->width < 1 || cam->height < 1) return vfail("invalid size");
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  /* reset, keep the struct's allocation discipline (gs_state_free frees all) */
  free(s->means2D); free(s->depths); free(s->radii); free(s->conic_opacity); free(s->rgb);
  free(s->tiles_touched); free(s->keys); free(s->values); free(s->ranges);
  free(s->out_color); free(s->final_T); free(s->n_contrib);
  memset(s, 0, offsetof(gs_state, tap_count));
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
  if (!s->means2D || !s->depths || !s->radii || !s->conic_opacity || !s->rgb ||
      !s->tiles_touched || !s->ranges || !s->out_color || !s->final_T || !s->n_contrib)
    return vfail("out of memory");
  for (int i = 0; i < P; ++i)
    gs_i_preprocess_one(i, means3D, scales, rotations, opacities, colors, cam, s);
  /* (depth, index) order of the visible Gaussians: stable radix sort of the
   * depth bits (depth > 0.2, so the bits order like the floats) */
  int64_t nvis = 0;
  for (int i = 0; i < P; ++i) nvis += s->radii[i] > 0;
  uint32_t* dk = malloc(sizeof(uint32_t) * (size_t)(nvis ? nvis : 1));
  uint32_t* order = malloc(sizeof(uint32_t) * (size_t)(nvis ? nvis : 1));
  int32_t* rects = malloc(sizeof(int32_t) * 4 * np);
  uint64_t* cnt = calloc((size_t)ntiles + 1, sizeof(uint64_t));
  int64_t* diff = calloc((size_t)(s->tiles_x + 1) * (size_t)(s->tiles_y + 1), sizeof(int64_t));
  if (!dk || !order || !rects || !cnt || !diff) {
    free(dk); free(order); free(rects); free(cnt); free(diff);
    return vfail("out of memory");
  }
  int64_t k = 0;
  const int dx1 = s->tiles_x + 1;
  for (int i = 0; i < P; ++i) {
    if (s->radii[i] <= 0) continue;
    memcpy(&dk[k], &s->depths[i], 4);
    order[k++] = (uint32_t)i;
    int32_t* r = rects + 4 * (size_t)i;
    gs_i_rect_of(s, i, r);
    /* 2D difference grid of the tile rectangles -> per-tile counts */
    diff[(size_t)r[1] * dx1 + r[0]]++;
    diff[(size_t)r[1] * dx1 + r[2]]--;
    diff[(size_t)r[3] * dx1 + r[0]]--;
    diff[(size_t)r[3] * dx1 + r[2]]++;
  }
  if (radix32(dk, order, nvis)) {
    free(dk); free(order); free(rects); free(cnt); free(diff);
    return 1;
  }
  free(dk);
  for (int y = 0; y <= s->tiles_y; ++y)
    for (int x = 0; x <= s->tiles_x; ++x) {
      int64_t v = diff[(size_t)y * dx1 + x];
      if (x > 0) v += diff[(size_t)y * dx1 + x - 1];
      if (y > 0) v += diff[(size_t)(y - 1) * dx1 + x];
      if (x > 0 && y > 0) v -= diff[(size_t)(y - 1) * dx1 + x - 1];
      diff[(size_t)y * dx1 + x] = v;
    }
  uint64_t total = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int64_t c = diff[(size_t)(t / s->tiles_x) * dx1 + (t % s->tiles_x)];
    cnt[t] = total;
    total += (uint64_t)c;
  }
  free(diff);
  if (total > 0xffffffffull) {
    free(order); free(rects); free(cnt);
    return vfail("more than 2^32 instances");
  }
  for (int t = 0; t < ntiles; ++t) {
    const uint64_t e = t + 1 < ntiles ? cnt[t + 1] : total;
    if (e > cnt[t]) {
      s->ranges[2 * t] = (uint32_t)cnt[t];
      s->ranges[2 * t + 1] = (uint32_t)e;
    }
  }
  s->num_rendered = (int64_t)total;
  s->values = malloc(sizeof(uint32_t) * (size_t)(total ? total : 1));
  s->keys = with_keys ? malloc(sizeof(uint64_t) * (size_t)(total ? total : 1)) : NULL;
  if (!s->values || (with_keys && !s->keys)) {
    free(order); free(rects); free(cnt);
    return vfail("out of memory");
  }
  pthread_t th[64];
  fill_job jobs[64];
  const int nt = threads < s->tiles_y ? threads : s->tiles_y;
  for (int t = 0; t < nt; ++t) {
    jobs[t] = (fill_job){s, order, rects, nvis, cnt, s->values, s->keys,
                         (int)((int64_t)s->tiles_y * t / nt),
                         (int)((int64_t)s->tiles_y * (t + 1) / nt)};
    pthread_create(&th[t], NULL, fill_worker, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(order);
  free(rects);
  free(cnt);
  return 0;
}

/* ----------------------------------------------------- per-Gaussian data */

/* The blend kernels' staged conic (raster_blend.cu scale_conic). */
static const float kConicScale = -0.5f * 1.4426950408889634f;
static const float kAlphaMin = 1.0f / 255.0f;
static const float kTMin = 0.0001f;

typedef struct {
  float mx, my;
  float A, B2, Cc;   /* k a, (2k) b, k c */
  float o;
  float pthr;        /* power < pthr => o 2^power < 1/255 beyond any ex2 error */
  float a, b, c;     /* raw conic */
  float col[3];
  double ex, ey;     /* conservative alpha >= 1/255 half-extents (pixels) */
  int dead;          /* opacity too small to ever reach 1/255 */
} vg;

/* What the front-to-back walk reads, gathered per tile in list order (the
 * list is in depth order, ids are random: this keeps the walk sequential). A
 * dead Gaussian gets ex = -1 (every pixel is outside it). */
typedef struct {
  float mx, my, A, B2, Cc, o, pthr, ex, ey;
} wg;

static void stage_gauss(const gs_state* s, int id, vg* g) {
  const float* co = s->conic_opacity + 4 * (size_t)id;
  g->mx = s->means2D[2 * (size_t)id];
  g->my = s->means2D[2 * (size_t)id + 1];
  g->a = co[0];
  g->b = co[1];
  g->c = co[2];
  g->o = co[3];
  g->A = kConicScale * co[0];
  g->B2 = (2.0f * kConicScale) * co[1];
  g->Cc = kConicScale * co[2];
  for (int ch = 0; ch < 3; ++ch) g->col[ch] = s->rgb[3 * (size_t)id + ch];
  const double o = co[3];
  g->dead = o * (1.0 + 1.0 / 65536.0) < 1.0 / 255.0;
  g->pthr = g->dead ? 0.0f : (float)(log2(1.0 / (255.0 * o)) - 0.01);
  /* q = a dx^2 + 2 b dx dy + c dy^2 <= tau, tau = 2 ln(255 o); inflated well
   * beyond the fp32 rounding of power; ill-conditioned conics: no culling */
  const double a = co[0], b = co[1], c = co[2];
  const double det = a * c - b * b;
  if (g->dead || !(a > 0.0) || !(c > 0.0) || !(det > 1e-4 * a * c)) {
    g->ex = g->ey = INFINITY;
  } else {
    const double tau = 2.0 * log(255.0 * o) * 1.25 + 1.0;
    g->ex = sqrt(tau * c / det) + 1.0;
    g->ey = sqrt(tau * a / det) + 1.0;
  }
}

/* ------------------------------------------------------------ one pixel */

typedef struct {
  uint32_t pos;  /* list position (tile-relative) */
  int kind;      /* 0 alpha test, 1 termination test */
} dpoint;

static int dp_less(dpoint a, dpoint b) { return a.pos < b.pos || (a.pos == b.pos && a.kind < b.kind); }

typedef struct {
  dpoint flips[MAX_AMB];
  int nflips;
  /* results */
  uint32_t nc;        /* last blended list position, 1-based */
  int64_t nblend;
  double T, C[3], Cmag[3], eT;
  dpoint amb[MAX_AMB];
  int namb;           /* ambiguous points after the last flip (truncated at MAX_AMB) */
  int amb_overflow;
  int64_t namb_total; /* all ambiguous points met on the walk */
  int namb_alpha, namb_term;
} world;

typedef struct {
  uint32_t pos;
  double G, alpha, Tb;  /* Tb: transmittance in front of the Gaussian */
  float dx32, dy32;
} blended;

typedef struct {
  const gs_state* s;
  const vg* g;
  const wg* tg;           /* the tile's walk data, by list position */
  const uint32_t* list;   /* the tile's list */
  uint32_t len;
  float pfx, pfy;
} pctx;

/* Walk one pixel front to back in world w (its flips forced). When bl is not
 * NULL the blended Gaussians are recorded there. */
static void walk(const pctx* c, world* w, blended* bl) {
  float T32 = 1.0f;
  double Td = 1.0, eT = 0.0;
  w->nc = 0;
  w->nblend = 0;
  w->C[0] = w->C[1] = w->C[2] = 0.0;
  w->Cmag[0] = w->Cmag[1] = w->Cmag[2] = 0.0;
  w->namb = 0;
  w->amb_overflow = 0;
  w->namb_total = 0;
  w->namb_alpha = w->namb_term = 0;
  const dpoint last = w->nflips ? w->flips[w->nflips - 1] : (dpoint){0, -1};
  int fi = 0;  /* next flip to meet */
  for (uint32_t pos = 0; pos < c->len; ++pos) {
    const wg* g = c->tg + pos;
    const float dx = g->mx - c->pfx, dy = g->my - c->pfy;
    if (!(fabsf(dx) <= g->ex) || !(fabsf(dy) <= g->ey)) continue;
    const float dxx = dx * dx;
    const float power = fmaf(fmaf(g->Cc, dy, g->B2 * dx), dy, g->A * dxx);
    if (!(power <= 0.0f)) continue;
    if (power < g->pthr) continue;
    const float G = exp2f(power);
    const float Go = G * g->o;
    int a = Go >= kAlphaMin;
    if (fabs((double)Go - (double)kAlphaMin) <= ldexp((double)kAlphaMin, -18)) {
      const dpoint p = {pos, 0};
      w->namb_total++;
      w->namb_alpha++;
      if (fi < w->nflips && w->flips[fi].pos == pos && w->flips[fi].kind == 0) {
        a = !a;
        fi++;
      } else if (w->nflips == 0 || dp_less(last, p)) {
        if (w->namb < MAX_AMB) w->amb[w->namb++] = p;
        else w->amb_overflow = 1;
      }
    }
    if (!a) continue;
    const float alpha = fminf(0.99f, Go);
    const float testT = T32 * (1.0f - alpha);
    const double inc = 12.0 * (double)alpha / (1.0 - (double)alpha) + 3.0;
    int b = testT >= kTMin;
    if (fabs((double)testT - (double)kTMin) <= 2.0 * (eT + inc) * U_F32 * (double)kTMin) {
      const dpoint p = {pos, 1};
      w->namb_total++;
      w->namb_term++;
      if (fi < w->nflips && w->flips[fi].pos == pos && w->flips[fi].kind == 1) {
        b = !b;
        fi++;
      } else if (w->nflips == 0 || dp_less(last, p)) {
        if (w->namb < MAX_AMB) w->amb[w->namb++] = p;
        else w->amb_overflow = 1;
      }
    }
    if (!b) break;  /* terminates: this and later Gaussians do not blend */
    const double Gd = exp2((double)power);
    const double ad = fmin(0.99, Gd * (double)g->o);
    if (bl) {
      blended* e = bl + w->nblend;
      e->pos = pos;
      e->G = Gd;
      e->alpha = ad;
      e->Tb = Td;
      e->dx32 = dx;
      e->dy32 = dy;
    }
    const float* col = c->g[c->list[pos]].col;
    for (int ch = 0; ch < 3; ++ch) {
      w->C[ch] += (double)col[ch] * ad * Td;
      w->Cmag[ch] += fabs((double)col[ch]) * ad * Td;
    }
    Td *= 1.0 - ad;
    T32 = testT;
    eT += inc;
    w->nc = pos + 1;
    w->nblend++;
  }
  w->T = Td;
  w->eT = eT;
}

/* ------------------------------------------------------------ the verify */

typedef struct {
  const gs_state* s;
  const gs_camera* cam;
  const float* dL;
  const uint32_t* gpu_nc;
  const float* gpu_T;
  const float* gpu_img;
  double kappa;
  const vg* g;
  gs_verify_out* out;
  int tid, nthreads;
  /* per-thread accumulators */
  double *grad, *bound, *gabs;
  int32_t* npix;
  gs_verify_report rep;
  pthread_mutex_t* mu;
  int failed;
} vjob;

static double pix_E(double eT) { return 2.0 * eT + 64.0; }

/* Backward of one pixel in exact-ish arithmetic over its blended list. With
 * acc == NULL the per-Gaussian terms go to terms[nb*9] (slack computation). */
static void pixel_backward(vjob* jb, const pctx* c, const blended* bl, int64_t nb, double Tf,
                           double E, const float* dLp, double* terms) {
  const gs_camera* cam = jb->cam;
  const double bgdot = cam->bg[0] * (double)dLp[0] + cam->bg[1] * (double)dLp[1] +
                       cam->bg[2] * (double)dLp[2];
  const double bgabs = fabs(cam->bg[0] * (double)dLp[0]) + fabs(cam->bg[1] * (double)dLp[1]) +
                       fabs(cam->bg[2] * (double)dLp[2]);
  const double hw = 0.5 * (double)jb->s->W, hh = 0.5 * (double)jb->s->H;
  double S = 0.0, Smag = 0.0;
  for (int64_t k = nb - 1; k >= 0; --k) {
    const blended* e = bl + k;
    const uint32_t id = c->list[e->pos];
    const vg* g = c->g + id;
    const double dx = (double)g->mx - (double)c->pfx, dy = (double)g->my - (double)c->pfy;
    const double al = e->alpha, T = e->Tb, G = e->G, o = g->o;
    double CD = 0.0, CDabs = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
      CD += (double)g->col[ch] * (double)dLp[ch];
      CDabs += fabs((double)g->col[ch] * (double)dLp[ch]);
    }
    const double dLa = T * (CD - S) - Tf * bgdot / (1.0 - al);
    const double dLam = T * (CDabs + Smag) + Tf * bgabs / (1.0 - al);
    const double q = G * o * dLa, qm = G * o * dLam;
    const double a = g->a, b = g->b, cc = g->c;
    const double t[GS_NPARAM] = {-q * (a * dx + b * dy) * hw,
                                 -q * (cc * dy + b * dx) * hh,
                                 -0.5 * q * dx * dx,
                                 -0.5 * q * dx * dy,
                                 -0.5 * q * dy * dy,
                                 G * dLa,
                                 al * T * (double)dLp[0],
                                 al * T * (double)dLp[1],
                                 al * T * (double)dLp[2]};
    if (terms) {
      memcpy(terms + k * GS_NPARAM, t, sizeof t);
    } else {
      const double m[GS_NPARAM] = {qm * (fabs(a * dx) + fabs(b * dy)) * hw,
                                   qm * (fabs(cc * dy) + fabs(b * dx)) * hh,
                                   0.5 * qm * dx * dx,
                                   0.5 * qm * fabs(dx * dy),
                                   0.5 * qm * dy * dy,
                                   G * dLam,
                                   al * T * fabs((double)dLp[0]),
                                   al * T * fabs((double)dLp[1]),
                                   al * T * fabs((double)dLp[2])};
      double* gr = jb->grad + (size_t)id * GS_NPARAM;
      double* bo = jb->bound + (size_t)id * GS_NPARAM;
      double* ga = jb->gabs + (size_t)id * GS_NPARAM;
      for (int p = 0; p < GS_NPARAM; ++p) {
        gr[p] += t[p];
        bo[p] += E * m[p];
        ga[p] += fabs(t[p]);
      }
      jb->npix[id]++;
    }
    S = al * CD + (1.0 - al) * S;
    Smag = al * CDabs + (1.0 - al) * Smag;
  }
}

/* distance of world w to the GPU's outputs at pixel pix (<= 1: consistent) */
static double world_dist(const vjob* jb, const world* w, int pix, int HW) {
  if (w->nc != jb->gpu_nc[pix]) return INFINITY;
  const double E = pix_E(w->eT) * jb->kappa * U_F32;
  double d = fabs(w->T - (double)jb->gpu_T[pix]) / (E * w->T + 1e-30);
  for (int ch = 0; ch < 3; ++ch) {
    const double want = w->C[ch] + w->T * jb->cam->bg[ch];
    const double mag = w->Cmag[ch] + w->T * fabs(jb->cam->bg[ch]);
    const double dd = fabs(want - (double)jb->gpu_img[ch * HW + pix]) / (E * mag + 1e-30);
    if (dd > d) d = dd;
  }
  return d;
}

typedef struct {
  int64_t cap;
  wg* tg;
  blended* bl;
  blended* bl2;
  double* terms;
  double* terms2;
  int64_t blcap;
  world worlds[MAX_WORLDS];
} vbuf;

static int vbuf_reserve(vbuf* b, int64_t n) {
  if (n <= b->cap) return 0;
  free(b->tg);
  b->tg = malloc(sizeof(wg) * (size_t)n);
  if (!b->tg) return 1;
  free(b->bl); free(b->bl2); free(b->terms); free(b->terms2);
  b->bl = malloc(sizeof(blended) * (size_t)n);
  b->bl2 = malloc(sizeof(blended) * (size_t)n);
  b->terms = malloc(sizeof(double) * GS_NPARAM * (size_t)n);
  b->terms2 = malloc(sizeof(double) * GS_NPARAM * (size_t)n);
  if (!b->bl || !b->bl2 || !b->terms || !b->terms2) return 1;
  b->cap = n;
  return 0;
}

static void vbuf_free(vbuf* b) {
  free(b->tg);
  free(b->bl); free(b->bl2); free(b->terms); free(b->terms2);
}

static void record_flips(vjob* jb, const world* w, const pctx* c, int pix) {
  gs_verify_out* o = jb->out;
  pthread_mutex_lock(jb->mu);
  for (int f = 0; f < w->nflips; ++f) {
    if (o->flips && o->nflip_rec < o->flip_cap) {
      gs_flip* r = o->flips + o->nflip_rec++;
      r->pixel = pix;
      r->position = w->flips[f].pos;
      r->gaussian = (int32_t)c->list[w->flips[f].pos];
      r->kind = w->flips[f].kind;
    }
  }
  pthread_mutex_unlock(jb->mu);
}

/* Unresolved pixel: the GPU's outputs fit more than one world. Add, per
 * Gaussian and parameter, the spread between the chosen world's terms and
 * each other consistent world's into grad_slack. */
static void add_slack(vjob* jb, vbuf* b, const pctx* c, const world* best, const world* other,
                      const float* dLp) {
  world wb = *best, wo = *other;
  walk(c, &wb, b->bl);
  walk(c, &wo, b->bl2);
  pixel_backward(jb, c, b->bl, wb.nblend, wb.T, 0.0, dLp, b->terms);
  pixel_backward(jb, c, b->bl2, wo.nblend, wo.T, 0.0, dLp, b->terms2);
  double* sl = jb->out->grad_slack;
  pthread_mutex_lock(jb->mu);
  int64_t i = 0, j = 0;
  while (i < wb.nblend || j < wo.nblend) {
    const uint32_t pi = i < wb.nblend ? b->bl[i].pos : 0xffffffffu;
    const uint32_t pj = j < wo.nblend ? b->bl2[j].pos : 0xffffffffu;
    const uint32_t pos = pi < pj ? pi : pj;
    const uint32_t id = c->list[pos];
    for (int p = 0; p < GS_NPARAM; ++p) {
      const double x = pi == pos ? b->terms[i * GS_NPARAM + p] : 0.0;
      const double y = pj == pos ? b->terms2[j * GS_NPARAM + p] : 0.0;
      sl[(size_t)id * GS_NPARAM + p] += fabs(x - y);
    }
    if (pi == pos) ++i;
    if (pj == pos) ++j;
  }
  pthread_mutex_unlock(jb->mu);
}

static void verify_tile(vjob* jb, vbuf* b, int tile) {
  const gs_state* s = jb->s;
  const uint32_t rs = s->ranges[2 * tile], re = s->ranges[2 * tile + 1];
  const int64_t L = (int64_t)re - rs;
  const int HW = s->H * s->W;
  const int tx0 = (tile % s->tiles_x) * GS_TILE, ty0 = (tile / s->tiles_x) * GS_TILE;
  if (vbuf_reserve(b, L > 0 ? L : 1)) { jb->failed = 1; return; }
  const uint32_t* list = s->values + rs;
  for (int64_t j = 0; j < L; ++j) {
    const vg* g = jb->g + list[j];
    wg* t = b->tg + j;
    t->mx = g->mx;
    t->my = g->my;
    t->A = g->A;
    t->B2 = g->B2;
    t->Cc = g->Cc;
    t->o = g->o;
    t->pthr = g->pthr;
    t->ex = g->dead ? -1.0f : (isinf(g->ex) ? INFINITY : (float)g->ex);
    t->ey = g->dead ? -1.0f : (isinf(g->ey) ? INFINITY : (float)g->ey);
  }
  gs_verify_out* o = jb->out;
  for (int r = 0; r < GS_TILE; ++r) {
    const int py = ty0 + r;
    if (py >= s->H) break;
    for (int cx = 0; cx < GS_TILE; ++cx) {
      const int px = tx0 + cx;
      if (px >= s->W) break;
      const int pix = py * s->W + px;
      pctx c = {s, jb->g, b->tg, list, (uint32_t)L, (float)px, (float)py};
      float dLp[3] = {0.0f, 0.0f, 0.0f};
      if (jb->dL)
        for (int ch = 0; ch < 3; ++ch) dLp[ch] = jb->dL[ch * HW + pix];
      /* enumerate worlds depth-first */
      int nw = 1, capped = 0;
      b->worlds[0].nflips = 0;
      for (int wi = 0; wi < nw; ++wi) {
        walk(&c, &b->worlds[wi], wi == 0 ? b->bl : NULL);
        if (b->worlds[wi].amb_overflow) capped = 1;
        for (int k = 0; k < b->worlds[wi].namb; ++k) {
          if (nw == MAX_WORLDS || b->worlds[wi].nflips == MAX_AMB) { capped = 1; break; }
          world* nwp = &b->worlds[nw++];
          memcpy(nwp->flips, b->worlds[wi].flips, sizeof(dpoint) * (size_t)b->worlds[wi].nflips);
          nwp->nflips = b->worlds[wi].nflips;
          nwp->flips[nwp->nflips++] = b->worlds[wi].amb[k];
        }
      }
      const world* w0 = &b->worlds[0];
      jb->rep.amb_alpha += w0->namb_alpha;
      jb->rep.amb_term += w0->namb_term;
      jb->rep.pairs_default += w0->nblend;
      if (nw > jb->rep.max_worlds) jb->rep.max_worlds = nw;
      int best = 0;
      uint8_t st = 0;
      if (nw > 1) {
        jb->rep.pix_ambiguous++;
        st = 1;
      }
      if (capped) {
        jb->rep.pix_world_cap++;
        st = 5;
      }
      if (!jb->gpu_nc && nw > 1) {
        /* nothing to match: every world is possible; its spread becomes slack */
        for (int wi = 1; wi < nw; ++wi) {
          add_slack(jb, b, &c, &b->worlds[0], &b->worlds[wi], dLp);
          if (o->image_slack)
            for (int ch = 0; ch < 3; ++ch) {
              const double d = fabs(b->worlds[wi].C[ch] + b->worlds[wi].T * jb->cam->bg[ch] -
                                    w0->C[ch] - w0->T * jb->cam->bg[ch]);
              if (d > o->image_slack[ch * HW + pix]) o->image_slack[ch * HW + pix] = d;
            }
        }
        walk(&c, &b->worlds[0], b->bl);  /* add_slack reused the buffer */
      }
      if (jb->gpu_nc) {
        double bd = INFINITY, second = INFINITY;
        for (int wi = 0; wi < nw; ++wi) {
          const double d = world_dist(jb, &b->worlds[wi], pix, HW);
          if (d < bd) { second = bd; bd = d; best = wi; }
          else if (d < second) second = d;
        }
        if (!(bd <= 1.0)) {
          jb->rep.pix_nomatch++;
          st = 4;
          best = 0;
        } else if (second <= 1.0) {
          jb->rep.pix_unresolved++;
          if (st != 5) st = 3;
          for (int wi = 0; wi < nw; ++wi)
            if (wi != best && world_dist(jb, &b->worlds[wi], pix, HW) <= 1.0)
              add_slack(jb, b, &c, &b->worlds[best], &b->worlds[wi], dLp);
        } else if (best != 0) {
          jb->rep.pix_flipped++;
          jb->rep.flips += b->worlds[best].nflips;
          if (st != 5) st = 2;
        }
        if (best != 0) record_flips(jb, &b->worlds[best], &c, pix);
      }
      world wsel = b->worlds[best];
      if (best != 0) walk(&c, &wsel, b->bl);
      jb->rep.pairs += wsel.nblend;
      const double E = pix_E(wsel.eT);
      if (o->status) o->status[pix] = st;
      if (o->n_contrib) o->n_contrib[pix] = wsel.nc;
      if (o->final_T) o->final_T[pix] = wsel.T;
      if (o->epix) o->epix[pix] = E;
      for (int ch = 0; ch < 3; ++ch) {
        if (o->image) o->image[ch * HW + pix] = wsel.C[ch] + wsel.T * jb->cam->bg[ch];
        if (o->image_mag)
          o->image_mag[ch * HW + pix] = wsel.Cmag[ch] + wsel.T * fabs(jb->cam->bg[ch]);
      }
      if (jb->dL) pixel_backward(jb, &c, b->bl, wsel.nblend, wsel.T, E, dLp, NULL);
    }
  }
}

static void* verify_worker(void* arg) {
  vjob* jb = arg;
  vbuf b;
  memset(&b, 0, sizeof b);
  const int ntiles = jb->s->tiles_x * jb->s->tiles_y;
  for (int tile = jb->tid; tile < ntiles && !jb->failed; tile += jb->nthreads)
    verify_tile(jb, &b, tile);
  vbuf_free(&b);
  return NULL;
}

typedef struct {
  vjob* jobs;
  int njobs;
  gs_verify_out* out;
  size_t lo, hi;
} rjob;

static void* reduce_worker(void* arg) {
  rjob* r = arg;
  for (size_t i = r->lo; i < r->hi; ++i) {
    double g = 0.0, bo = 0.0, ga = 0.0;
    for (int t = 0; t < r->njobs; ++t) {
      g += r->jobs[t].grad[i];
      bo += r->jobs[t].bound[i];
      ga += r->jobs[t].gabs[i];
    }
    if (r->out->grad) r->out->grad[i] = g;
    if (r->out->grad_bound) r->out->grad_bound[i] = bo;
    if (r->out->grad_abs) r->out->grad_abs[i] = ga;
    if (r->out->npix && i % GS_NPARAM == 0) {
      int32_t n = 0;
      for (int t = 0; t < r->njobs; ++t) n += r->jobs[t].npix[i / GS_NPARAM];
      r->out->npix[i / GS_NPARAM] = n;
    }
  }
  return NULL;
}

int gs_verify(const gs_state* s, const gs_camera* cam, const float* dL_dpixels,
              const uint32_t* gpu_n_contrib, const float* gpu_final_T, const float* gpu_image,
              double kappa, gs_verify_out* out, gs_verify_report* rep, int threads) {
  if (!s || !cam || !out || !rep) return vfail("null argument");
  if (!s->ranges || !s->values) return vfail("gs_verify before gs_forward_lists / gs_forward");
  if ((gpu_n_contrib != NULL) != (gpu_final_T != NULL) ||
      (gpu_n_contrib != NULL) != (gpu_image != NULL))
    return vfail("gpu_n_contrib, gpu_final_T and gpu_image go together");
  if (!(kappa > 0.0)) return vfail("kappa must be > 0");
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  memset(rep, 0, sizeof *rep);
  out->nflip_rec = 0;
  const size_t P = (size_t)s->P, words = P * GS_NPARAM;
  if (out->grad_slack) memset(out->grad_slack, 0, words * sizeof(double));
  if (out->image_slack)
    memset(out->image_slack, 0, (size_t)s->W * s->H * 3 * sizeof(double));
  vg* g = malloc(sizeof(vg) * (P ? P : 1));
  if (!g) return vfail("out of memory");
  for (size_t i = 0; i < P; ++i)
    if (s->radii[i] > 0) stage_gauss(s, (int)i, &g[i]);
    else memset(&g[i], 0, sizeof(vg)), g[i].dead = 1;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  pthread_t th[64];
  vjob* jobs = calloc((size_t)threads, sizeof(vjob));
  if (!jobs) { free(g); return vfail("out of memory"); }
  int oom = 0;
  for (int t = 0; t < threads; ++t) {
    vjob* jb = &jobs[t];
    jb->s = s;
    jb->cam = cam;
    jb->dL = dL_dpixels;
    jb->gpu_nc = gpu_n_contrib;
    jb->gpu_T = gpu_final_T;
    jb->gpu_img = gpu_image;
    jb->kappa = kappa;
    jb->g = g;
    jb->out = out;
    jb->tid = t;
    jb->nthreads = threads;
    jb->mu = &mu;
    jb->grad = calloc(words ? words : 1, sizeof(double));
    jb->bound = calloc(words ? words : 1, sizeof(double));
    jb->gabs = calloc(words ? words : 1, sizeof(double));
    jb->npix = calloc(P ? P : 1, sizeof(int32_t));
    if (!jb->grad || !jb->bound || !jb->gabs || !jb->npix) oom = 1;
  }
  if (!oom) {
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, verify_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    rjob rj[64];
    for (int t = 0; t < threads; ++t) {
      rj[t] = (rjob){jobs, threads, out, words * (size_t)t / (size_t)threads,
                     words * (size_t)(t + 1) / (size_t)threads};
      /* npix is written at i % 9 == 0: keep chunk borders on Gaussian borders */
      rj[t].lo -= rj[t].lo % GS_NPARAM;
      if (t + 1 < threads) rj[t].hi -= rj[t].hi % GS_NPARAM;
      pthread_create(&th[t], NULL, reduce_worker, &rj[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  }
  int failed = oom;
  for (int t = 0; t < threads; ++t) {
    vjob* jb = &jobs[t];
    failed |= jb->failed;
    rep->pairs += jb->rep.pairs;
    rep->pairs_default += jb->rep.pairs_default;
    rep->amb_alpha += jb->rep.amb_alpha;
    rep->amb_term += jb->rep.amb_term;
    rep->pix_ambiguous += jb->rep.pix_ambiguous;
    rep->pix_flipped += jb->rep.pix_flipped;
    rep->flips += jb->rep.flips;
    rep->pix_unresolved += jb->rep.pix_unresolved;
    rep->pix_nomatch += jb->rep.pix_nomatch;
    rep->pix_world_cap += jb->rep.pix_world_cap;
    if (jb->rep.max_worlds > rep->max_worlds) rep->max_worlds = jb->rep.max_worlds;
    free(jb->grad); free(jb->bound); free(jb->gabs); free(jb->npix);
  }
  rep->nflip_rec = out->nflip_rec;
  free(jobs);
  free(g);
  if (failed) return vfail("out of memory");
  return 0;
}
