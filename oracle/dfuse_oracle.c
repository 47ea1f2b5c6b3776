/*
 * dfuse_oracle.c -- TEST INFRASTRUCTURE ONLY (see dfuse_oracle.h).
 *
 * Plain-C restatement of the reference's per-frame hot path. Every function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj/include/dfuse/). Arithmetic is written in the
 * reference's evaluation order; build with -ffp-contract=off and no -march so
 * that no FMA contraction happens. Single thread,
 * sequential reductions in raster order, exactly like the reference.
 *
 * Pinned: tests/test_oracle_pin.py compares every orc_* against the ref_*
 * build of the reference headers bit for bit; tests/test_oracle_kats.py
 * replays the reference's own KATs (tests/test_semidense.cpp,
 * tests/test_fusion.cpp) against it.
 */
#include "dfuse_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define INF (1.0 / 0.0)

/* ------------------------------------------------------------------------
 * host geometry: geometry.hpp:44-67, semidense.hpp:101-106, with the
 * quaternion arithmetic of include/compat/Eigen/Geometry */
typedef struct {
  double w, x, y, z;
} quat;

static quat q_mul(quat a, quat b) {
  quat r;
  r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
  r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
  r.y = a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z;
  r.z = a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x;
  return r;
}

static quat q_normalized(quat q) {
  const double n = sqrt(((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w);
  if (!(n > 0.0)) return q;
  quat r = {q.w / n, q.x / n, q.y / n, q.z / n};
  return r;
}

static quat q_conj(quat q) {
  quat r = {q.w, -q.x, -q.y, -q.z};
  return r;
}

static void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

/* q * v = v + w*uv + qv x uv, uv = 2 (qv x v) */
static void q_rot(quat q, const double v[3], double o[3]) {
  const double qv[3] = {q.x, q.y, q.z};
  double uv[3], c2[3];
  cross3(qv, v, uv);
  uv[0] = uv[0] + uv[0];
  uv[1] = uv[1] + uv[1];
  uv[2] = uv[2] + uv[2];
  cross3(qv, uv, c2);
  for (int i = 0; i < 3; ++i) o[i] = (v[i] + q.w * uv[i]) + c2[i];
}

typedef struct {
  quat q;
  double t[3];
} pose;

/* Pose::inverse, geometry.hpp:52-55 */
static pose pose_inverse(pose p) {
  pose r;
  r.q = q_conj(p.q);
  double rt[3];
  q_rot(r.q, p.t, rt);
  r.t[0] = -rt[0];
  r.t[1] = -rt[1];
  r.t[2] = -rt[2];
  return r;
}

/* compose, geometry.hpp:65-67 */
static pose pose_compose(pose a, pose b) {
  pose r;
  r.q = q_normalized(q_mul(a.q, b.q));
  double rt[3];
  q_rot(a.q, b.t, rt);
  for (int i = 0; i < 3; ++i) r.t[i] = rt[i] + a.t[i];
  return r;
}

static void q_to_matrix(quat q, double R[9]) {
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  R[0] = 1.0 - (tyy + tzz);
  R[1] = txy - twz;
  R[2] = txz + twy;
  R[3] = txy + twz;
  R[4] = 1.0 - (txx + tzz);
  R[5] = tyz - twx;
  R[6] = txz - twy;
  R[7] = tyz + twx;
  R[8] = 1.0 - (txx + tyy);
}

int orc_make_epipolar_geometry(const double q0[4], const double t0[3], const double q1[4],
                               const double t1[3], const dfuse_intrinsics* K, dfuse_epigeom* out) {
  pose T0 = {{q0[0], q0[1], q0[2], q0[3]}, {t0[0], t0[1], t0[2]}};
  pose T1 = {{q1[0], q1[1], q1[2], q1[3]}, {t1[0], t1[1], t1[2]}};
  const pose T10 = pose_compose(pose_inverse(T1), T0); /* semidense.hpp:103 */
  const pose T01 = pose_compose(pose_inverse(T0), T1); /* semidense.hpp:104 */
  q_to_matrix(T10.q, out->R_10);
  for (int i = 0; i < 3; ++i) {
    out->t_10[i] = T10.t[i];
    out->t_01[i] = T01.t[i];
  }
  out->K = *K;
  return DFUSE_OK;
}

/* ------------------------------------------------------------------------
 * image sampling: image.hpp:23-40 */
static int can_sample(int w, int h, double x, double y) {
  return x >= 0.0 && x <= w - 1.0 && y >= 0.0 && y <= h - 1.0;
}

static double sample_unchecked(const float* img, int w, double x, double y) {
  const int x0 = (int)floor(x);
  const int y0 = (int)floor(y);
  const double ax = x - x0;
  const double ay = y - y0;
  const int x1 = (ax > 0.0) ? x0 + 1 : x0;
  const int y1 = (ay > 0.0) ? y0 + 1 : y0;
  const double v00 = img[(size_t)y0 * w + x0];
  const double v10 = img[(size_t)y0 * w + x1];
  const double v01 = img[(size_t)y1 * w + x0];
  const double v11 = img[(size_t)y1 * w + x1];
  return (1.0 - ay) * ((1.0 - ax) * v00 + ax * v10) + ay * ((1.0 - ax) * v01 + ax * v11);
}

/* texture_mask, semidense.hpp:77-91. The subtraction is float (C++ float -
 * float), the 0.5 product double. */
int orc_texture_mask(const float* img, int w, int h, double threshold, uint8_t* mask) {
  if (threshold <= 0.0) return DFUSE_E_INVALID_ARGUMENT;
  if (w <= 0 || h <= 0) return DFUSE_E_INVALID_ARGUMENT;
  memset(mask, 0, (size_t)w * h);
  const double t2 = threshold * threshold;
  for (int y = 1; y < h - 1; ++y)
    for (int x = 1; x < w - 1; ++x) {
      const float dx = img[(size_t)y * w + x + 1] - img[(size_t)y * w + x - 1];
      const float dy = img[(size_t)(y + 1) * w + x] - img[(size_t)(y - 1) * w + x];
      const double gx = 0.5 * (double)dx;
      const double gy = 0.5 * (double)dy;
      if (gx * gx + gy * gy > t2) mask[(size_t)y * w + x] = 1;
    }
  return DFUSE_OK;
}

/* ------------------------------------------------------------------------
 * glibc hypot (the function std::hypot resolves to in the reference build,
 * semidense.hpp:312): Borges' corrected hypot without FMA, as in glibc >= 2.35
 * sysdeps/ieee754/dbl-64/e_hypot.c (non-FMA kernel). Verified equal to this
 * image's libm hypot on 2e7 random pairs (tests/test_oracle_pin.py repeats a
 * smaller check). */
static double hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

double orc_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return INF;
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay / 0x1p-54) return ax + ay;
    return hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
  }
  if (ay <= ax * 0x1p-54) return ax + ay;
  return hypot_kernel(ax, ay);
}

/* ------------------------------------------------------------------------
 * epipolar search: semidense.hpp:108-379 */
typedef struct {
  double rays[5][3];
  double ref_intensity[5];
} stencil5;

/* R_10 * v, shim order ((r0 v0 + r1 v1) + r2 v2) */
static void mat3_vec(const double R[9], const double v[3], double o[3]) {
  for (int i = 0; i < 3; ++i) o[i] = (R[3 * i] * v[0] + R[3 * i + 1] * v[1]) + R[3 * i + 2] * v[2];
}

/* make_stencil, semidense.hpp:126-139 */
static int make_stencil(const dfuse_epigeom* g, const float* I0, double x, double y, double dx,
                        double dy, stencil5* s) {
  const int w = g->K.width, h = g->K.height;
  for (int j = 0; j < 5; ++j) {
    const double off = (double)(j - 2);
    const double px = x + off * dx;
    const double py = y + off * dy;
    if (!can_sample(w, h, px, py)) return 0;
    s->ref_intensity[j] = sample_unchecked(I0, w, px, py);
    const double ray[3] = {(px - g->K.cx) / g->K.fx, (py - g->K.cy) / g->K.fy, 1.0};
    mat3_vec(g->R_10, ray, s->rays[j]);
  }
  return 1;
}

enum { STEP_OK = 0, STEP_BEHIND = 1, STEP_OOB = 2 };

/* stencil_error, semidense.hpp:144-155 */
static int stencil_error(const dfuse_epigeom* g, const float* I1, const stencil5* s, double d,
                         double e[5]) {
  const int w = g->K.width, h = g->K.height;
  for (int j = 0; j < 5; ++j) {
    const double p0 = d * s->rays[j][0] + g->t_10[0];
    const double p1 = d * s->rays[j][1] + g->t_10[1];
    const double p2 = d * s->rays[j][2] + g->t_10[2];
    if (p2 <= 0.0) return STEP_BEHIND;
    const double u = g->K.fx * p0 / p2 + g->K.cx;
    const double v = g->K.fy * p1 / p2 + g->K.cy;
    if (!can_sample(w, h, u, v)) return STEP_OOB;
    e[j] = sample_unchecked(I1, w, u, v) - s->ref_intensity[j];
  }
  return STEP_OK;
}

/* project_center, semidense.hpp:158-164 */
static int project_center(const dfuse_epigeom* g, const double a[3], double d, double* ux,
                          double* uy) {
  const double p0 = d * a[0] + g->t_10[0];
  const double p1 = d * a[1] + g->t_10[1];
  const double p2 = d * a[2] + g->t_10[2];
  if (p2 <= 0.0) return 0;
  *ux = g->K.fx * p0 / p2 + g->K.cx;
  *uy = g->K.fy * p1 / p2 + g->K.cy;
  return 1;
}

/* depth_from_position, semidense.hpp:168-183 */
static int depth_from_position(const dfuse_epigeom* g, const double a[3], double ux, double uy,
                               double lx, double ly, double* d) {
  double num, den;
  if (fabs(lx) >= fabs(ly)) {
    const double alpha = ux - g->K.cx;
    num = g->K.fx * g->t_10[0] - alpha * g->t_10[2];
    den = alpha * a[2] - g->K.fx * a[0];
  } else {
    const double beta = uy - g->K.cy;
    num = g->K.fy * g->t_10[1] - beta * g->t_10[2];
    den = beta * a[2] - g->K.fy * a[1];
  }
  if (fabs(den) < 1e-15) return 0;
  *d = num / den;
  return isfinite(*d) && *d > 0.0;
}

/* clip_segment (Liang-Barsky), semidense.hpp:187-209 */
static int clip_segment(double p0x, double p0y, double p1x, double p1y, double xmin, double xmax,
                        double ymin, double ymax, double* t0, double* t1) {
  *t0 = 0.0;
  *t1 = 1.0;
  const double dx = p1x - p0x, dy = p1y - p0y;
  const double p[4] = {-dx, dx, -dy, dy};
  const double q[4] = {p0x - xmin, xmax - p0x, p0y - ymin, ymax - p0y};
  for (int i = 0; i < 4; ++i) {
    if (p[i] == 0.0) {
      if (q[i] < 0.0) return 0;
    } else {
      const double r = q[i] / p[i];
      if (p[i] < 0.0) {
        if (r > *t1) return 0;
        if (r > *t0) *t0 = r;
      } else {
        if (r < *t0) return 0;
        if (r < *t1) *t1 = r;
      }
    }
  }
  return 1;
}

/* search_depth, semidense.hpp:277-379. *best / *nsteps report the internal
 * SSD argmin and step count (-1 where the search did not get there). */
static int search_one(const dfuse_epigeom* g, const float* I0, const float* I1, double x, double y,
                      int has_prior, double pdepth, double psigma, const dfuse_search_cfg* cfg,
                      dfuse_obs* obs, int* best_out, int* nsteps_out) {
  *best_out = -1;
  *nsteps_out = -1;
  /* g.t_10.norm() < 1e-12, semidense.hpp:287 */
  const double tn = sqrt((g->t_10[0] * g->t_10[0] + g->t_10[1] * g->t_10[1]) +
                         g->t_10[2] * g->t_10[2]);
  if (tn < 1e-12) return DFUSE_EPI_DEGENERATE_BASELINE;

  /* epipolar_dir_in_keyframe, semidense.hpp:113-116 */
  double dx = g->K.fx * g->t_01[0] + (g->K.cx - x) * g->t_01[2];
  double dy = g->K.fy * g->t_01[1] + (g->K.cy - y) * g->t_01[2];
  const double dn = sqrt(dx * dx + dy * dy);
  if (dn < 1e-9) return DFUSE_EPI_DEGENERATE_BASELINE;
  dx = dx / dn;
  dy = dy / dn;

  stencil5 s;
  if (!make_stencil(g, I0, x, y, dx, dy, &s)) return DFUSE_EPI_OUT_OF_BOUNDS;
  const double* a = s.rays[2]; /* center_ray, semidense.hpp:137 */

  double d_lo, d_hi; /* semidense.hpp:297-305 */
  if (has_prior) {
    d_lo = pdepth - 2.0 * psigma;
    if (d_lo < 1e-4) d_lo = 1e-4; /* std::max(x, 1e-4) returns x unless 1e-4 > x */
    d_hi = pdepth + 2.0 * psigma;
  } else {
    d_lo = cfg->min_depth;
    d_hi = cfg->max_depth;
  }
  if (!(d_hi > d_lo)) return DFUSE_EPI_NO_MINIMUM;

  double ulx, uly, uhx, uhy;
  if (!project_center(g, a, d_lo, &ulx, &uly) || !project_center(g, a, d_hi, &uhx, &uhy))
    return DFUSE_EPI_BEHIND_CAMERA;

  const double seg_len = orc_hypot(uhx - ulx, uhy - uly);
  if (seg_len < 2.0) return DFUSE_EPI_DEGENERATE_BASELINE;

  double t0, t1;
  if (!clip_segment(ulx, uly, uhx, uhy, 1.0, g->K.width - 2.0, 1.0, g->K.height - 2.0, &t0, &t1))
    return DFUSE_EPI_OUT_OF_BOUNDS;
  const double s_begin = t0 * seg_len;
  const double s_end = t1 * seg_len;
  if (s_end - s_begin < 2.0) return DFUSE_EPI_OUT_OF_BOUNDS;

  const double e1x = (uhx - ulx) / seg_len, e1y = (uhy - uly) / seg_len;
  const int n_steps = (int)floor(s_end - s_begin) + 1;
  *nsteps_out = n_steps;

  double* ssd = (double*)calloc((size_t)n_steps, sizeof(double));
  double* depths = (double*)calloc((size_t)n_steps, sizeof(double));
  unsigned char* ok = (unsigned char*)calloc((size_t)n_steps, 1);
  double e[5];
  for (int k = 0; k < n_steps; ++k) { /* semidense.hpp:328-339 */
    const double sk = s_begin + k;
    const double ukx = ulx + sk * e1x, uky = uly + sk * e1y;
    double dk;
    if (!depth_from_position(g, a, ukx, uky, e1x, e1y, &dk)) continue;
    if (stencil_error(g, I1, &s, dk, e) != STEP_OK) continue;
    double sum = 0.0;
    for (int j = 0; j < 5; ++j) sum += e[j] * e[j];
    ssd[k] = sum;
    depths[k] = dk;
    ok[k] = 1;
  }

  int best = -1; /* semidense.hpp:344-351 */
  double best_ssd = INF;
  for (int k = 0; k < n_steps; ++k)
    if (ok[k] && ssd[k] < best_ssd) {
      best = k;
      best_ssd = ssd[k];
    }
  *best_out = best;
  int status = DFUSE_EPI_OK;
  if (best <= 0 || best + 1 >= n_steps || !ok[best - 1] || !ok[best + 1]) {
    status = DFUSE_EPI_NO_MINIMUM;
    goto done;
  }
  if (sqrt(best_ssd / 5.0) > cfg->max_rms_error) {
    status = DFUSE_EPI_NO_MINIMUM;
    goto done;
  }
  {
    const double denom = ssd[best - 1] - 2.0 * ssd[best] + ssd[best + 1];
    if (denom <= 0.0) {
      status = DFUSE_EPI_NO_MINIMUM;
      goto done;
    }
    const double offset = 0.5 * (ssd[best - 1] - ssd[best + 1]) / denom;
    const double s_star = s_begin + best + offset;
    const double usx = ulx + s_star * e1x, usy = uly + s_star * e1y;
    double d_star;
    if (!depth_from_position(g, a, usx, usy, e1x, e1y, &d_star)) {
      status = DFUSE_EPI_NO_MINIMUM;
      goto done;
    }
    double e_lo[5], e_hi[5];
    if (stencil_error(g, I1, &s, depths[best - 1], e_lo) != STEP_OK ||
        stencil_error(g, I1, &s, depths[best + 1], e_hi) != STEP_OK) {
      status = DFUSE_EPI_OUT_OF_BOUNDS;
      goto done;
    }
    if (depths[best + 1] == depths[best - 1]) {
      status = DFUSE_EPI_DEGENERATE_JACOBIAN;
      goto done;
    }
    /* jacobian_fd, semidense.hpp:253-261 */
    double J[5];
    const double inv = 1.0 / (depths[best + 1] - depths[best - 1]);
    for (int j = 0; j < 5; ++j) J[j] = (e_hi[j] - e_lo[j]) * inv;
    /* observation_variance, semidense.hpp:267-272 */
    double jtj = 0.0;
    for (int j = 0; j < 5; ++j) jtj += J[j] * J[j];
    const double var = (jtj < 1e-12) ? -1.0 : 1.0 / jtj;
    if (var <= 0.0) {
      status = DFUSE_EPI_DEGENERATE_JACOBIAN;
      goto done;
    }
    stencil_error(g, I1, &s, depths[best], e); /* semidense.hpp:376 */
    obs->x = x;
    obs->y = y;
    obs->depth = d_star;
    for (int j = 0; j < 5; ++j) {
      obs->error5[j] = e[j];
      obs->jacobian[j] = J[j];
    }
    obs->variance = var;
  }
done:
  free(ssd);
  free(depths);
  free(ok);
  return status;
}

int orc_search_depth(const dfuse_epigeom* g, const float* I0, const float* I1, int n,
                     const double* px, const double* prior, const uint8_t* has_prior,
                     const dfuse_search_cfg* cfg, int32_t* status, dfuse_obs* obs, int32_t* best,
                     int32_t* n_steps) {
  for (int i = 0; i < n; ++i) {
    const int hp = prior != NULL && (has_prior == NULL || has_prior[i]);
    int b, ns;
    dfuse_obs o;
    memset(&o, 0, sizeof o);
    status[i] = search_one(g, I0, I1, px[2 * i], px[2 * i + 1], hp, hp ? prior[2 * i] : 0.0,
                           hp ? prior[2 * i + 1] : 0.0, cfg, &o, &b, &ns);
    obs[i] = o;
    if (best) best[i] = b;
    if (n_steps) n_steps[i] = ns;
  }
  return DFUSE_OK;
}

/* update_semidense, semidense.hpp:393-417 (applied in place, after checking
 * every observation lies inside the raster). */
static void fuse_one(double* depth, double* variance, uint8_t* valid, size_t i, double d,
                     double v) {
  if (!valid[i]) {
    depth[i] = d;
    variance[i] = v;
    valid[i] = 1;
    return;
  }
  const double sigma_prior = sqrt(variance[i]);
  if (fabs(d - depth[i]) > 5.0 * sigma_prior) return;
  const double info = 1.0 / variance[i] + 1.0 / v;
  depth[i] = (depth[i] / variance[i] + d / v) / info;
  variance[i] = 1.0 / info;
}

int orc_update_semidense(int w, int h, double* depth, double* variance, uint8_t* valid,
                         int32_t* inlier_count, int n_obs, const dfuse_obs* obs) {
  for (int k = 0; k < n_obs; ++k) {
    const long px = lround(obs[k].x), py = lround(obs[k].y);
    if (!(px >= 0 && px < w && py >= 0 && py < h)) return DFUSE_E_OUT_OF_BOUNDS;
  }
  for (int k = 0; k < n_obs; ++k) {
    const size_t i = (size_t)lround(obs[k].y) * w + (size_t)lround(obs[k].x);
    fuse_one(depth, variance, valid, i, obs[k].depth, obs[k].variance);
  }
  int count = 0;
  for (size_t i = 0; i < (size_t)w * h; ++i) count += valid[i] ? 1 : 0;
  *inlier_count = count;
  return DFUSE_OK;
}

/* stereo_scan (pipeline.hpp:157-190) followed by update_semidense when any
 * observation was made (pipeline.hpp:207-212). */
int orc_stereo_update(const dfuse_epigeom* g, const float* I0, const float* I1,
                      const uint8_t* mask, const dfuse_search_cfg* cfg, double* depth,
                      double* variance, uint8_t* valid, int32_t* inlier_count, int32_t* n_obs,
                      int8_t* status, int32_t* best, int32_t* n_steps, dfuse_obs* obs_out) {
  const int w = g->K.width, h = g->K.height;
  const size_t P = (size_t)w * h;
  dfuse_obs* obs = (dfuse_obs*)malloc(P * sizeof(dfuse_obs));
  int n = 0;
  for (size_t i = 0; i < P; ++i) {
    if (status) status[i] = DFUSE_EPI_NOT_SEARCHED;
    if (best) best[i] = -1;
    if (n_steps) n_steps[i] = -1;
  }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      if (!mask[i]) continue;
      const int hp = valid[i] != 0; /* pipeline.hpp:172-174 */
      const double pd = hp ? depth[i] : 0.0, ps = hp ? sqrt(variance[i]) : 0.0;
      int b, ns;
      dfuse_obs o;
      const int st = search_one(g, I0, I1, (double)x, (double)y, hp, pd, ps, cfg, &o, &b, &ns);
      if (status) status[i] = (int8_t)st;
      if (best) best[i] = b;
      if (n_steps) n_steps[i] = ns;
      if (st == DFUSE_EPI_OK) obs[n++] = o;
    }
  *n_obs = n;
  if (obs_out) memcpy(obs_out, obs, (size_t)n * sizeof(dfuse_obs));
  int rc = DFUSE_OK;
  if (n > 0) rc = orc_update_semidense(w, h, depth, variance, valid, inlier_count, n, obs);
  free(obs);
  return rc;
}

/* ------------------------------------------------------------------------
 * fusion: fusion.hpp:44-454 */
typedef struct {
  int net, grad, scale;
} terms;

static terms terms_for(int mode) { /* fusion.hpp:151-158 */
  terms t = {1, 1, 1};
  if (mode == DFUSE_MODE_NOPAIRWISE) t.grad = 0;
  if (mode == DFUSE_MODE_LSSCALE) {
    t.net = 0;
    t.scale = 0;
  }
  return t;
}

static int bad_mode(int mode) { return mode < 0 || mode > 2; }

/* huber_weight / huber_cost, fusion.hpp:79-90; a delta <= 0 is reported
 * through *err (the reference throws InvalidArgument). */
static double huber_weight(double r, double delta, int* err) {
  if (delta <= 0.0) *err = DFUSE_E_INVALID_ARGUMENT;
  const double a = fabs(r);
  return a <= delta ? 1.0 : delta / a;
}
static double huber_cost(double r, double delta) {
  const double a = fabs(r);
  return a <= delta ? r * r : delta * (2.0 * a - delta);
}
/* semi_log_variance, fusion.hpp:98-100 */
static double semi_log_variance(double variance, double depth) {
  const double v = variance / (depth * depth);
  return v < 1e-4 ? 1e-4 : v; /* std::max(v, 1e-4) */
}

#define PRED(c) (in->pred[c])

int orc_assemble_normal_equations(const dfuse_fusion_inputs* in, const double* ld, double scale,
                                  const dfuse_robust_cfg* cfg, int mode, double* diag,
                                  double* right, double* down, double* b) {
  if (bad_mode(mode)) return DFUSE_E_INVALID_ARGUMENT;
  const terms sel = terms_for(mode);
  const int w = in->width, h = in->height;
  const size_t P = (size_t)w * h;
  for (size_t i = 0; i < P; ++i) diag[i] = right[i] = down[i] = b[i] = 0.0;
  const double ln_s = sel.scale ? log(scale) : 0.0;
  int err = 0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const double l = ld[i];
      if (sel.net) {
        const double r = l - PRED(0)[i];
        const double wi = huber_weight(r, cfg->delta_net, &err) / PRED(1)[i];
        diag[i] += wi;
        b[i] -= wi * r;
      }
      if (in->semi_valid[i]) {
        const double r = l - ln_s - log(in->semi_depth[i]);
        const double R = semi_log_variance(in->semi_variance[i], in->semi_depth[i]);
        const double wi = huber_weight(r, cfg->delta_semi, &err) / R;
        diag[i] += wi;
        b[i] -= wi * r;
      }
      if (sel.grad && x + 1 < w) {
        const double r = ld[i + 1] - l - PRED(2)[i];
        const double wi = huber_weight(r, cfg->delta_grad, &err) / PRED(3)[i];
        diag[i] += wi;
        diag[i + 1] += wi;
        right[i] -= wi;
        b[i] += wi * r;
        b[i + 1] -= wi * r;
      }
      if (sel.grad && y + 1 < h) {
        const double r = ld[i + w] - l - PRED(4)[i];
        const double wi = huber_weight(r, cfg->delta_grad, &err) / PRED(5)[i];
        diag[i] += wi;
        diag[i + w] += wi;
        down[i] -= wi;
        b[i] += wi * r;
        b[i + w] -= wi * r;
      }
    }
  return err;
}

static double cost_at(const dfuse_fusion_inputs* in, const double* ld, double scale,
                      const dfuse_robust_cfg* cfg, terms sel) {
  const int w = in->width, h = in->height;
  const double ln_s = sel.scale ? log(scale) : 0.0;
  double cost = 0.0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const double l = ld[i];
      if (sel.net) cost += huber_cost(l - PRED(0)[i], cfg->delta_net) / PRED(1)[i];
      if (in->semi_valid[i])
        cost += huber_cost(l - ln_s - log(in->semi_depth[i]), cfg->delta_semi) /
                semi_log_variance(in->semi_variance[i], in->semi_depth[i]);
      if (sel.grad && x + 1 < w)
        cost += huber_cost(ld[i + 1] - l - PRED(2)[i], cfg->delta_grad) / PRED(3)[i];
      if (sel.grad && y + 1 < h)
        cost += huber_cost(ld[i + w] - l - PRED(4)[i], cfg->delta_grad) / PRED(5)[i];
    }
  return cost;
}

int orc_total_cost(const dfuse_fusion_inputs* in, const double* ld, double scale,
                   const dfuse_robust_cfg* cfg, int mode, double* cost) {
  if (bad_mode(mode)) return DFUSE_E_INVALID_ARGUMENT;
  *cost = cost_at(in, ld, scale, cfg, terms_for(mode));
  return DFUSE_OK;
}

int orc_cost_gradient(const dfuse_fusion_inputs* in, const double* ld, double scale,
                      const dfuse_robust_cfg* cfg, int mode, double* cost, double* g,
                      double* g_lns) {
  if (bad_mode(mode)) return DFUSE_E_INVALID_ARGUMENT;
  const terms sel = terms_for(mode);
  const int w = in->width, h = in->height;
  const size_t P = (size_t)w * h;
  const double ln_s = sel.scale ? log(scale) : 0.0;
  int err = 0;
  double c = 0.0, gs = 0.0;
  for (size_t i = 0; i < P; ++i) g[i] = 0.0;
#define RHO_PRIME(r, d) (2.0 * huber_weight((r), (d), &err) * (r))
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const double l = ld[i];
      if (sel.net) {
        const double r = l - PRED(0)[i];
        c += huber_cost(r, cfg->delta_net) / PRED(1)[i];
        g[i] += RHO_PRIME(r, cfg->delta_net) / PRED(1)[i];
      }
      if (in->semi_valid[i]) {
        const double R = semi_log_variance(in->semi_variance[i], in->semi_depth[i]);
        const double r = l - ln_s - log(in->semi_depth[i]);
        c += huber_cost(r, cfg->delta_semi) / R;
        const double d = RHO_PRIME(r, cfg->delta_semi) / R;
        g[i] += d;
        if (sel.scale) gs -= d;
      }
      if (sel.grad && x + 1 < w) {
        const double r = ld[i + 1] - l - PRED(2)[i];
        c += huber_cost(r, cfg->delta_grad) / PRED(3)[i];
        const double d = RHO_PRIME(r, cfg->delta_grad) / PRED(3)[i];
        g[i + 1] += d;
        g[i] -= d;
      }
      if (sel.grad && y + 1 < h) {
        const double r = ld[i + w] - l - PRED(4)[i];
        c += huber_cost(r, cfg->delta_grad) / PRED(5)[i];
        const double d = RHO_PRIME(r, cfg->delta_grad) / PRED(5)[i];
        g[i + w] += d;
        g[i] -= d;
      }
    }
#undef RHO_PRIME
  *cost = c;
  *g_lns = gs;
  return err;
}

/* StencilMatrix::apply, fusion.hpp:120-135 */
int orc_stencil_apply(int w, int h, const double* diag, const double* right, const double* down,
                      const double* x, double* y) {
  for (int yy = 0; yy < h; ++yy)
    for (int xx = 0; xx < w; ++xx) {
      const size_t i = (size_t)yy * w + xx;
      double v = diag[i] * x[i];
      if (xx + 1 < w) v += right[i] * x[i + 1];
      if (xx > 0) v += right[i - 1] * x[i - 1];
      if (yy + 1 < h) v += down[i] * x[i + w];
      if (yy > 0) v += down[i - w] * x[i - w];
      y[i] = v;
    }
  return DFUSE_OK;
}

/* solve_depth_step, fusion.hpp:316-368 */
int orc_solve_depth_step(int w, int h, const double* diag, const double* right,
                         const double* down, const double* b, const dfuse_robust_cfg* cfg,
                         double* x, int32_t* iterations) {
  const size_t n = (size_t)w * h;
  int its = 0;
  for (size_t i = 0; i < n; ++i) x[i] = 0.0;
  double bnorm2 = 0.0;
  for (size_t i = 0; i < n; ++i) bnorm2 += b[i] * b[i];
  if (iterations) *iterations = 0;
  if (bnorm2 == 0.0) return DFUSE_OK;
  for (size_t i = 0; i < n; ++i)
    if (!(diag[i] > 0.0)) return DFUSE_E_CG_DIVERGENCE;
  double* r = (double*)malloc(n * sizeof(double));
  double* z = (double*)malloc(n * sizeof(double));
  double* p = (double*)malloc(n * sizeof(double));
  double* q = (double*)malloc(n * sizeof(double));
  int rc = DFUSE_OK;
  memcpy(r, b, n * sizeof(double));
  for (size_t i = 0; i < n; ++i) z[i] = r[i] / diag[i];
  memcpy(p, z, n * sizeof(double));
  double rz = 0.0;
  for (size_t i = 0; i < n; ++i) rz += r[i] * z[i];
  const double tol2 = cfg->cg_tol * cfg->cg_tol * bnorm2;
  double prev = bnorm2;
  int streak = 0;
  for (int it = 0; it < cfg->cg_max_iters; ++it) {
    its = it + 1;
    orc_stencil_apply(w, h, diag, right, down, p, q);
    double pq = 0.0;
    for (size_t i = 0; i < n; ++i) pq += p[i] * q[i];
    if (!(pq > 0.0)) {
      rc = DFUSE_E_CG_DIVERGENCE;
      break;
    }
    const double alpha = rz / pq;
    double rn = 0.0;
    for (size_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
      rn += r[i] * r[i];
    }
    if (rn <= tol2) break;
    if (rn > prev) {
      if (++streak >= 10) {
        rc = DFUSE_E_CG_DIVERGENCE;
        break;
      }
    } else {
      streak = 0;
    }
    prev = rn;
    double rz_new = 0.0;
    for (size_t i = 0; i < n; ++i) {
      z[i] = r[i] / diag[i];
      rz_new += r[i] * z[i];
    }
    const double beta = rz_new / rz;
    rz = rz_new;
    for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  if (iterations) *iterations = its;
  free(r);
  free(z);
  free(p);
  free(q);
  return rc;
}

/* solve_scale_step, fusion.hpp:373-391 */
static int scale_step(const dfuse_fusion_inputs* in, const double* ld, double scale,
                      const dfuse_robust_cfg* cfg, double* out) {
  if (in->inlier_count <= 0) return DFUSE_E_NO_SEMIDENSE_SUPPORT;
  const size_t P = (size_t)in->width * in->height;
  int err = 0;
  double ln_s = log(scale);
  for (int round = 0; round < 3; ++round) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < P; ++i) {
      if (!in->semi_valid[i]) continue;
      const double offset = ld[i] - log(in->semi_depth[i]);
      const double R = semi_log_variance(in->semi_variance[i], in->semi_depth[i]);
      const double wi = huber_weight(offset - ln_s, cfg->delta_semi, &err) / R;
      num += wi * offset;
      den += wi;
    }
    ln_s = num / den;
  }
  *out = exp(ln_s);
  return err;
}

int orc_solve_scale_step(const dfuse_fusion_inputs* in, const double* ld, double scale,
                         const dfuse_robust_cfg* cfg, double* out) {
  return scale_step(in, ld, scale, cfg, out);
}

/* optimize, fusion.hpp:402-454. Transactional like the reference (it works
 * on a copy and returns a new state). */
int orc_optimize(const dfuse_fusion_inputs* in, double* log_depth, double* scale_io,
                 int32_t* iteration, const dfuse_robust_cfg* cfg, int mode,
                 dfuse_solver_stats* stats) {
  if (bad_mode(mode)) return DFUSE_E_INVALID_ARGUMENT;
  const int w = in->width, h = in->height;
  const size_t P = (size_t)w * h;
  const terms sel = terms_for(mode);
  const int ls_mode = mode == DFUSE_MODE_LSSCALE;
  const int depth_solvable = !ls_mode || in->inlier_count > 0;
  double* st = (double*)malloc(P * sizeof(double));
  double* trial = (double*)malloc(P * sizeof(double));
  double* diag = (double*)malloc(P * sizeof(double));
  double* right = (double*)malloc(P * sizeof(double));
  double* down = (double*)malloc(P * sizeof(double));
  double* b = (double*)malloc(P * sizeof(double));
  double* delta = (double*)malloc(P * sizeof(double));
  memcpy(st, log_depth, P * sizeof(double));
  double scale = *scale_io;
  int iter = *iteration;
  int rc = DFUSE_OK;
  if (stats) {
    memset(stats, 0, sizeof *stats);
    for (int k = 0; k < DFUSE_STATS_MAX_GN; ++k) {
      stats->pcg_iters[k] = -1;
      stats->scale_step[k] = -1.0;
      stats->depth_step[k] = -1.0;
    }
  }
  for (int it = 0; it < cfg->gn_iterations; ++it) {
    if (!ls_mode && cfg->estimate_scale && in->inlier_count > 0) { /* fusion.hpp:411-425 */
      double s_new;
      rc = scale_step(in, st, scale, cfg, &s_new);
      if (rc) goto out;
      const double c0 = cost_at(in, st, scale, cfg, sel);
      if (stats) stats->cost_evals++;
      const double dlns = log(s_new) - log(scale);
      double step = 1.0, accepted = 0.0;
      for (int half = 0; half <= 5; ++half) {
        const double ts = exp(log(scale) + step * dlns);
        if (stats) stats->cost_evals++;
        if (cost_at(in, st, ts, cfg, sel) <= c0) {
          scale = ts;
          accepted = step;
          break;
        }
        step *= 0.5;
      }
      if (stats && it < DFUSE_STATS_MAX_GN) stats->scale_step[it] = accepted;
    }
    if (depth_solvable) { /* fusion.hpp:426-441 */
      rc = orc_assemble_normal_equations(in, st, scale, cfg, mode, diag, right, down, b);
      if (rc) goto out;
      int32_t its = 0;
      rc = orc_solve_depth_step(w, h, diag, right, down, b, cfg, delta, &its);
      if (stats) {
        stats->pcg_total += its;
        if (it < DFUSE_STATS_MAX_GN) stats->pcg_iters[it] = its;
      }
      if (rc) goto out;
      const double c0 = cost_at(in, st, scale, cfg, sel);
      if (stats) stats->cost_evals++;
      double step = 1.0, accepted = 0.0;
      for (int half = 0; half <= 5; ++half) {
        for (size_t i = 0; i < P; ++i) trial[i] = st[i] + step * delta[i];
        if (stats) stats->cost_evals++;
        if (cost_at(in, trial, scale, cfg, sel) <= c0) {
          memcpy(st, trial, P * sizeof(double));
          accepted = step;
          break;
        }
        step *= 0.5;
      }
      if (stats && it < DFUSE_STATS_MAX_GN) stats->depth_step[it] = accepted;
    }
    iter += 1;
    if (stats) stats->gn_done = it + 1;
  }
  if (ls_mode) { /* fusion.hpp:445-452 */
    double sum = 0.0;
    for (size_t i = 0; i < P; ++i) sum += PRED(0)[i] - st[i];
    const double offset = sum / (double)P;
    for (size_t i = 0; i < P; ++i) st[i] += offset;
    scale = exp(offset);
  }
  memcpy(log_depth, st, P * sizeof(double));
  *scale_io = scale;
  *iteration = iter;
out:
  free(st);
  free(trial);
  free(diag);
  free(right);
  free(down);
  free(b);
  free(delta);
  return rc;
}

/* ------------------------------------------------------------------------
 * KAT helpers */

/* photometric_error_5pt, semidense.hpp:227-243 */
int orc_photometric_error_5pt(const dfuse_epigeom* g, const float* I0, const float* I1, double x,
                              double y, double d, double e[5]) {
  double dx = g->K.fx * g->t_01[0] + (g->K.cx - x) * g->t_01[2];
  double dy = g->K.fy * g->t_01[1] + (g->K.cy - y) * g->t_01[2];
  const double n = sqrt(dx * dx + dy * dy);
  if (n < 1e-12) {
    dx = 1.0;
    dy = 0.0;
  } else {
    dx = dx / n;
    dy = dy / n;
  }
  stencil5 s;
  if (!make_stencil(g, I0, x, y, dx, dy, &s)) return DFUSE_EPI_OUT_OF_BOUNDS;
  switch (stencil_error(g, I1, &s, d, e)) {
    case STEP_BEHIND: return DFUSE_EPI_BEHIND_CAMERA;
    case STEP_OOB: return DFUSE_EPI_OUT_OF_BOUNDS;
    default: break;
  }
  return DFUSE_EPI_OK;
}

/* jacobian_fd, semidense.hpp:253-261 */
int orc_jacobian_fd(const double e_lo[5], const double e_hi[5], double d_lo, double d_hi,
                    double J[5]) {
  if (d_hi == d_lo) return DFUSE_E_ZERO_BASELINE_STEP;
  const double inv = 1.0 / (d_hi - d_lo);
  for (int j = 0; j < 5; ++j) J[j] = (e_hi[j] - e_lo[j]) * inv;
  return DFUSE_OK;
}

/* observation_variance, semidense.hpp:267-272 */
double orc_observation_variance(const double J[5]) {
  double jtj = 0.0;
  for (int j = 0; j < 5; ++j) jtj += J[j] * J[j];
  if (jtj < 1e-12) return -1.0;
  return 1.0 / jtj;
}

/* huber_weight / huber_cost, fusion.hpp:79-90 */
int orc_huber(double r, double delta, double* weight, double* cost) {
  int err = 0;
  *weight = huber_weight(r, delta, &err);
  *cost = huber_cost(r, delta);
  return err;
}

/* residual_semi, fusion.hpp:51-53 */
double orc_residual_semi(double ln_d, double s, double d_semi) {
  return ln_d - log(s) - log(d_semi);
}

double orc_semi_log_variance(double variance, double depth) {
  return semi_log_variance(variance, depth);
}

/* should_create_keyframe, semidense.hpp:419-424 */
int orc_should_create_keyframe(const double q_kf[4], const double t_kf[3], const double q_cur[4],
                               const double t_cur[3], double median, int inlier_count,
                               double lambda_trans, int lambda_inliers, int* out) {
  if (median <= 0.0) return DFUSE_E_NON_POSITIVE_DEPTH;
  pose a = {{q_kf[0], q_kf[1], q_kf[2], q_kf[3]}, {t_kf[0], t_kf[1], t_kf[2]}};
  pose b = {{q_cur[0], q_cur[1], q_cur[2], q_cur[3]}, {t_cur[0], t_cur[1], t_cur[2]}};
  const pose rel = pose_compose(pose_inverse(a), b);
  const double trans =
      sqrt((rel.t[0] * rel.t[0] + rel.t[1] * rel.t[1]) + rel.t[2] * rel.t[2]);
  *out = trans / median > lambda_trans || inlier_count < lambda_inliers;
  return DFUSE_OK;
}

/* focal_adjust, predictions.hpp:148-157: log_depth += log(test/source)
 * unless the focal lengths are equal */
int orc_focal_adjust(int w, int h, double* log_depth, double source_focal, double test_focal) {
  if (test_focal <= 0.0 || source_focal <= 0.0) return DFUSE_E_NON_POSITIVE_FOCAL;
  if (test_focal == source_focal) return DFUSE_OK;
  const double shift = log(test_focal / source_focal);
  for (long i = 0; i < (long)w * h; ++i) log_depth[i] += shift;
  return DFUSE_OK;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* detail::median_predicted_depth, pipeline.hpp:94-99: exp of the element
 * std::nth_element places at n/2 (= the (n/2)-th smallest) */
double orc_median_predicted_depth(const double* log_depth, long n) {
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(v, log_depth, sizeof(double) * (size_t)n);
  qsort(v, (size_t)n, sizeof(double), cmp_double);
  const double m = v[n / 2];
  free(v);
  return exp(m);
}

/* pct_within_10 (eval.hpp:34-46): 100 * correct / valid-gt, with the
 * boundary-inclusive 0.10 + 1e-12 threshold (eval.hpp:29); NULL est_valid =
 * every estimate defined. Returns NoValidGroundTruth on an empty gt mask. */
int orc_pct_within_10(long n, const double* est, const uint8_t* est_valid, const double* gt,
                      const uint8_t* gt_valid, double* out) {
  long n_gt = 0, n_ok = 0;
  for (long i = 0; i < n; ++i) {
    if (!gt_valid[i]) continue;
    ++n_gt;
    if (est_valid && !est_valid[i]) continue;
    if (fabs(est[i] - gt[i]) / gt[i] <= 0.10 + 1e-12) ++n_ok;
  }
  if (n_gt == 0) return DFUSE_E_NO_VALID_GROUND_TRUTH;
  *out = 100.0 * (double)n_ok / (double)n_gt;
  return DFUSE_OK;
}

/* median_abs_rel (eval.hpp:52-68): the element nth_element puts at n/2 of
 * |est - gt| / gt over pixels where both are defined; 0 when there are none */
double orc_median_abs_rel(long n, const double* est, const uint8_t* est_valid, const double* gt,
                          const uint8_t* gt_valid) {
  double* r = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  long m = 0;
  for (long i = 0; i < n; ++i) {
    if (!gt_valid[i]) continue;
    if (est_valid && !est_valid[i]) continue;
    r[m++] = fabs(est[i] - gt[i]) / gt[i];
  }
  double out = 0.0;
  if (m > 0) {
    qsort(r, (size_t)m, sizeof(double), cmp_double);
    out = r[m / 2];
  }
  free(r);
  return out;
}

/* export_depth_image (eval.hpp:221-226) through save_depth_png's
 * quantisation (depth_io.hpp:61-62): round(exp(ld) * scale) clamped to
 * [0, 65535] */
void orc_export_depth_u16(long n, const double* log_depth, double depth_scale, uint16_t* out) {
  for (long i = 0; i < n; ++i) {
    double s = round(exp(log_depth[i]) * depth_scale);
    s = s < 0.0 ? 0.0 : (s > 65535.0 ? 65535.0 : s);
    out[i] = (uint16_t)s;
  }
}
