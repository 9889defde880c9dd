/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference
 * voxmap per-frame path in Sequential mode (see voxmap_oracle.h for how it is
 * pinned). Built with -ffp-contract=off like the reference
 * (proj/src/CMakeLists.txt:33-35). Paths are relative to /root/reference.
 *
 * Eigen-dependent operation orders follow the in-repo
 * Eigen subset: Matrix3d*Vector3d rows are left-to-right dot products,
 * squaredNorm of a 3-vector is (d0^2 + d1^2) + d2^2.
 */
#include "voxmap_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PI_ 3.14159265358979323846

static size_t cells_of(const int32_t d[3]) {
  return (size_t)d[0] * (size_t)d[1] * (size_t)d[2];
}

/* proj/src/kernels/kernels_scalar.cpp:10-16 */
void vo_merge(uint8_t* local, const uint8_t* ms, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const uint8_t m = ms[i];
    if (m == 0) continue;
    local[i] = (m == 3) ? 0 : m;
  }
}

/* proj/src/kernels/kernels_scalar.cpp:25-35: t + R p, floor(/vs), clamp, int32.
 * x86 truncation of NaN yields INT32_MIN (cvttsd2si). */
static int32_t vox_axis(double acc, double vs) {
  double f = floor(acc / vs);
  f = f < -1e9 ? -1e9 : f;  /* std::max(f, -1e9) */
  f = 1e9 < f ? 1e9 : f;    /* std::min(f, 1e9) */
  if (f != f) return INT32_MIN;
  return (int32_t)f;
}

void vo_transform_voxelize(const double* xs, const double* ys, const double* zs, size_t n,
                           const double* R, const double* t, double vs, int32_t* cx,
                           int32_t* cy, int32_t* cz) {
  int32_t* out[3] = {cx, cy, cz};
  for (size_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      double acc = t[a];
      acc += R[3 * a + 0] * xs[i];
      acc += R[3 * a + 1] * ys[i];
      acc += R[3 * a + 2] * zs[i];
      out[a][i] = vox_axis(acc, vs);
    }
  }
}

/* CameraModel::validate (proj/src/geometry.cpp:28-41) */
static int camera_ok(const vxm_camera* c) {
  if (c->width <= 0 || c->height <= 0) return 0;
  if (!(c->fov_x > 0.0) || !(c->fov_x < PI_) || !(c->fov_y > 0.0) || !(c->fov_y < PI_)) return 0;
  if (!(c->max_depth > 0.0) || !isfinite(c->max_depth)) return 0;
  return 1;
}

/* back_project_rows (proj/src/geometry.cpp:43-61), whole image */
long long vo_depth_to_cloud(const vxm_camera* cam, const float* depth, double* xs, double* ys,
                            double* zs) {
  if (!camera_ok(cam)) return -1;
  const double fx = (cam->width / 2.0) / tan(cam->fov_x / 2.0);
  const double fy = (cam->height / 2.0) / tan(cam->fov_y / 2.0);
  const double cx = cam->width / 2.0, cy = cam->height / 2.0;
  long long n = 0;
  for (int v = 0; v < cam->height; ++v) {
    for (int u = 0; u < cam->width; ++u) {
      const float d = depth[(size_t)v * cam->width + u];
      if (!(isfinite(d) && d > 0.0f)) continue; /* DepthImage::valid_depth */
      const double D = (double)d;
      if (D > cam->max_depth) continue;
      xs[n] = (u + 0.5 - cx) / fx * D;
      ys[n] = (v + 0.5 - cy) / fy * D;
      zs[n] = D;
      ++n;
    }
  }
  return n;
}

/* populate_occupied (proj/src/integrator.cpp:45-103), Sequential */
int vo_populate(const vxm_grid_spec* g, uint8_t* ms, const double* xs, const double* ys,
                const double* zs, size_t n, const vxm_pose* t_vc, int vox_inf,
                vxm_populate_stats* st) {
  if (vox_inf < 0) return -1;
  const int r = vox_inf, dx = g->dims[0], dy = g->dims[1], dz = g->dims[2];
  uint64_t outside = 0, total = 0;
  for (size_t i = 0; i < n; ++i) {
    /* PointCloud::add drops non-finite points (geometry.hpp:84-89) */
    if (!isfinite(xs[i]) || !isfinite(ys[i]) || !isfinite(zs[i])) continue;
    ++total;
    int32_t c[3];
    vo_transform_voxelize(xs + i, ys + i, zs + i, 1, t_vc->rotation, t_vc->translation,
                          g->vox_size, &c[0], &c[1], &c[2]);
    if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[0] >= dx || c[1] >= dy || c[2] >= dz) {
      ++outside;
      continue;
    }
    const int x0 = c[0] - r < 0 ? 0 : c[0] - r, x1 = c[0] + r > dx - 1 ? dx - 1 : c[0] + r;
    const int y0 = c[1] - r < 0 ? 0 : c[1] - r, y1 = c[1] + r > dy - 1 ? dy - 1 : c[1] + r;
    const int z0 = c[2] - r < 0 ? 0 : c[2] - r, z1 = c[2] + r > dz - 1 ? dz - 1 : c[2] + r;
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) ms[(size_t)x + (size_t)y * dx + (size_t)z * dx * dy] = 2;
  }
  if (st) {
    st->points_total = total;
    st->points_outside = outside;
  }
  return 0;
}

/* bundle_dimensions (proj/src/raytracer.cpp:8-21) */
int vo_bundle_dimensions(const vxm_camera* cam, double depth, double vs, int32_t out[3]) {
  if (!camera_ok(cam) || !(depth > 0.0) || !isfinite(depth) || !(vs > 0.0) || !isfinite(vs)) return -1;
  long vd = lround(depth / vs);
  out[0] = vd < 1 ? 1 : (int32_t)vd;
  out[1] = 2 * (int32_t)lround(tan(cam->fov_x / 2.0) * out[0]) + 1;
  out[2] = 2 * (int32_t)lround(tan(cam->fov_y / 2.0) * out[0]) + 1;
  return 0;
}

/* walk_ray (proj/include/voxmap/raytracer.hpp:76-118) + traverse_ray
 * (proj/src/raytracer.cpp:63-96) for one ray, writing into ms. */
static void traverse(const vxm_grid_spec* g, uint8_t* ms, const double start[3],
                     const double dir_in[3], double max_dist, vxm_trace_stats* st) {
  const double vs = g->vox_size;
  const int dx = g->dims[0], dy = g->dims[1], dz = g->dims[2];
  const double n2 = (dir_in[0] * dir_in[0] + dir_in[1] * dir_in[1]) + dir_in[2] * dir_in[2];
  double dir[3];
  for (int a = 0; a < 3; ++a) dir[a] = n2 > 0.0 ? dir_in[a] / sqrt(n2) : dir_in[a];
  int cur[3], step[3];
  double tmax[3], tdelta[3];
  for (int a = 0; a < 3; ++a) {
    cur[a] = (int)floor(start[a] / vs);
    if (dir[a] > 0.0) {
      step[a] = 1;
      tmax[a] = ((cur[a] + 1) * vs - start[a]) / dir[a];
      tdelta[a] = vs / dir[a];
    } else if (dir[a] < 0.0) {
      step[a] = -1;
      tmax[a] = (cur[a] * vs - start[a]) / dir[a];
      tdelta[a] = vs / -dir[a];
    } else {
      step[a] = 0;
      tmax[a] = INFINITY;
      tdelta[a] = INFINITY;
    }
  }
  st->rays_traced += 1;
  uint8_t val = 1;
  int entered = 0;
  for (;;) {
    /* visit(cur) */
    if (cur[0] < 0 || cur[1] < 0 || cur[2] < 0 || cur[0] >= dx || cur[1] >= dy || cur[2] >= dz) {
      if (entered) return;
      st->voxels_skipped_out_of_bounds += 1;
    } else {
      entered = 1;
      uint8_t* cell = ms + (size_t)cur[0] + (size_t)cur[1] * dx + (size_t)cur[2] * dx * dy;
      if (*cell == 2) {
        val = 3;
      } else {
        *cell = val;
        if (val == 1) st->voxels_freed += 1;
        else st->voxels_marked_unknown_traced += 1;
      }
    }
    int axis;
    if (tmax[0] <= tmax[1] && tmax[0] <= tmax[2]) axis = 0;
    else if (tmax[1] <= tmax[2]) axis = 1;
    else axis = 2;
    if (tmax[axis] >= max_dist - 1e-10) return;
    cur[axis] += step[axis];
    tmax[axis] += tdelta[axis];
  }
}

/* trace_bundle (proj/src/raytracer.cpp:35-61, 98-105), Sequential */
int vo_trace_bundle(const vxm_grid_spec* g, uint8_t* ms, const int32_t b[3],
                    const vxm_pose* t_vc, vxm_trace_stats* st) {
  if (b[0] < 1 || b[1] < 1 || b[2] < 1 || b[1] % 2 == 0 || b[2] % 2 == 0) return -1;
  const double vs = g->vox_size;
  const double* R = t_vc->rotation;
  const int hw = (b[1] - 1) / 2, hh = (b[2] - 1) / 2;
  memset(st, 0, sizeof(*st));
  for (int yi = -hh; yi <= hh; ++yi) {
    for (int xi = -hw; xi <= hw; ++xi) {
      const double v[3] = {xi * vs, yi * vs, b[0] * vs};
      double dir[3];
      for (int a = 0; a < 3; ++a) dir[a] = (R[3 * a] * v[0] + R[3 * a + 1] * v[1]) + R[3 * a + 2] * v[2];
      const double max_dist =
          vs * sqrt((double)xi * xi + (double)yi * yi + (double)b[0] * b[0]);
      /* validate_ray (raytracer.cpp:23-33) */
      if (!isfinite(dir[0]) || !isfinite(dir[1]) || !isfinite(dir[2]) || !isfinite(max_dist)) return -1;
      if (dir[0] == 0.0 && dir[1] == 0.0 && dir[2] == 0.0) return -1;
      if (!(max_dist > 0.0)) return -1;
      traverse(g, ms, t_vc->translation, dir, max_dist, st);
    }
  }
  return 0;
}

/* bresenham_line (raytracer.hpp:136-194) + bresenham_trace_image
 * (raytracer.cpp:120-161), Sequential. */
static void visit_pp(const vxm_grid_spec* g, uint8_t* ms, const int c[3], const int end[3],
                     vxm_trace_stats* st) {
  if (c[0] == end[0] && c[1] == end[1] && c[2] == end[2]) return;
  const int dx = g->dims[0], dy = g->dims[1], dz = g->dims[2];
  if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[0] >= dx || c[1] >= dy || c[2] >= dz) {
    st->voxels_skipped_out_of_bounds += 1;
    return;
  }
  uint8_t* cell = ms + (size_t)c[0] + (size_t)c[1] * dx + (size_t)c[2] * dx * dy;
  if (*cell != 2) {
    *cell = 1;
    st->voxels_freed += 1;
  }
}

static void bresenham(const vxm_grid_spec* g, uint8_t* ms, const int from[3], const int to[3],
                      vxm_trace_stats* st) {
  int p[3] = {from[0], from[1], from[2]};
  int d[3], s[3];
  for (int a = 0; a < 3; ++a) {
    d[a] = abs(to[a] - p[a]);
    s[a] = to[a] > p[a] ? 1 : -1;
  }
  int drive, o1, o2;
  if (d[0] >= d[1] && d[0] >= d[2]) { drive = 0; o1 = 1; o2 = 2; }
  else if (d[1] >= d[0] && d[1] >= d[2]) { drive = 1; o1 = 0; o2 = 2; }
  else { drive = 2; o1 = 1; o2 = 0; }
  int p1 = 2 * d[o1] - d[drive], p2 = 2 * d[o2] - d[drive];
  while (p[drive] != to[drive]) {
    visit_pp(g, ms, p, to, st);
    if (p1 >= 0) { p[o1] += s[o1]; p1 -= 2 * d[drive]; }
    if (p2 >= 0) { p[o2] += s[o2]; p2 -= 2 * d[drive]; }
    p1 += 2 * d[o1];
    p2 += 2 * d[o2];
    p[drive] += s[drive];
  }
  visit_pp(g, ms, to, to, st);
}

int vo_trace_per_pixel(const vxm_grid_spec* g, uint8_t* ms, const double* xs, const double* ys,
                       const double* zs, size_t n, const vxm_pose* t_vc, vxm_trace_stats* st) {
  const double vs = g->vox_size;
  const double* R = t_vc->rotation;
  const double* t = t_vc->translation;
  memset(st, 0, sizeof(*st));
  if (!isfinite(t[0]) || !isfinite(t[1]) || !isfinite(t[2])) return -1;
  /* world_to_voxel(t_vc.translation) (grid.cpp:54-62) */
  const int cam[3] = {(int)floor(t[0] / vs), (int)floor(t[1] / vs), (int)floor(t[2] / vs)};
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(xs[i]) || !isfinite(ys[i]) || !isfinite(zs[i])) continue;
    /* RigidTransform::apply: (R p) + t, rows left to right */
    double w[3];
    for (int a = 0; a < 3; ++a) w[a] = ((R[3 * a] * xs[i] + R[3 * a + 1] * ys[i]) + R[3 * a + 2] * zs[i]) + t[a];
    const int end[3] = {(int)floor(w[0] / vs), (int)floor(w[1] / vs), (int)floor(w[2] / vs)};
    st->rays_traced += 1;
    bresenham(g, ms, cam, end, st);
  }
  return 0;
}

/* shift_grid_by (proj/src/grid.cpp:81-108) */
void vo_shift(const int32_t dims[3], const uint8_t* in, uint8_t* out, const int32_t off[3]) {
  const int dx = dims[0], dy = dims[1], dz = dims[2];
  memset(out, 0, cells_of(dims));
  for (int z = 0; z < dz; ++z)
    for (int y = 0; y < dy; ++y)
      for (int x = 0; x < dx; ++x) {
        const int sx = x + off[0], sy = y + off[1], sz = z + off[2];
        if (sx < 0 || sy < 0 || sz < 0 || sx >= dx || sy >= dy || sz >= dz) continue;
        out[(size_t)x + (size_t)y * dx + (size_t)z * dx * dy] =
            in[(size_t)sx + (size_t)sy * dx + (size_t)sz * dx * dy];
      }
}

/* ------------------------------------------------------------------ pipeline */

struct vo_pipeline {
  vxm_config cfg;
  double origin[3];
  uint8_t* local;
  uint8_t* ms;
  uint8_t* tmp;
  double *xs, *ys, *zs;
  size_t cap;
};

/* PipelineConfig::validate (pipeline.cpp:33-42) */
vo_pipeline* vo_pipeline_create(const vxm_config* cfg) {
  if (!camera_ok(&cfg->camera) || cfg->vox_inf < 0) return NULL;
  if (!(cfg->depth > 0.0) || cfg->depth > cfg->camera.max_depth) return NULL;
  const size_t n = cells_of(cfg->grid.dims);
  if (n == 0) return NULL;
  vo_pipeline* p = (vo_pipeline*)calloc(1, sizeof(vo_pipeline));
  p->cfg = *cfg;
  memcpy(p->origin, cfg->grid.origin, sizeof(p->origin));
  p->local = (uint8_t*)calloc(n, 1);
  p->ms = (uint8_t*)calloc(n, 1);
  p->tmp = (uint8_t*)calloc(n, 1);
  return p;
}

void vo_pipeline_destroy(vo_pipeline* p) {
  if (!p) return;
  free(p->local);
  free(p->ms);
  free(p->tmp);
  free(p->xs);
  free(p->ys);
  free(p->zs);
  free(p);
}

/* RigidTransform::is_valid(1e-6) (geometry.cpp:17-22), Eigen-subset order */
static int pose_valid(const vxm_pose* q, double tol) {
  for (int i = 0; i < 9; ++i) if (!isfinite(q->rotation[i])) return 0;
  for (int i = 0; i < 3; ++i) if (!isfinite(q->translation[i])) return 0;
#define RR(i, j) q->rotation[3 * (i) + (j)]
  double worst = 0.0;
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      double acc = RR(0, i) * RR(0, j);
      acc = acc + RR(1, i) * RR(1, j);
      acc = acc + RR(2, i) * RR(2, j);
      double d = fabs(acc - (i == j ? 1.0 : 0.0));
      if ((i == 0 && j == 0) || d > worst) worst = d;
    }
  if (worst > tol) return 0;
  const double det = RR(0, 0) * (RR(1, 1) * RR(2, 2) - RR(2, 1) * RR(1, 2)) -
                     RR(1, 0) * (RR(0, 1) * RR(2, 2) - RR(2, 1) * RR(0, 2)) +
                     RR(2, 0) * (RR(0, 1) * RR(1, 2) - RR(1, 1) * RR(0, 2));
#undef RR
  return fabs(det - 1.0) <= tol;
}

/* MappingPipeline::integrate (pipeline.cpp:74-117) */
int vo_pipeline_integrate_cloud(vo_pipeline* p, const double* xs, const double* ys,
                                const double* zs, size_t n, const vxm_pose* t_wc, vxm_stats* st) {
  if (!pose_valid(t_wc, 1e-6)) return -1;
  const vxm_grid_spec* g0 = &p->cfg.grid;
  const size_t N = cells_of(g0->dims);
  const double vs = g0->vox_size;
  memset(st, 0, sizeof(*st));
  memset(p->ms, 0, N);
  vxm_grid_spec g = *g0;
  memcpy(g.origin, p->origin, sizeof(g.origin));
  /* camera_to_grid_transform = compose(T(-origin), t_wc) (pipeline.cpp:63-66) */
  vxm_pose t_vc;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) {
      double acc = (i == 0 ? 1.0 : 0.0) * t_wc->rotation[j];
      acc = acc + (i == 1 ? 1.0 : 0.0) * t_wc->rotation[3 + j];
      acc = acc + (i == 2 ? 1.0 : 0.0) * t_wc->rotation[6 + j];
      t_vc.rotation[3 * i + j] = acc;
    }
    double acc = (i == 0 ? 1.0 : 0.0) * t_wc->translation[0];
    acc = acc + (i == 1 ? 1.0 : 0.0) * t_wc->translation[1];
    acc = acc + (i == 2 ? 1.0 : 0.0) * t_wc->translation[2];
    t_vc.translation[i] = acc + (-p->origin[i]);
  }
  vxm_populate_stats ps;
  vo_populate(&g, p->ms, xs, ys, zs, n, &t_vc, p->cfg.vox_inf, &ps);
  st->points_total = ps.points_total;
  st->points_outside = ps.points_outside;
  vxm_trace_stats ts;
  if (p->cfg.tracer_mode == VXM_TRACER_BUNDLED) {
    int32_t b[3];
    vo_bundle_dimensions(&p->cfg.camera, p->cfg.depth, vs, b);
    vo_trace_bundle(&g, p->ms, b, &t_vc, &ts);
  } else {
    vo_trace_per_pixel(&g, p->ms, xs, ys, zs, n, &t_vc, &ts);
  }
  st->rays_traced = ts.rays_traced;
  st->voxels_freed = ts.voxels_freed;
  st->voxels_marked_unknown_traced = ts.voxels_marked_unknown_traced;
  st->voxels_skipped_out_of_bounds = ts.voxels_skipped_out_of_bounds;
  vo_merge(p->local, p->ms, N);
  /* recentring (pipeline.cpp:102-112; grid.cpp:110-117) */
  int drift = 0;
  double half[3];
  for (int a = 0; a < 3; ++a) {
    half[a] = (double)(g0->dims[a] / 2) * vs;
    if (fabs(t_wc->translation[a] - (p->origin[a] + half[a])) >= vs) drift = 1;
  }
  if (drift) {
    int32_t off[3];
    for (int a = 0; a < 3; ++a) off[a] = (int32_t)lround(((t_wc->translation[a] - half[a]) - p->origin[a]) / vs);
    if (off[0] || off[1] || off[2]) {
      vo_shift(g0->dims, p->local, p->tmp, off);
      uint8_t* t = p->local;
      p->local = p->tmp;
      p->tmp = t;
      for (int a = 0; a < 3; ++a) {
        p->origin[a] = p->origin[a] + (double)off[a] * vs;
        st->shift_offset[a] = off[a];
      }
      st->shifted = 1;
    }
  }
  for (size_t i = 0; i < N; ++i) {
    st->occupied_count += p->local[i] == 2;
    st->freed_count += p->local[i] == 1;
  }
  memcpy(st->origin, p->origin, sizeof(st->origin));
  return 0;
}

int vo_pipeline_integrate_depth(vo_pipeline* p, const float* depth, const vxm_pose* t_wc,
                                vxm_stats* st) {
  const size_t npix = (size_t)p->cfg.camera.width * p->cfg.camera.height;
  if (p->cap < npix) {
    free(p->xs);
    free(p->ys);
    free(p->zs);
    p->xs = (double*)malloc(sizeof(double) * npix);
    p->ys = (double*)malloc(sizeof(double) * npix);
    p->zs = (double*)malloc(sizeof(double) * npix);
    p->cap = npix;
  }
  const long long n = vo_depth_to_cloud(&p->cfg.camera, depth, p->xs, p->ys, p->zs);
  if (n < 0) return -1;
  return vo_pipeline_integrate_cloud(p, p->xs, p->ys, p->zs, (size_t)n, t_wc, st);
}

void vo_pipeline_local(const vo_pipeline* p, uint8_t* cells, double origin[3]) {
  memcpy(cells, p->local, cells_of(p->cfg.grid.dims));
  memcpy(origin, p->origin, sizeof(double) * 3);
}
