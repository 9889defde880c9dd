// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A flat C shim over the UNMODIFIED reference voxmap library (built from
// /root/reference/proj/src by oracle/Makefile.ref) so that Python tests,
// golden-fixture generation and bench.py's reference arm can drive the
// reference's own code path through ctypes. Structs are the vxm.h PODs.
// Every function returns 0 on success, -1 on a reference exception (message
// in ref_last_error()).

#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "../include/vxm.h"
#include "voxmap/grid.hpp"
#include "voxmap/grid_io.hpp"
#include "voxmap/integrator.hpp"
#include "voxmap/kernels/kernels.hpp"
#include "voxmap/pipeline.hpp"
#include "voxmap/raytracer.hpp"
#include "voxmap/sim/render.hpp"
#include "voxmap/sim/scene.hpp"
#include "voxmap/sim/trajectory.hpp"

using namespace voxmap;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

GridSpec to_spec(const vxm_grid_spec& g) {
  GridSpec s = GridSpec::create(g.size[0], g.size[1], g.size[2], g.vox_size,
                                Eigen::Vector3d(g.origin[0], g.origin[1], g.origin[2]));
  // Honour the caller's dims (they come from the same lround formula).
  s.dims_x = g.dims[0];
  s.dims_y = g.dims[1];
  s.dims_z = g.dims[2];
  return s;
}

CameraModel to_cam(const vxm_camera& c) {
  CameraModel cam;
  cam.fov_x = c.fov_x;
  cam.fov_y = c.fov_y;
  cam.width = c.width;
  cam.height = c.height;
  cam.max_depth = c.max_depth;
  return cam;
}

RigidTransform to_pose(const vxm_pose& p) {
  RigidTransform t;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t.rotation(i, j) = p.rotation[3 * i + j];
  t.translation = Eigen::Vector3d(p.translation[0], p.translation[1], p.translation[2]);
  return t;
}

void from_pose(const RigidTransform& t, vxm_pose* p) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p->rotation[3 * i + j] = t.rotation(i, j);
  for (int i = 0; i < 3; ++i) p->translation[i] = t.translation[i];
}

PointCloud to_cloud(const double* xs, const double* ys, const double* zs, size_t n) {
  PointCloud c;
  c.reserve(n);
  for (size_t i = 0; i < n; ++i) c.add(xs[i], ys[i], zs[i]);
  return c;
}

void fill_stats(const PipelineStats& s, const GridSpec& spec, vxm_stats* out) {
  std::memset(out, 0, sizeof(*out));
  out->points_total = s.populate.points_total;
  out->points_outside = s.populate.points_outside;
  out->rays_traced = s.trace.rays_traced;
  out->voxels_freed = s.trace.voxels_freed;
  out->voxels_marked_unknown_traced = s.trace.voxels_marked_unknown_traced;
  out->voxels_skipped_out_of_bounds = s.trace.voxels_skipped_out_of_bounds;
  out->occupied_count = s.occupied_count;
  out->freed_count = s.freed_count;
  out->shifted = s.shifted ? 1 : 0;
  for (int a = 0; a < 3; ++a) {
    out->shift_offset[a] = s.shift_offset[a];
    out->origin[a] = spec.origin[a];
  }
  out->populate_us = s.populate_us;
  out->trace_us = s.trace_us;
  out->merge_us = s.merge_us;
  out->shift_us = s.shift_us;
}

struct RefPipeline {
  MappingPipeline pipeline;
  CameraModel cam;
  ExecutionMode mode;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

const char* ref_dispatch_isa(void) { return kernels::dispatch().isa; }

int ref_grid_spec_create_centered(double sx, double sy, double sz, double vs,
                                  const double center[3], vxm_grid_spec* out) {
  return guarded([&] {
    const GridSpec s =
        GridSpec::create_centered(sx, sy, sz, vs, Eigen::Vector3d(center[0], center[1], center[2]));
    out->size[0] = s.grid_size_x;
    out->size[1] = s.grid_size_y;
    out->size[2] = s.grid_size_z;
    out->vox_size = s.vox_size;
    out->dims[0] = s.dims_x;
    out->dims[1] = s.dims_y;
    out->dims[2] = s.dims_z;
    out->pad_ = 0;
    for (int a = 0; a < 3; ++a) out->origin[a] = s.origin[a];
  });
}

int ref_bundle_dimensions(const vxm_camera* cam, double depth, double vs, int32_t out[3]) {
  return guarded([&] {
    const RayBundle b = bundle_dimensions(to_cam(*cam), depth, vs);
    out[0] = b.vox_depth;
    out[1] = b.vox_width;
    out[2] = b.vox_height;
  });
}

int ref_look_along_x(const double pos[3], vxm_pose* out) {
  return guarded([&] { from_pose(sim::look_along_x(Eigen::Vector3d(pos[0], pos[1], pos[2])), out); });
}

// scene_kind: 0 empty, 1 wall (5.5 m), 2 box_field(seed); boxes != NULL
// overrides with nboxes explicit AABBs (minx miny minz maxx maxy maxz each).
int ref_render_depth(int scene_kind, uint64_t seed, const double* boxes, int nboxes,
                     const vxm_pose* t_wc, const vxm_camera* cam, int parallel, float* out) {
  return guarded([&] {
    sim::Scene scene;
    if (boxes) {
      for (int i = 0; i < nboxes; ++i) {
        const double* b = boxes + 6 * i;
        scene.boxes.push_back({{b[0], b[1], b[2]}, {b[3], b[4], b[5]}});
      }
    } else if (scene_kind == 1) {
      scene = sim::Scene::wall();
    } else if (scene_kind == 2) {
      scene = sim::Scene::box_field(seed);
    }
    const DepthImage img = sim::render_depth(
        scene, to_pose(*t_wc), to_cam(*cam),
        parallel ? ExecutionMode::DataParallel : ExecutionMode::Sequential);
    std::memcpy(out, img.depths.data(), img.depths.size() * sizeof(float));
  });
}

int ref_box_field(uint64_t seed, double* boxes_out, int* nboxes) {
  return guarded([&] {
    const sim::Scene s = sim::Scene::box_field(seed);
    *nboxes = static_cast<int>(s.boxes.size());
    for (size_t i = 0; i < s.boxes.size(); ++i) {
      for (int a = 0; a < 3; ++a) {
        boxes_out[6 * i + a] = s.boxes[i].min[a];
        boxes_out[6 * i + 3 + a] = s.boxes[i].max[a];
      }
    }
  });
}

int ref_depth_to_cloud(const vxm_camera* cam, const float* depth, int parallel, double* xs,
                       double* ys, double* zs, size_t* n_out) {
  return guarded([&] {
    DepthImage img(cam->width, cam->height);
    std::memcpy(img.depths.data(), depth, img.depths.size() * sizeof(float));
    const PointCloud c = depth_to_cloud(
        img, to_cam(*cam), parallel ? ExecutionMode::DataParallel : ExecutionMode::Sequential);
    for (size_t i = 0; i < c.size(); ++i) {
      xs[i] = c.xs()[i];
      ys[i] = c.ys()[i];
      zs[i] = c.zs()[i];
    }
    *n_out = c.size();
  });
}

void ref_merge(uint8_t* local, const uint8_t* ms, size_t n, int use_dispatch) {
  (use_dispatch ? kernels::dispatch() : kernels::scalar_table()).merge(local, ms, n);
}

void ref_transform_voxelize(const double* xs, const double* ys, const double* zs, size_t n,
                            const double* r, const double* t, double vs, int32_t* cx,
                            int32_t* cy, int32_t* cz, int use_dispatch) {
  (use_dispatch ? kernels::dispatch() : kernels::scalar_table())
      .transform_voxelize(xs, ys, zs, n, r, t, vs, cx, cy, cz);
}

int ref_populate(const vxm_grid_spec* g, uint8_t* ms, const double* xs, const double* ys,
                 const double* zs, size_t n, const vxm_pose* t_vc, int vox_inf, int parallel,
                 vxm_populate_stats* st) {
  return guarded([&] {
    VoxelGrid grid(to_spec(*g));
    std::memcpy(grid.raw(), ms, grid.size());
    const PopulateStats s = populate_occupied(
        grid, to_cloud(xs, ys, zs, n), to_pose(*t_vc), IntegratorConfig{vox_inf},
        parallel ? ExecutionMode::DataParallel : ExecutionMode::Sequential);
    std::memcpy(ms, grid.raw(), grid.size());
    st->points_total = s.points_total;
    st->points_outside = s.points_outside;
  });
}

int ref_trace_bundle(const vxm_grid_spec* g, uint8_t* ms, const int32_t bundle[3],
                     const vxm_pose* t_vc, int parallel, vxm_trace_stats* st) {
  return guarded([&] {
    VoxelGrid grid(to_spec(*g));
    std::memcpy(grid.raw(), ms, grid.size());
    const RayBundle b{bundle[0], bundle[1], bundle[2]};
    const TraceStats s =
        trace_bundle(grid, b, to_pose(*t_vc), g->vox_size,
                     parallel ? ExecutionMode::DataParallel : ExecutionMode::Sequential);
    std::memcpy(ms, grid.raw(), grid.size());
    st->rays_traced = s.rays_traced;
    st->voxels_freed = s.voxels_freed;
    st->voxels_marked_unknown_traced = s.voxels_marked_unknown_traced;
    st->voxels_skipped_out_of_bounds = s.voxels_skipped_out_of_bounds;
  });
}

int ref_trace_per_pixel(const vxm_grid_spec* g, uint8_t* ms, const double* xs,
                        const double* ys, const double* zs, size_t n, const vxm_pose* t_vc,
                        vxm_trace_stats* st) {
  return guarded([&] {
    VoxelGrid grid(to_spec(*g));
    std::memcpy(grid.raw(), ms, grid.size());
    const TraceStats s = bresenham_trace_image(grid, to_cloud(xs, ys, zs, n), to_pose(*t_vc),
                                               ExecutionMode::Sequential);
    std::memcpy(ms, grid.raw(), grid.size());
    st->rays_traced = s.rays_traced;
    st->voxels_freed = s.voxels_freed;
    st->voxels_marked_unknown_traced = s.voxels_marked_unknown_traced;
    st->voxels_skipped_out_of_bounds = s.voxels_skipped_out_of_bounds;
  });
}

// grid_io (proj/src/grid_io.cpp): the reference's own VOXGRID1 writer/reader
int ref_write_grid(const vxm_grid_spec* g, const uint8_t* cells, const char* path) {
  return guarded([&] {
    VoxelGrid grid(to_spec(*g));
    std::memcpy(grid.raw(), cells, grid.size());
    write_grid(grid, std::string(path));
  });
}

int ref_read_grid(const char* path, vxm_grid_spec* g, uint8_t* cells, size_t capacity) {
  return guarded([&] {
    const VoxelGrid grid = read_grid(std::string(path));
    const GridSpec& s = grid.spec();
    g->size[0] = s.grid_size_x;
    g->size[1] = s.grid_size_y;
    g->size[2] = s.grid_size_z;
    g->vox_size = s.vox_size;
    g->dims[0] = s.dims_x;
    g->dims[1] = s.dims_y;
    g->dims[2] = s.dims_z;
    g->pad_ = 0;
    for (int a = 0; a < 3; ++a) g->origin[a] = s.origin[a];
    if (cells && capacity >= grid.size()) std::memcpy(cells, grid.raw(), grid.size());
  });
}

int ref_shift(const vxm_grid_spec* g, const uint8_t* in, uint8_t* out, const int32_t off[3]) {
  return guarded([&] {
    VoxelGrid grid(to_spec(*g));
    std::memcpy(grid.raw(), in, grid.size());
    const VoxelGrid s = shift_grid_by(grid, Eigen::Vector3i(off[0], off[1], off[2]));
    std::memcpy(out, s.raw(), s.size());
  });
}

void* ref_pipeline_create(const vxm_config* cfg, int parallel) {
  try {
    PipelineConfig pc;
    pc.grid = to_spec(cfg->grid);
    pc.camera = to_cam(cfg->camera);
    pc.integrator.vox_inf = cfg->vox_inf;
    pc.depth = cfg->depth;
    pc.tracer_mode =
        cfg->tracer_mode == VXM_TRACER_PER_PIXEL ? TracerMode::PerPixelBaseline : TracerMode::Bundled;
    pc.parallelism = parallel ? ExecutionMode::DataParallel : ExecutionMode::Sequential;
    return new RefPipeline{MappingPipeline(pc), pc.camera, pc.parallelism};
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_pipeline_destroy(void* p) { delete static_cast<RefPipeline*>(p); }

int ref_pipeline_integrate_cloud(void* p, const double* xs, const double* ys, const double* zs,
                                 size_t n, const vxm_pose* t_wc, vxm_stats* out) {
  return guarded([&] {
    auto* rp = static_cast<RefPipeline*>(p);
    MeasurementFrame f;
    f.cloud = to_cloud(xs, ys, zs, n);
    f.t_wc = to_pose(*t_wc);
    const PipelineStats s = rp->pipeline.integrate(f);
    fill_stats(s, rp->pipeline.local_grid().spec(), out);
  });
}

// depth_to_cloud (in the pipeline's mode) followed by integrate, as every
// reference caller does (tools/voxmap_cli.cpp:117-126, sim/bench.cpp:242-249).
int ref_pipeline_integrate_depth(void* p, const float* depth, const vxm_pose* t_wc,
                                 vxm_stats* out) {
  return guarded([&] {
    auto* rp = static_cast<RefPipeline*>(p);
    DepthImage img(rp->cam.width, rp->cam.height);
    std::memcpy(img.depths.data(), depth, img.depths.size() * sizeof(float));
    MeasurementFrame f;
    f.cloud = depth_to_cloud(img, rp->cam, rp->mode);
    f.t_wc = to_pose(*t_wc);
    const PipelineStats s = rp->pipeline.integrate(f);
    fill_stats(s, rp->pipeline.local_grid().spec(), out);
  });
}

int ref_pipeline_local(void* p, uint8_t* cells, double origin[3]) {
  return guarded([&] {
    const VoxelGrid& g = static_cast<RefPipeline*>(p)->pipeline.local_grid();
    std::memcpy(cells, g.raw(), g.size());
    for (int a = 0; a < 3; ++a) origin[a] = g.spec().origin[a];
  });
}

}  // extern "C"
