// voxmap public API, B200 edition.
//
// One header carries the whole per-frame API surface the reference exposes in
// proj/include/voxmap/{voxel_state,exec,grid,geometry,integrator,raytracer,
// pipeline}.hpp and kernels/kernels.hpp; the files with those names next to
// this one just include it, so existing `#include "voxmap/pipeline.hpp"`
// callers compile unchanged. Names, signatures, argument meaning and the
// exception contract (std::invalid_argument for violated preconditions) are
// the reference's; the work behind populate_occupied, trace_bundle,
// bresenham_trace_image, merge_grids, shift_grid_by, depth_to_cloud and
// MappingPipeline::integrate runs on an sm_100a GPU through the C-ABI in
// include/vxm.h. There is no CPU implementation of those: without a GPU they
// throw std::runtime_error.
//
// ExecutionMode is accepted everywhere for source compatibility; the GPU
// result always equals the reference's Sequential mode byte for byte.
#pragma once

#include <Eigen/Core>
#include <Eigen/Geometry>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <iosfwd>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "vxm.h"

namespace voxmap {

// ------------------------------------------------------------ states, modes

enum class VoxelState : std::uint8_t { Unknown = 0, Free = 1, Occupied = 2, UnknownTraced = 3 };
const char* to_string(VoxelState s);

enum class ExecutionMode { Sequential, DataParallel };
enum class TracerMode { Bundled, PerPixelBaseline };
const char* to_string(ExecutionMode m);
const char* to_string(TracerMode m);

// ------------------------------------------------------------------- grids

struct VoxelCoord {
  int x = 0, y = 0, z = 0;
  friend bool operator==(const VoxelCoord&, const VoxelCoord&) = default;
};

struct GridSpec {
  double grid_size_x = 0.0, grid_size_y = 0.0, grid_size_z = 0.0;
  double vox_size = 0.0;
  int dims_x = 0, dims_y = 0, dims_z = 0;
  Eigen::Vector3d origin = Eigen::Vector3d::Zero();

  static GridSpec create(double size_x, double size_y, double size_z, double vox_size,
                         const Eigen::Vector3d& origin = Eigen::Vector3d::Zero());
  static GridSpec create_centered(double size_x, double size_y, double size_z, double vox_size,
                                  const Eigen::Vector3d& center);

  std::size_t cell_count() const {
    return static_cast<std::size_t>(dims_x) * static_cast<std::size_t>(dims_y) *
           static_cast<std::size_t>(dims_z);
  }
  Eigen::Vector3d half_extent() const {
    return Eigen::Vector3d(dims_x / 2, dims_y / 2, dims_z / 2) * vox_size;
  }
  Eigen::Vector3d center() const { return origin + half_extent(); }
  bool in_bounds(const VoxelCoord& c) const {
    return c.x >= 0 && c.x < dims_x && c.y >= 0 && c.y < dims_y && c.z >= 0 && c.z < dims_z;
  }
  bool same_layout(const GridSpec& o) const {
    return dims_x == o.dims_x && dims_y == o.dims_y && dims_z == o.dims_z &&
           vox_size == o.vox_size && origin == o.origin;
  }
  vxm_grid_spec to_c() const;
};

inline std::size_t linear_index_unchecked(const VoxelCoord& c, const GridSpec& s) {
  const auto dx = static_cast<std::size_t>(s.dims_x), dy = static_cast<std::size_t>(s.dims_y);
  return static_cast<std::size_t>(c.x) + static_cast<std::size_t>(c.y) * dx +
         static_cast<std::size_t>(c.z) * dx * dy;
}
inline std::optional<std::size_t> linear_index(const VoxelCoord& c, const GridSpec& s) {
  if (!s.in_bounds(c)) return std::nullopt;
  return linear_index_unchecked(c, s);
}

VoxelCoord world_to_voxel(const Eigen::Vector3d& p_grid, const GridSpec& spec);

class VoxelGrid {
 public:
  explicit VoxelGrid(GridSpec spec);
  const GridSpec& spec() const { return spec_; }
  std::size_t size() const { return cells_.size(); }
  VoxelState at(const VoxelCoord& c) const { return cells_[linear_index_unchecked(c, spec_)]; }
  void set(const VoxelCoord& c, VoxelState v) { cells_[linear_index_unchecked(c, spec_)] = v; }
  VoxelState operator[](std::size_t i) const { return cells_[i]; }
  std::span<const VoxelState> cells() const { return cells_; }
  std::span<VoxelState> cells() { return cells_; }
  std::uint8_t* raw() { return reinterpret_cast<std::uint8_t*>(cells_.data()); }
  const std::uint8_t* raw() const { return reinterpret_cast<const std::uint8_t*>(cells_.data()); }
  void reset();
  std::size_t count(VoxelState v) const;
  void set_origin(const Eigen::Vector3d& origin) { spec_.origin = origin; }
  friend bool operator==(const VoxelGrid& a, const VoxelGrid& b) {
    return a.spec_.same_layout(b.spec_) && a.cells_ == b.cells_;
  }

 private:
  GridSpec spec_;
  std::vector<VoxelState> cells_;
};

VoxelGrid shift_grid_by(const VoxelGrid& grid, const Eigen::Vector3i& offset_voxels);

// grid_io (proj/include/voxmap/grid_io.hpp:10-17): VOXGRID1 dumps, host only;
// std::runtime_error on I/O or format errors.
void write_grid(const VoxelGrid& grid, std::ostream& out);
void write_grid(const VoxelGrid& grid, const std::string& path);
VoxelGrid read_grid(std::istream& in);
VoxelGrid read_grid(const std::string& path);
VoxelGrid shift_grid(const VoxelGrid& grid, const Eigen::Vector3d& new_center);
Eigen::Vector3i shift_offset_for_center(const GridSpec& spec, const Eigen::Vector3d& new_center);

// ---------------------------------------------------------------- geometry

struct RigidTransform {
  Eigen::Matrix3d rotation = Eigen::Matrix3d::Identity();
  Eigen::Vector3d translation = Eigen::Vector3d::Zero();

  static RigidTransform identity() { return {}; }
  static RigidTransform from_translation(const Eigen::Vector3d& t) {
    return {Eigen::Matrix3d::Identity(), t};
  }
  static RigidTransform from_rotation(const Eigen::Matrix3d& r,
                                      const Eigen::Vector3d& t = Eigen::Vector3d::Zero()) {
    return {r, t};
  }
  Eigen::Vector3d apply(const Eigen::Vector3d& p) const;
  RigidTransform inverse() const {
    return {rotation.transpose(), -(rotation.transpose() * translation)};
  }
  bool is_valid(double tol = 1e-9) const;
  vxm_pose to_c() const;
};

RigidTransform compose(const RigidTransform& a, const RigidTransform& b);
inline RigidTransform operator*(const RigidTransform& a, const RigidTransform& b) {
  return compose(a, b);
}
inline Eigen::Vector3d camera_center_in_grid(const RigidTransform& t_vc) { return t_vc.translation; }

struct CameraModel {
  double fov_x = 0.0, fov_y = 0.0;  // radians
  int width = 0, height = 0;
  double max_depth = 0.0;
  void validate() const;
  double focal_x() const { return (width / 2.0) / std::tan(fov_x / 2.0); }
  double focal_y() const { return (height / 2.0) / std::tan(fov_y / 2.0); }
  vxm_camera to_c() const { return vxm_camera{fov_x, fov_y, width, height, max_depth}; }
};

class PointCloud {
 public:
  void reserve(std::size_t n) {
    xs_.reserve(n);
    ys_.reserve(n);
    zs_.reserve(n);
  }
  void add(double x, double y, double z) {
    if (!std::isfinite(x) || !std::isfinite(y) || !std::isfinite(z)) return;
    xs_.push_back(x);
    ys_.push_back(y);
    zs_.push_back(z);
  }
  void add(const Eigen::Vector3d& p) { add(p.x(), p.y(), p.z()); }
  std::size_t size() const { return xs_.size(); }
  bool empty() const { return xs_.empty(); }
  Eigen::Vector3d point(std::size_t i) const { return {xs_[i], ys_[i], zs_[i]}; }
  std::span<const double> xs() const { return xs_; }
  std::span<const double> ys() const { return ys_; }
  std::span<const double> zs() const { return zs_; }

 private:
  std::vector<double> xs_, ys_, zs_;
};

struct DepthImage {
  int width = 0, height = 0;
  std::vector<float> depths;
  DepthImage() = default;
  DepthImage(int w, int h) : width(w), height(h), depths(static_cast<std::size_t>(w) * h, 0.0f) {}
  float at(int u, int v) const { return depths[static_cast<std::size_t>(v) * width + u]; }
  float& at(int u, int v) { return depths[static_cast<std::size_t>(v) * width + u]; }
  static bool valid_depth(float d) { return std::isfinite(d) && d > 0.0f; }
};

PointCloud depth_to_cloud(const DepthImage& img, const CameraModel& cam,
                          ExecutionMode mode = ExecutionMode::Sequential);

// -------------------------------------------------------------- integrator

struct IntegratorConfig {
  int vox_inf = 2;
  void validate() const;
};

struct PopulateStats {
  std::uint64_t points_total = 0;
  std::uint64_t points_outside = 0;
};

PopulateStats populate_occupied(VoxelGrid& ms_grid, const PointCloud& cloud,
                                const RigidTransform& t_vc, const IntegratorConfig& cfg,
                                ExecutionMode mode = ExecutionMode::Sequential);

// --------------------------------------------------------------- raytracer

struct RayBundle {
  int vox_depth = 0, vox_width = 0, vox_height = 0;
  std::size_t ray_count() const {
    return static_cast<std::size_t>(vox_width) * static_cast<std::size_t>(vox_height);
  }
};

RayBundle bundle_dimensions(const CameraModel& cam, double depth, double vox_size);

struct Ray {
  Eigen::Vector3d start = Eigen::Vector3d::Zero();
  Eigen::Vector3d dir = Eigen::Vector3d::Zero();
  double max_dist = 0.0;
};

void validate_ray(const Ray& ray);

struct TraceStats {
  std::uint64_t rays_traced = 0;
  std::uint64_t voxels_freed = 0;
  std::uint64_t voxels_marked_unknown_traced = 0;
  std::uint64_t voxels_skipped_out_of_bounds = 0;
  TraceStats& operator+=(const TraceStats& o) {
    rays_traced += o.rays_traced;
    voxels_freed += o.voxels_freed;
    voxels_marked_unknown_traced += o.voxels_marked_unknown_traced;
    voxels_skipped_out_of_bounds += o.voxels_skipped_out_of_bounds;
    return *this;
  }
};

std::vector<Ray> generate_rays(const RayBundle& bundle, const RigidTransform& t_vc, double vox_size);

inline constexpr double kTraversalStopEpsilon = 1e-10;

// Host-side single-ray utilities (header templates in the reference too);
// the per-frame tracer never uses them: it runs as K3 on the GPU.
template <typename Visitor>
void walk_ray(const Ray& ray, double vox_size, Visitor&& visit) {
  const Eigen::Vector3d u = ray.dir.normalized();
  int cur[3], step[3];
  double tmax[3], tdelta[3];
  for (int a = 0; a < 3; ++a) {
    cur[a] = static_cast<int>(std::floor(ray.start[a] / vox_size));
    if (u[a] > 0.0) {
      step[a] = 1;
      tmax[a] = ((cur[a] + 1) * vox_size - ray.start[a]) / u[a];
      tdelta[a] = vox_size / u[a];
    } else if (u[a] < 0.0) {
      step[a] = -1;
      tmax[a] = (cur[a] * vox_size - ray.start[a]) / u[a];
      tdelta[a] = vox_size / -u[a];
    } else {
      step[a] = 0;
      tmax[a] = tdelta[a] = std::numeric_limits<double>::infinity();
    }
  }
  if (!visit(VoxelCoord{cur[0], cur[1], cur[2]})) return;
  while (true) {
    const int a = (tmax[0] <= tmax[1] && tmax[0] <= tmax[2]) ? 0 : (tmax[1] <= tmax[2] ? 1 : 2);
    if (tmax[a] >= ray.max_dist - kTraversalStopEpsilon) return;
    cur[a] += step[a];
    tmax[a] += tdelta[a];
    if (!visit(VoxelCoord{cur[0], cur[1], cur[2]})) return;
  }
}

template <typename Visitor>
void bresenham_line(const VoxelCoord& from, const VoxelCoord& to, Visitor&& visit) {
  int p[3] = {from.x, from.y, from.z};
  const int e[3] = {to.x, to.y, to.z};
  int d[3], s[3];
  for (int a = 0; a < 3; ++a) {
    d[a] = std::abs(e[a] - p[a]);
    s[a] = e[a] > p[a] ? 1 : -1;
  }
  const int k = (d[0] >= d[1] && d[0] >= d[2]) ? 0 : (d[1] >= d[0] && d[1] >= d[2]) ? 1 : 2;
  const int o1 = k == 1 ? 0 : 1, o2 = k == 2 ? 0 : 2;
  int e1 = 2 * d[o1] - d[k], e2 = 2 * d[o2] - d[k];
  while (p[k] != e[k]) {
    if (!visit(VoxelCoord{p[0], p[1], p[2]})) return;
    if (e1 >= 0) { p[o1] += s[o1]; e1 -= 2 * d[k]; }
    if (e2 >= 0) { p[o2] += s[o2]; e2 -= 2 * d[k]; }
    e1 += 2 * d[o1];
    e2 += 2 * d[o2];
    p[k] += s[k];
  }
  visit(to);
}

TraceStats traverse_ray(VoxelGrid& ms_grid, const Ray& ray);
TraceStats trace_bundle(VoxelGrid& ms_grid, const RayBundle& bundle, const RigidTransform& t_vc,
                        double vox_size, ExecutionMode mode = ExecutionMode::Sequential);
TraceStats bresenham_trace_image(VoxelGrid& ms_grid, const PointCloud& cloud,
                                 const RigidTransform& t_vc,
                                 ExecutionMode mode = ExecutionMode::Sequential);

// ---------------------------------------------------------------- pipeline

struct PipelineConfig {
  GridSpec grid;
  CameraModel camera;
  IntegratorConfig integrator;
  double depth = 6.5;
  TracerMode tracer_mode = TracerMode::Bundled;
  ExecutionMode parallelism = ExecutionMode::DataParallel;
  void validate() const;
};

struct MeasurementFrame {
  PointCloud cloud;
  RigidTransform t_wc;
  double timestamp = 0.0;
};

struct PipelineStats {
  double populate_us = 0.0, trace_us = 0.0, merge_us = 0.0, shift_us = 0.0;
  TraceStats trace;
  PopulateStats populate;
  std::uint64_t occupied_count = 0;
  std::uint64_t freed_count = 0;
  bool shifted = false;
  Eigen::Vector3i shift_offset = Eigen::Vector3i::Zero();
};

void merge_grids(VoxelGrid& loc_grid, const VoxelGrid& ms_grid,
                 ExecutionMode mode = ExecutionMode::Sequential);
RigidTransform camera_to_grid_transform(const RigidTransform& t_wc,
                                        const Eigen::Vector3d& grid_origin);

class MappingPipeline {
 public:
  explicit MappingPipeline(PipelineConfig cfg, int device = 0);
  MappingPipeline(PipelineConfig cfg, const Eigen::Vector3d& initial_position, int device = 0);
  ~MappingPipeline();
  MappingPipeline(MappingPipeline&&) noexcept;
  MappingPipeline& operator=(MappingPipeline&&) noexcept;

  PipelineStats integrate(const MeasurementFrame& frame);
  // Extension: the fused depth path (depth_to_cloud folded into the first
  // kernel); equal to integrate({depth_to_cloud(depth, camera), t_wc}).
  PipelineStats integrate_depth(const DepthImage& depth, const RigidTransform& t_wc);
  // Extension: multi-frame pipelining. Equal to calling integrate_depth on
  // each (depths[i], poses[i]) in order, bit for bit, but the populate and
  // ray-cast stages of up to kMaxFramesPerCall frames run concurrently and
  // one chain kernel folds their merges and shifts.
  static constexpr int kMaxFramesPerCall = 64;
  std::vector<PipelineStats> integrate_depth_sequence(const std::vector<DepthImage>& depths,
                                                      const std::vector<RigidTransform>& poses);

  const VoxelGrid& local_grid() const;
  const PipelineConfig& config() const { return cfg_; }
  // Extension (checkpoint/resume): continue from a saved
  // local grid, e.g. read_grid(path) of an earlier write_grid(local_grid()).
  // Its dims and vox_size must match the configuration's grid.
  void restore_local_grid(const VoxelGrid& grid);
  // Extension (asynchronous checkpoint): write the local grid as it stands now
  // to a VOXGRID1 file (as write_grid(local_grid(), path) would) without
  // stalling integration: device -> pinned copy on a side stream, file written
  // by a host thread. snapshot_wait() joins it and throws std::runtime_error
  // if the write failed.
  void save_snapshot_async(const std::string& path);
  void snapshot_wait();

 private:
  PipelineConfig cfg_;
  int device_ = 0;
  vxm_ctx* ctx_ = nullptr;      // single-frame context
  vxm_ctx* seq_ctx_ = nullptr;  // multi-frame context, created on first use
  bool seq_active_ = false;     // which context holds the current local grid
  mutable VoxelGrid local_;
  mutable bool local_stale_ = false;
  PipelineStats finish(const vxm_stats& s);
  void activate(bool sequence);
};

// ------------------------------------------------------------ kernel table

namespace kernels {
using MergeFn = void (*)(std::uint8_t* local, const std::uint8_t* measurement, std::size_t n);
using TransformVoxelizeFn = void (*)(const double* xs, const double* ys, const double* zs,
                                     std::size_t n, const double* rotation,
                                     const double* translation, double vox_size,
                                     std::int32_t* cx, std::int32_t* cy, std::int32_t* cz);
struct KernelTable {
  MergeFn merge = nullptr;
  TransformVoxelizeFn transform_voxelize = nullptr;
  const char* isa = "scalar";
};
// cuda_table(): the sm_100a implementation (isa "cuda-sm100a"), which
// dispatch() returns and every pipeline path uses. scalar_table(): the
// reference's portable host table (isa "scalar"), for callers that ask for it
// by name (the reference's test_kernels checks dispatch() against it).
const KernelTable& cuda_table();
const KernelTable& scalar_table();
const KernelTable& dispatch();
}  // namespace kernels

}  // namespace voxmap
