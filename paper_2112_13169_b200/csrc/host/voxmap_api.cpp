// Host side of the voxmap drop-in API (include/voxmap/b200_api.hpp).
//
// Host arithmetic (grid placement, transforms, bundle sizes, shift offsets)
// follows the reference formula for formula (citations inline). Everything
// that touches grid contents goes through the C-ABI of libvxm.so
// (include/vxm.h) and runs on the GPU.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <numbers>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>

#include "voxgrid_format.hpp"
#include "voxmap/b200_api.hpp"
#include "voxmap/sim/trajectory.hpp"

namespace voxmap {

namespace {

[[noreturn]] void raise(int rc) {
  const std::string msg = vxm_last_error();
  if (rc == VXM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("vxm error " + std::to_string(rc) + ": " + msg);
}

void check(int rc) {
  if (rc != VXM_OK) raise(rc);
}

}  // namespace

const char* to_string(VoxelState s) {
  switch (s) {
    case VoxelState::Unknown: return "unknown";
    case VoxelState::Free: return "free";
    case VoxelState::Occupied: return "occupied";
    case VoxelState::UnknownTraced: return "unknown_traced";
  }
  return "invalid";
}
const char* to_string(ExecutionMode m) {
  return m == ExecutionMode::Sequential ? "sequential" : "parallel";
}
const char* to_string(TracerMode m) { return m == TracerMode::Bundled ? "bundled" : "per-pixel"; }

// ------------------------------------------------------------------ grids

// GridSpec::create (proj/src/grid.cpp:17-42)
GridSpec GridSpec::create(double sx, double sy, double sz, double vs, const Eigen::Vector3d& origin) {
  vxm_grid_spec c{};
  const double o[3] = {origin.x(), origin.y(), origin.z()};
  check(vxm_grid_spec_create(sx, sy, sz, vs, o, &c));
  GridSpec s;
  s.grid_size_x = c.size[0];
  s.grid_size_y = c.size[1];
  s.grid_size_z = c.size[2];
  s.vox_size = c.vox_size;
  s.dims_x = c.dims[0];
  s.dims_y = c.dims[1];
  s.dims_z = c.dims[2];
  s.origin = origin;
  return s;
}

// GridSpec::create_centered (grid.cpp:44-52)
GridSpec GridSpec::create_centered(double sx, double sy, double sz, double vs,
                                   const Eigen::Vector3d& center) {
  GridSpec s = create(sx, sy, sz, vs);
  s.origin = center - s.half_extent();
  if (!s.origin.allFinite()) throw std::invalid_argument("grid center must be finite");
  return s;
}

vxm_grid_spec GridSpec::to_c() const {
  vxm_grid_spec c{};
  c.size[0] = grid_size_x;
  c.size[1] = grid_size_y;
  c.size[2] = grid_size_z;
  c.vox_size = vox_size;
  c.dims[0] = dims_x;
  c.dims[1] = dims_y;
  c.dims[2] = dims_z;
  for (int a = 0; a < 3; ++a) c.origin[a] = origin[a];
  return c;
}

// world_to_voxel (grid.cpp:54-62)
VoxelCoord world_to_voxel(const Eigen::Vector3d& p, const GridSpec& spec) {
  if (!p.allFinite()) throw std::invalid_argument("world_to_voxel: non-finite point");
  return {static_cast<int>(std::floor(p.x() / spec.vox_size)),
          static_cast<int>(std::floor(p.y() / spec.vox_size)),
          static_cast<int>(std::floor(p.z() / spec.vox_size))};
}

VoxelGrid::VoxelGrid(GridSpec spec) : spec_(spec), cells_(spec.cell_count(), VoxelState::Unknown) {}

void VoxelGrid::reset() { std::memset(cells_.data(), 0, cells_.size()); }

std::size_t VoxelGrid::count(VoxelState v) const {
  std::size_t n = 0;
  for (VoxelState c : cells_) n += c == v;
  return n;
}

// shift_grid_by (grid.cpp:81-108): origin moves by offset*vox_size, the
// cells are gathered on the GPU.
VoxelGrid shift_grid_by(const VoxelGrid& grid, const Eigen::Vector3i& offset) {
  GridSpec spec = grid.spec();
  spec.origin = grid.spec().origin + offset.cast<double>() * grid.spec().vox_size;
  VoxelGrid out(spec);
  const int32_t dims[3] = {spec.dims_x, spec.dims_y, spec.dims_z};
  const int32_t off[3] = {offset.x(), offset.y(), offset.z()};
  check(vxm_shift_grid(dims, grid.raw(), out.raw(), off));
  return out;
}

// shift_offset_for_center (grid.cpp:110-117)
Eigen::Vector3i shift_offset_for_center(const GridSpec& spec, const Eigen::Vector3d& new_center) {
  const Eigen::Vector3d ideal_origin = new_center - spec.half_extent();
  const Eigen::Vector3d delta = (ideal_origin - spec.origin) / spec.vox_size;
  return Eigen::Vector3i(static_cast<int>(std::lround(delta.x())), static_cast<int>(std::lround(delta.y())),
                         static_cast<int>(std::lround(delta.z())));
}

VoxelGrid shift_grid(const VoxelGrid& grid, const Eigen::Vector3d& new_center) {
  if (!new_center.allFinite()) throw std::invalid_argument("shift_grid: non-finite center");
  return shift_grid_by(grid, shift_offset_for_center(grid.spec(), new_center));
}

// --------------------------------------------------------------- geometry

Eigen::Vector3d RigidTransform::apply(const Eigen::Vector3d& p) const {
  if (!p.allFinite()) throw std::invalid_argument("RigidTransform::apply: non-finite point");
  return rotation * p + translation;
}

// RigidTransform::is_valid (geometry.cpp:17-22)
bool RigidTransform::is_valid(double tol) const {
  if (!rotation.allFinite() || !translation.allFinite()) return false;
  const Eigen::Matrix3d gram = rotation.transpose() * rotation;
  if ((gram - Eigen::Matrix3d::Identity()).cwiseAbs().maxCoeff() > tol) return false;
  return std::abs(rotation.determinant() - 1.0) <= tol;
}

vxm_pose RigidTransform::to_c() const {
  vxm_pose p{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p.rotation[3 * i + j] = rotation(i, j);
  for (int i = 0; i < 3; ++i) p.translation[i] = translation[i];
  return p;
}

// compose (geometry.cpp:24-26)
RigidTransform compose(const RigidTransform& a, const RigidTransform& b) {
  return {a.rotation * b.rotation, a.rotation * b.translation + a.translation};
}

// CameraModel::validate (geometry.cpp:28-41)
void CameraModel::validate() const {
  if (width <= 0 || height <= 0)
    throw std::invalid_argument("CameraModel: width and height must be positive");
  if (!(fov_x > 0.0) || !(fov_x < std::numbers::pi) || !(fov_y > 0.0) || !(fov_y < std::numbers::pi))
    throw std::invalid_argument("CameraModel: FOV must lie in (0, pi)");
  if (!(max_depth > 0.0) || !std::isfinite(max_depth))
    throw std::invalid_argument("CameraModel: max_depth must be positive and finite");
}

// depth_to_cloud (geometry.cpp:64-99): ordered compaction on the GPU
PointCloud depth_to_cloud(const DepthImage& img, const CameraModel& cam, ExecutionMode) {
  cam.validate();
  if (img.width != cam.width || img.height != cam.height)
    throw std::invalid_argument("depth_to_cloud: image size does not match camera model");
  if (img.depths.size() != static_cast<std::size_t>(img.width) * img.height)
    throw std::invalid_argument("depth_to_cloud: depth buffer size mismatch");
  const std::size_t npix = img.depths.size();
  std::vector<double> xs(npix), ys(npix), zs(npix);
  std::size_t n = 0;
  const vxm_camera c = cam.to_c();
  check(vxm_depth_to_cloud(&c, img.depths.data(), xs.data(), ys.data(), zs.data(), &n));
  PointCloud cloud;
  cloud.reserve(n);
  for (std::size_t i = 0; i < n; ++i) cloud.add(xs[i], ys[i], zs[i]);
  return cloud;
}

// ------------------------------------------------------------- integrator

void IntegratorConfig::validate() const {
  if (vox_inf < 0) throw std::invalid_argument("IntegratorConfig: vox_inf must be non-negative");
}

// populate_occupied (integrator.cpp:45-103)
PopulateStats populate_occupied(VoxelGrid& ms, const PointCloud& cloud, const RigidTransform& t_vc,
                                const IntegratorConfig& cfg, ExecutionMode) {
  cfg.validate();
  const vxm_grid_spec g = ms.spec().to_c();
  const vxm_pose p = t_vc.to_c();
  vxm_populate_stats st{};
  check(vxm_populate_occupied(&g, ms.raw(), cloud.xs().data(), cloud.ys().data(), cloud.zs().data(),
                              cloud.size(), &p, cfg.vox_inf, &st));
  return {st.points_total, st.points_outside};
}

// -------------------------------------------------------------- raytracer

// bundle_dimensions (raytracer.cpp:8-21)
RayBundle bundle_dimensions(const CameraModel& cam, double depth, double vox_size) {
  cam.validate();
  const vxm_camera c = cam.to_c();
  int32_t b[3];
  check(vxm_bundle_dimensions(&c, depth, vox_size, b));
  return {b[0], b[1], b[2]};
}

// validate_ray (raytracer.cpp:23-33)
void validate_ray(const Ray& ray) {
  if (!ray.start.allFinite() || !ray.dir.allFinite() || !std::isfinite(ray.max_dist))
    throw std::invalid_argument("Ray: non-finite field");
  if (ray.dir.isZero(0.0)) throw std::invalid_argument("Ray: direction must be non-zero");
  if (!(ray.max_dist > 0.0)) throw std::invalid_argument("Ray: max_dist must be positive");
}

// generate_rays (raytracer.cpp:35-61); the GPU tracer derives the same rays
// from (xi, yi) on the fly and never materialises this vector.
std::vector<Ray> generate_rays(const RayBundle& b, const RigidTransform& t_vc, double vs) {
  if (b.vox_depth < 1 || b.vox_width < 1 || b.vox_height < 1 || b.vox_width % 2 == 0 ||
      b.vox_height % 2 == 0)
    throw std::invalid_argument("generate_rays: bundle dimensions must be positive and odd");
  if (!(vs > 0.0)) throw std::invalid_argument("generate_rays: vox_size must be positive");
  const int hw = (b.vox_width - 1) / 2, hh = (b.vox_height - 1) / 2;
  std::vector<Ray> rays;
  rays.reserve(b.ray_count());
  for (int yi = -hh; yi <= hh; ++yi) {
    for (int xi = -hw; xi <= hw; ++xi) {
      Ray r;
      r.start = t_vc.translation;
      r.dir = t_vc.rotation * Eigen::Vector3d(xi * vs, yi * vs, b.vox_depth * vs);
      r.max_dist = vs * std::sqrt(static_cast<double>(xi) * xi + static_cast<double>(yi) * yi +
                                  static_cast<double>(b.vox_depth) * b.vox_depth);
      rays.push_back(r);
    }
  }
  return rays;
}

// traverse_ray (raytracer.cpp:63-96): single-ray host utility
TraceStats traverse_ray(VoxelGrid& ms, const Ray& ray) {
  validate_ray(ray);
  const GridSpec& spec = ms.spec();
  TraceStats st;
  st.rays_traced = 1;
  std::uint8_t val = 1;
  bool entered = false;
  walk_ray(ray, spec.vox_size, [&](const VoxelCoord& c) {
    if (!spec.in_bounds(c)) {
      if (entered) return false;
      ++st.voxels_skipped_out_of_bounds;
      return true;
    }
    entered = true;
    std::uint8_t& cell = ms.raw()[linear_index_unchecked(c, spec)];
    if (cell == 2) {
      val = 3;
    } else {
      cell = val;
      (val == 1 ? st.voxels_freed : st.voxels_marked_unknown_traced) += 1;
    }
    return true;
  });
  return st;
}

// trace_bundle (raytracer.cpp:98-118), Sequential semantics, on the GPU
TraceStats trace_bundle(VoxelGrid& ms, const RayBundle& b, const RigidTransform& t_vc, double vs,
                        ExecutionMode) {
  const vxm_grid_spec g = ms.spec().to_c();
  const int32_t bundle[3] = {b.vox_depth, b.vox_width, b.vox_height};
  const vxm_pose p = t_vc.to_c();
  vxm_trace_stats st{};
  check(vxm_trace_bundle(&g, ms.raw(), bundle, &p, vs, &st));
  return {st.rays_traced, st.voxels_freed, st.voxels_marked_unknown_traced,
          st.voxels_skipped_out_of_bounds};
}

// bresenham_trace_image (raytracer.cpp:120-161), on the GPU
TraceStats bresenham_trace_image(VoxelGrid& ms, const PointCloud& cloud, const RigidTransform& t_vc,
                                 ExecutionMode) {
  const vxm_grid_spec g = ms.spec().to_c();
  const vxm_pose p = t_vc.to_c();
  vxm_trace_stats st{};
  check(vxm_trace_per_pixel(&g, ms.raw(), cloud.xs().data(), cloud.ys().data(), cloud.zs().data(),
                            cloud.size(), &p, &st));
  return {st.rays_traced, st.voxels_freed, st.voxels_marked_unknown_traced,
          st.voxels_skipped_out_of_bounds};
}

// --------------------------------------------------------------- pipeline

// PipelineConfig::validate (pipeline.cpp:33-42)
void PipelineConfig::validate() const {
  camera.validate();
  integrator.validate();
  if (grid.cell_count() == 0) throw std::invalid_argument("PipelineConfig: empty grid");
  if (!(depth > 0.0) || depth > camera.max_depth)
    throw std::invalid_argument("PipelineConfig: depth must lie in (0, camera.max_depth]");
}

// merge_grids (pipeline.cpp:44-61)
void merge_grids(VoxelGrid& loc, const VoxelGrid& ms, ExecutionMode) {
  if (!loc.spec().same_layout(ms.spec())) throw std::invalid_argument("merge_grids: grid layouts differ");
  check(vxm_merge_grids(loc.raw(), ms.raw(), loc.size()));
}

// camera_to_grid_transform (pipeline.cpp:63-66)
RigidTransform camera_to_grid_transform(const RigidTransform& t_wc, const Eigen::Vector3d& origin) {
  return compose(RigidTransform::from_translation(-origin), t_wc);
}

namespace {
PipelineConfig validated(PipelineConfig cfg) {
  cfg.validate();
  return cfg;
}
PipelineConfig recentered(PipelineConfig cfg, const Eigen::Vector3d& position) {
  cfg.grid = GridSpec::create_centered(cfg.grid.grid_size_x, cfg.grid.grid_size_y, cfg.grid.grid_size_z,
                                       cfg.grid.vox_size, position);
  return cfg;
}
}  // namespace

MappingPipeline::MappingPipeline(PipelineConfig cfg, int device)
    : cfg_(validated(std::move(cfg))), device_(device), local_(cfg_.grid) {
  vxm_config c{};
  c.grid = cfg_.grid.to_c();
  c.camera = cfg_.camera.to_c();
  c.vox_inf = cfg_.integrator.vox_inf;
  c.tracer_mode = cfg_.tracer_mode == TracerMode::Bundled ? VXM_TRACER_BUNDLED : VXM_TRACER_PER_PIXEL;
  c.depth = cfg_.depth;
  check(vxm_create(&c, 1, device, 0, &ctx_));
}

MappingPipeline::MappingPipeline(PipelineConfig cfg, const Eigen::Vector3d& initial_position, int device)
    : MappingPipeline(recentered(std::move(cfg), initial_position), device) {}

MappingPipeline::~MappingPipeline() {
  if (ctx_) vxm_destroy(ctx_);
  if (seq_ctx_) vxm_destroy(seq_ctx_);
}

MappingPipeline::MappingPipeline(MappingPipeline&& o) noexcept
    : cfg_(std::move(o.cfg_)), device_(o.device_), ctx_(std::exchange(o.ctx_, nullptr)),
      seq_ctx_(std::exchange(o.seq_ctx_, nullptr)), seq_active_(o.seq_active_), local_(std::move(o.local_)),
      local_stale_(o.local_stale_) {}

MappingPipeline& MappingPipeline::operator=(MappingPipeline&& o) noexcept {
  if (this != &o) {
    if (ctx_) vxm_destroy(ctx_);
    if (seq_ctx_) vxm_destroy(seq_ctx_);
    cfg_ = std::move(o.cfg_);
    device_ = o.device_;
    ctx_ = std::exchange(o.ctx_, nullptr);
    seq_ctx_ = std::exchange(o.seq_ctx_, nullptr);
    seq_active_ = o.seq_active_;
    local_ = std::move(o.local_);
    local_stale_ = o.local_stale_;
  }
  return *this;
}

// Moves the local grid (cells + origin) to the context that runs next.
void MappingPipeline::activate(bool sequence) {
  if (sequence == seq_active_) return;
  if (sequence && !seq_ctx_) {
    vxm_config c{};
    c.grid = cfg_.grid.to_c();
    c.camera = cfg_.camera.to_c();
    c.vox_inf = cfg_.integrator.vox_inf;
    c.tracer_mode = cfg_.tracer_mode == TracerMode::Bundled ? VXM_TRACER_BUNDLED : VXM_TRACER_PER_PIXEL;
    c.depth = cfg_.depth;
    check(vxm_create_multi(&c, 1, kMaxFramesPerCall, device_, 0, &seq_ctx_));
  }
  std::vector<std::uint8_t> cells(local_.size());
  double origin[3];
  check(vxm_download_local(sequence ? ctx_ : seq_ctx_, 0, cells.data(), origin));
  check(vxm_upload_local(sequence ? seq_ctx_ : ctx_, 0, cells.data(), origin));
  seq_active_ = sequence;
}

PipelineStats MappingPipeline::finish(const vxm_stats& s) {
  PipelineStats st;
  st.populate_us = s.populate_us;
  st.trace_us = s.trace_us;
  st.merge_us = s.merge_us;
  st.shift_us = s.shift_us;
  st.populate = {s.points_total, s.points_outside};
  st.trace = {s.rays_traced, s.voxels_freed, s.voxels_marked_unknown_traced,
              s.voxels_skipped_out_of_bounds};
  st.occupied_count = s.occupied_count;
  st.freed_count = s.freed_count;
  st.shifted = s.shifted != 0;
  st.shift_offset = Eigen::Vector3i(s.shift_offset[0], s.shift_offset[1], s.shift_offset[2]);
  local_.set_origin(Eigen::Vector3d(s.origin[0], s.origin[1], s.origin[2]));
  local_stale_ = true;
  return st;
}

// MappingPipeline::integrate (pipeline.cpp:74-117)
PipelineStats MappingPipeline::integrate(const MeasurementFrame& frame) {
  if (!frame.t_wc.is_valid(1e-6)) throw std::invalid_argument("MeasurementFrame: invalid transform");
  const vxm_pose p = frame.t_wc.to_c();
  vxm_stats s{};
  activate(false);
  check(vxm_integrate_cloud(ctx_, frame.cloud.xs().data(), frame.cloud.ys().data(),
                            frame.cloud.zs().data(), frame.cloud.size(), &p, &s));
  return finish(s);
}

PipelineStats MappingPipeline::integrate_depth(const DepthImage& depth, const RigidTransform& t_wc) {
  if (depth.width != cfg_.camera.width || depth.height != cfg_.camera.height ||
      depth.depths.size() != static_cast<std::size_t>(depth.width) * depth.height)
    throw std::invalid_argument("depth_to_cloud: image size does not match camera model");
  if (!t_wc.is_valid(1e-6)) throw std::invalid_argument("MeasurementFrame: invalid transform");
  const vxm_pose p = t_wc.to_c();
  vxm_stats s{};
  activate(false);
  check(vxm_integrate_depth(ctx_, depth.depths.data(), &p, &s));
  return finish(s);
}

std::vector<PipelineStats> MappingPipeline::integrate_depth_sequence(const std::vector<DepthImage>& depths,
                                                                     const std::vector<RigidTransform>& poses) {
  if (depths.size() != poses.size()) throw std::invalid_argument("integrate_depth_sequence: one pose per frame");
  const std::size_t npix = static_cast<std::size_t>(cfg_.camera.width) * cfg_.camera.height;
  for (std::size_t i = 0; i < depths.size(); ++i) {
    const DepthImage& d = depths[i];
    if (d.width != cfg_.camera.width || d.height != cfg_.camera.height || d.depths.size() != npix)
      throw std::invalid_argument("depth_to_cloud: image size does not match camera model");
    if (!poses[i].is_valid(1e-6)) throw std::invalid_argument("MeasurementFrame: invalid transform");
  }
  std::vector<PipelineStats> out;
  out.reserve(depths.size());
  if (depths.empty()) return out;
  activate(true);
  std::vector<float> buf;
  std::vector<vxm_pose> p;
  std::vector<vxm_stats> st;
  for (std::size_t i0 = 0; i0 < depths.size(); i0 += kMaxFramesPerCall) {
    const std::size_t n = std::min<std::size_t>(kMaxFramesPerCall, depths.size() - i0);
    buf.resize(n * npix);
    p.resize(n);
    st.assign(n, vxm_stats{});
    for (std::size_t j = 0; j < n; ++j) {
      std::copy(depths[i0 + j].depths.begin(), depths[i0 + j].depths.end(), buf.begin() + j * npix);
      p[j] = poses[i0 + j].to_c();
    }
    check(vxm_integrate_depth_frames(seq_ctx_, buf.data(), p.data(), static_cast<int32_t>(n), st.data()));
    for (std::size_t j = 0; j < n; ++j) out.push_back(finish(st[j]));
  }
  return out;
}

const VoxelGrid& MappingPipeline::local_grid() const {
  if (local_stale_) {
    double origin[3];
    check(vxm_download_local(seq_active_ ? seq_ctx_ : ctx_, 0, local_.raw(), origin));
    local_.set_origin(Eigen::Vector3d(origin[0], origin[1], origin[2]));
    local_stale_ = false;
  }
  return local_;
}

// ---------------------------------------------------------------- grid io

void write_grid(const VoxelGrid& grid, std::ostream& out) {
  const GridSpec& g = grid.spec();
  const int dims[3] = {g.dims_x, g.dims_y, g.dims_z};
  const double origin[3] = {g.origin.x(), g.origin.y(), g.origin.z()};
  const std::string h = vxm_io::voxgrid_header(dims, g.vox_size, origin);
  out.write(h.data(), static_cast<std::streamsize>(h.size()));
  out.write(reinterpret_cast<const char*>(grid.raw()), static_cast<std::streamsize>(grid.size()));
  if (!out) throw std::runtime_error("write_grid: stream write failed");
}

void write_grid(const VoxelGrid& grid, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("write_grid: cannot open " + path);
  write_grid(grid, out);
}

VoxelGrid read_grid(std::istream& in) {
  // Consumes exactly the header (eight formatted fields and the one
  // character after them) and the cell bytes, leaving the stream positioned
  // after the grid as grid_io.cpp:31-63 does, so several grids (or a grid and
  // other data) can follow each other on one stream.
  vxm_io::VoxgridHeader h;
  std::string magic;
  in >> magic >> h.dims[0] >> h.dims[1] >> h.dims[2] >> h.vox_size >> h.origin[0] >> h.origin[1] >> h.origin[2];
  if (!in || magic != "VOXGRID1") throw std::runtime_error("read_grid: bad header");
  if (h.dims[0] <= 0 || h.dims[1] <= 0 || h.dims[2] <= 0 || !(h.vox_size > 0.0))
    throw std::runtime_error("read_grid: invalid dimensions");
  in.ignore(1);  // the newline ending the header
  std::string buf(h.cells(), '\0');
  in.read(buf.data(), static_cast<std::streamsize>(buf.size()));
  if (in.gcount() != static_cast<std::streamsize>(buf.size())) throw std::runtime_error("read_grid: truncated cell data");
  h.data_offset = 0;
  const std::string err = vxm_io::check_voxgrid_cells(buf.data(), buf.size(), h);
  if (!err.empty()) throw std::runtime_error(err);
  GridSpec spec;
  spec.dims_x = h.dims[0];
  spec.dims_y = h.dims[1];
  spec.dims_z = h.dims[2];
  spec.vox_size = h.vox_size;
  spec.grid_size_x = h.dims[0] * h.vox_size;
  spec.grid_size_y = h.dims[1] * h.vox_size;
  spec.grid_size_z = h.dims[2] * h.vox_size;
  spec.origin = Eigen::Vector3d(h.origin[0], h.origin[1], h.origin[2]);
  VoxelGrid grid(spec);
  std::memcpy(grid.raw(), buf.data() + h.data_offset, grid.size());
  return grid;
}

VoxelGrid read_grid(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("read_grid: cannot open " + path);
  return read_grid(in);
}

void MappingPipeline::restore_local_grid(const VoxelGrid& grid) {
  const GridSpec& a = grid.spec();
  const GridSpec& b = cfg_.grid;
  if (a.dims_x != b.dims_x || a.dims_y != b.dims_y || a.dims_z != b.dims_z || a.vox_size != b.vox_size)
    throw std::invalid_argument("restore_local_grid: grid layout differs from the pipeline's");
  const double origin[3] = {a.origin.x(), a.origin.y(), a.origin.z()};
  check(vxm_upload_local(seq_active_ ? seq_ctx_ : ctx_, 0, grid.raw(), origin));
  local_ = grid;
  local_stale_ = false;
}

void MappingPipeline::save_snapshot_async(const std::string& path) {
  check(vxm_snapshot_save_async(seq_active_ ? seq_ctx_ : ctx_, 0, path.c_str()));
}

void MappingPipeline::snapshot_wait() {
  for (vxm_ctx* c : {ctx_, seq_ctx_})
    if (c) check(vxm_snapshot_wait(c));
}

// ----------------------------------------------------------- kernel table

namespace kernels {
const KernelTable& cuda_table() {
  static const KernelTable t{vxm_kernel_merge, vxm_kernel_transform_voxelize, "cuda-sm100a"};
  return t;
}
// The reference's portable table (kernels_scalar.cpp:10-37), kept for
// callers that ask for it by name, e.g. as the baseline the reference's own
// test_kernels compares the dispatched table against. Nothing in this library
// selects it: dispatch() and every pipeline path run the sm_100a kernels.
namespace {
void merge_host(std::uint8_t* local, const std::uint8_t* measurement, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) {
    const std::uint8_t m = measurement[i];
    if (m != 0) local[i] = m == 3 ? 0 : m;
  }
}
void transform_voxelize_host(const double* xs, const double* ys, const double* zs, std::size_t n,
                             const double* rotation, const double* translation, double vox_size, std::int32_t* cx,
                             std::int32_t* cy, std::int32_t* cz) {
  std::int32_t* const out[3] = {cx, cy, cz};
  for (std::size_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      // ((t + R x) + R y) + R z, then floor of the true quotient, clamped
      double acc = translation[a];
      acc += rotation[3 * a] * xs[i];
      acc += rotation[3 * a + 1] * ys[i];
      acc += rotation[3 * a + 2] * zs[i];
      const double f = std::floor(acc / vox_size);
      out[a][i] = static_cast<std::int32_t>(std::min(std::max(f, -1e9), 1e9));
    }
  }
}
}  // namespace

const KernelTable& scalar_table() {
  static const KernelTable t{merge_host, transform_voxelize_host, "scalar"};
  return t;
}
const KernelTable& dispatch() { return cuda_table(); }
}  // namespace kernels

// ----------------------------------------------------------- pose helpers

namespace sim {
RigidTransform look_along_x(const Eigen::Vector3d& position) {
  Eigen::Matrix3d r;
  r(0, 0) = 0.0;  r(0, 1) = 0.0;  r(0, 2) = 1.0;
  r(1, 0) = -1.0; r(1, 1) = 0.0;  r(1, 2) = 0.0;
  r(2, 0) = 0.0;  r(2, 1) = -1.0; r(2, 2) = 0.0;
  return RigidTransform::from_rotation(r, position);
}

std::vector<RigidTransform> sweep_trajectory(const Eigen::Vector3d& start, const Eigen::Vector3d& end, int frames) {
  if (frames < 1) throw std::invalid_argument("sweep_trajectory: frames must be >= 1");
  std::vector<RigidTransform> poses;
  poses.reserve(static_cast<std::size_t>(frames));
  const Eigen::Vector3d span = end - start;
  for (int i = 0; i < frames; ++i) {
    const double s = frames == 1 ? 0.0 : static_cast<double>(i) / (frames - 1);
    poses.push_back(look_along_x(start + s * span));
  }
  return poses;
}
}  // namespace sim

}  // namespace voxmap
