// The reference's own unit cases (proj/tests/test_{kernels,integrator,
// raytracer,pipeline,grid_core}.cpp) written against the drop-in C++ API:
// same includes, same names, same known answers; the work runs on the GPU
// through libvoxmap_b200.so -> libvxm.so. Exit status = number of failures.
// Built by paper_2112_13169_b200/build.py, run by tests/test_dropin_cpp.py.

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "voxmap/kernels/kernels.hpp"
#include "voxmap/pipeline.hpp"

using namespace voxmap;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                             \
  do {                                                                       \
    if (c) {                                                                 \
      ++g_pass;                                                              \
    } else {                                                                 \
      ++g_fail;                                                              \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, ex)                                            \
  do {                                                                       \
    bool thrown_ = false;                                                    \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const ex&) {                                                    \
      thrown_ = true;                                                        \
    }                                                                        \
    CHECK(thrown_);                                                          \
  } while (0)

constexpr double kDeg = M_PI / 180.0;

static RigidTransform look_along_x(const Eigen::Vector3d& p) {
  Eigen::Matrix3d r;
  r.col(0) = Eigen::Vector3d(0.0, -1.0, 0.0);
  r.col(1) = Eigen::Vector3d(0.0, 0.0, -1.0);
  r.col(2) = Eigen::Vector3d(1.0, 0.0, 0.0);
  return RigidTransform::from_rotation(r, p);
}

static PipelineConfig small_config() {
  PipelineConfig cfg;
  cfg.grid = GridSpec::create_centered(6.0, 6.0, 3.0, 0.15, Eigen::Vector3d::Zero());
  cfg.camera = CameraModel{85.0 * kDeg, 101.0 * kDeg, 320, 240, 6.5};
  cfg.integrator = IntegratorConfig{0};
  cfg.depth = 4.0;
  cfg.parallelism = ExecutionMode::Sequential;
  return cfg;
}

static PointCloud wall_cloud(double depth) {
  PointCloud c;
  for (int j = -28; j <= 28; ++j)
    for (int i = -28; i <= 28; ++i) c.add(i * 0.05, j * 0.05, depth);
  return c;
}

static void kernels_cases() {
  const kernels::KernelTable& t = kernels::dispatch();
  CHECK(std::string(t.isa) == "cuda-sm100a");
  std::uint8_t loc[16], ms[16];
  for (int i = 0; i < 16; ++i) {
    loc[i] = static_cast<std::uint8_t>(i % 4);
    ms[i] = static_cast<std::uint8_t>(i / 4);
  }
  t.merge(loc, ms, 16);
  for (int i = 0; i < 16; ++i) {
    const int l = i % 4, m = i / 4;
    CHECK(loc[i] == (m == 0 ? l : (m == 3 ? 0 : m)));
  }
  t.merge(loc, ms, 0);  // n = 0 is allowed
  // floor semantics and the clamp (test_kernels.cpp:63-87)
  const double xs[5] = {0.05, 0.15, -0.05, 1e12, -1e12}, zs[5] = {0.0, 0.25, 0.0, 0.0, 0.0};
  const double ys[5] = {0, 0, 0, 0, 0};
  const double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, tr[3] = {0, 0, 0};
  std::int32_t cx[5], cy[5], cz[5];
  t.transform_voxelize(xs, ys, zs, 5, R, tr, 0.1, cx, cy, cz);
  CHECK(cx[0] == 0 && cx[1] == 1 && cx[2] == -1);
  CHECK(cz[0] == 0 && cz[1] == 2 && cz[2] == 0);
  CHECK(cx[3] == 1000000000 && cx[4] == -1000000000);
}

static void integrator_cases() {
  const GridSpec spec = GridSpec::create(1.5, 1.5, 1.5, 0.15);  // 10^3
  {
    VoxelGrid g(spec);
    PointCloud c;
    c.add(0.16, 0.0, 0.31);
    const PopulateStats st = populate_occupied(g, c, RigidTransform::identity(), IntegratorConfig{0});
    CHECK(st.points_total == 1 && st.points_outside == 0);
    CHECK(g.count(VoxelState::Occupied) == 1);
    CHECK(g.at({1, 0, 2}) == VoxelState::Occupied);
  }
  {
    VoxelGrid g(spec);
    PointCloud c;
    c.add(0.80, 0.80, 0.80);
    populate_occupied(g, c, RigidTransform::identity(), IntegratorConfig{2});
    CHECK(g.count(VoxelState::Occupied) == 125);
    CHECK(g.at({3, 3, 3}) == VoxelState::Occupied && g.at({7, 7, 7}) == VoxelState::Occupied);
    CHECK(g.at({2, 5, 5}) == VoxelState::Unknown);
  }
  {
    VoxelGrid g(spec);
    PointCloud c;
    c.add(0.01, 0.01, 0.01);
    populate_occupied(g, c, RigidTransform::identity(), IntegratorConfig{2});
    CHECK(g.count(VoxelState::Occupied) == 27);
  }
  {
    VoxelGrid g(spec);
    PointCloud c;
    c.add(-0.01, 0.30, 0.30);
    const PopulateStats st = populate_occupied(g, c, RigidTransform::identity(), IntegratorConfig{2});
    CHECK(st.points_outside == 1 && g.count(VoxelState::Occupied) == 0);
  }
  CHECK_THROWS_AS(IntegratorConfig{-1}.validate(), std::invalid_argument);
}

static void raytracer_cases() {
  const CameraModel cam{85.0 * kDeg, 101.0 * kDeg, 320, 240, 6.5};
  const RayBundle b = bundle_dimensions(cam, 6.5, 0.15);
  CHECK(b.vox_depth == 43 && b.vox_width == 79 && b.vox_height == 105 && b.ray_count() == 8295);
  CHECK_THROWS_AS(bundle_dimensions(cam, 0.0, 0.15), std::invalid_argument);
  // an empty grid traced by a bundle only ever writes Free
  VoxelGrid g(GridSpec::create(4.8, 4.8, 4.8, 0.15));
  const TraceStats st = trace_bundle(g, RayBundle{16, 13, 13}, look_along_x({0.3, 2.4, 2.4}), 0.15);
  CHECK(st.rays_traced == 169);
  CHECK(st.voxels_marked_unknown_traced == 0);
  CHECK(g.count(VoxelState::Free) > 0 && g.count(VoxelState::UnknownTraced) == 0);
}

static void pipeline_cases() {
  {
    MappingPipeline p(small_config());
    MeasurementFrame f;
    f.cloud = wall_cloud(2.0);
    f.t_wc = look_along_x(Eigen::Vector3d::Zero());
    const PipelineStats st = p.integrate(f);
    const VoxelGrid& local = p.local_grid();
    CHECK(st.occupied_count > 0 && st.trace.voxels_marked_unknown_traced > 0);
    for (int x = 21; x <= 32; ++x) CHECK(local.at({x, 20, 10}) == VoxelState::Free);
    CHECK(local.at({33, 20, 10}) == VoxelState::Occupied);
    for (int x = 34; x < 40; ++x) CHECK(local.at({x, 20, 10}) == VoxelState::Unknown);
    CHECK(st.occupied_count == local.count(VoxelState::Occupied));
    CHECK(st.freed_count == local.count(VoxelState::Free));
    f.cloud = wall_cloud(2.75);
    p.integrate(f);
    CHECK(p.local_grid().at({33, 20, 10}) == VoxelState::Free);
    CHECK(p.local_grid().at({38, 20, 10}) == VoxelState::Occupied);
  }
  {
    PipelineConfig cfg = small_config();
    MappingPipeline p(cfg);
    MeasurementFrame f;
    f.t_wc = look_along_x({0.05, 0.0, 0.0});
    CHECK(!p.integrate(f).shifted);
    const GridSpec before = p.local_grid().spec();
    f.t_wc = look_along_x({0.4, 0.0, 0.0});
    const PipelineStats st = p.integrate(f);
    CHECK(st.shifted && st.shift_offset == Eigen::Vector3i(3, 0, 0));
    CHECK(st.shift_offset == shift_offset_for_center(before, {0.4, 0.0, 0.0}));
    CHECK(p.local_grid().spec().origin.isApprox(before.origin + Eigen::Vector3d(0.45, 0, 0)));
  }
  {
    MappingPipeline p(small_config());
    MeasurementFrame f;
    f.t_wc.rotation = Eigen::Matrix3d::Identity() * 2.0;
    CHECK_THROWS_AS(p.integrate(f), std::invalid_argument);
  }
  {
    // the fused depth entry equals integrate(depth_to_cloud(depth))
    PipelineConfig cfg = small_config();
    cfg.integrator.vox_inf = 1;
    MappingPipeline a(cfg), b(cfg);
    DepthImage img(320, 240);
    for (int v = 0; v < 240; ++v)
      for (int u = 0; u < 320; ++u) img.at(u, v) = (u / 40 + v / 30) % 3 == 0 ? 0.0f : 1.5f + 0.004f * u;
    const RigidTransform pose = look_along_x({0.02, -0.1, 0.03});
    MeasurementFrame f;
    f.cloud = depth_to_cloud(img, cfg.camera);
    f.t_wc = pose;
    const PipelineStats sa = a.integrate(f);
    const PipelineStats sb = b.integrate_depth(img, pose);
    CHECK(sa.populate.points_total == sb.populate.points_total);
    CHECK(sa.trace.voxels_freed == sb.trace.voxels_freed);
    CHECK(a.local_grid() == b.local_grid());
  }
  {
    // extension: integrate_depth_sequence == integrate_depth frame by frame,
    // across the 64-frame call boundary, interleaved with single frames
    PipelineConfig cfg = small_config();
    cfg.integrator.vox_inf = 2;
    MappingPipeline seq(cfg), one(cfg);
    std::vector<DepthImage> imgs;
    std::vector<RigidTransform> poses;
    for (int k = 0; k < 70; ++k) {
      DepthImage img(320, 240);
      for (int v = 0; v < 240; ++v)
        for (int u = 0; u < 320; ++u)
          img.at(u, v) = ((u + 3 * k) / 40 + v / 30) % 4 == 0 ? 0.0f : 1.2f + 0.003f * u + 0.01f * (k % 5);
      imgs.push_back(img);
      poses.push_back(look_along_x({0.04 * (k % 9), 0.11 * k - 3.0, 0.02 * (k % 3)}));
    }
    const std::vector<PipelineStats> ss = seq.integrate_depth_sequence(imgs, poses);
    bool same = ss.size() == imgs.size();
    for (std::size_t k = 0; k < imgs.size() && same; ++k) {
      const PipelineStats so = one.integrate_depth(imgs[k], poses[k]);
      same = so.occupied_count == ss[k].occupied_count && so.freed_count == ss[k].freed_count &&
             so.trace.voxels_freed == ss[k].trace.voxels_freed && so.shifted == ss[k].shifted &&
             so.shift_offset == ss[k].shift_offset && so.populate.points_total == ss[k].populate.points_total;
    }
    CHECK(same);
    CHECK(seq.local_grid() == one.local_grid());
    CHECK(seq.local_grid().spec().origin == one.local_grid().spec().origin);
    const PipelineStats a1 = seq.integrate_depth(imgs[3], poses[60]);
    const PipelineStats b1 = one.integrate_depth(imgs[3], poses[60]);
    CHECK(a1.freed_count == b1.freed_count);
    CHECK(seq.local_grid() == one.local_grid());
    CHECK_THROWS_AS(seq.integrate_depth_sequence(imgs, {}), std::invalid_argument);
  }
}

static void gridio_cases() {
  // VOXGRID1 round trip (grid_io.hpp) and checkpoint/resume of a pipeline
  PipelineConfig cfg = small_config();
  MappingPipeline a(cfg);
  DepthImage img(320, 240);
  for (int v = 0; v < 240; ++v)
    for (int u = 0; u < 320; ++u) img.at(u, v) = (u / 40 + v / 30) % 3 == 0 ? 0.0f : 1.5f + 0.004f * u;
  a.integrate_depth(img, look_along_x({0.0, 0.2, 0.0}));
  a.integrate_depth(img, look_along_x({0.1, 0.4, 0.0}));
  const std::string path = "/tmp/vxm_dropin_snapshot.vox";
  write_grid(a.local_grid(), path);
  const VoxelGrid back = read_grid(path);
  CHECK(back == a.local_grid());
  CHECK(back.spec().origin == a.local_grid().spec().origin);
  MappingPipeline b(cfg);
  b.restore_local_grid(back);
  const PipelineStats sa = a.integrate_depth(img, look_along_x({0.2, 0.55, 0.0}));
  const PipelineStats sb = b.integrate_depth(img, look_along_x({0.2, 0.55, 0.0}));
  CHECK(sa.freed_count == sb.freed_count && sa.occupied_count == sb.occupied_count);
  CHECK(a.local_grid() == b.local_grid());
  CHECK_THROWS_AS(read_grid(std::string("/tmp/definitely_missing_grid.vox")), std::runtime_error);
  VoxelGrid other(GridSpec::create(1.0, 1.0, 1.0, 0.1));
  CHECK_THROWS_AS(b.restore_local_grid(other), std::invalid_argument);
}

static void grid_cases() {
  const GridSpec spec = GridSpec::create_centered(15.0, 15.0, 3.0, 0.15, Eigen::Vector3d::Zero());
  CHECK(spec.dims_x == 100 && spec.dims_y == 100 && spec.dims_z == 20);
  CHECK(linear_index_unchecked({3, 2, 1}, GridSpec::create(15.0, 15.0, 3.0, 0.15)) == 10203);
  VoxelGrid g(GridSpec::create(16 * 0.15, 16 * 0.15, 16 * 0.15, 0.15));
  for (std::size_t i = 0; i < g.size(); ++i) g.raw()[i] = static_cast<std::uint8_t>((i * 7) % 4);
  const Eigen::Vector3i off(3, -2, 1);
  const VoxelGrid s = shift_grid_by(g, off);
  CHECK(s.at({0, 2, 0}) == g.at({3, 0, 1}));
  CHECK(s.at({15, 0, 0}) == VoxelState::Unknown);
  const VoxelGrid back = shift_grid_by(s, -off);
  CHECK(back.spec().origin.isApprox(g.spec().origin));
  CHECK_THROWS_AS(GridSpec::create(0.0, 1.0, 1.0, 0.1), std::invalid_argument);
}

int main() {
  try {
    kernels_cases();
    integrator_cases();
    raytracer_cases();
    pipeline_cases();
    grid_cases();
    gridio_cases();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "FAIL: uncaught %s\n", e.what());
    ++g_fail;
  }
  std::printf("drop-in C++ cases: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
