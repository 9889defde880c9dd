// ORACLE / CPU BASELINE ONLY — the reference arm of bench.py.
//
// Runs the UNMODIFIED reference voxmap library (oracle/_ref, built from
// /root/reference/proj/src) on the same synthetic workload as bench.py: S
// independent sensor streams, each a Sequential MappingPipeline (the
// bit-exact mode), one frame per stream per step. Streams are spread over T
// host threads (one Sequential pipeline per core). Each
// frame is depth_to_cloud + integrate, as the reference's callers do
// (tools/voxmap_cli.cpp:117-126). Frames come from the reference's own
// generator: render_depth(box_field(seed), look_along_x(pose)), rendered
// before timing.
//
// Frame rule shared with bench.py: pool of P poses y_j = y0 + 0.1001 j;
// stream s at step k uses pool frame (s + k) mod P.
//
// Prints one JSON object: frames/s over the timed steps, per-frame latency
// percentiles (linear interpolation as proj/src/sim/bench.cpp:19-25).
//
// Parity dumps (bench.py and tests/test_gpu_bench_parity.py compare the GPU
// against them): --dump-stats FILE writes, for every step (warm-up steps
// included) and stream, the nine PipelineStats counters as int64
// (points_total, points_outside, rays_traced, voxels_freed,
// voxels_marked_unknown_traced, voxels_skipped_out_of_bounds,
// occupied_count, freed_count, shifted); --dump-grids FILE writes every
// stream's final local grid (cells) followed by all origins (3 doubles each).
//
// Latency mode (--latency-frames N > 0): one stream, N frames of the pool
// rule (stream 0), depth_to_cloud + integrate timed per frame after 5
// warm-up frames as sim::measure does (proj/src/sim/bench.cpp:44-55), with
// --parallel 0 (Sequential, one core) or 1 (DataParallel, OpenMP over
// --threads threads, AVX2 kernels via dispatch()).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <omp.h>
#include <string>
#include <thread>
#include <vector>

#include "voxmap/pipeline.hpp"
#include "voxmap/sim/render.hpp"
#include "voxmap/sim/scene.hpp"
#include "voxmap/sim/trajectory.hpp"

using namespace voxmap;
using Clock = std::chrono::steady_clock;

namespace {

double arg_d(int argc, char** argv, const char* k, double def) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], k) == 0) return std::atof(argv[i + 1]);
  return def;
}

double percentile(std::vector<double> v, double q) {
  std::sort(v.begin(), v.end());
  const double pos = q * static_cast<double>(v.size() - 1);
  const auto lo = static_cast<size_t>(pos);
  const size_t hi = std::min(lo + 1, v.size() - 1);
  return v[lo] + (pos - static_cast<double>(lo)) * (v[hi] - v[lo]);
}

}  // namespace

int main(int argc, char** argv) {
  const int W = static_cast<int>(arg_d(argc, argv, "--width", 640));
  const int H = static_cast<int>(arg_d(argc, argv, "--height", 480));
  const double vs = arg_d(argc, argv, "--vox", 0.1);
  const double gx = arg_d(argc, argv, "--gx", 10.0), gy = arg_d(argc, argv, "--gy", 10.0),
               gz = arg_d(argc, argv, "--gz", 5.0);
  const double depth = arg_d(argc, argv, "--depth", 5.0);
  const int vox_inf = static_cast<int>(arg_d(argc, argv, "--vox-inf", 2));
  const int S = static_cast<int>(arg_d(argc, argv, "--streams", 64));
  const int K = static_cast<int>(arg_d(argc, argv, "--steps", 4));
  const int WU = static_cast<int>(arg_d(argc, argv, "--warmup", 1));
  const int P = static_cast<int>(arg_d(argc, argv, "--pool", 16));
  const double y0 = arg_d(argc, argv, "--y0", -0.8);
  const unsigned seed = static_cast<unsigned>(arg_d(argc, argv, "--seed", 1));
  int T = static_cast<int>(arg_d(argc, argv, "--threads", 0));
  if (T <= 0) T = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int T_all = T;
  T = std::min(T, S);
  const int lat_frames = static_cast<int>(arg_d(argc, argv, "--latency-frames", 0));
  const bool parallel = arg_d(argc, argv, "--parallel", 0) != 0;
  const char* dump_stats = nullptr;
  const char* dump_grids = nullptr;
  for (int i = 1; i + 1 < argc; ++i) {
    if (std::strcmp(argv[i], "--dump-stats") == 0) dump_stats = argv[i + 1];
    if (std::strcmp(argv[i], "--dump-grids") == 0) dump_grids = argv[i + 1];
  }

  CameraModel cam;
  cam.fov_x = 85.0 * std::numbers::pi / 180.0;
  cam.fov_y = 101.0 * std::numbers::pi / 180.0;
  cam.width = W;
  cam.height = H;
  cam.max_depth = depth;

  // frame pool (reference renderer, untimed)
  const sim::Scene scene = sim::Scene::box_field(seed);
  std::vector<RigidTransform> poses(P);
  std::vector<DepthImage> frames(P);
  for (int j = 0; j < P; ++j) poses[j] = sim::look_along_x(Eigen::Vector3d(0.0, y0 + 0.1001 * j, 0.0));
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (int j = t; j < P; j += T) frames[j] = sim::render_depth(scene, poses[j], cam, ExecutionMode::Sequential);
      });
    for (auto& x : th) x.join();
  }

  PipelineConfig pc;
  pc.camera = cam;
  pc.integrator.vox_inf = vox_inf;
  pc.depth = depth;
  pc.tracer_mode = TracerMode::Bundled;
  pc.parallelism = ExecutionMode::Sequential;

  if (lat_frames > 0) {
    const ExecutionMode mode = parallel ? ExecutionMode::DataParallel : ExecutionMode::Sequential;
    omp_set_num_threads(parallel ? T_all : 1);
    PipelineConfig c = pc;
    c.parallelism = mode;
    c.grid = GridSpec::create_centered(gx, gy, gz, vs, poses[0].translation);
    MappingPipeline pipe(c);
    std::vector<double> us;
    us.reserve(static_cast<size_t>(lat_frames));
    constexpr int kWarm = 5;  // sim::measure's warm-up
    for (int k = 0; k < kWarm + lat_frames; ++k) {
      const int j = k % P;
      const auto f0 = Clock::now();
      MeasurementFrame f;
      f.cloud = depth_to_cloud(frames[j], cam, mode);
      f.t_wc = poses[j];
      pipe.integrate(f);
      const double t = std::chrono::duration<double, std::micro>(Clock::now() - f0).count();
      if (k >= kWarm) us.push_back(t);
    }
    double sum = 0.0;
    for (double v : us) sum += v;
    std::printf(
        "{\"mode\": \"%s\", \"frames\": %d, \"threads\": %d, \"p50_ms\": %.4f, \"p99_ms\": %.4f, "
        "\"mean_ms\": %.4f}\n",
        parallel ? "DataParallel" : "Sequential", lat_frames, parallel ? T_all : 1, percentile(us, 0.5) / 1000.0,
        percentile(us, 0.99) / 1000.0, sum / us.size() / 1000.0);
    return 0;
  }
  std::vector<MappingPipeline> pipes;
  pipes.reserve(S);
  for (int s = 0; s < S; ++s) {
    PipelineConfig c = pc;
    c.grid = GridSpec::create_centered(gx, gy, gz, vs, poses[s % P].translation);
    pipes.emplace_back(c);
  }

  std::vector<std::vector<double>> lat(T);
  std::atomic<unsigned long long> checksum{0};
  std::vector<long long> stats_dump(dump_stats ? static_cast<size_t>(WU + K) * S * 9 : 0);
  auto run_steps = [&](int k0, int nsteps, bool record) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        unsigned long long cs = 0;
        for (int k = k0; k < k0 + nsteps; ++k) {
          for (int s = t; s < S; s += T) {
            const int j = (s + k) % P;
            const auto f0 = Clock::now();
            MeasurementFrame f;
            f.cloud = depth_to_cloud(frames[j], cam, ExecutionMode::Sequential);
            f.t_wc = poses[j];
            const PipelineStats st = pipes[s].integrate(f);
            const double us = std::chrono::duration<double, std::micro>(Clock::now() - f0).count();
            if (record) lat[t].push_back(us);
            cs += st.occupied_count * 1000003ull + st.freed_count;
            if (dump_stats) {
              long long* d = &stats_dump[(static_cast<size_t>(k) * S + s) * 9];
              d[0] = static_cast<long long>(st.populate.points_total);
              d[1] = static_cast<long long>(st.populate.points_outside);
              d[2] = static_cast<long long>(st.trace.rays_traced);
              d[3] = static_cast<long long>(st.trace.voxels_freed);
              d[4] = static_cast<long long>(st.trace.voxels_marked_unknown_traced);
              d[5] = static_cast<long long>(st.trace.voxels_skipped_out_of_bounds);
              d[6] = static_cast<long long>(st.occupied_count);
              d[7] = static_cast<long long>(st.freed_count);
              d[8] = st.shifted ? 1 : 0;
            }
          }
        }
        checksum += cs;
      });
    for (auto& x : th) x.join();
  };
  run_steps(0, WU, false);
  const auto t0 = Clock::now();
  run_steps(WU, K, true);
  const double secs = std::chrono::duration<double>(Clock::now() - t0).count();
  std::vector<double> all;
  for (auto& v : lat) all.insert(all.end(), v.begin(), v.end());
  if (dump_stats) {
    FILE* f = std::fopen(dump_stats, "wb");
    if (!f || std::fwrite(stats_dump.data(), sizeof(long long), stats_dump.size(), f) != stats_dump.size()) return 2;
    std::fclose(f);
  }
  if (dump_grids) {
    FILE* f = std::fopen(dump_grids, "wb");
    if (!f) return 2;
    for (int s = 0; s < S; ++s) {
      const VoxelGrid& g = pipes[s].local_grid();
      if (std::fwrite(g.raw(), 1, g.size(), f) != g.size()) return 2;
    }
    for (int s = 0; s < S; ++s) {
      const Eigen::Vector3d o = pipes[s].local_grid().spec().origin;
      const double od[3] = {o.x(), o.y(), o.z()};
      if (std::fwrite(od, sizeof(double), 3, f) != 3) return 2;
    }
    std::fclose(f);
  }
  std::printf(
      "{\"frames\": %d, \"seconds\": %.6f, \"frames_per_s\": %.3f, \"p50_ms\": %.4f, \"p99_ms\": %.4f, "
      "\"threads\": %d, \"streams\": %d, \"steps\": %d, \"checksum\": %llu}\n",
      S * K, secs, S * K / secs, percentile(all, 0.5) / 1000.0, percentile(all, 0.99) / 1000.0, T, S,
      K, static_cast<unsigned long long>(checksum.load()));
  return 0;
}
