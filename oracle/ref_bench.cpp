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

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numbers>
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
  T = std::min(T, S);

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
  std::vector<MappingPipeline> pipes;
  pipes.reserve(S);
  for (int s = 0; s < S; ++s) {
    PipelineConfig c = pc;
    c.grid = GridSpec::create_centered(gx, gy, gz, vs, poses[s % P].translation);
    pipes.emplace_back(c);
  }

  std::vector<std::vector<double>> lat(T);
  std::atomic<unsigned long long> checksum{0};
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
  std::printf(
      "{\"frames\": %d, \"seconds\": %.6f, \"frames_per_s\": %.3f, \"p50_ms\": %.4f, \"p99_ms\": %.4f, "
      "\"threads\": %d, \"streams\": %d, \"steps\": %d, \"checksum\": %llu}\n",
      S * K, secs, S * K / secs, percentile(all, 0.5) / 1000.0, percentile(all, 0.99) / 1000.0, T, S,
      K, static_cast<unsigned long long>(checksum.load()));
  return 0;
}
