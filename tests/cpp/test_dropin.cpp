// C++ drop-in check: the reference's own known-answer tests
// (proj/tests/test_semidense.cpp, test_fusion.cpp, test_pipeline.cpp),
// restated against include/dfuse/*.hpp, which forward to the CUDA library.
// Built and run by tests/test_cpp_dropin.py; exit code = failed checks.
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <vector>
#include <random>

#include "dfuse/session.hpp"

using namespace dfuse;

static int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(cond)) {                                                        \
      ++g_failed;                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
    }                                                                     \
  } while (0)

template <class F>
static bool throws_code(F&& f, Err code) {
  try {
    f();
  } catch (const Error& e) {
    return e.code() == code;
  }
  return false;
}

// analytic slanted textured plane (the reference fixture's construction,
// tests/support/synthetic.hpp:25-72, restated)
struct Plane {
  CameraIntrinsics K{200.0, 200.0, 127.5, 95.5, 256, 192};
  double z0 = 2.0, ax = 0.25, ay = -0.15, env_gain = 2.2, env_bias = 0.5;
  double tex(double u, double v) const {
    const double base = 0.5 + 0.17 * std::sin(1.3 * u - 0.7 * v);
    const double s = std::sin(2.3 * u + 1.1 * v) * std::sin(1.7 * v - 0.9 * u + 0.4);
    const double env = std::clamp(env_gain * s + env_bias, 0.0, 1.0);
    const double hi = 0.13 * std::sin(31.0 * u + 7.0 * v) + 0.11 * std::sin(23.0 * u - 17.0 * v) +
                      0.08 * std::sin(43.0 * u + 29.0 * v);
    return std::clamp(base + env * hi, 0.02, 0.98);
  }
  IntensityImage render(const Eigen::Vector3d& origin, Raster<double>* depth = nullptr) const {
    IntensityImage img(K.width, K.height);
    for (int y = 0; y < K.height; ++y)
      for (int x = 0; x < K.width; ++x) {
        const Eigen::Vector3d d((x - K.cx) / K.fx, (y - K.cy) / K.fy, 1.0);
        const Eigen::Vector3d n(-ax, -ay, 1.0);
        const double t = (z0 - n.dot(origin)) / n.dot(d);
        const Eigen::Vector3d P = origin + t * d;
        img.raster().at(x, y) = static_cast<float>(tex(P.x(), P.y()));
        if (depth) depth->at(x, y) = t;
      }
    return img;
  }
};

static Pose translated(double x, double y = 0.0) {
  Pose p;
  p.translation = Eigen::Vector3d(x, y, 0.0);
  return p;
}

static void semidense_kats() {
  // test_semidense.cpp:51-78
  IntensityImage flat(32, 24, 0.5f);
  const Mask m0 = texture_mask(flat, 0.02);
  int any = 0;
  for (std::size_t i = 0; i < m0.size(); ++i) any += m0[i];
  CHECK(any == 0);
  IntensityImage step(16, 8, 0.0f);
  for (int y = 0; y < 8; ++y)
    for (int x = 8; x < 16; ++x) step.raster().at(x, y) = 0.5f;
  const Mask m1 = texture_mask(step, 0.1);
  bool ok = true;
  for (int y = 0; y < 8; ++y)
    for (int x = 0; x < 16; ++x)
      ok = ok && (m1.at(x, y) == ((y >= 1 && y <= 6 && (x == 7 || x == 8)) ? 1 : 0));
  CHECK(ok);
  CHECK(throws_code([] { texture_mask(IntensityImage(8, 8, 0.f), 0.0); }, Err::InvalidArgument));

  // test_semidense.cpp:80-88, 113-136
  Plane sc;
  sc.ax = sc.ay = 0.0;
  sc.env_gain = 10.0;
  const IntensityImage I0 = sc.render(Eigen::Vector3d::Zero());
  std::array<double, 5> e{};
  CHECK(photometric_error_5pt(I0, I0, {100.5, 80.25}, 1.7, Pose::identity(), Pose::identity(),
                              sc.K, e) == EpipolarStatus::Ok);
  for (double v : e) CHECK(std::abs(v) < 1e-12);
  const auto r0 = search_depth(I0, I0, {100, 90}, std::nullopt, Pose::identity(),
                               Pose::identity(), sc.K);
  CHECK(r0.status == EpipolarStatus::DegenerateBaseline);
  sc.K = {100.0, 100.0, 127.5, 95.5, 256, 192};
  const IntensityImage J0 = sc.render(Eigen::Vector3d::Zero());
  const IntensityImage J1 = sc.render(Eigen::Vector3d(0.1, 0, 0));
  // strongest-gradient pixel away from the borders (test_semidense.cpp:33-47)
  PixelCoord strong{64, 64};
  double best = -1.0;
  const Raster<float>& v = J0.raster();
  for (int y = 20; y < J0.height() - 20; ++y)
    for (int x = 20; x < J0.width() - 20; ++x) {
      const double gx = 0.5 * (v.at(x + 1, y) - v.at(x - 1, y));
      const double gy = 0.5 * (v.at(x, y + 1) - v.at(x, y - 1));
      if (gx * gx + gy * gy > best) {
        best = gx * gx + gy * gy;
        strong = {double(x), double(y)};
      }
    }
  const auto r1 = search_depth(J0, J1, strong, std::nullopt, Pose::identity(), translated(0.1),
                               sc.K, SearchConfig{1.0, 4.0});
  CHECK(r1.ok());
  CHECK(r1.obs.depth > 1.95 && r1.obs.depth < 2.05 && r1.obs.variance > 0.0);

  // test_semidense.cpp:174-203 (host helpers)
  const std::array<double, 5> e1{0.1, 0.1, 0.1, 0.1, 0.1}, e2{0.2, 0.2, 0.2, 0.2, 0.2};
  const auto J = jacobian_fd(e1, e2, 2.0, 2.05);
  CHECK(std::abs(J[0] - 2.0) < 1e-9);
  CHECK(throws_code([&] { jacobian_fd(e1, e2, 2.0, 2.0); }, Err::ZeroBaselineStep));
  CHECK(std::abs(observation_variance({1, 1, 1, 1, 1}) - 0.2) < 1e-15);
  CHECK(observation_variance({0, 0, 0, 0, 0}) < 0.0);

  // test_semidense.cpp:205-222
  SemiDenseMap map = SemiDenseMap::empty(8, 6);
  map = update_semidense(std::move(map), {{{2, 3}, 2.0, {}, {}, 0.04}});
  CHECK(map.inlier_count == 1 && map.depth.at(2, 3) == 2.0 && map.variance.at(2, 3) == 0.04);
  map = update_semidense(std::move(map), {{{2, 3}, 2.2, {}, {}, 0.04}});
  CHECK(std::abs(map.depth.at(2, 3) - 2.1) < 1e-12 && std::abs(map.variance.at(2, 3) - 0.02) < 1e-12);
  SemiDenseMap gate = SemiDenseMap::empty(8, 6);
  gate = update_semidense(std::move(gate), {{{1, 1}, 2.0, {}, {}, 0.0001}});
  gate = update_semidense(std::move(gate), {{{1, 1}, 10.0, {}, {}, 0.04}});
  CHECK(gate.depth.at(1, 1) == 2.0 && gate.variance.at(1, 1) == 0.0001);

  // test_semidense.cpp:238-261 (host)
  SemiDenseMap pol = SemiDenseMap::empty(4, 4);
  pol.inlier_count = 500;
  CHECK(!should_create_keyframe(Pose::identity(), Pose::identity(), 2.0, pol, {0.1, 100}));
  CHECK(should_create_keyframe(Pose::identity(), translated(0.4), 2.0, pol, {0.1, 100}));
}

struct Problem {
  FusionState st;
  SemiDenseMap semi;
  PredictionSet pred;
};

static Problem blank(int w, int h) {  // test_fusion.cpp:16-29
  Problem p;
  p.st = {Raster<double>(w, h, 0.0), 1.0, 0};
  p.semi = SemiDenseMap::empty(w, h);
  p.pred = {Raster<double>(w, h, 0.0), Raster<double>(w, h, 1.0), Raster<double>(w, h, 0.0),
            Raster<double>(w, h, 1.0), Raster<double>(w, h, 0.0), Raster<double>(w, h, 1.0),
            200.0};
  return p;
}

static RobustConfig quadratic() {  // test_fusion.cpp:31-37
  RobustConfig c;
  c.delta_semi = c.delta_net = c.delta_grad = 1e9;
  c.cg_tol = 1e-12;
  c.cg_max_iters = 1000;
  return c;
}

static void fusion_kats() {
  {  // test_fusion.cpp:76-83
    Problem p = blank(1, 1);
    p.st.log_depth[0] = 0.25;
    p.pred.log_depth[0] = 0.05;
    const auto eq = assemble_normal_equations(p.st, p.semi, p.pred, {}, FusionMode::Full);
    CHECK(std::abs(eq.H.diag[0] - 1.0) < 1e-15 && std::abs(eq.b[0] + 0.2) < 1e-15);
  }
  {  // test_fusion.cpp:85-99
    Problem p = blank(2, 1);
    p.pred.log_depth[0] = 0.4;
    p.pred.log_depth_var[0] = 1e-10;
    p.pred.log_depth_var[1] = 1e12;
    p.pred.grad_x[0] = std::log(2.0);
    RobustConfig c = quadratic();
    c.gn_iterations = 3;
    c.estimate_scale = false;
    const FusionState out = optimize(p.st, p.semi, p.pred, c, FusionMode::Full);
    CHECK(std::abs(out.log_depth[0] - 0.4) < 1e-8);
    CHECK(std::abs(out.log_depth[1] - (0.4 + std::log(2.0))) < 1e-6);
  }
  {  // test_fusion.cpp:120-125
    Problem p = blank(3, 3);
    const auto eq = assemble_normal_equations(p.st, p.semi, p.pred, {}, FusionMode::Full);
    for (double v : solve_depth_step(eq, {})) CHECK(v == 0.0);
  }
  {  // test_fusion.cpp:162-196
    RobustConfig c;
    c.delta_semi = 10.0;
    Problem q = blank(2, 1);
    q.semi.valid[0] = q.semi.valid[1] = 1;
    q.semi.inlier_count = 2;
    q.semi.depth[0] = q.semi.depth[1] = 1.0;
    q.semi.variance[0] = 1.0;
    q.semi.variance[1] = 1.0 / 3.0;
    q.st.log_depth[0] = std::log(2.0);
    const double s = solve_scale_step(q.st, q.semi, c);
    CHECK(std::abs(s - 1.189207) < 1e-6);
    CHECK(throws_code([&] { solve_scale_step(q.st, SemiDenseMap::empty(2, 1), c); },
                      Err::NoSemiDenseSupport));
  }
  {  // test_fusion.cpp:226-239
    Problem p = blank(1, 1);
    p.semi.valid[0] = 1;
    p.semi.depth[0] = 1.0;
    p.semi.variance[0] = 1.0;
    p.semi.inlier_count = 1;
    p.pred.log_depth[0] = 1.0;
    p.st.log_depth[0] = 1.0;
    RobustConfig c = quadratic();
    c.estimate_scale = false;
    c.gn_iterations = 2;
    CHECK(std::abs(optimize(p.st, p.semi, p.pred, c, FusionMode::Full).log_depth[0] - 0.5) < 1e-9);
  }
  {  // test_fusion.cpp:354-359, 392-398
    std::mt19937_64 rng(12);
    std::uniform_real_distribution<double> u(0.5, 2.0);
    Problem p = blank(6, 4);
    for (std::size_t i = 0; i < 24; ++i) p.st.log_depth[i] = std::log(u(rng));
    const auto eq = assemble_normal_equations(p.st, p.semi, p.pred, {}, FusionMode::NoPairwise);
    bool zero = true;
    for (double v : eq.H.right) zero = zero && v == 0.0;
    for (double v : eq.H.down) zero = zero && v == 0.0;
    CHECK(zero);
    const FusionState s = init_state(p.pred);
    CHECK(s.log_depth == p.pred.log_depth && s.scale == 1.0 && s.iteration == 0);
  }
  {  // test_fusion.cpp:400-411
    NormalEquations eq;
    eq.H = StencilMatrix(2, 2);
    eq.b.assign(4, 1.0);
    eq.H.diag = {1.0, 0.0, 1.0, 1.0};
    CHECK(throws_code([&] { solve_depth_step(eq, {}); }, Err::CgDivergence));
  }
  {  // StencilMatrix::apply against the definition (fusion.hpp:120-135)
    StencilMatrix H(3, 2);
    for (int i = 0; i < 6; ++i) {
      H.diag[i] = 2.0 + i;
      H.right[i] = -0.5;
      H.down[i] = -0.25;
    }
    const double x[6] = {1, 2, 3, 4, 5, 6};
    double y[6];
    H.apply(x, y);
    CHECK(y[0] == 2.0 * 1 + -0.5 * 2 + -0.25 * 4);
    CHECK(y[4] == 6.0 * 5 + -0.5 * 6 + -0.5 * 4 + -0.25 * 2);
  }
}

static void session_kats() {  // test_pipeline.cpp:57-73, 92-102
  Plane sc;
  Raster<double> gt(sc.K.width, sc.K.height, 0.0);
  const IntensityImage I0 = sc.render(Eigen::Vector3d::Zero(), &gt);
  PredictionSet pred{Raster<double>(sc.K.width, sc.K.height, 0.0),
                     Raster<double>(sc.K.width, sc.K.height, 0.04),
                     Raster<double>(sc.K.width, sc.K.height, 0.0),
                     Raster<double>(sc.K.width, sc.K.height, 0.0025),
                     Raster<double>(sc.K.width, sc.K.height, 0.0),
                     Raster<double>(sc.K.width, sc.K.height, 0.0025), sc.K.fx};
  for (int y = 0; y < sc.K.height; ++y)
    for (int x = 0; x < sc.K.width; ++x) {
      pred.log_depth.at(x, y) = static_cast<float>(std::log(gt.at(x, y)));
      if (x + 1 < sc.K.width)
        pred.grad_x.at(x, y) = static_cast<float>(std::log(gt.at(x + 1, y) / gt.at(x, y)));
      if (y + 1 < sc.K.height)
        pred.grad_y.at(x, y) = static_cast<float>(std::log(gt.at(x, y + 1) / gt.at(x, y)));
    }
  DeviceKeyframe kf(sc.K, I0, pred, 0.02);
  const FusionState st0 = kf.fusion();
  CHECK(st0.iteration == 0 && st0.scale == 1.0 && st0.log_depth == pred.log_depth);
  RobustConfig robust;
  const auto r = kf.process_frame(Pose::identity(), translated(0.04), sc.render({0.04, 0, 0}),
                                  SearchConfig{1.0, 4.0}, robust, FusionMode::Full);
  CHECK(r.observations > 1000);
  CHECK(r.inlier_count == r.observations);
  CHECK(kf.fusion().iteration == robust.gn_iterations);
  const auto r2 = kf.process_frame(Pose::identity(), Pose::identity(), I0, SearchConfig{1.0, 4.0},
                                   robust, FusionMode::Full);
  CHECK(r2.observations == 0 && kf.fusion().iteration == 2 * robust.gn_iterations);

  // the pipelined host-frame path gives the synchronous path's states
  {
    DeviceKeyframe ka(sc.K, I0, pred, 0.02), kb(sc.K, I0, pred, 0.02);
    const IntensityImage f1 = sc.render({0.04, 0, 0}), f2 = sc.render({0.03, 0.01, 0});
    const auto g1 = make_epipolar_geometry(Pose::identity(), translated(0.04), sc.K);
    const auto g2 = make_epipolar_geometry(Pose::identity(), translated(0.03, 0.01), sc.K);
    ka.process_frame(g1, f1, SearchConfig{1.0, 4.0}, robust, FusionMode::Full);
    const FusionState s1 = ka.fusion();
    const auto ra = ka.process_frame(g2, f2, SearchConfig{1.0, 4.0}, robust, FusionMode::Full);
    const FusionState s2 = ka.fusion();
    std::vector<double> o1(s1.log_depth.size()), o2(s1.log_depth.size());
    kb.submit_frame(g1, f1.raster().data(), SearchConfig{1.0, 4.0}, robust, FusionMode::Full,
                    o1.data());
    kb.submit_frame(g2, f2.raster().data(), SearchConfig{1.0, 4.0}, robust, FusionMode::Full,
                    o2.data());
    const auto rb = kb.finish();
    CHECK(rb.observations == ra.observations && rb.stereo_frames == 2);
    CHECK(std::equal(o1.begin(), o1.end(), s1.log_depth.data()));
    CHECK(std::equal(o2.begin(), o2.end(), s2.log_depth.data()));
  }

  // make_keyframe from a DFPRED file (pipeline.hpp:133-147): written the way
  // save_predictions does (predictions.hpp:125-145), read back on the device
  const std::string path = "/tmp/dfuse_dropin_test.dfpred";
  {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    const uint32_t head[5] = {1u, (uint32_t)sc.K.width, (uint32_t)sc.K.height, 6u,
                              (uint32_t)std::lround(sc.K.fx * 1000.0)};
    out.write("DFPR", 4);
    out.write(reinterpret_cast<const char*>(head), sizeof head);  // little-endian host
    const Raster<double>* ch[6] = {&pred.log_depth, &pred.log_depth_var, &pred.grad_x,
                                   &pred.grad_x_var, &pred.grad_y,       &pred.grad_y_var};
    std::vector<float> buf(pred.log_depth.size());
    for (const Raster<double>* c : ch) {
      for (std::size_t i = 0; i < buf.size(); ++i) buf[i] = static_cast<float>((*c)[i]);
      out.write(reinterpret_cast<const char*>(buf.data()), buf.size() * 4);
    }
  }
  DeviceKeyframe kd(sc.K, I0, path, 0.02);
  CHECK(kd.fusion().log_depth == pred.log_depth);
  std::vector<double> v(pred.log_depth.data(), pred.log_depth.data() + pred.log_depth.size());
  std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
  CHECK(kd.median_depth() == std::exp(v[v.size() / 2]));
  // retirement (semidense.hpp:419-424): a fresh keyframe has no inliers
  CHECK(kd.should_create_keyframe(Pose::identity(), Pose::identity()));
  CHECK(!kd.should_create_keyframe(Pose::identity(), Pose::identity(), KeyframePolicy{0.07, 0}));
  bool threw = false;
  try {
    DeviceKeyframe missing(sc.K, I0, std::string("/nonexistent/x.dfpred"), 0.02);
  } catch (const Error& e) {
    threw = e.code() == Err::MissingFile;
  }
  CHECK(threw);
}

int main() {
  semidense_kats();
  fusion_kats();
  session_kats();
  std::printf("%d checks, %d failed\n", g_checks, g_failed);
  return g_failed;
}
