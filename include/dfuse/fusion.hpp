// dfuse/fusion.hpp -- drop-in for proj/include/dfuse/fusion.hpp:13-454.
//
// Same types, names and signatures. assemble_normal_equations, total_cost,
// cost_gradient, StencilMatrix::apply, solve_depth_step, solve_scale_step
// and optimize run on the GPU (the whole optimize() is one persistent kernel,
// csrc/fusion.cu). The scalar residual / Huber helpers stay inline.
#pragma once

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "dfuse/device.hpp"
#include "dfuse/predictions.hpp"
#include "dfuse/raster.hpp"
#include "dfuse/semidense.hpp"

namespace dfuse {

struct FusionState {
  Raster<double> log_depth;
  double scale = 1.0;
  int iteration = 0;
};

struct RobustConfig {
  double delta_semi = 0.3;
  double delta_net = 0.3;
  double delta_grad = 0.1;
  int gn_iterations = 10;
  double cg_tol = 1e-6;
  int cg_max_iters = 200;
  bool estimate_scale = true;

  dfuse_robust_cfg c_abi() const {
    return {delta_semi, delta_net, delta_grad, cg_tol, gn_iterations, cg_max_iters,
            estimate_scale ? 1 : 0, 0};
  }
};

enum class FusionMode { Full, NoPairwise, LeastSquaresScale };

inline const char* to_string(FusionMode m) {
  switch (m) {
    case FusionMode::Full: return "full";
    case FusionMode::NoPairwise: return "nopairwise";
    case FusionMode::LeastSquaresScale: return "lsscale";
  }
  return "?";
}

inline FusionState init_state(const PredictionSet& pred) { return {pred.log_depth, 1.0, 0}; }

inline double residual_semi(double ln_d, double s, double d_semi) {
  return ln_d - std::log(s) - std::log(d_semi);
}
inline double residual_net(double ln_d, double ln_d_net) { return ln_d - ln_d_net; }
inline double residual_grad(double ln_d_nbr, double ln_d, double g) { return ln_d_nbr - ln_d - g; }

enum class GradAxis { X, Y };

inline double residual_grad_at(const Raster<double>& log_depth, int x, int y, GradAxis axis,
                               double g) {
  if (axis == GradAxis::X) {
    if (x + 1 >= log_depth.width())
      throw Error(Err::BorderPixel, "no right neighbour at x=" + std::to_string(x));
    return residual_grad(log_depth.at(x + 1, y), log_depth.at(x, y), g);
  }
  if (y + 1 >= log_depth.height())
    throw Error(Err::BorderPixel, "no lower neighbour at y=" + std::to_string(y));
  return residual_grad(log_depth.at(x, y + 1), log_depth.at(x, y), g);
}

inline double huber_weight(double r, double delta) {
  if (delta <= 0.0) throw Error(Err::InvalidArgument, "huber delta must be > 0");
  const double a = std::abs(r);
  return a <= delta ? 1.0 : delta / a;
}

inline double huber_cost(double r, double delta) {
  const double a = std::abs(r);
  return a <= delta ? r * r : delta * (2.0 * a - delta);
}

inline constexpr double kSemiLogVarianceFloor = 1e-4;

inline double semi_log_variance(double variance, double depth) {
  return std::max(variance / (depth * depth), kSemiLogVarianceFloor);
}

struct StencilMatrix {
  int width = 0, height = 0;
  std::vector<double> diag, right, down;

  StencilMatrix() = default;
  StencilMatrix(int w, int h)
      : width(w), height(h),
        diag(static_cast<std::size_t>(w) * h, 0.0),
        right(static_cast<std::size_t>(w) * h, 0.0),
        down(static_cast<std::size_t>(w) * h, 0.0) {}

  std::size_t size() const { return diag.size(); }

  void apply(const double* x, double* y) const {
    device::check(dfuse_stencil_apply(device::ctx(), width, height, diag.data(), right.data(),
                                      down.data(), x, y),
                  "StencilMatrix::apply");
  }
};

struct NormalEquations {
  StencilMatrix H;
  std::vector<double> b;
};

struct CostGradient {
  double cost = 0.0;
  std::vector<double> wrt_log_depth;
  double wrt_ln_scale = 0.0;
};

namespace detail {

inline int mode_of(FusionMode m) {
  return m == FusionMode::NoPairwise ? DFUSE_MODE_NOPAIRWISE
                                     : (m == FusionMode::LeastSquaresScale ? DFUSE_MODE_LSSCALE
                                                                           : DFUSE_MODE_FULL);
}

inline dfuse_fusion_inputs inputs_of(const FusionState& state, const SemiDenseMap& semi,
                                     const PredictionSet& pred) {
  require_same_size(state.log_depth, semi.depth, "fusion state vs semi-dense map");
  require_same_size(state.log_depth, pred.log_depth, "fusion state vs predictions");
  dfuse_fusion_inputs in;
  in.width = state.log_depth.width();
  in.height = state.log_depth.height();
  in.semi_depth = semi.depth.data();
  in.semi_variance = semi.variance.data();
  in.semi_valid = semi.valid.data();
  in.inlier_count = semi.inlier_count;
  in.reserved = 0;
  const Raster<double>* ch[6] = {&pred.log_depth, &pred.log_depth_var, &pred.grad_x,
                                 &pred.grad_x_var, &pred.grad_y, &pred.grad_y_var};
  for (int c = 0; c < 6; ++c) {
    require_same_size(state.log_depth, *ch[c], "fusion state vs predictions");
    in.pred[c] = ch[c]->data();
  }
  return in;
}

}  // namespace detail

inline NormalEquations assemble_normal_equations(const FusionState& state,
                                                 const SemiDenseMap& semi,
                                                 const PredictionSet& pred,
                                                 const RobustConfig& cfg, FusionMode mode) {
  const dfuse_fusion_inputs in = detail::inputs_of(state, semi, pred);
  NormalEquations eq;
  eq.H = StencilMatrix(in.width, in.height);
  eq.b.assign(eq.H.size(), 0.0);
  const dfuse_robust_cfg c = cfg.c_abi();
  device::check(dfuse_assemble_normal_equations(device::ctx(), &in, state.log_depth.data(),
                                                state.scale, &c, detail::mode_of(mode),
                                                eq.H.diag.data(), eq.H.right.data(),
                                                eq.H.down.data(), eq.b.data()),
                "assemble_normal_equations");
  return eq;
}

inline double total_cost(const FusionState& state, const SemiDenseMap& semi,
                         const PredictionSet& pred, const RobustConfig& cfg, FusionMode mode) {
  const dfuse_fusion_inputs in = detail::inputs_of(state, semi, pred);
  const dfuse_robust_cfg c = cfg.c_abi();
  double cost = 0.0;
  device::check(dfuse_total_cost(device::ctx(), &in, state.log_depth.data(), state.scale, &c,
                                 detail::mode_of(mode), &cost),
                "total_cost");
  return cost;
}

inline CostGradient cost_gradient(const FusionState& state, const SemiDenseMap& semi,
                                  const PredictionSet& pred, const RobustConfig& cfg,
                                  FusionMode mode) {
  const dfuse_fusion_inputs in = detail::inputs_of(state, semi, pred);
  const dfuse_robust_cfg c = cfg.c_abi();
  CostGradient g;
  g.wrt_log_depth.assign(state.log_depth.size(), 0.0);
  device::check(dfuse_cost_gradient(device::ctx(), &in, state.log_depth.data(), state.scale, &c,
                                    detail::mode_of(mode), &g.cost, g.wrt_log_depth.data(),
                                    &g.wrt_ln_scale),
                "cost_gradient");
  return g;
}

inline std::vector<double> solve_depth_step(const NormalEquations& eq, const RobustConfig& cfg) {
  std::vector<double> delta(eq.b.size(), 0.0);
  const dfuse_robust_cfg c = cfg.c_abi();
  int32_t its = 0;
  device::check(dfuse_solve_depth_step(device::ctx(), eq.H.width, eq.H.height, eq.H.diag.data(),
                                       eq.H.right.data(), eq.H.down.data(), eq.b.data(), &c,
                                       delta.data(), &its),
                "solve_depth_step");
  return delta;
}

inline double solve_scale_step(const FusionState& state, const SemiDenseMap& semi,
                               const RobustConfig& cfg) {
  require_same_size(state.log_depth, semi.depth, "fusion state vs semi-dense map");
  dfuse_fusion_inputs in;
  in.width = state.log_depth.width();
  in.height = state.log_depth.height();
  in.semi_depth = semi.depth.data();
  in.semi_variance = semi.variance.data();
  in.semi_valid = semi.valid.data();
  in.inlier_count = semi.inlier_count;
  in.reserved = 0;
  for (auto& p : in.pred) p = nullptr;  // not read by the scale step
  const dfuse_robust_cfg c = cfg.c_abi();
  double s = 0.0;
  device::check(dfuse_solve_scale_step(device::ctx(), &in, state.log_depth.data(), state.scale,
                                       &c, &s),
                "solve_scale_step");
  return s;
}

inline FusionState optimize(const FusionState& state, const SemiDenseMap& semi,
                            const PredictionSet& pred, const RobustConfig& cfg, FusionMode mode) {
  const dfuse_fusion_inputs in = detail::inputs_of(state, semi, pred);
  const dfuse_robust_cfg c = cfg.c_abi();
  FusionState out = state;
  int32_t iteration = state.iteration;
  device::check(dfuse_optimize(device::ctx(), &in, out.log_depth.data(), &out.scale, &iteration,
                               &c, detail::mode_of(mode), nullptr),
                "optimize");
  out.iteration = iteration;
  return out;
}

}  // namespace dfuse
