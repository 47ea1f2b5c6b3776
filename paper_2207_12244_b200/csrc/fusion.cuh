// fusion.cuh -- launch interface of the fusion optimiser (fusion.cu)
#pragma once

#include "common.cuh"

namespace dfuse_cuda {

enum FusionOp { OP_OPTIMIZE = 0, OP_PCG = 1, OP_COST = 2, OP_ASSEMBLE = 3, OP_SCALE = 4 };

// fusion state scalars kept on the device between optimize() calls of a
// keyframe session (FusionState::scale/iteration + which ld buffer is live)
struct FusionStateDev {
  double scale;
  int iteration;
  int cur;
};

struct FusionControl {
  int status;
  int ld_final;   // which ld buffer holds the result
  int iteration;
  int pcg_last;
  double scale;
  double value[2];
  dfuse_solver_stats stats;
};

struct FusionArgs {
  int W, H;
  const double* pred[6];
  const double* sd;
  const double* sv;
  const uint8_t* svalid;
  int inlier_count;
  const int* inlier_dev;  // if set, overrides inlier_count (device-resident session)
  double dsemi, dnet, dgrad, cg_tol;
  int gn, cg_max, est_scale, mode;
  int op;
  double* ld[2];
  double scale0;              // OP_COST / OP_ASSEMBLE / OP_SCALE / gradient
  const FusionStateDev* st_in;  // OP_OPTIMIZE input state
  FusionStateDev* st_out;       // OP_OPTIMIZE output state (= input on error)
  double* diag;
  double* right;
  double* down;
  double* b;
  double* x;
  double* r;
  double* p[2];
  double* q;
  double* partials;   // [2][grid][4]
  unsigned* barrier;  // arrive counter (zeroed before each launch)
  FusionControl* ctl;
};

int fusion_grid(dfuse_ctx* ctx);
void launch_fusion(dfuse_ctx* ctx, FusionArgs& a, int grid);
void launch_gradient(dfuse_ctx* ctx, FusionArgs& a, int grid, double* g);
void launch_stencil_apply(dfuse_ctx* ctx, int W, int H, const double* diag, const double* right,
                          const double* down, const double* x, double* y);

}  // namespace dfuse_cuda
