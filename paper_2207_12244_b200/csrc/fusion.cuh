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

// one CTA's published partial sums for the grid all-reduce (fusion.cu)
struct ReduceSlot {
  double v[4];
  unsigned long long tag;
  unsigned long long pad[3];
};

struct FusionControl {
  int status;
  int ld_final;   // which ld buffer holds the result
  int iteration;
  int pcg_last;
  double scale;
  double value[2];
  long long trace[16];  // SM cycles per phase, CTA 0 (DFUSE_TRACE=1)
  // all-reduce phase and LL flag counters carried from one launch to the next
  // (FusionArgs::persist_sync): flags keep growing, so no launch has to clear
  // the slot and halo words the previous one left behind
  unsigned sync_phase, sync_ll;
  dfuse_solver_stats stats;
};

// Row-band decomposition of one keyframe: band g
// owns rows [y0, y1). Each band's planes are separate allocations covering
// rows [y0 - 1, y1 + 1) whose base pointers are shifted so that global pixel
// indices address them; the planes read at i - W / i + W get their halo row
// from the neighbour band, which writes its boundary row into both its own
// plane and ours (a remote store when bands live on different GPUs).
enum HaloPlane { HP_LD0, HP_LD1, HP_X, HP_Z, HP_DOWN, HP_P0, HP_P1, HP_IV2, HP_COUNT };
struct BandNb {
  double* up[HP_COUNT];  // the band above's plane (whose bottom halo row is our row y0), or null
  double* dn[HP_COUNT];  // the band below's plane (whose top halo row is our row y1 - 1), or null
};

struct FusionArgs {
  int W, H;
  const double* pred[6];
  // float32 copies of prediction planes 1..5 (log_depth_var, grad_x,
  // grad_x_var, grad_y, grad_y_var) when their values are float-exact, as
  // DFPRED values always are (predictions.hpp:16-17, 201-203); pred[0] (the
  // log-depth, shifted by focal_adjust in double) stays fp64. pred_f32 = 1:
  // the sweeps read these (24 instead of 48 bytes of prediction data per
  // pixel and sweep) and form the reciprocal variances on the fly, with the
  // same div_nr as the per-call planes: bit-identical results (modes in
  // fusion_impl.cuh, SweepPlanesT).
  const float* predf[6];
  int pred_f32_ok;  // predf holds every value exactly (set at keyframe creation)
  int pred_f32;     // the sweeps' plane mode (SweepPlanesT), set per launch
  const double* sd;
  const double* sv;
  const uint8_t* svalid;
  // per-call planes, filled by the kernel prologue (sweep_prologue)
  double* lnsd;     // log(semi depth), 0 where the semi map has no value
  double* irs;      // 1 / semi_log_variance(variance, depth), 0 likewise
  double* ivar[3];  // 1 / log_depth_var, 1 / grad_x_var, 1 / grad_y_var
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
  double* z;  // streaming PCG: z = r/diag (null: the resident path keeps z on chip)
  double* p[2];
  double* q;
  ReduceSlot* slots;  // [2][grid] all-reduce slots (+1)
  unsigned long long base_tag;  // unique per launch (set by launch_*)
  unsigned long long* halo;     // resident PCG LL halo words [3][P][2], or null
  int tiles_x, tiles_y, tw_max, th_max, ppt;  // resident-PCG tiling (set by launch_fusion)
  int diag_repeat, diag_sweep;  // OP_PCG diagnostics (DFUSE_PCG_REPEAT)
  int pcg_variant;  // resident PCG: 0 pipelined (default), 1 Chronopoulos-Gear, 2 two all-reduces
  int trace;  // record per-phase cycle counts of the resident PCG in ctl->trace
  int stage_n;  // > 0: scale rounds 1-2 read round 0's values from shared memory
  int persist_sync;  // continue the LL flags of ctl (no per-launch clearing)
  int* session_counters;  // keyframe session: [1] n_obs of this frame, [5] stereo_frames
  long long* dbg;  // DFUSE_TRACE=2: per-CTA phase times [grid][8]
  FusionControl* ctl;
  // row band (banded launches; otherwise y0 = 0, y1 = H, ctas = 0 = the grid)
  int band_y0, band_y1, band_cta0, band_ctas;
  const BandNb* nb;  // null unless banded
};

int fusion_grid(dfuse_ctx* ctx);
size_t fusion_slots_bytes(int grid);
size_t fusion_halo_bytes(long P);
bool fusion_resident_possible(long P, int grid);
float sync_bench(dfuse_ctx* ctx, int n, int variant, int grid);
void launch_fusion(dfuse_ctx* ctx, FusionArgs& a, int grid);
void launch_gradient(dfuse_ctx* ctx, FusionArgs& a, int grid, double* g);
// row-band optimize: args_dev[nband] (device), one cooperative launch of
// nband * cpr CTAs (fusion.cu, k_fusion_banded)
// (bands band0 .. band0 + nlocal - 1 of nband; sys: bands on several GPUs)
// args_host: the host copy of the local bands' args (one local band runs
// the parameter-space kernel k_fusion_band1)
void launch_fusion_banded(dfuse_ctx* ctx, const FusionArgs* args_dev,
                          unsigned long long* const* rank_slots_dev, int nband, int cpr,
                          int band0, int nlocal, int sys, const FusionArgs* args_host);
size_t band_rank_slots_bytes(int nband);
int band_ctas_per_sm();  // resident CTAs per SM of k_fusion_banded
void launch_stencil_apply(dfuse_ctx* ctx, int W, int H, const double* diag, const double* right,
                          const double* down, const double* x, double* y);

}  // namespace dfuse_cuda
