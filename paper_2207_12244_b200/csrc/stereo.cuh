// stereo.cuh -- launch interface of the stereo front end (stereo.cu)
#pragma once

#include "common.cuh"

namespace dfuse_cuda {

// the scalar outcome of one search; the observation itself is written to
// the warp's shared slot (stereo.cu, Stencil::obs)
struct SearchResult {
  int status;
  int best;
  int n_steps;
};

// a pixel of the scan that reaches the step loop (stereo.cu)
struct StereoItem;

struct StereoArgs {
  dfuse_epigeom g;
  dfuse_search_cfg cfg;
  const float* I0;
  const float* I1;
  cudaTextureObject_t tex1;  // set by launch_stereo (frame_texture)
  double wm1, hm1;           // width - 1.0, height - 1.0 (set by launch_stereo)
  int n_items;
  int* work_counter;
  // scan mode: masked-pixel list + semi map (in/out)
  const int* list;
  double* depth;
  double* variance;
  uint8_t* valid;
  int* n_obs;
  int* n_installed;
  unsigned long long* step_count;  // optional: epipolar steps of all searches
  // list mode: pixels and optional priors
  const double* px;
  const double* prior;
  const uint8_t* has_prior;
  // optional outputs (slot = raster index in scan mode, item in list mode)
  void* status;  // int8 (scan) / int32 (list)
  int32_t* best;
  int32_t* n_steps;
  dfuse_obs* obs;
  uint8_t* obs_flag;
  // scan mode: the searches queued by the preamble (set by launch_stereo)
  StereoItem* queue;
  int* queue_count;
};

void launch_photometric(dfuse_ctx* ctx, const dfuse_epigeom& g, const float* I0, const float* I1,
                        double x, double y, double d, double* out);
void launch_texture_mask(dfuse_ctx* ctx, const float* img, int w, int h, double threshold,
                         uint8_t* mask);
// list = indices i (+ index_offset) of the set mask[i], i < P, in any order
void launch_mask_list(dfuse_ctx* ctx, const uint8_t* mask, long P, int* list, int* count,
                      long index_offset = 0);
// counter_zeroed: the caller already cleared a.work_counter on the stream
void launch_stereo(dfuse_ctx* ctx, const StereoArgs& a, bool list_mode,
                   bool counter_zeroed = false);
void launch_count_valid(dfuse_ctx* ctx, const uint8_t* valid, long P, int* out);
// float32 copies of prediction planes 1..5 over [0, n) (the caller shifts
// the pointers); *inexact += the values that do not survive the round trip
// through float (then the fp64 planes must be used)
void launch_pred_narrow(dfuse_ctx* ctx, const double* const* planes64, float* const* planes32,
                        long n, int* inexact);
void launch_compact_obs(dfuse_ctx* ctx, const uint8_t* flag, const dfuse_obs* dense, long P,
                        int* block_scratch, dfuse_obs* out);
void launch_update_list(dfuse_ctx* ctx, const dfuse_obs* obs, int n, int w, int h, int* head,
                        int* link, int* bad, double* depth, double* variance, uint8_t* valid);

}  // namespace dfuse_cuda
