// fusion.cu -- host side of the fusion optimiser and its small kernels
// (k_fusion_banded, k_gradient, k_stencil_apply, k_sync_bench). The device
// code and the design notes are in fusion_impl.cuh; the k_fusion<PPT, VAR>
// instantiations live in fusion_part_*.cu.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "fusion_impl.cuh"

namespace dfuse_cuda {

// optimize() over row bands: CTAs [b cpr, (b+1) cpr)
// of this launch run band band0 + b with that band's FusionArgs, the
// streaming PCG and the two-level all-reduce of BandCtx. One launch holding
// every band is the single-GPU form of the multi-GPU layout (the bands'
// planes are separate allocations that exchange halo rows and band totals
// only through the BandNb pointers and the level-2 LL arrays, which on
// several GPUs are peer mappings).
struct BandLaunch {
  const FusionArgs* args;                  // [nband]
  unsigned long long* const* rank_slots;   // [nband] level-2 LL arrays
  int nband, cpr, band0, sys;
};

#ifndef DFUSE_BAND_MINB
#define DFUSE_BAND_MINB 2  // CTAs per SM of the row-band solve (bands.cu sizes its grid by it)
#endif
__global__ void __launch_bounds__(FT, DFUSE_BAND_MINB) k_fusion_banded(BandLaunch L) {
  __shared__ FusionArgs s_args;  // fields survive the L1 invalidation of every fence
  const int band = L.band0 + (int)(blockIdx.x / L.cpr);
  if (threadIdx.x == 0) s_args = L.args[band];
  __syncthreads();
  const FusionArgs& a = s_args;
  BandCtx c;
  c.slots = a.slots;
  c.G = (unsigned)L.cpr;
  c.base_tag = 0;
  // LL flags continue from the band's previous launch (persist_sync): the
  // slots are never cleared between launches, so no rank has to touch an
  // array a peer may already be posting into. Every band runs the same
  // all-reduces, so every band's control block carries the same phase.
  c.phase = a.persist_sync ? a.ctl->sync_phase : 0u;
  c.syncs = 0;
  c.ll_next = 1;
  c.me = blockIdx.x % L.cpr;
  c.band = band;
  c.nband = L.nband;
  c.rank_slots = L.rank_slots;
  c.sys = L.sys;
  const Range rg = my_range<true>(a);  // the band's CTAs walk it interleaved
  const Sel sel = terms_for(a.mode);
  FusionControl* ctl = a.ctl;
  const bool leader = c.me == 0 && threadIdx.x == 0;  // each band's own control block
  if (c.me == 0) {
    for (int k = threadIdx.x; k < DFUSE_STATS_MAX_GN; k += FT) {
      ctl->stats.pcg_iters[k] = -1;
      ctl->stats.scale_step[k] = -1.0;
      ctl->stats.depth_step[k] = -1.0;
    }
    __syncthreads();
  }
  sweep_prologue(a, rg);
  // fenced (the per-call planes and their halo rows are read at i-1, i-W),
  // and the inlier count of the whole keyframe: each band holds its own
  double v[1] = {c.me == 0 && threadIdx.x == 0 ? (double)*a.inlier_dev : 0.0};
  grid_allreduce(c, v);
  __syncthreads();
  if (threadIdx.x == 0) {
    s_args.inlier_count = (int)v[0];
    s_args.inlier_dev = nullptr;
  }
  __syncthreads();
  int status = 0;
  optimize_body<0, 0>(c, a, rg, sel, leader, status);
  if (leader) {
    ctl->status = status;
    ctl->stats.grid_syncs = c.syncs;
    if (a.persist_sync) ctl->sync_phase = c.phase;
  }
}

// One band in this launch (one band per GPU, or a one-band keyframe): the
// band's FusionArgs travel as a kernel parameter, like k_fusion's, so every
// field is a constant-bank operand; k_fusion_banded's shared-memory copy
// made each one a register load and spilled 2 KB per thread at the
// 64-register cap.
struct BandLaunch1 {
  FusionArgs a;
  unsigned long long* const* rank_slots;  // [nband] level-2 LL arrays
  int nband, cpr, band, sys;
};

__global__ void __launch_bounds__(FT, DFUSE_BAND_MINB) k_fusion_band1(BandLaunch1 L) {
  const FusionArgs& a = L.a;
  BandCtx c;
  c.slots = a.slots;
  c.G = (unsigned)L.cpr;
  c.base_tag = 0;
  c.phase = a.persist_sync ? a.ctl->sync_phase : 0u;  // as k_fusion_banded
  c.syncs = 0;
  c.ll_next = 1;
  c.me = blockIdx.x;
  c.band = L.band;
  c.nband = L.nband;
  c.rank_slots = L.rank_slots;
  c.sys = L.sys;
  const Range rg = my_range<true>(a);
  const Sel sel = terms_for(a.mode);
  FusionControl* ctl = a.ctl;
  const bool leader = c.me == 0 && threadIdx.x == 0;
  if (c.me == 0) {
    for (int k = threadIdx.x; k < DFUSE_STATS_MAX_GN; k += FT) {
      ctl->stats.pcg_iters[k] = -1;
      ctl->stats.scale_step[k] = -1.0;
      ctl->stats.depth_step[k] = -1.0;
    }
    __syncthreads();
  }
  sweep_prologue(a, rg);
  double v[1] = {c.me == 0 && threadIdx.x == 0 ? (double)*a.inlier_dev : 0.0};
  grid_allreduce(c, v);  // fenced, and the keyframe's inlier count
  int status = 0;
  optimize_body<0, 0>(c, a, rg, sel, leader, status, (int)v[0]);
  if (leader) {
    ctl->status = status;
    ctl->stats.grid_syncs = c.syncs;
    if (a.persist_sync) ctl->sync_phase = c.phase;
  }
}

void launch_fusion_banded(dfuse_ctx* ctx, const FusionArgs* args_dev,
                          unsigned long long* const* rank_slots_dev, int nband, int cpr,
                          int band0, int nlocal, int sys, const FusionArgs* args_host) {
  if (nlocal == 1 && args_host) {
    BandLaunch1 L{*args_host, rank_slots_dev, nband, cpr, band0, sys};
    void* argv[] = {&L};
    DF_CUDA(cudaLaunchCooperativeKernel((const void*)k_fusion_band1, dim3(cpr), dim3(FT), argv, 0,
                                        ctx->stream));
    DF_LAUNCHED(ctx);
    return;
  }
  BandLaunch L{args_dev, rank_slots_dev, nband, cpr, band0, sys};
  void* argv[] = {&L};
  DF_CUDA(cudaLaunchCooperativeKernel((const void*)k_fusion_banded, dim3(nlocal * cpr), dim3(FT),
                                      argv, 0, ctx->stream));
  DF_LAUNCHED(ctx);
}

int band_ctas_per_sm() { return DFUSE_BAND_MINB; }

size_t band_rank_slots_bytes(int nband) {
  return sizeof(unsigned long long) * kSlotWords * 8 * (size_t)nband;
}

// cost_gradient in gather form (fusion.hpp:274-305). The gradient at pixel
// i receives, in the reference's order: +d_y of i-W, +d_x of i-1, net,
// semi, -d_x of i, -d_y of i. Cost and d/d ln s are grid reductions.
__global__ void __launch_bounds__(FT, 1) k_gradient(FusionArgs a, double* g) {
  GridCtx c{a.slots, gridDim.x, a.base_tag, 0u, 0, 1u};
  const Range rg = my_range(a);
  const Sel sel = terms_for(a.mode);
  const double ln_s = sel.scale ? log(a.scale0) : 0.0;
  const int W = a.W, H = a.H;
  const double* ld = a.ld[0];
  PlainLd L{ld};
  double cost = 0.0, gs = 0.0;
  for (int i = rg.first(FT); i < rg.end; i += rg.stride(FT)) {
    const int y = i / W, x = i - y * W;
    const double li = ld[i];
    double gi = 0.0;
    if (sel.grad && y > 0) {
      const int j = i - W;
      const double r = li - ld[j] - a.pred[4][j];
      gi += 2.0 * huber_w(r, a.dgrad) * r / a.pred[5][j];
    }
    if (sel.grad && x > 0) {
      const int j = i - 1;
      const double r = li - ld[j] - a.pred[2][j];
      gi += 2.0 * huber_w(r, a.dgrad) * r / a.pred[3][j];
    }
    if (sel.net) {
      const double r = li - a.pred[0][i];
      gi += 2.0 * huber_w(r, a.dnet) * r / a.pred[1][i];
    }
    if (a.svalid[i]) {
      const double R = semi_logvar(a.sv[i], a.sd[i]);  // fusion.hpp:95-100
      const double r = li - ln_s - log(a.sd[i]);
      const double d = 2.0 * huber_w(r, a.dsemi) * r / R;
      gi += d;
      if (sel.scale) gs -= d;
    }
    if (sel.grad && x + 1 < W) {
      const double r = ld[i + 1] - li - a.pred[2][i];
      gi -= 2.0 * huber_w(r, a.dgrad) * r / a.pred[3][i];
    }
    if (sel.grad && y + 1 < H) {
      const double r = ld[i + W] - li - a.pred[4][i];
      gi -= 2.0 * huber_w(r, a.dgrad) * r / a.pred[5][i];
    }
    g[i] = gi;
    cost += pixel_cost_exact(a, sel, i, x, y, L, li, ln_s);
  }
  double v[2] = {cost, gs};
  grid_allreduce(c, v);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ctl->value[0] = v[0];
    a.ctl->value[1] = v[1];
    a.ctl->status = 0;
  }
}

// StencilMatrix::apply, fusion.hpp:120-135
__global__ void k_stencil_apply(int W, int H, const double* __restrict__ diag,
                                const double* __restrict__ right, const double* __restrict__ down,
                                const double* __restrict__ xv, double* __restrict__ yv) {
  const long P = (long)W * H;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long)gridDim.x * blockDim.x) {
    const int yy = (int)(i / W), xx = (int)(i - (long)yy * W);
    double v = diag[i] * xv[i];
    if (xx + 1 < W) v += right[i] * xv[i + 1];
    if (xx > 0) v += right[i - 1] * xv[i - 1];
    if (yy + 1 < H) v += down[i] * xv[i + W];
    if (yy > 0) v += down[i - W] * xv[i - W];
    yv[i] = v;
  }
}

// microbenchmark of the grid all-reduce (dfuse_debug_sync_bench)
template <int VARIANT>
__global__ void __launch_bounds__(FT, 1) k_sync_bench(ReduceSlot* slots, unsigned long long tag,
                                                      int n, double* out) {
  GridCtx c{slots, gridDim.x, tag, 0u, 0, 1u};
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    double v[2] = {1.0, (double)threadIdx.x};
    grid_allreduce<2, VARIANT != 10, VARIANT>(c, v);
    acc += v[0];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = acc;
}

// Two-level all-reduce over CTA pairs (clusters of 2; microbenchmark
// variants 11 and 12): the odd CTA of a pair sends its partial to the even
// one through distributed shared memory (one LL pair per value); the even
// CTA posts the pair's sum as one LL slot. Variant 11: every CTA polls the
// G/2 pair slots. Variant 12: only the even CTAs poll, and each forwards the
// total to its partner through distributed shared memory.
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
template <bool WEAK>
__device__ __forceinline__ void dsmem_put_v2(void* local_addr, unsigned rank, unsigned long long a,
                                             unsigned long long b) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(local_addr);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  if (WEAK)
    asm volatile("st.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(ra), "l"(a), "l"(b)
                 : "memory");
  else
    asm volatile("st.relaxed.cluster.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(ra), "l"(a),
                 "l"(b)
                 : "memory");
}
template <bool WEAK>
__device__ __forceinline__ double smem_ll_wait(const unsigned long long* p, unsigned flag) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(p);
  unsigned long long w0, w1;
  do {
    if (WEAK)
      asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                   : "=l"(w0), "=l"(w1)
                   : "r"(la)
                   : "memory");
    else
      asm volatile("ld.relaxed.cluster.shared::cta.v2.u64 {%0, %1}, [%2];"
                   : "=l"(w0), "=l"(w1)
                   : "r"(la)
                   : "memory");
  } while ((unsigned)(w0 >> 32) != flag || (unsigned)(w1 >> 32) != flag);
  return ll_value(w0, w1);
}

template <int NV, int VARIANT>
__device__ void pair_allreduce(GridCtx& c, double (&v)[NV]) {
  __shared__ double red[FW * 4];
  __shared__ double pol[kPollWarps * 4];
  __shared__ __align__(16) unsigned long long box[2][4][2];  // [0] partial in, [1] total in
  constexpr bool WEAK = VARIANT >= 13;  // weak DSMEM store, volatile local poll
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned rank = cluster_rank(), pair = blockIdx.x >> 1, P2 = c.G >> 1;
  const unsigned flag = c.phase + 1;
  double t[NV];
  cta_partial(v, t, red);
  if (wid == 0 && lane < NV) {
    double tk = t[0];
#pragma unroll
    for (int k = 1; k < NV; ++k)
      if (lane == k) tk = t[k];
    if (rank == 1) {
      dsmem_put_v2<WEAK>(&box[0][lane][0], 0, ll_word(tk, 0, flag), ll_word(tk, 1, flag));
    } else {
      const double other = smem_ll_wait<WEAK>(&box[0][lane][0], flag);
      const double ps = tk + other;  // rank order
      st_relaxed_v2(ll_slot(c, c.phase, lane, pair), ll_word(ps, 0, flag),
                    ll_word(ps, 1, flag));
    }
  }
  const bool poller = VARIANT == 11 || VARIANT == 13 || rank == 0;
  if (poller && wid < kPollWarps) {
    double acc[NV];
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = 0.0;
#pragma unroll
      for (int m = 0; m < kMaxPollSlots; ++m) {
        const unsigned b = lane + 32 * (wid + kPollWarps * m);
        if (b < P2) {
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            unsigned long long w0, w1;
            ld_relaxed_v2(ll_slot(c, c.phase, k, b), w0, w1);
            ok &= (unsigned)(w0 >> 32) == flag && (unsigned)(w1 >> 32) == flag;
            acc[k] += ll_value(w0, w1);
          }
        }
      }
      if (__all_sync(0xffffffffu, ok)) break;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = warp_sum(acc[k]);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) pol[wid * 4 + k] = acc[k];
  }
  if (VARIANT == 12 || VARIANT == 14) {
    if (rank == 0) {
      __syncthreads();
      if (wid == 0 && lane < NV) {
        double s = pol[lane];
        for (int w = 1; w < kPollWarps; ++w) s += pol[w * 4 + lane];
        dsmem_put_v2<WEAK>(&box[1][lane][0], 1, ll_word(s, 0, flag), ll_word(s, 1, flag));
      }
    } else if (wid == 0 && lane < NV) {
      const double s = smem_ll_wait<WEAK>(&box[1][lane][0], flag);
      pol[lane] = s;
      for (int w = 1; w < kPollWarps; ++w) pol[w * 4 + lane] = 0.0;
    }
  }
  __syncthreads();
  poll_total(pol, v);
  c.phase += 1;
  c.syncs += 1;
}

// variant 16: the pair stage as st.async into the even CTA's buffer,
// completing bytes on its mbarrier (hardware wait instead of a spin)
template <int NV>
__device__ void pair_allreduce_mbar(GridCtx& c, double (&v)[NV], unsigned long long* mbar,
                                    double* buf) {
  __shared__ double red[FW * 4];
  __shared__ double pol[kPollWarps * 4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned rank = cluster_rank(), pair = blockIdx.x >> 1, P2 = c.G >> 1;
  const unsigned flag = c.phase + 1;
  double t[NV];
  cta_partial(v, t, red);
  if (wid == 0) {
    double tk = t[0];
#pragma unroll
    for (int k = 1; k < NV; ++k)
      if (lane == k) tk = t[k];
    const unsigned mb = (unsigned)__cvta_generic_to_shared(mbar);
    if (rank == 1) {
      if (lane < NV) {
        const unsigned lb = (unsigned)__cvta_generic_to_shared(buf + lane);
        unsigned rb, rm;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rb) : "r"(lb));
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rm) : "r"(mb));
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rb),
            "l"(__double_as_longlong(tk)), "r"(rm)
            : "memory");
      }
    } else {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                     "r"(8 * NV)
                     : "memory");
      unsigned done = 0;
      const unsigned par = c.phase & 1;
      do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(mb), "r"(par)
            : "memory");
      } while (!done);
      if (lane < NV) {
        const double ps = tk + buf[lane];  // rank order
        st_relaxed_v2(ll_slot(c, c.phase, lane, pair), ll_word(ps, 0, flag),
                      ll_word(ps, 1, flag));
      }
    }
  }
  if (wid < kPollWarps) {
    double acc[NV];
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = 0.0;
      const unsigned b = lane + 32 * wid;
      if (b < P2) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          unsigned long long w0, w1;
          ld_relaxed_v2(ll_slot(c, c.phase, k, b), w0, w1);
          ok &= (unsigned)(w0 >> 32) == flag && (unsigned)(w1 >> 32) == flag;
          acc[k] += ll_value(w0, w1);
        }
      }
      if (__all_sync(0xffffffffu, ok)) break;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = warp_sum(acc[k]);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) pol[wid * 4 + k] = acc[k];
  }
  __syncthreads();
  poll_total(pol, v);
  c.phase += 1;
  c.syncs += 1;
}

template <int VARIANT>
__global__ void __launch_bounds__(FT, 1) k_sync_bench_pair(ReduceSlot* slots, int n, double* out) {
  GridCtx c{slots, gridDim.x, 0ull, 0u, 0, 1u};
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ double mbuf[4];
  if (VARIANT == 16) {
    if (threadIdx.x == 0) {
      const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
  }
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    double v[2] = {1.0, (double)threadIdx.x};
    if (VARIANT == 16)
      pair_allreduce_mbar<2>(c, v, &mbar, mbuf);
    else if (VARIANT == 15)  // the flat LL all-reduce under a cluster launch
      grid_allreduce<2, false, 10>(c, v);
    else
      pair_allreduce<2, VARIANT>(c, v);
    acc += v[0];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = acc;
  // no CTA leaves while its partner may still address its shared memory
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// ---------------------------------------------------------------------------
// host side
static unsigned long long next_tag() {
  static unsigned long long seq = 0;  // host-side launch sequence (one process)
  return (__atomic_add_fetch(&seq, 1ULL, __ATOMIC_RELAXED)) << 32;
}

constexpr size_t kMaxDynSmem = 227 * 1024;  // also in fusion_launch.cuh
// static shared memory of the resident kernels (all-reduce and ring prefetch
// staging, reduction scratch: 18 KB at 384 threads), kept out of the tile's
// dynamic budget
constexpr size_t kResidentStaticSmem = 20 * 1024;

int fusion_grid(dfuse_ctx* ctx) {
  int& occ = ctx->fusion_occ;
  if (occ <= 0) {
    // every grid-synchronising kernel is __launch_bounds__(FT, 1); these two
    // stand for the k_fusion instantiations of the fusion_part_*.cu units
    int o[2] = {0, 0};
    DF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o[0], k_fusion_banded, FT, 0));
    DF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o[1], k_gradient, FT, 0));
    occ = o[0] < o[1] ? o[0] : o[1];
    if (occ < 1) throw CudaFailure{cudaErrorLaunchOutOfResources, "k_fusion occupancy"};
  }
  int g = ctx->solver_ctas > 0 ? ctx->solver_ctas : ctx->num_sms;
  if (g > ctx->num_sms) g = ctx->num_sms;  // one CTA per SM: resident tiles need the SM's smem
  if (g > 32 * kPollWarps * kMaxPollSlots) g = 32 * kPollWarps * kMaxPollSlots;
  return g;
}

size_t fusion_slots_bytes(int grid) {
  grid *= 2;  // room for the streaming kernel's two CTAs per SM
  // LL slots (2 parities x 4 values x grid x 256 B) or the atomic-counter
  // microbenchmark variants' ReduceSlots, whichever is larger
  const size_t ll = sizeof(unsigned long long) * kSlotWords * 8 * (size_t)grid;
  const size_t tag = sizeof(ReduceSlot) * (2 * (size_t)grid + 1);
  return ll > tag ? ll : tag;
}

size_t fusion_halo_bytes(long P) { return sizeof(unsigned long long) * 6 * (size_t)P; }

bool fusion_resident_possible(long P, int grid) {
  return P <= (long)grid * DFUSE_PPT_HI * kResidentFT;  // coarse bound; plan_tiles decides
}

// tile partition for the resident PCG: tx x ty <= grid tiles, minimal
// largest tile, then minimal halo
void plan_tiles(FusionArgs& a, int grid) {
  static const int force_tx = getenv("DFUSE_TILES_X") ? atoi(getenv("DFUSE_TILES_X")) : 0;
  // Two cost models, measured: small tiles (<= 4 pixels per thread, latency
  // bound: C1 320x240) take the smallest largest tile, then the smallest
  // half perimeter (C1: 107x5 139 updates/s, 64x9 136). Large tiles take the
  // largest tile's pixels plus 1.5 x its half perimeter (halo ring, boundary
  // SpMV, boundary words), not narrower than 64 px, within the resident
  // capacity. C2 (640x480, 148 CTAs), updates/s at the reference defaults by
  // tiles_x: 3: 447, 4 (160x13): 466, 6: 473, 7 (92x23): 473, 9: 461,
  // 10: 444, 12 (54x40): 450 -- the second model picks 7.
  int bx = 1, by = 1;
  for (int model = 0; model < 2; ++model) {
    long best = -1;
    for (int tx = 1; tx <= grid && tx <= a.W; ++tx) {
      if (force_tx > 0 && tx != force_tx) continue;  // diagnostics: DFUSE_TILES_X
      int ty = grid / tx;
      if (ty > a.H) ty = a.H;
      if (ty < 1) break;
      const long tw = (a.W + tx - 1) / tx, th = (a.H + ty - 1) / ty;
      long cost;
      if (model == 0) {
        cost = tw * th * 64 + (tw + th);
      } else {
        cost = 2 * tw * th + 3 * (tw + th);
        if (tw < 64 && a.W >= 64) cost += 1L << 40;
        if (tw * th > (long)DFUSE_PPT_HI * kResidentFT) cost += 1L << 41;
      }
      if (best < 0 || cost < best) {
        best = cost;
        bx = tx;
        by = ty;
      }
    }
    const long T0 = (long)((a.W + bx - 1) / bx) * ((a.H + by - 1) / by);
    if (model == 0 && T0 <= 4L * kResidentFT) break;  // small tiles: model 0 stands
  }
  a.tiles_x = bx;
  a.tiles_y = by;
  a.tw_max = (a.W + bx - 1) / bx;
  a.th_max = (a.H + by - 1) / by;
  const long T = (long)a.tw_max * a.th_max;
  constexpr long R = kResidentFT;
  a.ppt = T <= 4 * R ? 4 : (T <= 5 * R ? 5 : (T <= DFUSE_PPT_HI * R ? DFUSE_PPT_HI : 0));
  if (a.ppt > 0 && pcg_tile_smem(a.ppt, a.tw_max, a.th_max) > kMaxDynSmem - kResidentStaticSmem)
    a.ppt = 0;
  // LL flags are 32-bit: the whole launch must fit
  if ((double)a.gn * ((double)a.cg_max + 2.0) > 2.0e9) a.ppt = 0;
  if (!a.halo) a.ppt = 0;
}

void launch_fusion(dfuse_ctx* ctx, FusionArgs& a, int grid) {
  plan_tiles(a, grid);
  if (ctx->force_streaming == 1) a.ppt = 0;
  // prediction planes (SweepPlanesT): the fp32 copies when streaming from HBM
  a.pred_f32 = a.pred_f32_ok && a.ppt == 0 ? 1 : 0;
  a.pcg_variant = ctx->force_streaming == 2 ? 2 : (ctx->force_streaming == 3 ? 1 : 0);
  {  // scale-round staging lives in the resident PCG's shared memory
    const long range = ((long)a.W * a.H + grid - 1) / grid;
    a.stage_n = (a.ppt > 0 && (size_t)(16 * range) <= pcg_tile_smem(a.ppt, a.tw_max, a.th_max))
                    ? (int)range
                    : 0;
  }
  a.base_tag = next_tag();
  // LL flags restart at 1 every launch: clear the slots and the halo words
  // (a session's launches continue the flags instead, FusionArgs::persist_sync)
  if (!a.persist_sync) {
    DF_CUDA(cudaMemsetAsync(a.slots, 0, fusion_slots_bytes(grid), ctx->stream));
    if (a.ppt > 0)
      DF_CUDA(cudaMemsetAsync(a.halo, 0, fusion_halo_bytes((long)a.W * a.H), ctx->stream));
  }
  a.trace = ctx->trace;
  if (ctx->trace && !DFUSE_TRACE_BUILD) {
    static bool told = false;
    if (!told)
      fprintf(stderr, "dfuse: DFUSE_TRACE needs the diagnostics build (make -C "
                      "paper_2207_12244_b200/csrc diag; DFUSE_LIB=.../libdfuse_cuda_diag.so)\n");
    told = true;
  }
  a.diag_repeat = ctx->diag_repeat;
  a.diag_sweep = ctx->diag_sweep;
  a.dbg = nullptr;
  const size_t dbg_n = ctx->trace >= 3 ? (size_t)256 * grid * 8 : (size_t)8 * grid;
  if (ctx->trace >= 2) {
    a.dbg = (long long*)scratch(ctx, S_TMP4, sizeof(long long) * dbg_n);
    DF_CUDA(cudaMemsetAsync(a.dbg, 0, sizeof(long long) * dbg_n, ctx->stream));
  }
  const int key = a.ppt * 10 + a.pcg_variant;
  switch (key) {
    case 40: launch_fusion_t<4, 0>(ctx, a, grid); break;
    case 41: launch_fusion_t<4, 1>(ctx, a, grid); break;
    case 42: launch_fusion_t<4, 2>(ctx, a, grid); break;
    case 50: launch_fusion_t<5, 0>(ctx, a, grid); break;
    case 51: launch_fusion_t<5, 1>(ctx, a, grid); break;
    case 52: launch_fusion_t<5, 2>(ctx, a, grid); break;
    case DFUSE_PPT_HI * 10: launch_fusion_t<DFUSE_PPT_HI, 0>(ctx, a, grid); break;
    case DFUSE_PPT_HI * 10 + 1: launch_fusion_t<DFUSE_PPT_HI, 1>(ctx, a, grid); break;
    case DFUSE_PPT_HI * 10 + 2: launch_fusion_t<DFUSE_PPT_HI, 2>(ctx, a, grid); break;
    default: {  // streaming: two CTAs per SM (k_fusion<0, 0> launch bounds)
      int g2 = 2 * grid;
      if (g2 > 32 * kPollWarps * kMaxPollSlots) g2 = 32 * kPollWarps * kMaxPollSlots;
      launch_fusion_t<0, 0>(ctx, a, g2);
      break;
    }
  }
  DF_LAUNCHED(ctx);
  if (ctx->trace) {  // diagnostics only (DFUSE_TRACE=1): per-phase cycles of the resident PCG
    long long tr[16];
    int its = 0;
    DF_CUDA(cudaMemcpyAsync(tr, a.ctl->trace, sizeof tr, cudaMemcpyDeviceToHost, ctx->stream));
    DF_CUDA(cudaMemcpyAsync(&its, &a.ctl->stats.pcg_total, sizeof its, cudaMemcpyDeviceToHost,
                            ctx->stream));
    DF_CUDA(cudaStreamSynchronize(ctx->stream));
    // PCG phases are SM cycles; convert with the clock measured over the solves
    const double ghz = tr[6] > 0 ? (double)tr[7] / (double)tr[6] : 1.0;
    double ns[6];
    for (int k = 0; k < 6; ++k) ns[k] = (double)tr[k] / ghz;
    fprintf(stderr,
            "dfuse trace (ppt %d, ns, CTA 0): ring %.0f spmv %.0f ar/wait_rz %.0f pq_upd %.0f "
            "ar_pq %.0f sweep %.0f | scale %lld strial %lld assemble %lld pcg %lld dtrial %lld "
            "(pcg its %d) sm_clock %.0f MHz | trial sweeps only: scale %lld depth %lld | "
            "prefetched all-reduce waits that polled (poll warps, all CTAs, cumulative) %lld\n",
            a.ppt, ns[0], ns[1], ns[2], ns[3], ns[4], ns[5], tr[8], tr[9], tr[10], tr[11], tr[12],
            its, 1e3 * ghz, tr[13], tr[14], tr[15]);
    if (a.dbg && ctx->trace >= 3) {  // each CTA's view of its all-reduces (SM cycles)
      std::vector<long long> h(dbg_n);
      DF_CUDA(cudaMemcpy(h.data(), a.dbg, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost));
      // per CTA: mean entry->publish, publish->done, done->exit, rounds
      std::vector<double> e2p, p2d, d2x, rounds;
      for (int b = 0; b < grid; ++b) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        int n = 0;
        for (int it = 0; it < 256; ++it) {
          const long long* r = h.data() + ((size_t)it * grid + b) * 8;
          if (!r[0] || !r[4]) continue;
          s0 += r[1] - r[0]; s1 += r[2] - r[1]; s2 += r[4] - r[2]; s3 += r[3]; ++n;
        }
        if (!n) continue;
        e2p.push_back(s0 / n / ghz); p2d.push_back(s1 / n / ghz); d2x.push_back(s2 / n / ghz);
        rounds.push_back(s3 / n);
      }
      auto stat = [](std::vector<double> v, const char* name) {
        if (v.empty()) return;
        std::sort(v.begin(), v.end());
        fprintf(stderr, "  all-reduce %s across CTAs: min %.0f median %.0f max %.0f\n", name, v[0],
                v[v.size() / 2], v.back());
      };
      stat(e2p, "entry->publish ns");
      stat(p2d, "publish->complete ns");
      stat(d2x, "complete->exit ns");
      stat(rounds, "poll rounds");
    } else if (a.dbg) {  // per-CTA spread of each phase
      std::vector<long long> h((size_t)8 * grid);
      DF_CUDA(cudaMemcpy(h.data(), a.dbg, sizeof(long long) * 8 * grid, cudaMemcpyDeviceToHost));
      for (int k = 0; k < 6; ++k) {
        std::vector<long long> col(grid);
        for (int b = 0; b < grid; ++b) col[b] = h[(size_t)b * 8 + k];
        std::sort(col.begin(), col.end());
        fprintf(stderr, "  phase %d across CTAs (ns): min %.0f median %.0f max %.0f\n", k,
                col[0] / ghz, col[grid / 2] / ghz, col[grid - 1] / ghz);
      }
    }
  }
}

void launch_gradient(dfuse_ctx* ctx, FusionArgs& a, int grid, double* g) {
  a.base_tag = next_tag();
  DF_CUDA(cudaMemsetAsync(a.slots, 0, fusion_slots_bytes(grid), ctx->stream));
  void* args[] = {&a, &g};
  DF_CUDA(cudaLaunchCooperativeKernel((const void*)k_gradient, dim3(grid), dim3(FT), args, 0,
                                      ctx->stream));
  DF_LAUNCHED(ctx);
}

float sync_bench(dfuse_ctx* ctx, int n, int variant, int grid) {
  if (grid <= 0 || grid > ctx->num_sms) grid = ctx->num_sms;
  const size_t bytes = fusion_slots_bytes(grid) + 256;
  ReduceSlot* slots = (ReduceSlot*)scratch(ctx, S_TMP4, bytes);
  double* out = (double*)scratch(ctx, S_TMP3, 64);
  DF_CUDA(cudaMemsetAsync(slots, 0, bytes, ctx->stream));
  unsigned long long tag = next_tag();
  void* args[] = {&slots, &tag, &n, &out};
  DF_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (variant >= 11 && variant <= 16) {  // clusters of 2 (grid rounded down to even)
    grid &= ~1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(FT);
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (variant == 11)
      DF_CUDA(cudaLaunchKernelEx(&cfg, k_sync_bench_pair<11>, slots, n, out));
    else if (variant == 12)
      DF_CUDA(cudaLaunchKernelEx(&cfg, k_sync_bench_pair<12>, slots, n, out));
    else if (variant == 13)
      DF_CUDA(cudaLaunchKernelEx(&cfg, k_sync_bench_pair<13>, slots, n, out));
    else if (variant == 14)
      DF_CUDA(cudaLaunchKernelEx(&cfg, k_sync_bench_pair<14>, slots, n, out));
    else if (variant == 15)
      DF_CUDA(cudaLaunchKernelEx(&cfg, k_sync_bench_pair<15>, slots, n, out));
    else
      DF_CUDA(cudaLaunchKernelEx(&cfg, k_sync_bench_pair<16>, slots, n, out));
  } else {
    const void* fn = variant == 2 ? (const void*)k_sync_bench<2> : (const void*)k_sync_bench<10>;
    DF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(FT), args, 0, ctx->stream));
  }
  DF_LAUNCHED(ctx);
  DF_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  DF_CUDA(cudaEventSynchronize(ctx->ev[1]));
  float ms = 0.f;
  DF_CUDA(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
  return ms;
}

void launch_stencil_apply(dfuse_ctx* ctx, int W, int H, const double* diag, const double* right,
                          const double* down, const double* x, double* y) {
  const long P = (long)W * H;
  long blocks = (P + 255) / 256;
  if (blocks > ctx->num_sms * 8L) blocks = ctx->num_sms * 8L;
  k_stencil_apply<<<(int)blocks, 256, 0, ctx->stream>>>(W, H, diag, right, down, x, y);
  DF_LAUNCHED(ctx);
}

}  // namespace dfuse_cuda
