// fusion.cu -- the probabilistic fusion optimiser on sm_100a.
//
// One persistent, cooperatively launched kernel (k_fusion) runs a whole
// optimize() call (fusion.hpp:402-454) on the device with no host round
// trips: the alternating scale / depth Gauss-Newton iterations, the Huber
// IRLS weights, the line searches and the Jacobi-PCG loop
// (fusion.hpp:316-368). Every CTA owns a contiguous range of pixels; the
// reductions the reference performs sequentially are done as deterministic
// trees (warp butterfly -> CTA -> fixed-order sum over per-CTA partials) and
// each one ends in a grid barrier, after which every CTA holds the same
// bits and takes the same control decision.
//
// Fused sweeps (each followed by exactly one grid barrier):
//   scale round 0  : Huber-weighted (num, den) of the scale IRLS + the
//                    scale block's c0 = total_cost(st)       fusion.hpp:378-389,413
//   scale rounds 1,2
//   scale trial    : total_cost at exp(ln s + step dlns)     fusion.hpp:416-424
//   assemble       : gather-form normal equations + b.b + r.z + diag>0 check
//                    + the depth block's c0                  fusion.hpp:171-222,319-332,429
//   PCG sweep A    : p = r/diag + beta p_prev (recomputed at the 4 neighbours,
//                    so no halo exchange), q = H p, p.q      fusion.hpp:339-343,358-365
//   PCG sweep B    : x += a p, r -= a q, r.r, z = r/diag, r.z   fusion.hpp:343-362
//   depth trial    : trial = st + step delta (written to the other ld
//                    buffer; accepted = pointer swap), cost  fusion.hpp:430-440
// The standalone API functions (assemble, cost, gradient, scale step, PCG)
// run the same kernel with a different op.
#include <math.h>

#include "common.cuh"
#include "fusion.cuh"

namespace dfuse_cuda {

constexpr int FT = 512;  // threads per CTA
constexpr int FW = FT / 32;

struct Sel {
  bool net, grad, scale;
};

__device__ __forceinline__ Sel terms_for(int mode) {  // fusion.hpp:151-158
  Sel s{true, true, true};
  if (mode == DFUSE_MODE_NOPAIRWISE) s.grad = false;
  if (mode == DFUSE_MODE_LSSCALE) {
    s.net = false;
    s.scale = false;
  }
  return s;
}

__device__ __forceinline__ double huber_w(double r, double delta) {  // fusion.hpp:79-83
  const double a = fabs(r);
  return a <= delta ? 1.0 : delta / a;
}
__device__ __forceinline__ double huber_c(double r, double delta) {  // fusion.hpp:87-90
  const double a = fabs(r);
  return a <= delta ? r * r : delta * (2.0 * a - delta);
}
__device__ __forceinline__ double semi_logvar(double v, double d) {  // fusion.hpp:98-100
  const double x = v / (d * d);
  return x < 1e-4 ? 1e-4 : x;
}

// ---------------------------------------------------------------------------
// grid barrier + deterministic all-reduce
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct GridCtx {
  unsigned* arrive;
  double* partials;  // [2][G][4]
  unsigned G;
  unsigned epoch;
  unsigned phase;
  int syncs;
};

__device__ __forceinline__ void grid_sync(GridCtx& c) {
  __syncthreads();
  c.epoch += 1;
  c.syncs += 1;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(c.arrive, 1u);
    const unsigned target = c.epoch * c.G;
    while (ld_acquire(c.arrive) < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

// Sum v[0..NV) over every thread of the grid. Order: per-thread sequential
// partials (caller) -> warp butterfly -> CTA (warp 0 over warp partials) ->
// fixed-order sum over the G CTA partials. Identical result in every thread.
template <int NV>
__device__ void grid_allreduce(GridCtx& c, double (&v)[NV]) {
  __shared__ double red[FW][4];
  __shared__ double bcast[4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[wid][k] = v[k];
  __syncthreads();
  double* part = c.partials + (size_t)(c.phase & 1) * c.G * 4;
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = lane < FW ? red[lane][k] : 0.0;
      t = warp_sum(t);
      if (lane == 0) part[(size_t)blockIdx.x * 4 + k] = t;
    }
  }
  grid_sync(c);
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = 0.0;
      for (unsigned b = lane; b < c.G; b += 32) t += __ldcg(part + (size_t)b * 4 + k);
      t = warp_sum(t);
      if (lane == 0) bcast[k] = t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = bcast[k];
  c.phase += 1;
}

// ---------------------------------------------------------------------------
// per-pixel terms (gather form)
struct PlainLd {
  const double* ld;
  __device__ __forceinline__ double operator()(int j) const { return ld[j]; }
};
struct TrialLd {  // trial.log_depth = st + step * delta, fusion.hpp:432-433
  const double* ld;
  const double* x;
  double step;
  __device__ __forceinline__ double operator()(int j) const { return ld[j] + step * x[j]; }
};

// total_cost's contribution of pixel i, fusion.hpp:234-250 (terms added in
// the reference's order into a per-pixel sum)
template <class LD>
__device__ __forceinline__ double pixel_cost(const FusionArgs& a, const Sel& sel, int i, int x,
                                             int y, const LD& L, double li, double ln_s) {
  double c = 0.0;
  if (sel.net) c += huber_c(li - a.pred[0][i], a.dnet) / a.pred[1][i];
  if (a.svalid[i])
    c += huber_c(li - ln_s - log(a.sd[i]), a.dsemi) / semi_logvar(a.sv[i], a.sd[i]);
  if (sel.grad && x + 1 < a.W) c += huber_c(L(i + 1) - li - a.pred[2][i], a.dgrad) / a.pred[3][i];
  if (sel.grad && y + 1 < a.H)
    c += huber_c(L(i + a.W) - li - a.pred[4][i], a.dgrad) / a.pred[5][i];
  return c;
}

struct Range {
  int beg, end;
};

__device__ __forceinline__ Range my_range(const FusionArgs& a) {
  const long P = (long)a.W * a.H;
  Range r;
  r.beg = (int)(P * blockIdx.x / gridDim.x);
  r.end = (int)(P * (blockIdx.x + 1) / gridDim.x);
  return r;
}

// ---------------------------------------------------------------------------
// sweeps
// scale IRLS round (fusion.hpp:379-388) [+ total_cost at ln_s_cost]
__device__ void sweep_scale(const FusionArgs& a, const Sel& sel, const Range& rg,
                            const double* ld, double ln_s, bool with_cost, double ln_s_cost,
                            double (&v)[4]) {
  double num = 0.0, den = 0.0, cost = 0.0;
  PlainLd L{ld};
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) {
    const double li = ld[i];
    if (a.svalid[i]) {
      const double offset = li - log(a.sd[i]);
      const double R = semi_logvar(a.sv[i], a.sd[i]);
      const double wi = huber_w(offset - ln_s, a.dsemi) / R;
      num += wi * offset;
      den += wi;
    }
    if (with_cost) {
      const int y = i / a.W, x = i - y * a.W;
      cost += pixel_cost(a, sel, i, x, y, L, li, ln_s_cost);
    }
  }
  v[0] = num;
  v[1] = den;
  v[2] = cost;
  v[3] = 0.0;
}

template <class LD>
__device__ double sweep_cost(const FusionArgs& a, const Sel& sel, const Range& rg, const LD& L,
                             double ln_s, double* write_trial) {
  double cost = 0.0;
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) {
    const int y = i / a.W, x = i - y * a.W;
    const double li = L(i);
    if (write_trial) write_trial[i] = li;
    cost += pixel_cost(a, sel, i, x, y, L, li, ln_s);
  }
  return cost;
}

// assemble_normal_equations in gather form (fusion.hpp:183-219). For pixel
// i the reference's scatter loop adds, in raster order of the contributing
// pixel: grad_y of i-W, grad_x of i-1, then net, semi, grad_x, grad_y of i.
// Also: PCG init (r = b, z = r/diag, r.z, b.b, diag > 0 check,
// fusion.hpp:319-332) and the depth block's c0 (fusion.hpp:429).
__device__ void sweep_assemble(const FusionArgs& a, const Sel& sel, const Range& rg,
                               const double* ld, double ln_s, bool store_b, double (&v)[4]) {
  double bn = 0.0, rz = 0.0, bad = 0.0, cost = 0.0;
  const int W = a.W, H = a.H;
  PlainLd L{ld};
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) {
    const int y = i / W, x = i - y * W;
    const double li = ld[i];
    double diag = 0.0, b = 0.0, right = 0.0, down = 0.0;
    if (sel.grad && y > 0) {
      const int j = i - W;
      const double r = li - ld[j] - a.pred[4][j];
      const double wi = huber_w(r, a.dgrad) / a.pred[5][j];
      diag += wi;
      b -= wi * r;
    }
    if (sel.grad && x > 0) {
      const int j = i - 1;
      const double r = li - ld[j] - a.pred[2][j];
      const double wi = huber_w(r, a.dgrad) / a.pred[3][j];
      diag += wi;
      b -= wi * r;
    }
    if (sel.net) {
      const double r = li - a.pred[0][i];
      const double wi = huber_w(r, a.dnet) / a.pred[1][i];
      diag += wi;
      b -= wi * r;
    }
    if (a.svalid[i]) {
      const double r = li - ln_s - log(a.sd[i]);
      const double R = semi_logvar(a.sv[i], a.sd[i]);
      const double wi = huber_w(r, a.dsemi) / R;
      diag += wi;
      b -= wi * r;
    }
    if (sel.grad && x + 1 < W) {
      const double r = ld[i + 1] - li - a.pred[2][i];
      const double wi = huber_w(r, a.dgrad) / a.pred[3][i];
      diag += wi;
      right -= wi;
      b += wi * r;
    }
    if (sel.grad && y + 1 < H) {
      const double r = ld[i + W] - li - a.pred[4][i];
      const double wi = huber_w(r, a.dgrad) / a.pred[5][i];
      diag += wi;
      down -= wi;
      b += wi * r;
    }
    a.diag[i] = diag;
    a.right[i] = right;
    a.down[i] = down;
    a.r[i] = b;
    if (store_b) a.b[i] = b;
    bn += b * b;
    if (!(diag > 0.0)) bad += 1.0;
    rz += b * (b / diag);
    cost += pixel_cost(a, sel, i, x, y, L, li, ln_s);
  }
  v[0] = bn;
  v[1] = rz;
  v[2] = bad;
  v[3] = cost;
}

// standalone PCG init from (diag, right, down, b)
__device__ void sweep_pcg_init(const FusionArgs& a, const Range& rg, double (&v)[4]) {
  double bn = 0.0, rz = 0.0, bad = 0.0;
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) {
    const double b = a.b[i], d = a.diag[i];
    a.r[i] = b;
    bn += b * b;
    if (!(d > 0.0)) bad += 1.0;
    rz += b * (b / d);
  }
  v[0] = bn;
  v[1] = rz;
  v[2] = bad;
  v[3] = 0.0;
}

// p at pixel j for iteration it: z_j + beta p_prev_j (fusion.hpp:360,365);
// at it == 0, p = z (fusion.hpp:329-330)
__device__ __forceinline__ double p_at(const FusionArgs& a, const double* pprev, double beta,
                                       bool first, int j) {
  const double z = a.r[j] / a.diag[j];
  return first ? z : z + beta * pprev[j];
}

// PCG sweep A: q = H p (StencilMatrix::apply order, fusion.hpp:127-132), p.q
__device__ double sweep_pcg_a(const FusionArgs& a, const Range& rg, int it, double beta) {
  const double* pprev = a.p[(it + 1) & 1];
  double* pcur = a.p[it & 1];
  const bool first = it == 0;
  const int W = a.W, H = a.H;
  double pq = 0.0;
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) {
    const int y = i / W, x = i - y * W;
    const double pi = p_at(a, pprev, beta, first, i);
    double v = a.diag[i] * pi;
    if (x + 1 < W) v += a.right[i] * p_at(a, pprev, beta, first, i + 1);
    if (x > 0) v += a.right[i - 1] * p_at(a, pprev, beta, first, i - 1);
    if (y + 1 < H) v += a.down[i] * p_at(a, pprev, beta, first, i + W);
    if (y > 0) v += a.down[i - W] * p_at(a, pprev, beta, first, i - W);
    pcur[i] = pi;
    a.q[i] = v;
    pq += pi * v;
  }
  return pq;
}

// PCG sweep B (fusion.hpp:345-362): returns (r.r, r.z)
__device__ void sweep_pcg_b(const FusionArgs& a, const Range& rg, int it, double alpha,
                            double (&v)[4]) {
  const double* pcur = a.p[it & 1];
  double rr = 0.0, rz = 0.0;
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) {
    const double xo = it == 0 ? 0.0 : a.x[i];
    a.x[i] = xo + alpha * pcur[i];
    const double r = a.r[i] - alpha * a.q[i];
    a.r[i] = r;
    rr += r * r;
    rz += r * (r / a.diag[i]);
  }
  v[0] = rr;
  v[1] = rz;
  v[2] = 0.0;
  v[3] = 0.0;
}

__device__ void sweep_zero_x(const FusionArgs& a, const Range& rg) {
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) a.x[i] = 0.0;
}

// Jacobi PCG after init (solve_depth_step, fusion.hpp:334-367). Returns the
// error code (0 ok); *its = iterations run.
__device__ int pcg_loop(GridCtx& c, const FusionArgs& a, const Range& rg, double bnorm2,
                        double rz, int* its) {
  const double tol2 = a.cg_tol * a.cg_tol * bnorm2;
  double prev = bnorm2;
  int streak = 0;
  double beta = 0.0;
  *its = 0;
  for (int it = 0; it < a.cg_max; ++it) {
    *its = it + 1;
    double v1[1] = {sweep_pcg_a(a, rg, it, beta)};
    grid_allreduce(c, v1);
    const double pq = v1[0];
    if (!(pq > 0.0)) return DFUSE_E_CG_DIVERGENCE;
    const double alpha = rz / pq;
    double v2[4];
    sweep_pcg_b(a, rg, it, alpha, v2);
    double v3[2] = {v2[0], v2[1]};
    grid_allreduce(c, v3);
    const double rn = v3[0];
    if (rn <= tol2) return 0;
    if (rn > prev) {
      if (++streak >= 10) return DFUSE_E_CG_DIVERGENCE;
    } else {
      streak = 0;
    }
    prev = rn;
    beta = v3[1] / rz;
    rz = v3[1];
  }
  return 0;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(FT, 1) k_fusion(FusionArgs a) {
  GridCtx c{a.barrier, a.partials, gridDim.x, 0u, 0u, 0};
  const Range rg = my_range(a);
  const Sel sel = terms_for(a.mode);
  FusionControl* ctl = a.ctl;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  int status = 0;
  if (blockIdx.x == 0) {  // only CTA 0 (its thread 0) writes ctl afterwards
    for (int k = threadIdx.x; k < DFUSE_STATS_MAX_GN; k += FT) {
      ctl->stats.pcg_iters[k] = -1;
      ctl->stats.scale_step[k] = -1.0;
      ctl->stats.depth_step[k] = -1.0;
    }
    __syncthreads();
  }

  if (a.op == OP_COST) {
    double v[1] = {sweep_cost(a, sel, rg, PlainLd{a.ld[0]}, sel.scale ? log(a.scale0) : 0.0,
                              nullptr)};
    grid_allreduce(c, v);
    if (leader) ctl->value[0] = v[0];
  } else if (a.op == OP_ASSEMBLE) {
    double v[4];
    sweep_assemble(a, sel, rg, a.ld[0], sel.scale ? log(a.scale0) : 0.0, true, v);
  } else if (a.op == OP_SCALE) {
    double ln_s = log(a.scale0);  // fusion.hpp:377
    for (int round = 0; round < 3; ++round) {
      double v[4];
      sweep_scale(a, sel, rg, a.ld[0], ln_s, false, 0.0, v);
      double w[2] = {v[0], v[1]};
      grid_allreduce(c, w);
      ln_s = w[0] / w[1];
    }
    if (leader) ctl->value[0] = exp(ln_s);
  } else if (a.op == OP_PCG) {
    double v[4];
    sweep_pcg_init(a, rg, v);
    double w[3] = {v[0], v[1], v[2]};
    grid_allreduce(c, w);
    int its = 0;
    if (w[0] == 0.0) {
      sweep_zero_x(a, rg);
    } else if (w[2] > 0.0) {
      status = DFUSE_E_CG_DIVERGENCE;
    } else {
      status = pcg_loop(c, a, rg, w[0], w[1], &its);
      if (its == 0) sweep_zero_x(a, rg);
    }
    if (leader) ctl->pcg_last = its;
  } else {  // OP_OPTIMIZE, fusion.hpp:402-454
    const FusionStateDev st0 = *a.st_in;
    double scale = st0.scale;
    int iteration = st0.iteration;
    int cur = st0.cur;
    const int inliers = a.inlier_dev ? *a.inlier_dev : a.inlier_count;
    const bool ls_mode = a.mode == DFUSE_MODE_LSSCALE;
    const bool depth_solvable = !ls_mode || inliers > 0;
    int cost_evals = 0, pcg_total = 0, gn_done = 0;
    for (int it = 0; it < a.gn && status == 0; ++it) {
      if (!ls_mode && a.est_scale && inliers > 0) {  // fusion.hpp:411-425
        const double ln_s0 = log(scale);
        double ln_s = ln_s0;
        double c0 = 0.0;
        for (int round = 0; round < 3; ++round) {
          double v[4];
          sweep_scale(a, sel, rg, a.ld[cur], ln_s, round == 0, sel.scale ? ln_s0 : 0.0, v);
          if (round == 0) {
            double w[3] = {v[0], v[1], v[2]};
            grid_allreduce(c, w);
            c0 = w[2];
            ln_s = w[0] / w[1];
          } else {
            double w[2] = {v[0], v[1]};
            grid_allreduce(c, w);
            ln_s = w[0] / w[1];
          }
        }
        cost_evals += 1;
        const double s_new = exp(ln_s);
        const double dlns = log(s_new) - log(scale);
        double step = 1.0, accepted = 0.0;
        for (int half = 0; half <= 5; ++half) {
          const double ts = exp(log(scale) + step * dlns);
          double v[1] = {sweep_cost(a, sel, rg, PlainLd{a.ld[cur]}, sel.scale ? log(ts) : 0.0,
                                    nullptr)};
          grid_allreduce(c, v);
          cost_evals += 1;
          if (v[0] <= c0) {
            scale = ts;
            accepted = step;
            break;
          }
          step *= 0.5;
        }
        if (leader && it < DFUSE_STATS_MAX_GN) ctl->stats.scale_step[it] = accepted;
      }
      if (depth_solvable) {  // fusion.hpp:426-441
        const double ln_s = sel.scale ? log(scale) : 0.0;
        double v[4];
        sweep_assemble(a, sel, rg, a.ld[cur], ln_s, false, v);
        grid_allreduce(c, v);
        const double c0 = v[3];
        cost_evals += 1;
        int its = 0;
        if (v[0] != 0.0) {
          if (v[2] > 0.0) {
            status = DFUSE_E_CG_DIVERGENCE;
          } else {
            status = pcg_loop(c, a, rg, v[0], v[1], &its);
          }
        }
        pcg_total += its;
        if (leader && it < DFUSE_STATS_MAX_GN) ctl->stats.pcg_iters[it] = its;
        if (status) break;
        double step = 1.0, accepted = 0.0;
        const bool xzero = its == 0;  // delta == 0 (b == 0 or cg_max_iters == 0)
        for (int half = 0; half <= 5; ++half) {
          double w[1];
          if (xzero)
            w[0] = sweep_cost(a, sel, rg, PlainLd{a.ld[cur]}, ln_s, a.ld[1 - cur]);
          else
            w[0] = sweep_cost(a, sel, rg, TrialLd{a.ld[cur], a.x, step}, ln_s, a.ld[1 - cur]);
          grid_allreduce(c, w);
          cost_evals += 1;
          if (w[0] <= c0) {
            cur = 1 - cur;
            accepted = step;
            break;
          }
          step *= 0.5;
        }
        if (leader && it < DFUSE_STATS_MAX_GN) ctl->stats.depth_step[it] = accepted;
      }
      iteration += 1;
      gn_done = it + 1;
    }
    if (status == 0 && ls_mode) {  // fusion.hpp:445-452
      double v[1] = {0.0};
      const double* ld = a.ld[cur];
      for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) v[0] += a.pred[0][i] - ld[i];
      grid_allreduce(c, v);
      const double offset = v[0] / (double)((long)a.W * a.H);
      double* ldw = a.ld[cur];
      for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) ldw[i] += offset;
      scale = exp(offset);
    }
    if (leader) {
      FusionStateDev out = st0;  // transactional: unchanged on error
      if (status == 0) {
        out.scale = scale;
        out.iteration = iteration;
        out.cur = cur;
      }
      *a.st_out = out;
      ctl->scale = out.scale;
      ctl->iteration = out.iteration;
      ctl->ld_final = out.cur;
      ctl->stats.gn_done = gn_done;
      ctl->stats.pcg_total = pcg_total;
      ctl->stats.cost_evals = cost_evals;
    }
  }
  if (leader) {
    ctl->status = status;
    ctl->stats.grid_syncs = c.syncs;
  }
}

// cost_gradient in gather form (fusion.hpp:274-305). The gradient at pixel
// i receives, in the reference's order: +d_y of i-W, +d_x of i-1, net,
// semi, -d_x of i, -d_y of i. Cost and d/d ln s are grid reductions.
__global__ void __launch_bounds__(FT, 1) k_gradient(FusionArgs a, double* g) {
  GridCtx c{a.barrier, a.partials, gridDim.x, 0u, 0u, 0};
  const Range rg = my_range(a);
  const Sel sel = terms_for(a.mode);
  const double ln_s = sel.scale ? log(a.scale0) : 0.0;
  const int W = a.W, H = a.H;
  const double* ld = a.ld[0];
  PlainLd L{ld};
  double cost = 0.0, gs = 0.0;
  for (int i = rg.beg + threadIdx.x; i < rg.end; i += FT) {
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
      const double R = semi_logvar(a.sv[i], a.sd[i]);
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
    cost += pixel_cost(a, sel, i, x, y, L, li, ln_s);
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

// ---------------------------------------------------------------------------
int fusion_grid(dfuse_ctx* ctx) {
  static int occ = -1;
  if (occ < 0) {
    DF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fusion, FT, 0));
    int occ2 = 0;
    DF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_gradient, FT, 0));
    if (occ2 < occ) occ = occ2;
    if (occ < 1) throw CudaFailure{cudaErrorLaunchOutOfResources, "k_fusion occupancy"};
  }
  int g = ctx->solver_ctas > 0 ? ctx->solver_ctas : ctx->num_sms;
  if (g > ctx->num_sms * occ) g = ctx->num_sms * occ;
  return g;
}

void launch_fusion(dfuse_ctx* ctx, FusionArgs& a, int grid) {
  DF_CUDA(cudaMemsetAsync(a.barrier, 0, sizeof(unsigned), ctx->stream));
  void* args[] = {&a};
  DF_CUDA(cudaLaunchCooperativeKernel((const void*)k_fusion, dim3(grid), dim3(FT), args, 0,
                                      ctx->stream));
  DF_LAUNCHED(ctx);
}

void launch_gradient(dfuse_ctx* ctx, FusionArgs& a, int grid, double* g) {
  DF_CUDA(cudaMemsetAsync(a.barrier, 0, sizeof(unsigned), ctx->stream));
  void* args[] = {&a, &g};
  DF_CUDA(cudaLaunchCooperativeKernel((const void*)k_gradient, dim3(grid), dim3(FT), args, 0,
                                      ctx->stream));
  DF_LAUNCHED(ctx);
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
