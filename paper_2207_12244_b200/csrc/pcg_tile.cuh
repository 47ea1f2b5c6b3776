// pcg_tile.cuh -- SM-resident Jacobi PCG (included by fusion.cu).
//
// Same iteration, stop rules and per-pixel expressions as solve_depth_step
// (fusion.hpp:316-368), up to algebraic rearrangements that change rounding
// at the ulp level only (tolerance parity):
//
//   pcg_resident     (default) one grid all-reduce per iteration. The
//                    direction product q = H p is carried by the recurrence
//                        p_k = z_k + beta_k p_{k-1},  q_k = H z_k + beta_k q_{k-1}
//                    and the curvature p_k.q_k by the Chronopoulos-Gear identity
//                        p_k.q_k = z_k.Hz_k - beta_k (r_k.z_k) / alpha_{k-1}
//                    (exact for a symmetric H with M^-1-orthogonal residuals),
//                    so (r.r, r.z, z.Hz) travel in ONE all-reduce that follows
//                    the SpMV.
//   pcg_resident_2r  two all-reduces per iteration: (p.q) as the reference
//                    computes it, and a split-phase (r.r, r.z) that overlaps
//                    the next SpMV. Kept as the A/B partner
//                    (dfuse_ctx_set_solver_path(ctx, 2)).
//
// CTA b owns tile b of a tiles_x x tiles_y partition. For the whole solve:
//   registers : r, z, p, q of PPT pixels per thread, their shared-memory
//               offsets and boundary flags
//   shared    : diag, 1/diag, the four off-diagonal couplings of every pixel
//               (right, left = right[i-1], down, up = down[i-W], zero where the
//               reference skips the term, fusion.hpp:128-131), x, and z with
//               a one-pixel halo
// Only the tile boundary of z leaves the SM: after each update sweep a CTA
// posts its boundary z as LL words {32-bit half, 32-bit flag} in a
// raster-indexed array and the neighbours rebuild their halo from them. The
// LL flags order that data, so the all-reduces of the loop need no fence.
//
// z = r/diag uses the reciprocal computed once per solve and one Markstein
// correction (q0 = r*(1/d); e = fma(-q0, d, r); z = fma(e, 1/d, q0)), which
// returns the IEEE quotient except in rare double-rounding corner cases.
#pragma once

// shared-memory carve-up and per-thread pixel map of one tile
template <int PPT>
struct PcgTile {
  TileGeo tg;
  int T, pw, ring_n;
  double *s_diag, *s_rdiag, *s_right, *s_left, *s_down, *s_up, *s_z, *s_x;
  int so_[PPT];  // offset in s_z
  int gi_[PPT];  // global pixel index (-1: no pixel); bit 30 set: tile boundary

  __device__ __forceinline__ int gi(int j) const { return gi_[j] & ~(1 << 30); }
  __device__ __forceinline__ bool boundary(int j) const { return gi_[j] & (1 << 30); }

  // load the tile's couplings, r, and z = r/diag; post boundary z with `flag`
  __device__ __forceinline__ void load(const FusionArgs& a, double (&rr_)[PPT], double (&zr)[PPT],
                                       unsigned long long* z_ll, unsigned flag) {
    extern __shared__ double dsm[];
    tg = my_tile(a);
    T = tg.tw * tg.th;
    const int TM = a.tw_max * a.th_max;
    s_diag = dsm;
    s_rdiag = dsm + TM;
    s_right = dsm + 2 * TM;
    s_left = dsm + 3 * TM;
    s_down = dsm + 4 * TM;
    s_up = dsm + 5 * TM;
    s_z = dsm + 6 * TM;  // (th+2) x (tw+2), halo included
    s_x = s_z + (a.th_max + 2) * (a.tw_max + 2);
    pw = tg.tw + 2;
    ring_n = T > 0 ? 2 * (tg.tw + tg.th) : 0;
    const int W = a.W, H = a.H;
    // halo entries outside the image stay 0 (their couplings are 0 too)
    for (int t = threadIdx.x; t < (tg.th + 2) * pw; t += FT) s_z[t] = 0.0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int k = threadIdx.x + FT * j;
      rr_[j] = zr[j] = 0.0;
      gi_[j] = -1;
      so_[j] = 0;
      if (k < T) {
        s_x[k] = 0.0;
        const int ly = k / tg.tw, lx = k - ly * tg.tw;
        const int gx = tg.x0 + lx, gy = tg.y0 + ly;
        const int g = gy * W + gx;
        const bool bd = lx == 0 || ly == 0 || lx == tg.tw - 1 || ly == tg.th - 1;
        gi_[j] = g | (bd ? (1 << 30) : 0);
        so_[j] = (ly + 1) * pw + lx + 1;
        const double d = __ldcg(a.diag + g);
        const double rd = 1.0 / d;
        s_diag[k] = d;
        s_rdiag[k] = rd;
        s_right[k] = gx + 1 < W ? __ldcg(a.right + g) : 0.0;
        s_left[k] = gx > 0 ? __ldcg(a.right + g - 1) : 0.0;
        s_down[k] = gy + 1 < H ? __ldcg(a.down + g) : 0.0;
        s_up[k] = gy > 0 ? __ldcg(a.down + g - W) : 0.0;
        const double r = __ldcg(a.r + g);
        rr_[j] = r;
        const double q0 = r * rd;  // z = r/diag, fusion.hpp:329
        const double z = __fma_rn(__fma_rn(-q0, d, r), rd, q0);
        zr[j] = z;
        s_z[so_[j]] = z;
        if (bd) ll_store(z_ll + 2 * (long)g, z, flag);
      }
    }
  }

  // halo ring of z (version `flag`) from the neighbours' LL words
  __device__ __forceinline__ void ring(const FusionArgs& a, const unsigned long long* z_ll,
                                       unsigned flag) const {
    for (int t = threadIdx.x; t < ring_n; t += FT) {
      int gx, gy, so;
      if (t < tg.tw) {
        gx = tg.x0 + t, gy = tg.y0 - 1, so = t + 1;
      } else if (t < 2 * tg.tw) {
        gx = tg.x0 + t - tg.tw, gy = tg.y0 + tg.th, so = (tg.th + 1) * pw + t - tg.tw + 1;
      } else if (t < 2 * tg.tw + tg.th) {
        gx = tg.x0 - 1, gy = tg.y0 + t - 2 * tg.tw, so = (t - 2 * tg.tw + 1) * pw;
      } else {
        gx = tg.x0 + tg.tw, gy = tg.y0 + t - 2 * tg.tw - tg.th,
        so = (t - 2 * tg.tw - tg.th + 1) * pw + tg.tw + 1;
      }
      if (gx >= 0 && gx < a.W && gy >= 0 && gy < a.H)
        s_z[so] = ll_wait(z_ll + 2 * ((long)gy * a.W + gx), flag);
    }
  }

  // w = H z, StencilMatrix::apply order (fusion.hpp:127-131), branch-free.
  // BOUNDARY selects the pass: false = interior pixels (own-tile z only, can
  // run before the halo ring arrives), true = tile-boundary pixels
  template <bool BOUNDARY>
  __device__ __forceinline__ void spmv(const double (&zr)[PPT], double (&wv)[PPT]) const {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (gi_[j] >= 0 && boundary(j) == BOUNDARY) {
        const int k = threadIdx.x + FT * j, so = so_[j];
        double v = s_diag[k] * zr[j];
        v += s_right[k] * s_z[so + 1];
        v += s_left[k] * s_z[so - 1];
        v += s_down[k] * s_z[so + pw];
        v += s_up[k] * s_z[so - pw];
        wv[j] = v;
      } else if (gi_[j] < 0) {
        wv[j] = 0.0;
      }
    }
  }

  // delta to the raster for the line search (x == 0 if no iteration ran)
  __device__ __forceinline__ void store_x(const FusionArgs& a) const {
#pragma unroll
    for (int j = 0; j < PPT; ++j)
      if (gi_[j] >= 0) a.x[gi(j)] = s_x[threadIdx.x + FT * j];
  }
};

// DFUSE_TRACE: thread 0 accumulates SM cycles per phase (CTA 0 -> ctl->trace,
// every CTA -> a.dbg[cta][phase] when DFUSE_TRACE=2); the host converts
// cycles to ns with the clock measured over the whole solve
struct PcgTrace {
  bool on;
  long long tr[6], t_last, t_start, c_start;
  __device__ __forceinline__ explicit PcgTrace(const FusionArgs& a)
      : on(a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || a.trace == 2)) {
    for (int k = 0; k < 6; ++k) tr[k] = 0;
    t_start = on ? df_now() : 0;
    t_last = c_start = on ? clock64() : 0;
  }
  __device__ __forceinline__ void mark(int k) {
    if (on) {
      const long long t = clock64();
      tr[k] += t - t_last;
      t_last = t;
    }
  }
  __device__ __forceinline__ void flush(const FusionArgs& a) {
    if (on && blockIdx.x == 0) {
      for (int k = 0; k < 6; ++k) a.ctl->trace[k] += tr[k];
      a.ctl->trace[6] += df_now() - t_start;   // ns
      a.ctl->trace[7] += clock64() - c_start;  // SM cycles -> effective clock
    }
    if (on && a.trace == 2)
      for (int k = 0; k < 6; ++k) a.dbg[blockIdx.x * 8 + k] += tr[k];
  }
};

// One all-reduce per iteration (Chronopoulos-Gear). Trace phases:
// 0 halo ring, 1 SpMV, 2 all-reduce, 5 update sweep.
template <int PPT>
__device__ int pcg_resident(GridCtx& c, const FusionArgs& a, double bnorm2, double rz, int* its) {
  PcgTile<PPT> t;
  unsigned long long* z_ll = a.halo;  // [P][2]
  // LL flags of this solve: z after v updates -> base + v + 1
  const unsigned base = c.ll_next;
  c.ll_next += (unsigned)a.cg_max + 2u;
  double rr_[PPT], zr[PPT], pr[PPT], qr[PPT];
  t.load(a, rr_, zr, z_ll, base + 1);
#pragma unroll
  for (int j = 0; j < PPT; ++j) pr[j] = qr[j] = 0.0;

  const double tol2 = a.cg_tol * a.cg_tol * bnorm2;
  double prev = bnorm2, beta = 0.0, alpha = 1.0;
  double rr_part = 0.0, rz_part = 0.0;
  int streak = 0, status = 0;
  *its = 0;
  PcgTrace trc(a);
  for (int it = 0; a.cg_max > 0; ++it) {
    // z is the version after `it` updates; w = H z
    const bool more = it < a.cg_max;
    double wv[PPT];
    double zw = 0.0;
    if (more) {
      __syncthreads();  // own-tile z of the last sweep
      t.template spmv<false>(zr, wv);  // interior while the halo travels
      trc.mark(1);
      t.ring(a, z_ll, base + (unsigned)it + 1u);
      __syncthreads();
      trc.mark(0);
      t.template spmv<true>(zr, wv);
#pragma unroll
      for (int j = 0; j < PPT; ++j) zw += zr[j] * wv[j];
      trc.mark(1);
    }
    double pq;
    if (it == 0) {
      double v[1] = {zw};
      grid_allreduce<1, false>(c, v);
      trc.mark(2);
      pq = v[0];  // p0 = z0, q0 = H z0
    } else {
      double v[3] = {rr_part, rz_part, zw};
      long long* rec = a.trace >= 3 && it <= 256
                           ? a.dbg + ((long)(it - 1) * gridDim.x + blockIdx.x) * 8
                           : nullptr;  // DFUSE_TRACE=3: every CTA's view of the exchange
      grid_allreduce<3, false>(c, v, rec);
      trc.mark(2);
      // finish iteration it-1: fusion.hpp:350-364
      const double rn = v[0];
      if (rn <= tol2) break;
      if (rn > prev) {
        if (++streak >= 10) {
          status = DFUSE_E_CG_DIVERGENCE;
          break;
        }
      } else {
        streak = 0;
      }
      prev = rn;
      if (!more) break;
      beta = v[1] / rz;
      rz = v[1];
      pq = v[2] - beta * rz / alpha;
    }
    if (!(pq > 0.0)) {  // fusion.hpp:342
      status = DFUSE_E_CG_DIVERGENCE;
      break;
    }
    alpha = rz / pq;
    *its = it + 1;
    // p = z + beta p, q = H z + beta q (p = z at it 0, fusion.hpp:329-330,
    // 364); x += alpha p, r -= alpha q, z = r/diag (fusion.hpp:345-359)
    rr_part = 0.0;
    rz_part = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (t.gi_[j] >= 0) {
        const int k = threadIdx.x + FT * j;
        const double p = it == 0 ? zr[j] : zr[j] + beta * pr[j];
        const double q = it == 0 ? wv[j] : wv[j] + beta * qr[j];
        pr[j] = p;
        qr[j] = q;
        t.s_x[k] = t.s_x[k] + alpha * p;
        const double r = rr_[j] - alpha * q;
        rr_[j] = r;
        rr_part += r * r;
        const double rd = t.s_rdiag[k];
        const double q0 = r * rd;
        const double z = __fma_rn(__fma_rn(-q0, t.s_diag[k], r), rd, q0);
        zr[j] = z;
        t.s_z[t.so_[j]] = z;
        rz_part += r * z;
        if (t.boundary(j)) ll_store(z_ll + 2 * (long)t.gi(j), z, base + (unsigned)it + 2u);
      }
    }
    trc.mark(5);
  }
  trc.flush(a);
  t.store_x(a);
  grid_sync(c);  // fenced: the trial sweeps read x at the neighbours
  return status;
}

// Two all-reduces per iteration: (p.q) exposed, (r.r, r.z) split-phase
// behind the next SpMV. Trace phases: 0 ring, 1 SpMV, 2 wait (r.r, r.z),
// 3 p/q update, 4 (p.q) all-reduce, 5 sweep B + publish.
template <int PPT>
__device__ int pcg_resident_2r(GridCtx& c, const FusionArgs& a, double bnorm2, double rz,
                               int* its) {
  PcgTile<PPT> t;
  unsigned long long* z_ll = a.halo;
  const unsigned base = c.ll_next;
  c.ll_next += (unsigned)a.cg_max + 2u;
  double rr_[PPT], zr[PPT], pr[PPT], qr[PPT];
  t.load(a, rr_, zr, z_ll, base + 1);
#pragma unroll
  for (int j = 0; j < PPT; ++j) pr[j] = qr[j] = 0.0;

  const double tol2 = a.cg_tol * a.cg_tol * bnorm2;
  double prev = bnorm2, beta = 0.0;
  int streak = 0, status = 0;
  bool pending = false;  // an (r.r, r.z) all-reduce has been published
  *its = 0;
  PcgTrace trc(a);
  for (int it = 0;; ++it) {
    const bool more = it < a.cg_max;
    double wv[PPT];  // H z of this iteration
    if (more) {
      __syncthreads();  // own-tile z of the last sweep
      t.template spmv<false>(zr, wv);  // interior while the halo travels
      trc.mark(1);
      t.ring(a, z_ll, base + (unsigned)it + 1u);
      __syncthreads();
      trc.mark(0);
      t.template spmv<true>(zr, wv);
      trc.mark(1);
    }
    if (pending) {  // finish iteration it-1: fusion.hpp:350-364
      double v2[2];
      grid_allreduce_wait(c, v2);
      pending = false;
      trc.mark(2);
      const double rn = v2[0];
      if (rn <= tol2) break;
      if (rn > prev) {
        if (++streak >= 10) {
          status = DFUSE_E_CG_DIVERGENCE;
          break;
        }
      } else {
        streak = 0;
      }
      prev = rn;
      beta = v2[1] / rz;
      rz = v2[1];
    }
    if (!more) break;
    *its = it + 1;
    double pq = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (t.gi_[j] >= 0) {
        const double p = it == 0 ? zr[j] : zr[j] + beta * pr[j];
        const double q = it == 0 ? wv[j] : wv[j] + beta * qr[j];
        pr[j] = p;
        qr[j] = q;
        pq += p * q;
      }
    }
    trc.mark(3);
    double v1[1] = {pq};
    grid_allreduce<1, false>(c, v1);
    trc.mark(4);
    if (!(v1[0] > 0.0)) {  // fusion.hpp:342
      status = DFUSE_E_CG_DIVERGENCE;
      break;
    }
    const double alpha = rz / v1[0];
    double rr = 0.0, rzn = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (t.gi_[j] >= 0) {
        const int k = threadIdx.x + FT * j;
        t.s_x[k] = t.s_x[k] + alpha * pr[j];
        const double r = rr_[j] - alpha * qr[j];
        rr_[j] = r;
        rr += r * r;
        const double rd = t.s_rdiag[k];
        const double q0 = r * rd;
        const double z = __fma_rn(__fma_rn(-q0, t.s_diag[k], r), rd, q0);
        zr[j] = z;
        t.s_z[t.so_[j]] = z;
        rzn += r * z;
        if (t.boundary(j)) ll_store(z_ll + 2 * (long)t.gi(j), z, base + (unsigned)it + 2u);
      }
    }
    double v2[2] = {rr, rzn};
    grid_allreduce_publish(c, v2);
    pending = true;
    trc.mark(5);
  }
  trc.flush(a);
  if (pending) {  // broke out before collecting: keep the phase counter in step
    double v2[2];
    grid_allreduce_wait(c, v2);
  }
  t.store_x(a);
  grid_sync(c);
  return status;
}

// shared memory of the resident PCG for a tw_max x th_max tile
inline size_t pcg_tile_smem(int tw_max, int th_max) {
  return sizeof(double) * (7 * (size_t)tw_max * th_max + (size_t)(th_max + 2) * (tw_max + 2));
}
