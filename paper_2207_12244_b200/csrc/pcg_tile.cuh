// pcg_tile.cuh -- SM-resident Jacobi PCG (included by fusion.cu).
//
// Same iteration, stop rules and per-pixel expressions as solve_depth_step
// (fusion.hpp:316-368), with one algebraic rearrangement: the search
// direction's product q = H p is carried by the recurrence
//     p_k = z_k + beta_k p_{k-1},   q_k = H z_k + beta_k q_{k-1}
// (H linear, so q_k = H p_k exactly in exact arithmetic). H z_k does not need
// beta_k, so each iteration's SpMV runs while the (r.r, r.z) all-reduce that
// produces beta_k is in flight (split-phase all-reduce): the SpMV leaves the
// critical path. Rounding differs from the reference's direct H p at the ulp
// level, inside the solver's tolerance parity.
//
// CTA b owns tile b of a tiles_x x tiles_y partition. For the whole solve:
//   registers : x, r, z, p, q of PPT pixels per thread, their shared-memory
//               offsets and boundary flags
//   shared    : diag, 1/diag, the four off-diagonal couplings of every pixel
//               (right, left = right[i-1], down, up = down[i-W], zero where the
//               reference skips the term, fusion.hpp:128-131), and z with a
//               one-pixel halo
// Only the tile boundary of z leaves the SM: after sweep B each CTA posts its
// boundary z as LL words {32-bit half, 32-bit flag} in a raster-indexed array
// and the neighbours rebuild their halo from them. The LL flags order that
// data, so the all-reduces of the loop need no memory fence.
//
// z = r/diag uses the reciprocal computed once per solve and one Markstein
// correction (q0 = r*(1/d); e = fma(-q0, d, r); z = fma(e, 1/d, q0)), which
// returns the IEEE quotient except in rare double-rounding corner cases.
#pragma once

template <int PPT>
__device__ int pcg_resident(GridCtx& c, const FusionArgs& a, double bnorm2, double rz, int* its) {
  extern __shared__ double dsm[];
  const TileGeo tg = my_tile(a);
  const int T = tg.tw * tg.th;
  const int TM = a.tw_max * a.th_max;
  double* s_diag = dsm;
  double* s_rdiag = dsm + TM;
  double* s_right = dsm + 2 * TM;
  double* s_left = dsm + 3 * TM;
  double* s_down = dsm + 4 * TM;
  double* s_up = dsm + 5 * TM;
  double* s_z = dsm + 6 * TM;  // (th+2) x (tw+2), halo included
  const int W = a.W, H = a.H, pw = tg.tw + 2;
  unsigned long long* z_ll = a.halo;  // [P][2]
  // LL flags of this solve: z after v updates -> base + v + 1
  const unsigned base = c.ll_next;
  c.ll_next += (unsigned)a.cg_max + 2u;

  // halo entries outside the image stay 0 (their couplings are 0 too)
  for (int t = threadIdx.x; t < (tg.th + 2) * pw; t += FT) s_z[t] = 0.0;
  __syncthreads();

  double* s_x = s_z + (a.th_max + 2) * (a.tw_max + 2);  // x lives in shared memory
  double rr_[PPT], zr[PPT], pr[PPT], qr[PPT];
  int so_[PPT];  // offset in s_z
  int gi_[PPT];  // global pixel index (-1: no pixel); bit 30 set: tile boundary
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int k = threadIdx.x + FT * j;
    rr_[j] = zr[j] = pr[j] = qr[j] = 0.0;
    if (k < T) s_x[k] = 0.0;
    gi_[j] = -1;
    so_[j] = 0;
    if (k < T) {
      const int ly = k / tg.tw, lx = k - ly * tg.tw;
      const int gx = tg.x0 + lx, gy = tg.y0 + ly;
      const int gi = gy * W + gx;
      const bool bd = lx == 0 || ly == 0 || lx == tg.tw - 1 || ly == tg.th - 1;
      gi_[j] = gi | (bd ? (1 << 30) : 0);
      so_[j] = (ly + 1) * pw + lx + 1;
      const double d = __ldcg(a.diag + gi);
      const double rd = 1.0 / d;
      s_diag[k] = d;
      s_rdiag[k] = rd;
      s_right[k] = gx + 1 < W ? __ldcg(a.right + gi) : 0.0;
      s_left[k] = gx > 0 ? __ldcg(a.right + gi - 1) : 0.0;
      s_down[k] = gy + 1 < H ? __ldcg(a.down + gi) : 0.0;
      s_up[k] = gy > 0 ? __ldcg(a.down + gi - W) : 0.0;
      const double r = __ldcg(a.r + gi);
      rr_[j] = r;
      const double q0 = r * rd;  // z = r/diag, fusion.hpp:329
      const double z = __fma_rn(__fma_rn(-q0, d, r), rd, q0);
      zr[j] = z;
      s_z[so_[j]] = z;
      if (bd) ll_store(z_ll + 2 * (long)gi, z, base + 1);
    }
  }

  const int ring_n = T > 0 ? 2 * (tg.tw + tg.th) : 0;
  const double tol2 = a.cg_tol * a.cg_tol * bnorm2;
  double prev = bnorm2, beta = 0.0;
  int streak = 0, status = 0;
  bool pending = false;  // an (r.r, r.z) all-reduce has been published
  *its = 0;
  // DFUSE_TRACE: thread 0 accumulates ns per phase (CTA 0 -> ctl->trace,
  // every CTA -> a.dbg[cta][phase] when DFUSE_TRACE=2)
  const bool tracer = a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || a.dbg);
  long long tr[6] = {0, 0, 0, 0, 0, 0}, t_last = tracer ? df_now() : 0;
  const long long t_start = t_last, c_start = tracer ? clock64() : 0;
#define DF_TRACE(k)               \
  if (tracer) {                   \
    const long long t_ = df_now(); \
    tr[k] += t_ - t_last;         \
    t_last = t_;                  \
  }
  for (int it = 0;; ++it) {
    const bool more = it < a.cg_max;
    double wv[PPT];  // H z of this iteration
    if (more) {
      // halo ring of z (the version after it updates) from the neighbours
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
        if (gx >= 0 && gx < W && gy >= 0 && gy < H)
          s_z[so] = ll_wait(z_ll + 2 * ((long)gy * W + gx), base + (unsigned)it + 1u);
      }
      __syncthreads();
      DF_TRACE(0);
      // w = H z, StencilMatrix::apply order (fusion.hpp:127-131), branch-free
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        wv[j] = 0.0;
        if (gi_[j] >= 0) {
          const int k = threadIdx.x + FT * j, so = so_[j];
          double v = s_diag[k] * zr[j];
          v += s_right[k] * s_z[so + 1];
          v += s_left[k] * s_z[so - 1];
          v += s_down[k] * s_z[so + pw];
          v += s_up[k] * s_z[so - pw];
          wv[j] = v;
        }
      }
      DF_TRACE(1);
    }
    if (pending) {  // finish iteration it-1: fusion.hpp:350-364
      double v2[2];
      grid_allreduce_wait(c, v2);
      pending = false;
      DF_TRACE(2);
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
    // p = z + beta p, q = H z + beta q (p = z at it 0, fusion.hpp:329-330)
    double pq = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (gi_[j] >= 0) {
        const double p = it == 0 ? zr[j] : zr[j] + beta * pr[j];
        const double q = it == 0 ? wv[j] : wv[j] + beta * qr[j];
        pr[j] = p;
        qr[j] = q;
        pq += p * q;
      }
    }
    DF_TRACE(3);
    double v1[1] = {pq};
    grid_allreduce<1, false>(c, v1);
    DF_TRACE(4);
    if (!(v1[0] > 0.0)) {  // fusion.hpp:342
      status = DFUSE_E_CG_DIVERGENCE;
      break;
    }
    const double alpha = rz / v1[0];
    // ---- sweep B (fusion.hpp:345-362)
    double rr = 0.0, rzn = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (gi_[j] >= 0) {
        const int k = threadIdx.x + FT * j;
        s_x[k] = s_x[k] + alpha * pr[j];
        const double r = rr_[j] - alpha * qr[j];
        rr_[j] = r;
        rr += r * r;
        const double rd = s_rdiag[k];
        const double q0 = r * rd;
        const double z = __fma_rn(__fma_rn(-q0, s_diag[k], r), rd, q0);
        zr[j] = z;
        s_z[so_[j]] = z;
        rzn += r * z;
        if (gi_[j] & (1 << 30))
          ll_store(z_ll + 2 * (long)(gi_[j] & ~(1 << 30)), z, base + (unsigned)it + 2u);
      }
    }
    double v2[2] = {rr, rzn};
    grid_allreduce_publish(c, v2);
    pending = true;
    DF_TRACE(5);
  }
#undef DF_TRACE
  if (tracer && blockIdx.x == 0) {
    for (int k = 0; k < 6; ++k) a.ctl->trace[k] += tr[k];
    a.ctl->trace[6] += df_now() - t_start;  // ns
    a.ctl->trace[7] += clock64() - c_start;  // SM cycles -> effective clock
  }
  if (tracer && a.dbg)
    for (int k = 0; k < 6; ++k) a.dbg[blockIdx.x * 8 + k] += tr[k];
  if (pending) {  // broke out before collecting: keep the phase counter in step
    double v2[2];
    grid_allreduce_wait(c, v2);
  }
  // delta to the raster for the line search (x == 0 if no iteration ran)
#pragma unroll
  for (int j = 0; j < PPT; ++j)
    if (gi_[j] >= 0) a.x[gi_[j] & ~(1 << 30)] = s_x[threadIdx.x + FT * j];
  grid_sync(c);  // fenced: the trial sweeps read x at the neighbours
  return status;
}

// shared memory of pcg_resident for a tw_max x th_max tile
inline size_t pcg_tile_smem(int tw_max, int th_max) {
  return sizeof(double) * (7 * (size_t)tw_max * th_max + (size_t)(th_max + 2) * (tw_max + 2));
}
