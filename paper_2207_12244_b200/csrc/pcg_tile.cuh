// pcg_tile.cuh -- SM-resident Jacobi PCG (included by fusion.cu).
//
// Same iteration, stop rules and per-pixel expression order as
// solve_depth_step (fusion.hpp:316-368). CTA b owns tile b of a
// tiles_x x tiles_y partition. For the whole solve:
//   registers : x, r, z = r/diag of PPT pixels per thread, their shared-memory
//               offsets and boundary flags
//   shared    : diag, 1/diag, the four off-diagonal couplings of every pixel
//               (right, left = right[i-1], down, up = down[i-W], zero where the
//               reference skips the term, fusion.hpp:128-131), q, and p with a
//               one-pixel halo
// so the SpMV is branch-free and the only traffic leaving the SM per
// iteration is the tile boundary: z (after sweep B) and p (sweep A, parity
// buffer) as LL words {32-bit half, 32-bit flag} in raster-indexed arrays.
// Each CTA rebuilds its halo as p = z + beta p_prev from the neighbours'
// words -- the owner's expression on the owner's bits, so halo and owner
// agree exactly -- and the LL flags order that data, so the two grid
// all-reduces per iteration (p.q; r.r and r.z) need no memory fence.
//
// z = r/diag uses the reciprocal computed once per solve and one Markstein
// correction (q0 = r*(1/d); e = fma(-q0, d, r); z = fma(e, 1/d, q0)), which
// returns the IEEE quotient except in rare double-rounding corner cases; the
// reference's sequential reductions already make the solver a tolerance
// (not bit) parity target.
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
  double* s_q = dsm + 6 * TM;
  double* s_p = dsm + 7 * TM;  // (th+2) x (tw+2), halo included
  const int W = a.W, H = a.H, pw = tg.tw + 2;
  const long P = (long)W * H;
  unsigned long long* z_ll = a.halo;  // [P][2]
  unsigned long long* p_ll[2] = {a.halo + 2 * P, a.halo + 4 * P};
  // LL flags of this solve: z version v -> base + v; p of iteration it -> base + it + 1
  const unsigned base = c.ll_next;
  c.ll_next += (unsigned)a.cg_max + 2u;

  // halo entries outside the image stay 0 (their couplings are 0 too)
  for (int t = threadIdx.x; t < (tg.th + 2) * pw; t += FT) s_p[t] = 0.0;

  double xr[PPT], rr_[PPT], zr[PPT];
  int so_[PPT];   // offset in s_p
  int gi_[PPT];   // global pixel index (-1: no pixel); bit 30 set: tile boundary
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int k = threadIdx.x + FT * j;
    xr[j] = rr_[j] = zr[j] = 0.0;
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
      zr[j] = __fma_rn(__fma_rn(-q0, d, r), rd, q0);
      if (bd) ll_store(z_ll + 2 * (long)gi, zr[j], base + 1);
    }
  }
  __syncthreads();

  const int ring_n = T > 0 ? 2 * (tg.tw + tg.th) : 0;
  const double tol2 = a.cg_tol * a.cg_tol * bnorm2;
  double prev = bnorm2, beta = 0.0;
  int streak = 0, status = 0;
  *its = 0;
  // DFUSE_TRACE: CTA 0 / thread 0 accumulates SM cycles per phase
  const bool tracer = a.trace && blockIdx.x == 0 && threadIdx.x == 0;
  long long tr[6] = {0, 0, 0, 0, 0, 0}, t_last = tracer ? df_now() : 0;
#define DF_TRACE(k)                 \
  if (tracer) {                     \
    const long long t_ = df_now(); \
    tr[k] += t_ - t_last;           \
    t_last = t_;                    \
  }
  for (int it = 0; it < a.cg_max; ++it) {
    *its = it + 1;
    const bool first = it == 0;
    // ---- sweep A: halo ring p = z + beta p_prev from the neighbours' LL words
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
      if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
        const long j = (long)gy * W + gx;
        const unsigned fz = base + (first ? 1u : (unsigned)it + 1u), fp = base + (unsigned)it;
        const unsigned long long* zw = z_ll + 2 * j;
        const unsigned long long* pwd = p_ll[(it + 1) & 1] + 2 * j;
        unsigned long long z0, z1, p0 = (unsigned long long)fp << 32, p1 = p0;
        for (;;) {  // all words in flight per round
#if DFUSE_LL_V2_HALO
          ld_relaxed_v2(zw, z0, z1);
          if (!first) ld_relaxed_v2(pwd, p0, p1);
#else
          z0 = ld_relaxed_u64(zw);
          z1 = ld_relaxed_u64(zw + 1);
          if (!first) {
            p0 = ld_relaxed_u64(pwd);
            p1 = ld_relaxed_u64(pwd + 1);
          }
#endif
          if ((unsigned)(z0 >> 32) == fz && (unsigned)(z1 >> 32) == fz &&
              (unsigned)(p0 >> 32) == fp && (unsigned)(p1 >> 32) == fp)
            break;
        }
        const double z = ll_value(z0, z1);
        s_p[so] = first ? z : z + beta * ll_value(p0, p1);
      }
    }
    DF_TRACE(0);
    // own p = z + beta p (fusion.hpp:360,365; p = z at it 0, fusion.hpp:329-330)
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (gi_[j] >= 0) {
        const double p = first ? zr[j] : zr[j] + beta * s_p[so_[j]];
        s_p[so_[j]] = p;
        if (gi_[j] & (1 << 30))
          ll_store(p_ll[it & 1] + 2 * (long)(gi_[j] & ~(1 << 30)), p, base + (unsigned)it + 1u);
      }
    }
    __syncthreads();
    DF_TRACE(1);
    // q = H p, StencilMatrix::apply order (fusion.hpp:127-131), branch-free
    double pq = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (gi_[j] >= 0) {
        const int k = threadIdx.x + FT * j, so = so_[j];
        const double pi = s_p[so];
        double v = s_diag[k] * pi;
        v += s_right[k] * s_p[so + 1];
        v += s_left[k] * s_p[so - 1];
        v += s_down[k] * s_p[so + pw];
        v += s_up[k] * s_p[so - pw];
        s_q[k] = v;
        pq += pi * v;
      }
    }
    DF_TRACE(2);
    double v1[1] = {pq};
    grid_allreduce<1, false>(c, v1);
    DF_TRACE(3);
    if (!(v1[0] > 0.0)) {
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
        xr[j] = xr[j] + alpha * s_p[so_[j]];
        const double r = rr_[j] - alpha * s_q[k];
        rr_[j] = r;
        rr += r * r;
        const double rd = s_rdiag[k];
        const double q0 = r * rd;
        const double z = __fma_rn(__fma_rn(-q0, s_diag[k], r), rd, q0);
        zr[j] = z;
        rzn += r * z;
        if (gi_[j] & (1 << 30))
          ll_store(z_ll + 2 * (long)(gi_[j] & ~(1 << 30)), z, base + (unsigned)it + 2u);
      }
    }
    DF_TRACE(4);
    double v2[2] = {rr, rzn};
    grid_allreduce<2, false>(c, v2);
    DF_TRACE(5);
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
#undef DF_TRACE
  if (tracer)
    for (int k = 0; k < 6; ++k) a.ctl->trace[k] += tr[k];
  // delta to the raster for the line search (x == 0 if no iteration ran)
#pragma unroll
  for (int j = 0; j < PPT; ++j)
    if (gi_[j] >= 0) a.x[gi_[j] & ~(1 << 30)] = xr[j];
  grid_sync(c);  // fenced: the trial sweeps read x at the neighbours
  return status;
}

// shared memory of pcg_resident for a tw_max x th_max tile
inline size_t pcg_tile_smem(int tw_max, int th_max) {
  return sizeof(double) * (7 * (size_t)tw_max * th_max + (size_t)(th_max + 2) * (tw_max + 2));
}
