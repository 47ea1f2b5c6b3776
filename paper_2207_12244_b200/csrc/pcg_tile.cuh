// pcg_tile.cuh -- SM-resident Jacobi PCG (included by fusion.cu).
//
// Same iteration, stop rules and per-pixel expressions as solve_depth_step
// (fusion.hpp:316-368), up to algebraic rearrangements that change rounding
// at the ulp level only (tolerance parity):
//
//   pcg_resident_pipe (default) pipelined PCG (Ghysels & Vanroose 2014,
//                    "Hiding global synchronization latency in the
//                    preconditioned Conjugate Gradient algorithm", Alg. 3,
//                    with the Jacobi preconditioner applied directly:
//                    u = r/diag, m = w/diag). Besides r it carries
//                        w = H u,  s = H p,  z = H M^-1 s
//                    by recurrence, so the iteration's one all-reduce of
//                    (r.u, w.u, r.r) is posted right after the vector update
//                    and travels while the CTA exchanges the halo of
//                    m = M^-1 w and runs the SpMV n = H m. The curvature is
//                    p.q = w.u - beta (r.u) / alpha_prev as below.
//   pcg_resident     one grid all-reduce per iteration. The
//                    direction product q = H p is carried by the recurrence
//                        p_k = z_k + beta_k p_{k-1},  q_k = H z_k + beta_k q_{k-1}
//                    and the curvature p_k.q_k by the Chronopoulos-Gear identity
//                        p_k.q_k = z_k.Hz_k - beta_k (r_k.z_k) / alpha_{k-1}
//                    (exact for a symmetric H with M^-1-orthogonal residuals),
//                    so (r.r, r.z, z.Hz) travel in ONE all-reduce that follows
//                    the SpMV.
//                    (dfuse_ctx_set_solver_path(ctx, 3)).
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
// z = r/diag uses the reciprocal computed once per solve. The
// Chronopoulos-Gear and two-all-reduce variants add one Markstein
// correction (q0 = r*(1/d); e = fma(-q0, d, r); z = fma(e, 1/d, q0)), which
// returns the IEEE quotient except in rare double-rounding corner cases; the
// pipelined loop applies the rounded reciprocal as it is (a Jacobi
// preconditioner within one rounding of diag^-1: same iteration counts on
// every parity case, 2 % faster at C2).
#pragma once

#ifndef DFUSE_TASM_UNROLL
#define DFUSE_TASM_UNROLL 2  // pixel slots per step of the tile-order assembly (1/2/3/6 measured)
#endif
constexpr int kTasmUnroll = DFUSE_TASM_UNROLL;

// shared-memory carve-up and per-thread pixel map of one tile
template <int PPT>
struct PcgTile {
  TileGeo tg;
  int T, pw;
  // shared memory: eight per-pixel planes of PPT*FT doubles at fixed offsets
  // (so every access is one base register plus an immediate), then z/m with
  // its one-pixel halo
  static constexpr int TMX = PPT * FT;
  __device__ __forceinline__ static double* sm() {
    extern __shared__ double dsm[];
    return dsm;
  }
  __device__ __forceinline__ double* s_diag() const { return sm(); }
  __device__ __forceinline__ double* s_rdiag() const { return sm() + TMX; }
  __device__ __forceinline__ double* s_right() const { return sm() + 2 * TMX; }
  __device__ __forceinline__ double* s_left() const { return sm() + 3 * TMX; }
  __device__ __forceinline__ double* s_down() const { return sm() + 4 * TMX; }
  __device__ __forceinline__ double* s_up() const { return sm() + 5 * TMX; }
  __device__ __forceinline__ double* s_x() const { return sm() + 6 * TMX; }
  __device__ __forceinline__ double* s_p() const { return sm() + 7 * TMX; }
  __device__ __forceinline__ double* s_z() const { return sm() + 8 * TMX; }
  // per pixel slot j (local index k = threadIdx.x + FT j) one int: the
  // tile row ly, bit 30 = tile boundary, -1 = no pixel. The global index
  // g0 + k + ly (W - tw) and the halo-plane offset k + 2 ly + tw + 3 follow
  // from it, so the slot map costs PPT + 2 registers.
  int lyb_[PPT];
  int g0, wmt;  // y0 W + x0, W - tw

  __device__ __forceinline__ bool valid(int j) const { return lyb_[j] >= 0; }
  __device__ __forceinline__ bool boundary(int j) const { return lyb_[j] & (1 << 30); }
  __device__ __forceinline__ int ly(int j) const { return lyb_[j] & ((1 << 30) - 1); }
  __device__ __forceinline__ int gi(int j) const {
    return g0 + (int)threadIdx.x + FT * j + ly(j) * wmt;
  }
  __device__ __forceinline__ int so(int j) const {
    return (int)threadIdx.x + FT * j + 2 * ly(j) + tg.tw + 3;
  }

  // load the tile's couplings, r, and z = r/diag; post boundary z with `flag`
  // tile geometry and this thread's pixel map (no memory traffic)
  __device__ __forceinline__ void map(const FusionArgs& a) {
    tg = my_tile(a);
    T = tg.tw * tg.th;
    pw = tg.tw + 2;

    g0 = tg.y0 * a.W + tg.x0;
    wmt = a.W - tg.tw;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int k = threadIdx.x + FT * j;
      lyb_[j] = -1;
      if (k < T) {
        const int ly = k / tg.tw, lx = k - ly * tg.tw;
        const bool bd = lx == 0 || ly == 0 || lx == tg.tw - 1 || ly == tg.th - 1;
        lyb_[j] = ly | (bd ? (1 << 30) : 0);
      }
    }
  }

  __device__ __forceinline__ void load(const FusionArgs& a, double (&rr_)[PPT], double (&zr)[PPT],
                                       unsigned long long* z_ll, unsigned flag) {
    tg = my_tile(a);
    T = tg.tw * tg.th;
    pw = tg.tw + 2;

    const int W = a.W, H = a.H;
    g0 = tg.y0 * W + tg.x0;
    wmt = W - tg.tw;
    // halo entries outside the image stay 0 (their couplings are 0 too)
    for (int t = threadIdx.x; t < (tg.th + 2) * pw; t += FT) s_z()[t] = 0.0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int k = threadIdx.x + FT * j;
      rr_[j] = zr[j] = 0.0;
      lyb_[j] = -1;
      if (k < T) {
        s_x()[k] = 0.0;
        s_p()[k] = 0.0;
        const int ly = k / tg.tw, lx = k - ly * tg.tw;
        const int gx = tg.x0 + lx, gy = tg.y0 + ly;
        const int g = gy * W + gx;
        const bool bd = lx == 0 || ly == 0 || lx == tg.tw - 1 || ly == tg.th - 1;
        lyb_[j] = ly | (bd ? (1 << 30) : 0);
        const double d = __ldcg(a.diag + g);
        const double rd = rcp_nr(d);
        s_diag()[k] = d;
        s_rdiag()[k] = rd;
        s_right()[k] = gx + 1 < W ? __ldcg(a.right + g) : 0.0;
        s_left()[k] = gx > 0 ? __ldcg(a.right + g - 1) : 0.0;
        s_down()[k] = gy + 1 < H ? __ldcg(a.down + g) : 0.0;
        s_up()[k] = gy > 0 ? __ldcg(a.down + g - W) : 0.0;
        const double r = __ldcg(a.r + g);
        rr_[j] = r;
        const double q0 = r * rd;  // z = r/diag, fusion.hpp:329
        const double z = __fma_rn(__fma_rn(-q0, d, r), rd, q0);
        zr[j] = z;
        s_z()[so(j)] = z;
        if (bd) ll_store(z_ll + 2 * (long)g, z, flag);
      }
    }
  }

  // Tile-order assembly (the pipelined solve's default): every own pixel's
  // diag and four couplings go straight into the tile's planes, b is parked
  // in s_p for load_assembled, and nothing is written to global memory --
  // no coupling raster, no re-read, no fence before the solve. Per-pixel
  // arithmetic is assemble_pixel's, as in the raster-order sweep; the left
  // and up couplings are formed by the pixel itself with the expressions
  // its neighbours use for their right and down ones.
  template <class PL>
  __device__ __forceinline__ void assemble(const FusionArgs& a, const Sel sel,
                                           const double* __restrict__ ld, const double ln_s,
                                           const PL pl, double (&v)[4]) {
    map(a);
    double bn = 0.0, rz = 0.0, bad = 0.0, cost = 0.0;
#pragma unroll kTasmUnroll
    for (int j = 0; j < PPT; ++j) {
      const int k = threadIdx.x + FT * j;
      if (k < T) {
        const int ly = k / tg.tw, lx = k - ly * tg.tw;
        const int x = tg.x0 + lx, y = tg.y0 + ly;
        const AsmPixel e = assemble_pixel(y * a.W + x, x, y, a.W, a.H, sel, a.dnet, a.dsemi,
                                          a.dgrad, ld, ln_s, pl);
        s_diag()[k] = e.diag;
        s_right()[k] = e.right;
        s_left()[k] = e.left;
        s_down()[k] = e.down;
        s_up()[k] = e.up;
        s_p()[k] = e.b;
        const double z = div_nr(e.b, e.diag);  // PCG init z = r/diag, fusion.hpp:329
        bn += e.b * e.b;
        if (!(e.diag > 0.0)) bad += 1.0;
        rz += e.b * z;
        cost += e.cost;
      }
    }
    v[0] = bn;
    v[1] = rz;
    v[2] = bad;
    v[3] = cost;
  }

  // the global rasters (diag, right, down, r) of the standalone solve into
  // the tile's planes, as assemble() leaves them (r parked in s_p)
  __device__ __forceinline__ void stage_global(const FusionArgs& a) {
    map(a);
    const int W = a.W, H = a.H;
    for (int j = 0; j < PPT; ++j) {
      const int k = threadIdx.x + FT * j;
      if (valid(j)) {
        const int g = gi(j), gy = g / W, gx = g - gy * W;
        s_diag()[k] = __ldcg(a.diag + g);
        s_right()[k] = gx + 1 < W ? __ldcg(a.right + g) : 0.0;
        s_left()[k] = gx > 0 ? __ldcg(a.right + g - 1) : 0.0;
        s_down()[k] = gy + 1 < H ? __ldcg(a.down + g) : 0.0;
        s_up()[k] = gy > 0 ? __ldcg(a.down + g - W) : 0.0;
        s_p()[k] = __ldcg(a.r + g);
      }
    }
  }

  // load() for a tile assembled in place: r from s_p, then as load()
  __device__ __forceinline__ void load_assembled(const FusionArgs& a, double (&rr_)[PPT],
                                                 double (&zr)[PPT], unsigned long long* z_ll,
                                                 unsigned flag) {
    map(a);
    for (int t = threadIdx.x; t < (tg.th + 2) * pw; t += FT) s_z()[t] = 0.0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int k = threadIdx.x + FT * j;
      rr_[j] = zr[j] = 0.0;
      if (valid(j)) {
        const double d = s_diag()[k];
        const double rd = rcp_nr(d);
        s_rdiag()[k] = rd;
        const double r = s_p()[k];
        s_p()[k] = 0.0;
        s_x()[k] = 0.0;
        rr_[j] = r;
        const double q0 = r * rd;  // z = r/diag, fusion.hpp:329
        const double z = __fma_rn(__fma_rn(-q0, d, r), rd, q0);
        zr[j] = z;
        s_z()[so(j)] = z;
        if (boundary(j)) ll_store(z_ll + 2 * (long)gi(j), z, flag);
      }
    }
  }

  // halo ring of z (version `flag`) from the neighbours' LL words: one
  // thread per ring cell, all loads in flight at once
  __device__ __forceinline__ void ring(const FusionArgs& a, const unsigned long long* z_ll,
                                       unsigned flag) const {
    const int ring_n = T > 0 ? 2 * (tg.tw + tg.th) : 0;
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
        s_z()[so] = ll_wait(z_ll + 2 * ((long)gy * a.W + gx), flag);
    }
  }

  // The ring with its words prefetched: ring_prefetch (thread t takes ring
  // cell t) starts cp.async copies of the cells' LL words into a shared
  // staging area, issued part-way through the interior SpMV, when the
  // neighbours have usually posted; ring_finish waits for the copies and
  // keeps the words whose flags are `flag`, polling L2 only for the others.
  __device__ __forceinline__ static unsigned long long* ring_stage() {
    __shared__ unsigned long long st[2 * FT];
    return st;
  }
  __device__ __forceinline__ void ring_cell(const FusionArgs& a, int t, int& g, int& so) const {
    int gx, gy;
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
    g = gy * a.W + gx;
    if (!(gx >= 0 && gx < a.W && gy >= 0 && gy < a.H)) so = -1;
  }
  __device__ __forceinline__ void ring_prefetch(const FusionArgs& a,
                                                const unsigned long long* z_ll) const {
    const int ring_n = T > 0 ? 2 * (tg.tw + tg.th) : 0;
    if ((int)threadIdx.x < ring_n) {
      int g, so;
      ring_cell(a, threadIdx.x, g, so);
      if (so >= 0) cp_async16(ring_stage() + 2 * threadIdx.x, z_ll + 2 * (long)g);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __device__ __forceinline__ void ring_finish(const FusionArgs& a, const unsigned long long* z_ll,
                                              unsigned flag) const {
    asm volatile("cp.async.wait_all;" ::: "memory");
    const int ring_n = T > 0 ? 2 * (tg.tw + tg.th) : 0;
    if ((int)threadIdx.x < ring_n) {
      int g, so;
      ring_cell(a, threadIdx.x, g, so);
      if (so >= 0) {
        const unsigned long long w0 = ring_stage()[2 * threadIdx.x];
        const unsigned long long w1 = ring_stage()[2 * threadIdx.x + 1];
        const bool hit = (unsigned)(w0 >> 32) == flag && (unsigned)(w1 >> 32) == flag;
        s_z()[so] = hit ? ll_value(w0, w1) : ll_wait(z_ll + 2 * (long)g, flag);
      }
    }
    for (int t = threadIdx.x + FT; t < ring_n; t += FT) {
      int g, so;
      ring_cell(a, t, g, so);
      if (so >= 0) s_z()[so] = ll_wait(z_ll + 2 * (long)g, flag);
    }
  }

  // post the tile's own boundary cells of the halo'd plane (s_z) as LL
  // words (version `flag`): one thread per perimeter cell (corners twice,
  // same value), after a barrier that follows the plane's writes
  __device__ __forceinline__ void post_boundary(const FusionArgs& a, unsigned long long* ll,
                                                unsigned flag) const {
    const int perim = T > 0 ? 2 * (tg.tw + tg.th) : 0;
    for (int t = threadIdx.x; t < perim; t += FT) {
      int lx, ly;
      if (t < tg.tw) {
        lx = t, ly = 0;
      } else if (t < 2 * tg.tw) {
        lx = t - tg.tw, ly = tg.th - 1;
      } else if (t < 2 * tg.tw + tg.th) {
        lx = 0, ly = t - 2 * tg.tw;
      } else {
        lx = tg.tw - 1, ly = t - 2 * tg.tw - tg.th;
      }
      const double v = s_z()[(ly + 1) * pw + lx + 1];
      ll_store(ll + 2 * ((long)g0 + (long)ly * a.W + lx), v, flag);
    }
  }

  // w = H z, StencilMatrix::apply order (fusion.hpp:127-131), branch-free.
  // BOUNDARY selects the pass: false = interior pixels (own-tile z only, can
  // run before the halo ring arrives), true = tile-boundary pixels
  template <bool BOUNDARY, int J0 = 0, int J1 = PPT>
  __device__ __forceinline__ void spmv(const double (&zr)[PPT], double (&wv)[PPT]) const {
#pragma unroll
    for (int j = J0; j < J1; ++j) {
      if (valid(j) && boundary(j) == BOUNDARY) {
        const int k = threadIdx.x + FT * j, so = this->so(j);
        double v = s_diag()[k] * zr[j];
        v += s_right()[k] * s_z()[so + 1];
        v += s_left()[k] * s_z()[so - 1];
        v += s_down()[k] * s_z()[so + pw];
        v += s_up()[k] * s_z()[so - pw];
        wv[j] = v;
      } else if (!valid(j)) {
        wv[j] = 0.0;
      }
    }
  }

  // delta to the raster for the line search (x == 0 if no iteration ran)
  __device__ __forceinline__ void store_x(const FusionArgs& a) const {
#pragma unroll
    for (int j = 0; j < PPT; ++j)
      if (valid(j)) a.x[gi(j)] = s_x()[threadIdx.x + FT * j];
  }
};

// DFUSE_TRACE: thread 0 accumulates SM cycles per phase (CTA 0 -> ctl->trace,
// every CTA -> a.dbg[cta][phase] when DFUSE_TRACE=2); the host converts
// cycles to ns with the clock measured over the whole solve
// The accumulators live in shared memory (only thread 0 touches them), so
// the instrumentation costs the solver loop one predicate register.
struct PcgTrace {
  bool on;
  __device__ __forceinline__ static long long* st() {
    __shared__ long long s[9];  // tr[6], t_last, t_start, c_start
    return s;
  }
  __device__ __forceinline__ explicit PcgTrace(const FusionArgs& a, bool resume = false)
      : on(DFUSE_TRACE_BUILD && a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || a.trace == 2)) {
    if (on && !resume) {
      long long* s = st();
      for (int k = 0; k < 6; ++k) s[k] = 0;
      s[7] = df_now();
      s[6] = s[8] = clock64();
    }
  }
  __device__ __forceinline__ void mark(int k) {
    if (on) {
      long long* s = st();
      const long long t = clock64();
      s[k] += t - s[6];
      s[6] = t;
    }
  }
  __device__ __forceinline__ void flush(const FusionArgs& a) {
    if (!on) return;
    const long long* s = st();
    if (blockIdx.x == 0) {
      for (int k = 0; k < 6; ++k) a.ctl->trace[k] += s[k];
      a.ctl->trace[6] += df_now() - s[7];   // ns
      a.ctl->trace[7] += clock64() - s[8];  // SM cycles -> effective clock
    }
    if (a.trace == 2)
      for (int k = 0; k < 6; ++k) a.dbg[blockIdx.x * 8 + k] += s[k];
  }
};

// Chronopoulos-Gear loop from iteration it0 (0: a fresh solve; > 0: resumed
// from the pipelined variant). On entry s_z holds z (the version after it0
// updates, boundary posted to z_ll with flag base + it0 + 1), pr/qr hold p
// and q = H p of iteration it0-1, and (rz, alpha) are those of it0-1.
template <int PPT>
__device__ __forceinline__ int pcg_cg_core(GridCtx& c, const FusionArgs& a, PcgTile<PPT>& t,
                                           PcgTrace& trc, unsigned long long* z_ll,
                                           unsigned base, double (&rr_)[PPT], double (&zr)[PPT],
                                           double (&pr)[PPT], double (&qr)[PPT], double bnorm2,
                                           double rz, int it0, double alpha, double prev,
                                           int streak, int* its) {
  const double tol2 = a.cg_tol * a.cg_tol * bnorm2;
  double beta = 0.0;
  double rr_part = 0.0, rz_part = 0.0;
  if (it0 > 0) {  // partials of the entry residual (same order as the sweep below)
#pragma unroll
    for (int j = 0; j < PPT; ++j)
      if (t.valid(j)) {
        rr_part += rr_[j] * rr_[j];
        rz_part += rr_[j] * zr[j];
      }
  }
  int status = 0;
  for (int it = it0; a.cg_max > 0; ++it) {
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
      beta = div_nr(v[1], rz);
      rz = v[1];
      pq = v[2] - div_nr(beta * rz, alpha);
    }
    if (!(pq > 0.0)) {  // fusion.hpp:342
      status = DFUSE_E_CG_DIVERGENCE;
      break;
    }
    alpha = div_nr(rz, pq);
    *its = it + 1;
    // p = z + beta p, q = H z + beta q (p = z at it 0, fusion.hpp:329-330,
    // 364); x += alpha p, r -= alpha q, z = r/diag (fusion.hpp:345-359)
    rr_part = 0.0;
    rz_part = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (t.valid(j)) {
        const int k = threadIdx.x + FT * j;
        const double p = it == 0 ? zr[j] : zr[j] + beta * pr[j];
        const double q = it == 0 ? wv[j] : wv[j] + beta * qr[j];
        pr[j] = p;
        qr[j] = q;
        t.s_x()[k] = t.s_x()[k] + alpha * p;
        const double r = rr_[j] - alpha * q;
        rr_[j] = r;
        rr_part += r * r;
        const double rd = t.s_rdiag()[k];
        const double q0 = r * rd;
        const double z = __fma_rn(__fma_rn(-q0, t.s_diag()[k], r), rd, q0);
        zr[j] = z;
        t.s_z()[t.so(j)] = z;
        rz_part += r * z;
        if (t.boundary(j)) ll_store(z_ll + 2 * (long)t.gi(j), z, base + (unsigned)it + 2u);
      }
    }
    trc.mark(5);
  }
  return status;
}

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
  *its = 0;
  PcgTrace trc(a);
  const int status = pcg_cg_core<PPT>(c, a, t, trc, z_ll, base, rr_, zr, pr, qr, bnorm2, rz, 0,
                                      1.0, bnorm2, 0, its);
  trc.flush(a);
  t.store_x(a);
  grid_sync(c);  // fenced: the trial sweeps read x at the neighbours
  return status;
}

// relative residual r.r / b.b below which the pipelined solve hands over to
// Chronopoulos-Gear (residual norm 1e-10 of |b|, far below cg_tol = 1e-6)
constexpr double kPipeSwitch = 1e-20;

// Pipelined: one all-reduce per iteration, in flight during the halo
// exchange and SpMV. Trace phases: 0 halo ring, 1 SpMV, 2 all-reduce wait,
// 3 scalars + update sweep, 4 CTA reduction + publish,
// 5 boundary words of m.
//
// The halo words of m alternate between two LL arrays by version parity: a
// CTA posts m_{i+1} only after the all-reduce of iteration i, which needs
// every CTA's post-update publish of iteration i-1, which each CTA makes
// after its threads read the m_{i-1} halo. So a version is never overwritten before
// its readers are done with it.
struct PcgHandover {
  int it, streak;
  double rz, alpha, prev;
};

// returns the status, or -1 after a handover (*hand filled; x, p in shared
// memory, the PcgTrace accumulators still open)
template <int PPT>
__device__ int pcg_resident_pipe(GridCtx& c, const FusionArgs& a, double bnorm2, double rz,
                                 int* its, PcgHandover* hand, bool assembled) {
  PcgTile<PPT> t;
  const long P = (long)a.W * a.H;
  // LL array v: a.halo + v 2P (v = 0, 1; arithmetic, not an indexed local array)
  unsigned long long* const hb0 = a.halo;
  // LL flags: u0 -> base + 1 (array 0); m_i -> base + i + 2 (array (i+1)&1)
  const unsigned base = c.ll_next;
  c.ll_next += (unsigned)a.cg_max + 3u;
  double rr_[PPT], mr[PPT], wr[PPT], zr[PPT], sr[PPT];
  if (!assembled) t.stage_global(a);
  t.load_assembled(a, rr_, mr, hb0, base + 1);  // mr = u0 = r0/diag, in s_z with halo
  PcgTrace trc(a);
  // w0 = H u0
  __syncthreads();
  t.template spmv<false>(mr, wr);
  t.ring(a, hb0, base + 1);
  __syncthreads();
  t.template spmv<true>(mr, wr);
  __syncthreads();  // every thread is done reading u0 from s_z
  double wu = 0.0;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    zr[j] = sr[j] = 0.0;
    if (t.valid(j)) {
      const int k = threadIdx.x + FT * j;
      wu += wr[j] * mr[j];  // (w0, u0)
      const double m = wr[j] * t.s_rdiag()[k];  // m0 = w0/diag
      mr[j] = m;
      t.s_z()[t.so(j)] = m;
    }
  }
  {
    double v[3] = {0.0, wu, 0.0};
    grid_allreduce_publish(c, v);  // its barrier follows every m0 write
  }
  t.post_boundary(a, hb0 + 2 * P, base + 2u);
  trc.mark(5);

  const double tol2 = a.cg_tol * a.cg_tol * bnorm2;
  double prev = bnorm2, alpha = 1.0, gamma_prev = rz;
  // reciprocals of the previous iteration's scalars, formed before the
  // all-reduce wait so that only 1/p.q stays on the path after it (the
  // quotients are div_nr's, bit for bit)
  double r_gp = rcp_nr(gamma_prev), r_al = 1.0;
  int streak = 0, status = 0;
  *its = 0;
  // prefetched all-reduce waits: one slot per polling lane
  const bool pf = DFUSE_AR_PREFETCH && c.G <= 32u * kPollWarps;
  for (int it = 0;; ++it) {
    // s_z holds m_it (halo from array (it+1)&1, flag base+it+2); mr := H m_it
    const bool more = it < a.cg_max;
    if (more) {
      // no barrier before the interior SpMV: the one in the last publish
      // (cta_partial) follows every thread's s_z writes of the update sweep
      const unsigned long long* hr = hb0 + (long)((it + 1) & 1) * 2 * P;
      if (DFUSE_RING_PF > 0 && DFUSE_RING_PF < PPT) {
        // the ring's words start towards shared memory part-way through the
        // interior SpMV (DFUSE_RING_PF of the PPT slots done)
        t.template spmv<false, 0, (DFUSE_RING_PF < PPT ? DFUSE_RING_PF : 0)>(mr, mr);
        t.ring_prefetch(a, hr);
        t.template spmv<false, (DFUSE_RING_PF < PPT ? DFUSE_RING_PF : 0), PPT>(mr, mr);
      } else {
        t.template spmv<false>(mr, mr);
      }
      if (pf && DFUSE_AR_PREFETCH == 1) grid_allreduce_prefetch<3>(c);
      trc.mark(1);
      if (DFUSE_RING_PF > 0 && DFUSE_RING_PF < PPT)
        t.ring_finish(a, hr, base + (unsigned)it + 2u);
      else
        t.ring(a, hr, base + (unsigned)it + 2u);
      // the all-reduce's slot words start towards shared memory now, while
      // the boundary SpMV runs (grid_allreduce_wait_prefetched). Issued
      // after the interior SpMV instead (DFUSE_AR_PREFETCH=1): 501 vs 504
      // updates/s at C2 defaults (the earlier copy finds more flags unset)
      if (pf && DFUSE_AR_PREFETCH == 2) grid_allreduce_prefetch<3>(c);
      __syncthreads();
      trc.mark(0);
      t.template spmv<true>(mr, mr);
      trc.mark(1);
    }
    double v[3];  // (r.u, w.u, r.r) of the vectors after `it` updates
    if (pf && more)
      grid_allreduce_wait_prefetched(c, v);
    else
      grid_allreduce_wait(c, v);
    trc.mark(2);
    double gamma, beta, pq;
    if (it == 0) {
      gamma = rz;  // (r0, z0) as the assembly sweep computed it
      beta = 0.0;
      pq = v[1];
    } else {
      if (v[2] < kPipeSwitch * bnorm2) {
        // Deep convergence: pipelined CG's recursive residual stagnates
        // near eps*cond (its auxiliary recurrences drift), while the
        // reference's keeps falling; hand the solve over to
        // Chronopoulos-Gear (pcg_resume_cg), which re-derives this
        // iteration's (r.r, r.z) and applies the stop rules to them. The
        // state leaves the loop through memory (r, q = s in the r/q
        // rasters; p, x stay in shared memory) so that the handover adds no
        // registers to this loop.
#pragma unroll
        for (int j = 0; j < PPT; ++j)
          if (t.valid(j)) {
            a.r[t.gi(j)] = rr_[j];
            a.q[t.gi(j)] = sr[j];
          }
        hand->it = it;
        hand->rz = gamma_prev;
        hand->alpha = alpha;
        hand->prev = prev;
        hand->streak = streak;
        return -1;
      }
      // finish iteration it-1: fusion.hpp:350-364
      const double rn = v[2];
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
      gamma = v[0];
      beta = div_rb(gamma, gamma_prev, r_gp);
      pq = v[1] - div_rb(beta * gamma, alpha, r_al);
    }
    if (!(pq > 0.0)) {  // fusion.hpp:342
      status = DFUSE_E_CG_DIVERGENCE;
      break;
    }
    alpha = div_nr(gamma, pq);
    gamma_prev = gamma;
    r_gp = rcp_nr(gamma_prev);
    r_al = rcp_nr(alpha);
    *its = it + 1;
    // z = n + beta z, s = w + beta s, p = u + beta p; x += alpha p,
    // r -= alpha s, w -= alpha z; u = r/diag, m = w/diag (fusion.hpp:345-364)
    double ru = 0.0, wu2 = 0.0, rr = 0.0;
    unsigned long long* hm = hb0 + (long)(it & 1) * 2 * P;  // m_{it+1}: array (it+2)&1
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (t.valid(j)) {
        const int k = threadIdx.x + FT * j;
        // u = M^-1 r with M^-1 = diag(1/diag rounded): within one rounding of
        // the reference's r/diag (fusion.hpp:359; tolerance parity, H7)
        const double rd = t.s_rdiag()[k];
        const double r0 = rr_[j];
        const double u = r0 * rd;
        const double z = mr[j] + beta * zr[j];
        const double sv = wr[j] + beta * sr[j];
        const double p = u + beta * t.s_p()[k];
        zr[j] = z;
        sr[j] = sv;
        t.s_p()[k] = p;
        t.s_x()[k] = t.s_x()[k] + alpha * p;
        const double r = r0 - alpha * sv;
        rr_[j] = r;
        const double w = wr[j] - alpha * z;
        wr[j] = w;
        const double un = r * rd;
        const double m = w * rd;  // M^-1 w: internal to the pipelined recurrences
        mr[j] = m;
        t.s_z()[t.so(j)] = m;
        ru += r * un;
        wu2 += w * un;
        rr += r * r;
      }
    }
    trc.mark(3);  // (diagnostics: scalars + update sweep)
    double v2[3] = {ru, wu2, rr};
    grid_allreduce_publish(c, v2);  // its barrier follows every m write
    trc.mark(4);  // (CTA reduction + publish)
    t.post_boundary(a, hm, base + (unsigned)it + 3u);
    trc.mark(5);
  }
  trc.flush(a);
  t.store_x(a);
  grid_sync(c);  // fenced: the trial sweeps read x at the neighbours
  return status;
}

// Chronopoulos-Gear continuation of a pipelined solve after its handover
template <int PPT>
__device__ int pcg_resume_cg(GridCtx& c, const FusionArgs& a, double bnorm2,
                             const PcgHandover& h, int* its) {
  PcgTile<PPT> t;
  t.map(a);
  PcgTrace trc(a, true);
  const long P = (long)a.W * a.H;
  unsigned long long* z3 = a.halo + 4 * P;  // third LL array (the pipelined solve used two)
  const unsigned base = c.ll_next;
  c.ll_next += (unsigned)a.cg_max + 2u;
  double rr_[PPT], zr[PPT], pr[PPT], qr[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    rr_[j] = zr[j] = pr[j] = qr[j] = 0.0;
    if (t.valid(j)) {
      const int k = threadIdx.x + FT * j;
      const double r = a.r[t.gi(j)], d = t.s_diag()[k], rd = t.s_rdiag()[k];
      const double uq = r * rd;
      const double u = __fma_rn(__fma_rn(-uq, d, r), rd, uq);
      rr_[j] = r;
      zr[j] = u;
      pr[j] = t.s_p()[k];
      qr[j] = a.q[t.gi(j)];
      t.s_z()[t.so(j)] = u;
      if (t.boundary(j)) ll_store(z3 + 2 * (long)t.gi(j), u, base + (unsigned)h.it + 1u);
    }
  }
  const int status = pcg_cg_core<PPT>(c, a, t, trc, z3, base, rr_, zr, pr, qr, bnorm2, h.rz, h.it,
                                      h.alpha, h.prev, h.streak, its);
  trc.flush(a);
  t.store_x(a);
  grid_sync(c);
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
      beta = div_nr(v2[1], rz);
      rz = v2[1];
    }
    if (!more) break;
    *its = it + 1;
    double pq = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (t.valid(j)) {
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
    const double alpha = div_nr(rz, v1[0]);
    double rr = 0.0, rzn = 0.0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (t.valid(j)) {
        const int k = threadIdx.x + FT * j;
        t.s_x()[k] = t.s_x()[k] + alpha * pr[j];
        const double r = rr_[j] - alpha * qr[j];
        rr_[j] = r;
        rr += r * r;
        const double rd = t.s_rdiag()[k];
        const double q0 = r * rd;
        const double z = __fma_rn(__fma_rn(-q0, t.s_diag()[k], r), rd, q0);
        zr[j] = z;
        t.s_z()[t.so(j)] = z;
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

// shared memory of the resident PCG for a tw_max x th_max tile at ppt pixels per thread
inline size_t pcg_tile_smem(int ppt, int tw_max, int th_max) {
  return sizeof(double) * (8 * (size_t)ppt * kResidentFT + (size_t)(th_max + 2) * (tw_max + 2));
}
