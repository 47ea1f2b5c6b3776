"""Test fixtures restated from the reference's test support code.

make_random_problem / blank_problem / quadratic_config follow
proj/include/dfuse/testing.hpp:29-65 and tests/test_fusion.cpp:16-37 (numpy's
PCG64 replaces std::mt19937_64, so the draws differ but the distributions
match). semi_from_groundtruth follows tests/support/synthetic.hpp:134-151.
"""
from __future__ import annotations

import numpy as np

from paper_2207_12244_b200._ffi import (FusionState, PredictionSet, RobustConfig, SemiDenseMap)
from paper_2207_12244_b200 import synth


def blank_problem(w, h):
    """test_fusion.cpp:16-29"""
    z = lambda v: np.full((h, w), float(v))
    state = FusionState(z(0.0), 1.0, 0)
    semi = SemiDenseMap.empty(w, h)
    pred = PredictionSet(z(0.0), z(1.0), z(0.0), z(1.0), z(0.0), z(1.0), source_focal=200.0)
    return state, semi, pred


def quadratic_config():
    """test_fusion.cpp:31-37"""
    return RobustConfig(delta_semi=1e9, delta_net=1e9, delta_grad=1e9, cg_tol=1e-12,
                        cg_max_iters=1000)


def make_random_problem(seed, w, h, semi_fraction=0.6, depth_lo=0.5, depth_hi=5.0,
                        outlier_fraction=0.0):
    """testing.hpp:29-65"""
    rng = np.random.default_rng(seed)
    u = lambda lo, hi, n=None: rng.uniform(lo, hi, n)
    P = w * h
    ld = np.log(u(depth_lo, depth_hi, P))
    pl = np.log(u(depth_lo, depth_hi, P))
    if outlier_fraction > 0:
        out = rng.uniform(0, 1, P) < outlier_fraction
        pl = pl + np.where(out, u(-4.0, 4.0, P), 0.0)
    pv = u(0.05, 1.0, P)
    gx, gxv = u(-0.2, 0.2, P), u(0.005, 0.1, P)
    gy, gyv = u(-0.2, 0.2, P), u(0.005, 0.1, P)
    valid = (rng.uniform(0, 1, P) < semi_fraction).astype(np.uint8)
    sd = np.where(valid, u(depth_lo, depth_hi, P), 0.0)
    sv = np.where(valid, u(1e-4, 5e-2, P), 0.0)
    rs = lambda a: a.reshape(h, w).copy()
    state = FusionState(rs(ld), float(u(0.5, 2.0)), 0)
    semi = SemiDenseMap(rs(sd), rs(sv), rs(valid), int(valid.sum()))
    pred = PredictionSet(rs(pl), rs(pv), rs(gx), rs(gxv), rs(gy), rs(gyv), source_focal=200.0)
    return state, semi, pred


def semi_from_groundtruth(gt, fraction, alpha, rel_noise, seed):
    """synthetic.hpp:134-151"""
    rng = np.random.default_rng(seed)
    h, w = gt.shape
    semi = SemiDenseMap.empty(w, h)
    pick = rng.uniform(0, 1, gt.shape) < fraction
    d_true = alpha * gt
    sigma = np.maximum(rel_noise * d_true, 1e-6)
    d = d_true + sigma * rng.normal(0, 1, gt.shape)
    d = np.where(d <= 0, d_true, d)
    semi.depth = np.where(pick, d, 0.0)
    semi.variance = np.where(pick, sigma * sigma, 0.0)
    semi.valid = pick.astype(np.uint8)
    semi.inlier_count = int(pick.sum())
    return semi


def synth_oracle(gt, sigma_d, sigma_g, seed, source_focal):
    """predictions.hpp:190-224 (uniform sigma; values quantised through float)"""
    rng = np.random.default_rng(seed)
    q = lambda v: np.asarray(v, np.float64).astype(np.float32).astype(np.float64)
    h, w = gt.shape
    lg = np.log(gt)
    ld = q(lg + sigma_d * rng.normal(0, 1, gt.shape))
    gx = np.zeros_like(gt)
    gy = np.zeros_like(gt)
    gx[:, :-1] = q(lg[:, 1:] - lg[:, :-1] + sigma_g * rng.normal(0, 1, (h, w - 1)))
    gy[:-1, :] = q(lg[1:, :] - lg[:-1, :] + sigma_g * rng.normal(0, 1, (h - 1, w)))
    dv = np.full(gt.shape, q(max(sigma_d * sigma_d, 1e-12)))
    gv = np.full(gt.shape, q(max(sigma_g * sigma_g, 1e-12)))
    return PredictionSet(ld, dv, gx, gv, gy, gv.copy(), source_focal=source_focal)


def sequence_inputs(spec, seed, frames=None):
    """Seeded BASELINE-style keyframe + tracked frames (paper_2207_12244_b200.synth)."""
    return synth.make_sequence(spec, seed, frames)


def rel_err(a, b, floor=1e-300):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0
