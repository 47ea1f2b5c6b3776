"""Pin the oracle to the reference: orc_* (plain-C restatement) must equal
ref_* (the reference's own headers compiled unmodified, oracle/_ref) bit for
bit on seeded inputs, for every function on the hot path. CPU only."""
import math

import numpy as np
import pytest

import oracle
from paper_2207_12244_b200 import synth
from paper_2207_12244_b200._ffi import (EPI_OK, OBS_DTYPE, DfuseError, NormalEquations,
                                        RobustConfig, SearchConfig, SemiDenseMap, init_state)
from helpers import make_random_problem

MODES = ["full", "nopairwise", "lsscale"]


def test_hypot_restatement_matches_libm():
    import ctypes
    import ctypes.util

    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(0)
    a = rng.uniform(-700, 700, 20000)
    b = np.concatenate([rng.uniform(-700, 700, 10000), rng.uniform(-1e-3, 1e-3, 10000)])
    specials = [(0.0, 0.0), (3.0, 4.0), (1e300, 1e300), (1e-310, 1e-310), (1e-300, 1.0),
                (math.inf, 1.0), (1.0, -math.inf)]
    for x, y in list(zip(a, b)) + specials:
        assert oracle.hypot(x, y) == libm.hypot(x, y)


def test_geometry(orc, ref):
    spec = synth.CONFIGS["C2"]
    rng = np.random.default_rng(1)
    for _ in range(200):
        q0, t0 = synth.random_pose(spec, rng)
        q1, t1 = synth.random_pose(spec, rng)
        assert bytes(orc.make_epipolar_geometry(q0, t0, q1, t1, spec.camera())) == bytes(
            ref.make_epipolar_geometry(q0, t0, q1, t1, spec.camera()))


def test_texture_mask(orc, ref):
    rng = np.random.default_rng(2)
    for (h, w) in [(1, 1), (3, 3), (24, 32), (97, 131)]:
        img = rng.uniform(0, 1, (h, w)).astype(np.float32)
        for thr in (0.01, 0.2):
            assert np.array_equal(orc.texture_mask(img, thr), ref.texture_mask(img, thr))
    with pytest.raises(DfuseError):
        orc.texture_mask(np.zeros((4, 4), np.float32), -1.0)
    with pytest.raises(DfuseError):
        ref.texture_mask(np.zeros((4, 4), np.float32), 0.0)


def test_search_depth_list(orc, ref):
    spec = synth.small_spec(128, 96, frames=2)
    seq = synth.make_sequence(spec, 3)
    rng = np.random.default_rng(4)
    n = 1500
    px = np.stack([rng.uniform(0, spec.width - 1, n), rng.uniform(0, spec.height - 1, n)], 1)
    px[: n // 2] = np.round(px[: n // 2])
    prior = np.stack([rng.uniform(0.2, 5, n), rng.uniform(0.001, 2.0, n)], 1)
    has = (rng.uniform(0, 1, n) < 0.5).astype(np.uint8)
    for q, t, I1 in seq.frames:
        g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
        for cfg in (SearchConfig(), SearchConfig(0.1, 20.0)):
            so, oo, _, _ = orc.search_depth(g, seq.I0, I1, px, prior, has, cfg)
            sr, orr, _, _ = ref.search_depth(g, seq.I0, I1, px, prior, has, cfg)
            assert np.array_equal(so, sr)
            ok = so == EPI_OK
            assert ok.sum() > 20
            assert oo[ok].tobytes() == orr[ok].tobytes()


@pytest.mark.parametrize("name", ["S", "C1"])
def test_stereo_update_sequence(orc, ref, name):
    spec = synth.small_spec(128, 96, frames=3) if name == "S" else synth.CONFIGS["C1"]
    seq = synth.make_sequence(spec, 5, frames=3)
    mask = orc.texture_mask(seq.I0, 0.02)
    so = SemiDenseMap.empty(spec.width, spec.height)
    sr = so.copy()
    for q, t, I1 in seq.frames:
        g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
        a = orc.stereo_update(g, seq.I0, I1, mask, so, spec.search)
        b = ref.stereo_update(g, seq.I0, I1, mask, sr, spec.search)
        assert a.n_obs == b.n_obs and a.n_obs > 0
        assert np.array_equal(a.status, b.status)
        assert a.obs.tobytes() == b.obs.tobytes()
        for f in ("depth", "variance", "valid"):
            assert getattr(a.semi, f).tobytes() == getattr(b.semi, f).tobytes()
        assert a.semi.inlier_count == b.semi.inlier_count
        so, sr = a.semi, b.semi


def test_update_semidense(orc, ref):
    rng = np.random.default_rng(6)
    w, h, n = 16, 9, 3000
    obs = np.zeros(n, OBS_DTYPE)
    obs["x"], obs["y"] = rng.integers(0, w, n), rng.integers(0, h, n)
    obs["depth"], obs["variance"] = rng.uniform(0.5, 4, n), rng.uniform(1e-3, 2.0, n)
    a = orc.update_semidense(SemiDenseMap.empty(w, h), obs)
    b = ref.update_semidense(SemiDenseMap.empty(w, h), obs)
    assert a.depth.tobytes() == b.depth.tobytes()
    assert a.variance.tobytes() == b.variance.tobytes()
    assert a.inlier_count == b.inlier_count
    bad = obs[:1].copy()
    bad["x"] = w
    for impl in (orc, ref):
        with pytest.raises(DfuseError) as e:
            impl.update_semidense(SemiDenseMap.empty(w, h), bad)
        assert e.value.code == "OutOfBounds"


def _problems():
    yield make_random_problem(11, 8, 6)
    yield make_random_problem(12, 23, 17, outlier_fraction=0.2)
    yield make_random_problem(13, 1, 1)
    yield make_random_problem(14, 1, 5)
    yield make_random_problem(15, 6, 1)


@pytest.mark.parametrize("mode", MODES)
def test_fusion_functions_bit_exact(orc, ref, mode):
    cfg = RobustConfig()
    for st, semi, pred in _problems():
        a = orc.assemble_normal_equations(st, semi, pred, cfg, mode)
        b = ref.assemble_normal_equations(st, semi, pred, cfg, mode)
        for f in ("diag", "right", "down", "b"):
            assert getattr(a, f).tobytes() == getattr(b, f).tobytes()
        assert orc.total_cost(st, semi, pred, cfg, mode) == ref.total_cost(st, semi, pred, cfg,
                                                                           mode)
        ca, ga, sa = orc.cost_gradient(st, semi, pred, cfg, mode)
        cb, gb, sb = ref.cost_gradient(st, semi, pred, cfg, mode)
        assert ca == cb and sa == sb and ga.tobytes() == gb.tobytes()
        x = np.random.default_rng(0).normal(size=st.log_depth.shape)
        assert orc.stencil_apply(a, x).tobytes() == ref.stencil_apply(a, x).tobytes()
        da, _ = orc.solve_depth_step(a, cfg)
        db, _ = ref.solve_depth_step(a, cfg)
        assert da.tobytes() == db.tobytes()
        if semi.inlier_count > 0:
            assert orc.solve_scale_step(st, semi, cfg) == ref.solve_scale_step(st, semi, cfg)
        oa = orc.optimize(st, semi, pred, cfg, mode)
        ob = ref.optimize(st, semi, pred, cfg, mode)
        assert oa.log_depth.tobytes() == ob.log_depth.tobytes()
        assert oa.scale == ob.scale and oa.iteration == ob.iteration


def test_optimize_on_keyframe_bit_exact(orc, ref):
    spec = synth.small_spec(96, 72, frames=2)
    seq = synth.make_sequence(spec, 7)
    mask = orc.texture_mask(seq.I0, 0.02)
    semi = SemiDenseMap.empty(spec.width, spec.height)
    st = init_state(seq.pred)
    for q, t, I1 in seq.frames:
        g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
        semi = orc.stereo_update(g, seq.I0, I1, mask, semi, spec.search).semi
        for regime in (RobustConfig(), RobustConfig(cg_tol=0.0, cg_max_iters=5)):
            a = orc.optimize(st, semi, seq.pred, regime)
            b = ref.optimize(st, semi, seq.pred, regime)
            assert a.log_depth.tobytes() == b.log_depth.tobytes() and a.scale == b.scale
        st = a


def test_error_paths_agree(orc, ref):
    st, semi, pred = make_random_problem(20, 5, 4)
    eq = orc.assemble_normal_equations(st, semi, pred)
    eq.diag[0, 1] = 0.0
    for impl in (orc, ref):
        with pytest.raises(DfuseError) as e:
            impl.solve_depth_step(eq)
        assert e.value.code == "CgDivergence"
        with pytest.raises(DfuseError) as e:
            impl.solve_scale_step(st, SemiDenseMap.empty(5, 4))
        assert e.value.code == "NoSemiDenseSupport"
        with pytest.raises(DfuseError) as e:
            impl.assemble_normal_equations(st, semi, pred, RobustConfig(delta_net=0.0))
        assert e.value.code == "InvalidArgument"
