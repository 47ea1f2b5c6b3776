"""The reference's own known-answer tests replayed against the oracle
(tests/test_semidense.cpp, tests/test_fusion.cpp, selftest.hpp). CPU only.
Each test cites the reference test it restates."""
import numpy as np
import pytest

import oracle
from paper_2207_12244_b200 import synth
from paper_2207_12244_b200._ffi import (EPI_DEGENERATE_BASELINE, EPI_OK, OBS_DTYPE, DfuseError,
                                        RobustConfig, SearchConfig, SemiDenseMap, init_state)
from helpers import (blank_problem, make_random_problem, quadratic_config,
                     semi_from_groundtruth, synth_oracle)

import ctypes as C


def _helper(impl, name, restype, argtypes):
    f = getattr(impl.lib, impl.prefix + name)
    f.restype = restype
    f.argtypes = argtypes
    return f


D5 = C.c_double * 5


# ------------------------------------------------------------------ semidense
def test_mask_constant_and_step(orc):  # test_semidense.cpp:51-78
    assert orc.texture_mask(np.full((24, 32), 0.5, np.float32), 0.02).sum() == 0
    img = np.zeros((8, 16), np.float32)
    img[:, 8:] = 0.5
    exp = np.zeros((8, 16), np.uint8)
    exp[1:7, 7:9] = 1
    assert np.array_equal(orc.texture_mask(img, 0.1), exp)
    with pytest.raises(DfuseError):
        orc.texture_mask(np.zeros((8, 8), np.float32), 0.0)


def _photometric(impl, g, I0, I1, x, y, d):
    f = _helper(impl, "photometric_error_5pt", C.c_int,
                [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double, D5])
    e = D5()
    I0 = np.ascontiguousarray(I0, np.float32)
    I1 = np.ascontiguousarray(I1, np.float32)
    st = f(C.byref(g), I0.ctypes.data, I1.ctypes.data, x, y, d, e)
    return st, np.array(e[:])


def test_photometric_identical_views(orc):  # test_semidense.cpp:80-88
    sc = synth.fronto_scene(200.0)
    I, _ = synth.render_view(sc)
    g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q, np.zeros(3),
                                   sc.camera)
    st, e = _photometric(orc, g, I, I, 100.5, 80.25, 1.7)
    assert st == EPI_OK and np.all(np.abs(e) < 1e-12)


def test_photometric_rendered_second_view(orc):  # test_semidense.cpp:90-111
    sc = synth.fronto_scene(200.0)
    I0, _ = synth.render_view(sc)
    I1, _ = synth.render_view(sc, synth.IDENTITY_Q, (0.1, 0, 0))
    g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                   np.array([0.1, 0, 0]), sc.camera)
    x, y = synth.strong_pixel(I0)
    st, e = _photometric(orc, g, I0, I1, x, y, 2.0)
    assert st == EPI_OK and np.all(np.abs(e) < 1e-3)
    st, e = _photometric(orc, g, I0, I1, x, y, 2.5)
    assert st == EPI_OK and np.abs(e).max() > 0.01


def test_search_kats(orc):  # test_semidense.cpp:113-136
    sc = synth.fronto_scene(200.0)
    I, _ = synth.render_view(sc)
    g0 = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q, np.zeros(3),
                                    sc.camera)
    st, _, _, _ = orc.search_depth(g0, I, I, np.array([[100.0, 90.0]]))
    assert st[0] == EPI_DEGENERATE_BASELINE
    sc = synth.fronto_scene(100.0)
    I0, _ = synth.render_view(sc)
    I1, _ = synth.render_view(sc, synth.IDENTITY_Q, (0.1, 0, 0))
    g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                   np.array([0.1, 0, 0]), sc.camera)
    st, obs, _, _ = orc.search_depth(g, I0, I1, np.array([synth.strong_pixel(I0)]),
                                     cfg=SearchConfig(1.0, 4.0))
    assert st[0] == EPI_OK and 1.95 < obs["depth"][0] < 2.05 and obs["variance"][0] > 0


def test_prior_window(orc):  # test_semidense.cpp:138-172
    sc = synth.fronto_scene(100.0)
    I0, _ = synth.render_view(sc)
    I1, _ = synth.render_view(sc, synth.IDENTITY_Q, (0.1, 0, 0))
    g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                   np.array([0.1, 0, 0]), sc.camera)
    px = np.array([synth.strong_pixel(I0)])
    st, _, _, _ = orc.search_depth(g, I0, I1, px, np.array([[2.0, 0.1]]))
    assert st[0] == EPI_DEGENERATE_BASELINE
    I1w, _ = synth.render_view(sc, synth.IDENTITY_Q, (0.25, 0, 0))
    gw = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                    np.array([0.25, 0, 0]), sc.camera)
    # The numpy restatement of the fixture's sinusoid texture is not bit-equal
    # to the C++ one, so the single strongest pixel can land on the RMS gate
    # (the reference build agrees with the oracle on it: test_oracle_pin).
    # Assert the property over the central region instead: the wider
    # baseline makes the +-2 sigma window searchable and recovers d = 2.
    ys, xs = np.mgrid[20:172:2, 20:236:2]
    pp = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.float64)
    prior = np.tile([2.0, 0.1], (len(pp), 1))
    st_n, _, _, _ = orc.search_depth(g, I0, I1, pp, prior)
    assert np.all(st_n == EPI_DEGENERATE_BASELINE)
    st, obs, _, _ = orc.search_depth(gw, I0, I1w, pp, prior)
    ok = st == EPI_OK
    assert ok.mean() > 0.9
    assert np.all((obs["depth"][ok] > 1.8 - 0.05) & (obs["depth"][ok] < 2.2 + 0.05))


def test_jacobian_and_variance(orc):  # test_semidense.cpp:174-203
    jac = _helper(orc, "jacobian_fd", C.c_int, [D5, D5, C.c_double, C.c_double, D5])
    var = _helper(orc, "observation_variance", C.c_double, [D5])
    e = D5(*[0.1] * 5)
    J = D5()
    assert jac(e, e, 1.0, 2.0, J) == 0 and all(v == 0.0 for v in J)
    hi = D5(*[0.2] * 5)
    assert jac(e, hi, 2.0, 2.05, J) == 0 and np.allclose(J[:], 2.0)
    assert jac(e, hi, 2.0, 2.0, J) == 6  # ZeroBaselineStep
    assert abs(var(D5(1, 1, 1, 1, 1)) - 0.2) < 1e-15
    assert abs(var(D5(2, 0, 0, 0, 0)) - 0.25) < 1e-15
    assert var(D5(0, 0, 0, 0, 0)) < 0
    rng = np.random.default_rng(5)
    for _ in range(100):
        j = rng.uniform(-1, 1, 5)
        v = var(D5(*j))
        if v > 0:
            assert abs(var(D5(*(2 * j))) - v / 4) <= 1e-12 * v


def _obs(x, y, d, v):
    o = np.zeros(1, OBS_DTYPE)
    o["x"], o["y"], o["depth"], o["variance"] = x, y, d, v
    return o


def test_update_semidense_kats(orc):  # test_semidense.cpp:205-236
    m = orc.update_semidense(SemiDenseMap.empty(8, 6), _obs(2, 3, 2.0, 0.04))
    assert m.inlier_count == 1 and m.depth[3, 2] == 2.0 and m.variance[3, 2] == 0.04
    m = orc.update_semidense(m, _obs(2, 3, 2.2, 0.04))
    assert abs(m.depth[3, 2] - 2.1) < 1e-12 and abs(m.variance[3, 2] - 0.02) < 1e-12
    gate = orc.update_semidense(SemiDenseMap.empty(8, 6), _obs(1, 1, 2.0, 0.0001))
    gate = orc.update_semidense(gate, _obs(1, 1, 10.0, 0.04))
    assert gate.depth[1, 1] == 2.0 and gate.variance[1, 1] == 0.0001
    rng = np.random.default_rng(17)
    for _ in range(200):
        d0, v0 = rng.uniform(0.5, 5.0), rng.uniform(1e-4, 1e-1)
        m = orc.update_semidense(SemiDenseMap.empty(2, 2), _obs(0, 0, d0, v0))
        v1 = rng.uniform(1e-4, 1e-1)
        m = orc.update_semidense(m, _obs(0, 0, d0 + 0.1 * np.sqrt(v0), v1))
        assert m.variance[0, 0] <= min(v0, v1) + 1e-15


def test_keyframe_policy(orc):  # test_semidense.cpp:238-261
    f = _helper(orc, "should_create_keyframe", C.c_int,
                [C.c_double * 4, C.c_double * 3, C.c_double * 4, C.c_double * 3, C.c_double,
                 C.c_int, C.c_double, C.c_int, C.POINTER(C.c_int)])
    I = (C.c_double * 4)(1, 0, 0, 0)
    Z = (C.c_double * 3)(0, 0, 0)

    def ask(t, inliers, lt, li):
        out = C.c_int(-1)
        assert f(I, Z, I, (C.c_double * 3)(t, 0, 0), 2.0, inliers, lt, li, C.byref(out)) == 0
        return bool(out.value)

    assert not ask(0.0, 500, 0.1, 100)
    assert ask(0.4, 500, 0.1, 100)
    assert ask(0.0, 0, 0.1, 100)
    trig = False
    for t in np.arange(0.0, 1.0, 0.05):
        now = ask(t, 10, 0.1, 0)
        if trig:
            assert now
        trig = trig or now
    assert trig


def test_two_view_coverage_and_accuracy(orc):  # test_semidense.cpp:263-294, acceptance C7
    sc = synth.PlaneScene()
    I0, gt = synth.render_view(sc)
    I1, _ = synth.render_view(sc, synth.IDENTITY_Q, (0.15, 0.002, 0.0))
    mask = orc.texture_mask(I0, 0.02)
    g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                   np.array([0.15, 0.002, 0.0]), sc.camera)
    ys, xs = np.nonzero(mask)
    px = np.stack([xs, ys], 1).astype(np.float64)
    st, obs, _, _ = orc.search_depth(g, I0, I1, px, cfg=SearchConfig(1.2, 3.5))
    ok = st == EPI_OK
    assert len(px) > 3000 and ok.mean() >= 0.9
    rel = np.abs(obs["depth"][ok] - gt[ys[ok], xs[ok]]) / gt[ys[ok], xs[ok]]
    assert np.median(rel) < 0.02


def test_depths_scale_with_trajectory(orc):  # test_semidense.cpp:328-355
    sc = synth.PlaneScene()
    I0, _ = synth.render_view(sc)
    I1, _ = synth.render_view(sc, synth.IDENTITY_Q, (0.15, 0, 0))
    alpha = 0.5
    g1 = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                    np.array([0.15, 0, 0]), sc.camera)
    g2 = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                    np.array([0.15 * alpha, 0, 0]), sc.camera)
    mask = orc.texture_mask(I0, 0.02)
    ys, xs = np.mgrid[5:190:3, 5:250:3]
    sel = mask[ys, xs] == 1
    px = np.stack([xs[sel], ys[sel]], 1).astype(np.float64)
    sa, oa, _, _ = orc.search_depth(g1, I0, I1, px, cfg=SearchConfig(1.2, 3.5))
    sb, ob, _, _ = orc.search_depth(g2, I0, I1, px, cfg=SearchConfig(1.2 * alpha, 3.5 * alpha))
    both = (sa == EPI_OK) & (sb == EPI_OK)
    assert both.sum() > 500
    da, db = oa["depth"][both], ob["depth"][both]
    assert (np.abs(db - alpha * da) / (alpha * da) < 0.01).mean() > 0.95


# ------------------------------------------------------------------ fusion
def test_huber_and_residuals(orc):  # test_fusion.cpp:41-74
    hub = _helper(orc, "huber", C.c_int,
                  [C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)])
    rs = _helper(orc, "residual_semi", C.c_double, [C.c_double, C.c_double, C.c_double])
    w, c = C.c_double(), C.c_double()

    def hw(r, d):
        rc = hub(r, d, C.byref(w), C.byref(c))
        return rc, w.value, c.value

    assert hw(0.0, 0.3)[1] == 1.0 and hw(0.3, 0.3)[1] == 1.0 and hw(-0.3, 0.3)[1] == 1.0
    assert abs(hw(0.9, 0.3)[1] - 1 / 3) < 1e-15
    assert hw(0.1, 0.0)[0] == 27  # InvalidArgument
    assert abs(hw(0.3, 0.3)[2] - 0.09) < 1e-15
    assert abs(hw(0.9, 0.3)[2] - 0.3 * (1.8 - 0.3)) < 1e-15
    assert abs(rs(np.log(2.0), 1.0, 2.0)) < 1e-15
    assert abs(rs(np.log(4.0), 2.0, 2.0)) < 1e-15
    assert abs(rs(1.0, 1.0, 1.0) - 1.0) < 1e-15


def test_assembly_single_pixel(orc):  # test_fusion.cpp:76-83
    st, semi, pred = blank_problem(1, 1)
    st.log_depth[0, 0], pred.log_depth[0, 0] = 0.25, 0.05
    eq = orc.assemble_normal_equations(st, semi, pred)
    assert abs(eq.diag[0, 0] - 1.0) < 1e-15 and abs(eq.b[0, 0] + 0.2) < 1e-15


def test_anchored_chain(orc):  # test_fusion.cpp:85-99
    st, semi, pred = blank_problem(2, 1)
    pred.log_depth[0, 0] = 0.4
    pred.log_depth_var[0, 0], pred.log_depth_var[0, 1] = 1e-10, 1e12
    pred.grad_x[0, 0] = np.log(2.0)
    cfg = quadratic_config()
    cfg.gn_iterations, cfg.estimate_scale = 3, False
    out = orc.optimize(st, semi, pred, cfg)
    assert abs(out.log_depth[0, 0] - 0.4) < 1e-8
    assert abs(out.log_depth[0, 1] - (0.4 + np.log(2.0))) < 1e-6


def test_variance_rescale_invariance(orc):  # test_fusion.cpp:101-118
    st, semi, pred = make_random_problem(19, 6, 4)
    cfg = quadratic_config()
    d1, _ = orc.solve_depth_step(orc.assemble_normal_equations(st, semi, pred, cfg), cfg)
    c = 7.3
    pred2 = pred.copy()
    pred2.log_depth_var *= c
    pred2.grad_x_var *= c
    pred2.grad_y_var *= c
    semi2 = semi.copy()
    semi2.variance = np.where(semi2.valid == 1, semi2.variance * c, semi2.variance)
    d2, _ = orc.solve_depth_step(orc.assemble_normal_equations(st, semi2, pred2, cfg), cfg)
    assert np.abs(d1 - d2).max() < 1e-9


def _dense(eq):
    h, w = eq.diag.shape
    n = w * h
    M = np.zeros((n, n))
    for y in range(h):
        for x in range(w):
            i = y * w + x
            M[i, i] = eq.diag[y, x]
            if x + 1 < w:
                M[i, i + 1] = M[i + 1, i] = eq.right[y, x]
            if y + 1 < h:
                M[i, i + w] = M[i + w, i] = eq.down[y, x]
    return M


def test_pcg_vs_dense_solve(orc):  # test_fusion.cpp:127-142 (testing.hpp:67-86)
    for inst in range(8):
        st, semi, pred = make_random_problem(400 + inst, 8, 6)
        cfg = RobustConfig(cg_tol=1e-10, cg_max_iters=500)
        eq = orc.assemble_normal_equations(st, semi, pred, cfg)
        d, _ = orc.solve_depth_step(eq, cfg)
        ref = np.linalg.solve(_dense(eq), eq.b.ravel())
        scale = max(1.0, np.abs(ref).max())
        assert np.abs(d.ravel() - ref).max() / scale < 1e-6


def test_spd_and_gershgorin(orc):  # test_fusion.cpp:338-352
    st, semi, pred = make_random_problem(1100, 8, 6)
    M = _dense(orc.assemble_normal_equations(st, semi, pred))
    assert np.abs(M - M.T).max() == 0.0
    off = np.abs(M).sum(1) - np.abs(np.diag(M))
    assert np.all(np.diag(M) > off)
    assert np.linalg.eigvalsh(M).min() > 0


def test_net_only_one_step(orc):  # test_fusion.cpp:144-160
    st, semi, pred = blank_problem(4, 3)
    rng = np.random.default_rng(9)
    pred.log_depth = rng.uniform(-1, 1, (3, 4))
    pred.grad_x_var[:] = pred.grad_y_var[:] = 1e12
    st.log_depth = rng.uniform(-1, 1, (3, 4))
    cfg = quadratic_config()
    cfg.gn_iterations, cfg.estimate_scale = 1, False
    out = orc.optimize(st, semi, pred, cfg, "nopairwise")
    assert np.abs(out.log_depth - pred.log_depth).max() < 1e-12


def test_scale_step_kats(orc):  # test_fusion.cpp:162-196
    cfg = RobustConfig(delta_semi=10.0)
    st, semi, pred = blank_problem(2, 2)
    semi.valid[:], semi.depth[:], semi.variance[:], semi.inlier_count = 1, 1.0, 0.01, 4
    assert abs(orc.solve_scale_step(st, semi, cfg) - 1.0) < 1e-12
    st.log_depth[:] = np.log(2.0)
    assert abs(orc.solve_scale_step(st, semi, cfg) - 2.0) < 2e-12
    st, semi, pred = blank_problem(2, 1)
    semi.valid[:], semi.inlier_count, semi.depth[:] = 1, 2, 1.0
    semi.variance[0, 0], semi.variance[0, 1] = 1.0, 1.0 / 3.0
    st.log_depth[0, 0] = np.log(2.0)
    s = orc.solve_scale_step(st, semi, cfg)
    assert abs(s - np.exp(np.log(2.0) / 4.0)) < 1e-12 and abs(s - 1.189207) < 1e-6
    with pytest.raises(DfuseError):
        orc.solve_scale_step(st, SemiDenseMap.empty(2, 1), cfg)


def test_zero_residual_fixed_point(orc):  # test_fusion.cpp:198-224
    w, h = 8, 6
    rng = np.random.default_rng(23)
    st, semi, pred = blank_problem(w, h)
    st.log_depth = np.log(rng.uniform(0.5, 4.0, (h, w)))
    pred.log_depth = st.log_depth.copy()
    pred.grad_x[:, :-1] = st.log_depth[:, 1:] - st.log_depth[:, :-1]
    pred.grad_y[:-1, :] = st.log_depth[1:, :] - st.log_depth[:-1, :]
    semi.valid[:], semi.depth, semi.variance[:] = 1, np.exp(st.log_depth), 0.01
    semi.inlier_count = w * h
    out = orc.optimize(st, semi, pred, RobustConfig(gn_iterations=1))
    assert orc.total_cost(out, semi, pred, RobustConfig(gn_iterations=1)) < 1e-10
    assert np.abs(out.log_depth - st.log_depth).max() < 1e-9
    assert abs(out.scale - 1.0) < 1e-9 and out.iteration == 1


def test_single_pixel_split(orc):  # test_fusion.cpp:226-239
    st, semi, pred = blank_problem(1, 1)
    semi.valid[:], semi.depth[:], semi.variance[:], semi.inlier_count = 1, 1.0, 1.0, 1
    pred.log_depth[:] = 1.0
    st.log_depth[:] = 1.0
    cfg = quadratic_config()
    cfg.estimate_scale, cfg.gn_iterations = False, 2
    assert abs(orc.optimize(st, semi, pred, cfg).log_depth[0, 0] - 0.5) < 1e-9


def test_scale_recovery(orc):  # test_fusion.cpp:241-254
    rng = np.random.default_rng(31)
    gt = rng.uniform(1.0, 3.0, (12, 16))
    pred = synth_oracle(gt, 0.05, 0.01, 77, 200.0)
    semi = semi_from_groundtruth(gt, 0.5, 0.5, 0.05, 78)
    out = orc.optimize(init_state(pred), semi, pred, RobustConfig())
    assert abs(out.scale - 2.0) < 0.05 * 2.0 and out.iteration == 10


def _near_kink(st, semi, pred, cfg, mode, i, margin=1e-3):  # testing.hpp:155-184
    h, w = st.log_depth.shape
    ld = st.log_depth.ravel()
    x, y = i % w, i // w
    use_net, use_grad = mode != "lsscale", mode != "nopairwise"
    ln_s = 0.0 if mode == "lsscale" else np.log(st.scale)
    near = lambda r, d: abs(abs(r) - d) <= margin
    gx, gy = pred.grad_x.ravel(), pred.grad_y.ravel()
    if use_net and near(ld[i] - pred.log_depth.ravel()[i], cfg.delta_net):
        return True
    if semi.valid.ravel()[i] and near(ld[i] - ln_s - np.log(semi.depth.ravel()[i]),
                                      cfg.delta_semi):
        return True
    if use_grad:
        if x + 1 < w and near(ld[i + 1] - ld[i] - gx[i], cfg.delta_grad):
            return True
        if x > 0 and near(ld[i] - ld[i - 1] - gx[i - 1], cfg.delta_grad):
            return True
        if y + 1 < h and near(ld[i + w] - ld[i] - gy[i], cfg.delta_grad):
            return True
        if y > 0 and near(ld[i] - ld[i - w] - gy[i - w], cfg.delta_grad):
            return True
    return False


@pytest.mark.parametrize("mode", ["full", "nopairwise"])
def test_gradient_vs_finite_differences(orc, mode):  # test_fusion.cpp:256-275, acceptance C1
    cfg = RobustConfig()
    for inst in range(5):
        st, semi, pred = make_random_problem(700 + inst, 8, 6, outlier_fraction=0.15)
        c, g, gs = orc.cost_gradient(st, semi, pred, cfg, mode)
        assert abs(c - orc.total_cost(st, semi, pred, cfg, mode)) <= 1e-12 * abs(c)
        hstep = 1e-5
        for i in range(st.log_depth.size):
            if _near_kink(st, semi, pred, cfg, mode, i):
                continue
            up, dn = st.copy(), st.copy()
            up.log_depth.ravel()[i] += hstep
            dn.log_depth.ravel()[i] -= hstep
            fd = (orc.total_cost(up, semi, pred, cfg, mode) -
                  orc.total_cost(dn, semi, pred, cfg, mode)) / (2 * hstep)
            assert abs(g.ravel()[i] - fd) / max(abs(fd), 1e-2) < 1e-4
        up, dn = st.copy(), st.copy()
        up.scale = np.exp(np.log(st.scale) + hstep)
        dn.scale = np.exp(np.log(st.scale) - hstep)
        fd = (orc.total_cost(up, semi, pred, cfg, mode) -
              orc.total_cost(dn, semi, pred, cfg, mode)) / (2 * hstep)
        assert abs(gs - fd) / max(abs(fd), 1e-2) < 1e-4


def test_scale_equivariance(orc):  # test_fusion.cpp:277-305
    st, semi, pred = make_random_problem(800, 6, 5)
    alpha = 0.25
    cfg = RobustConfig(cg_tol=1e-10, cg_max_iters=500)
    a = orc.optimize(st, semi, pred, cfg)
    s2 = semi.copy()
    s2.depth = np.where(s2.valid == 1, s2.depth * alpha, s2.depth)
    s2.variance = np.where(s2.valid == 1, s2.variance * alpha * alpha, s2.variance)
    start = st.copy()
    start.scale = st.scale / alpha
    b = orc.optimize(start, s2, pred, cfg)
    assert np.abs(a.log_depth - b.log_depth).max() < 1e-5
    assert abs(b.scale - a.scale / alpha) <= 1e-6 * abs(a.scale / alpha)


def test_monotone_cost(orc):  # test_fusion.cpp:307-321
    for inst in range(4):
        st, semi, pred = make_random_problem(900 + inst, 8, 6, outlier_fraction=0.2)
        cfg = RobustConfig(gn_iterations=1)
        cost = orc.total_cost(st, semi, pred, cfg)
        for _ in range(10):
            st = orc.optimize(st, semi, pred, cfg)
            nxt = orc.total_cost(st, semi, pred, cfg)
            assert nxt <= cost
            cost = nxt


def _dense_wls(semi, pred, scale, mode="full"):  # testing.hpp:91-122
    h, w = pred.log_depth.shape
    n = w * h
    A = np.zeros((n, n))
    rhs = np.zeros(n)
    ln_s = 0.0 if mode == "lsscale" else np.log(scale)

    def row(coeffs, target, weight):
        for i, ci in coeffs:
            for j, cj in coeffs:
                A[i, j] += weight * ci * cj
            rhs[i] += weight * ci * target

    for y in range(h):
        for x in range(w):
            i = y * w + x
            if mode != "lsscale":
                row([(i, 1.0)], pred.log_depth[y, x], 1.0 / pred.log_depth_var[y, x])
            if semi.valid[y, x]:
                R = max(semi.variance[y, x] / semi.depth[y, x] ** 2, 1e-4)
                row([(i, 1.0)], ln_s + np.log(semi.depth[y, x]), 1.0 / R)
            if mode != "nopairwise" and x + 1 < w:
                row([(i + 1, 1.0), (i, -1.0)], pred.grad_x[y, x], 1.0 / pred.grad_x_var[y, x])
            if mode != "nopairwise" and y + 1 < h:
                row([(i + w, 1.0), (i, -1.0)], pred.grad_y[y, x], 1.0 / pred.grad_y_var[y, x])
    return np.linalg.solve(A, rhs)


def test_quadratic_fixed_point_is_dense_wls(orc):  # test_fusion.cpp:323-336, acceptance C2
    for inst in range(6):
        w, h = 2 + inst % 3, 2 + (inst // 2) % 3
        st, semi, pred = make_random_problem(1000 + inst, w, h)
        cfg = quadratic_config()
        cfg.gn_iterations, cfg.estimate_scale = 3, False
        out = orc.optimize(st, semi, pred, cfg)
        ref = _dense_wls(semi, pred, st.scale)
        assert np.abs(out.log_depth.ravel() - ref).max() < 1e-8


def test_nopairwise_and_lsscale(orc):  # test_fusion.cpp:354-390
    st, semi, pred = make_random_problem(1200, 6, 4)
    eq = orc.assemble_normal_equations(st, semi, pred, RobustConfig(), "nopairwise")
    assert not eq.right.any() and not eq.down.any()
    rng = np.random.default_rng(41)
    w, h = 10, 8
    gt = rng.uniform(1.0, 3.0, (h, w))
    st, semi, pred = blank_problem(w, h)
    pred.log_depth = np.log(gt) + np.log(3.0)
    pred.grad_x[:, :-1] = np.log(gt[:, 1:]) - np.log(gt[:, :-1])
    pred.grad_y[:-1, :] = np.log(gt[1:, :]) - np.log(gt[:-1, :])
    pred.grad_x_var[:] = pred.grad_y_var[:] = 0.01
    semi.valid[:], semi.depth, semi.variance = 1, gt.copy(), 1e-4 * gt * gt
    semi.inlier_count = w * h
    st.log_depth = pred.log_depth.copy()
    out = orc.optimize(st, semi, pred, RobustConfig(), "lsscale")
    assert abs(out.scale - 3.0) < 0.03
    assert np.abs(out.log_depth - (np.log(gt) + np.log(3.0))).max() < 0.05


def test_init_state_and_divergence(orc):  # test_fusion.cpp:392-411
    st, semi, pred = make_random_problem(1300, 5, 4)
    s = init_state(pred)
    assert np.array_equal(s.log_depth, pred.log_depth) and s.scale == 1.0 and s.iteration == 0
    eq = orc.assemble_normal_equations(st, semi, pred)
    eq.diag = np.array([[1.0, 0.0], [1.0, 1.0]])
    eq.right = np.zeros((2, 2))
    eq.down = np.zeros((2, 2))
    eq.b = np.ones((2, 2))
    with pytest.raises(DfuseError) as e:
        orc.solve_depth_step(eq)
    assert e.value.code == "CgDivergence"
