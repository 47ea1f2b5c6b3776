"""GPU parity: the stereo front end (semidense.hpp, pipeline.hpp:157-212).

Bar (BASELINE.json north_star): texture masks, search
status, best-match index, step count and every double of the observations
bit-exact against the oracle (itself pinned bit-exactly to the reference
build, tests/test_oracle_pin.py); the updated semi-dense map bit-exact.
"""
import numpy as np
import pytest

from paper_2207_12244_b200 import synth
from paper_2207_12244_b200._ffi import (EPI_OK, EPI_DEGENERATE_BASELINE, OBS_DTYPE, DfuseError,
                                        SearchConfig, SemiDenseMap)

pytestmark = pytest.mark.gpu


def _seq(w=160, h=120, frames=3, seed=5, **kw):
    spec = synth.small_spec(w, h, frames=frames, **kw)
    return spec, synth.make_sequence(spec, seed)


# ---------------------------------------------------------------- texture_mask
def test_mask_constant_image_empty(gpu):  # test_semidense.cpp:51-55
    m = gpu.texture_mask(np.full((24, 32), 0.5, np.float32), 0.02)
    assert m.sum() == 0


def test_mask_step_edge(gpu):  # test_semidense.cpp:57-73
    img = np.zeros((8, 16), np.float32)
    img[:, 8:] = 0.5
    m = gpu.texture_mask(img, 0.1)
    exp = np.zeros((8, 16), np.uint8)
    exp[1:7, 7:9] = 1
    assert np.array_equal(m, exp)


def test_mask_rejects_nonpositive_threshold(gpu):  # test_semidense.cpp:75-78
    with pytest.raises(DfuseError) as e:
        gpu.texture_mask(np.zeros((8, 8), np.float32), 0.0)
    assert e.value.code == "InvalidArgument"


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_mask_bit_exact_full_size(gpu, orc, name):
    spec = synth.CONFIGS[name]
    seq = synth.make_sequence(spec, seed=11, frames=0)
    for thr in (0.02, 0.005, 0.1):
        assert np.array_equal(gpu.texture_mask(seq.I0, thr), orc.texture_mask(seq.I0, thr))


def test_mask_random_and_ragged(gpu, orc):
    rng = np.random.default_rng(3)
    for (h, w) in [(1, 1), (2, 3), (3, 3), (7, 129), (33, 17), (480, 641)]:
        img = rng.uniform(0, 1, (h, w)).astype(np.float32)
        assert np.array_equal(gpu.texture_mask(img, 0.2), orc.texture_mask(img, 0.2))


# ---------------------------------------------------------------- search_depth
def _geom(api, spec, q, t):
    return api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())


def test_geometry_identical(gpu, orc):
    spec = synth.CONFIGS["C2"]
    rng = np.random.default_rng(0)
    for _ in range(50):
        q, t = synth.random_pose(spec, rng)
        q0, t0 = synth.random_pose(spec, rng)
        a = gpu.make_epipolar_geometry(q0, t0, q, t, spec.camera())
        b = orc.make_epipolar_geometry(q0, t0, q, t, spec.camera())
        assert bytes(a) == bytes(b)


def test_search_list_bit_exact(gpu, orc):
    spec, seq = _seq(160, 120, frames=2, seed=9)
    rng = np.random.default_rng(1)
    n = 3000
    px = np.stack([rng.integers(0, spec.width, n), rng.integers(0, spec.height, n)], 1)
    px = px.astype(np.float64)
    px[:200] += rng.uniform(-0.5, 0.5, (200, 2))  # non-integer pixels too
    prior = np.stack([rng.uniform(0.3, 5.0, n), rng.uniform(0.001, 2.0, n)], 1)
    has = (rng.uniform(0, 1, n) < 0.5).astype(np.uint8)
    for (q, t, I1) in seq.frames:
        g = _geom(orc, spec, q, t)
        for cfg in (SearchConfig(), SearchConfig(0.1, 20.0), SearchConfig(1.0, 4.0, 0.2)):
            sg, og, bg, ng = gpu.search_depth(g, seq.I0, I1, px, prior, has, cfg)
            so, oo, bo, no = orc.search_depth(g, seq.I0, I1, px, prior, has, cfg)
            assert np.array_equal(sg, so)
            assert np.array_equal(bg, bo)
            assert np.array_equal(ng, no)
            ok = so == EPI_OK
            assert ok.sum() > 50
            assert og[ok].tobytes() == oo[ok].tobytes()


def test_search_zero_baseline(gpu):  # test_semidense.cpp:113-119
    sc = synth.fronto_scene(200.0)
    I, _ = synth.render_view(sc)
    g = gpu.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q, np.zeros(3),
                                   sc.camera)
    st, _, _, _ = gpu.search_depth(g, I, I, np.array([[100.0, 90.0]]))
    assert st[0] == EPI_DEGENERATE_BASELINE


def test_search_fronto_plane_kat(gpu):  # test_semidense.cpp:121-136
    sc = synth.fronto_scene(100.0)
    I0, _ = synth.render_view(sc)
    I1, _ = synth.render_view(sc, synth.IDENTITY_Q, (0.1, 0.0, 0.0))
    g = gpu.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), synth.IDENTITY_Q,
                                   np.array([0.1, 0, 0]), sc.camera)
    x = synth.strong_pixel(I0)
    st, obs, _, _ = gpu.search_depth(g, I0, I1, np.array([x]), cfg=SearchConfig(1.0, 4.0))
    assert st[0] == EPI_OK
    assert 1.95 < obs["depth"][0] < 2.05
    assert obs["variance"][0] > 0


# ---------------------------------------------------------------- fused scan + update
@pytest.mark.parametrize("name,seed", [("S", 2), ("C1", 4), ("C5", 6)])
def test_stereo_update_sequence_bit_exact(gpu, orc, name, seed):
    if name == "S":
        spec, seq = _seq(200, 150, frames=4, seed=seed)
    else:
        spec = synth.CONFIGS[name]
        seq = synth.make_sequence(spec, seed, frames=3)
    mask = orc.texture_mask(seq.I0, 0.02)
    sg = SemiDenseMap.empty(spec.width, spec.height)
    so = sg.copy()
    for (q, t, I1) in seq.frames:
        g = _geom(orc, spec, q, t)
        rg = gpu.stereo_update(g, seq.I0, I1, mask, sg, spec.search)
        ro = orc.stereo_update(g, seq.I0, I1, mask, so, spec.search)
        assert rg.n_obs == ro.n_obs
        assert np.array_equal(rg.status, ro.status)
        assert np.array_equal(rg.best, ro.best)
        assert np.array_equal(rg.n_steps, ro.n_steps)
        assert rg.obs.tobytes() == ro.obs.tobytes()
        for f in ("depth", "variance", "valid"):
            assert getattr(rg.semi, f).tobytes() == getattr(ro.semi, f).tobytes(), f
        assert rg.semi.inlier_count == ro.semi.inlier_count
        sg, so = rg.semi, ro.semi
    assert so.inlier_count > 0


def test_stereo_update_zero_baseline_keeps_count(gpu, orc):
    spec, seq = _seq(64, 48, frames=1)
    mask = orc.texture_mask(seq.I0, 0.02)
    semi = SemiDenseMap.empty(spec.width, spec.height)
    semi.inlier_count = 7  # inconsistent on purpose: no update -> no recount
    g = _geom(orc, spec, synth.IDENTITY_Q, np.zeros(3))
    r = gpu.stereo_update(g, seq.I0, seq.I0, mask, semi)
    assert r.n_obs == 0 and r.semi.inlier_count == 7
    assert np.all(r.status[mask == 1] == EPI_DEGENERATE_BASELINE)


# ---------------------------------------------------------------- update_semidense
def test_update_semidense_kats(gpu):  # test_semidense.cpp:205-222
    def ob(x, y, d, v):
        o = np.zeros(1, OBS_DTYPE)
        o["x"], o["y"], o["depth"], o["variance"] = x, y, d, v
        return o

    m = SemiDenseMap.empty(8, 6)
    m = gpu.update_semidense(m, ob(2, 3, 2.0, 0.04))
    assert m.inlier_count == 1 and m.depth[3, 2] == 2.0 and m.variance[3, 2] == 0.04
    m = gpu.update_semidense(m, ob(2, 3, 2.2, 0.04))
    assert abs(m.depth[3, 2] - 2.1) < 1e-12 and abs(m.variance[3, 2] - 0.02) < 1e-12
    gate = gpu.update_semidense(SemiDenseMap.empty(8, 6), ob(1, 1, 2.0, 0.0001))
    gate = gpu.update_semidense(gate, ob(1, 1, 10.0, 0.04))
    assert gate.depth[1, 1] == 2.0 and gate.variance[1, 1] == 0.0001
    with pytest.raises(DfuseError) as e:
        gpu.update_semidense(m, ob(8, 0, 1.0, 1.0))
    assert e.value.code == "OutOfBounds"


def test_update_semidense_duplicates_in_order(gpu, orc):
    rng = np.random.default_rng(4)
    w, h, n = 20, 10, 4000
    obs = np.zeros(n, OBS_DTYPE)
    obs["x"] = rng.integers(0, w, n)
    obs["y"] = rng.integers(0, h, n)
    obs["depth"] = rng.uniform(1, 3, n)
    obs["variance"] = rng.uniform(0.01, 1.0, n)
    a = gpu.update_semidense(SemiDenseMap.empty(w, h), obs)
    b = orc.update_semidense(SemiDenseMap.empty(w, h), obs)
    assert a.depth.tobytes() == b.depth.tobytes()
    assert a.variance.tobytes() == b.variance.tobytes()
    assert a.inlier_count == b.inlier_count
