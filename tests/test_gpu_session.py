"""GPU parity: the device-resident keyframe session (make_keyframe +
process_frame for tracked frames, pipeline.hpp:125-228) against the oracle
pipeline (stereo_update + optimize per frame)."""
import numpy as np
import pytest

from paper_2207_12244_b200 import api, synth
from paper_2207_12244_b200._ffi import DfuseError, RobustConfig, SemiDenseMap, init_state
from helpers import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["S", "C1"])
def test_session_matches_oracle_pipeline(gpu_ctx, orc, name):
    spec = synth.small_spec(160, 120, frames=3) if name == "S" else synth.CONFIGS["C1"]
    seq = synth.make_sequence(spec, 21, frames=3)
    cfg = RobustConfig(gn_iterations=spec.gn_iterations)
    kf = api.Keyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    st, semi, mask = kf.download()
    assert np.array_equal(mask, orc.texture_mask(seq.I0, 0.02))
    assert st.iteration == 0 and st.scale == 1.0 and semi.inlier_count == 0
    o_semi = SemiDenseMap.empty(spec.width, spec.height)
    o_st = init_state(seq.pred)
    for (q, t, I1) in seq.frames:
        g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
        # the session's stereo stage is bit-exact; feed the oracle's fusion
        # the session's input state each frame so tolerances do not compound
        g_st_before, _, _ = kf.download()
        res = kf.process_frame(g, I1, spec.search, cfg, "full")
        r = orc.stereo_update(g, seq.I0, I1, mask, o_semi, spec.search)
        o_semi = r.semi
        assert res.observations == r.n_obs
        assert res.inlier_count == o_semi.inlier_count
        g_st, g_semi, _ = kf.download()
        assert g_semi.depth.tobytes() == o_semi.depth.tobytes()
        assert g_semi.variance.tobytes() == o_semi.variance.tobytes()
        o_st = orc.optimize(g_st_before, o_semi, seq.pred, cfg)
        assert res.optimize_status == 0
        assert g_st.iteration == o_st.iteration
        assert rel_err(np.exp(g_st.log_depth), np.exp(o_st.log_depth)) < 1e-4
        assert rel_err(g_st.scale, o_st.scale) < 1e-4
    assert res.stereo_frames == len(seq.frames)
    kf.reset()
    st, semi, _ = kf.download()
    assert st.iteration == 0 and semi.inlier_count == 0
    assert np.array_equal(st.log_depth, seq.pred.log_depth)
    kf.close()


def test_launch_counter_moves(gpu_ctx):
    before = gpu_ctx.launch_count()
    gpu_ctx.api.texture_mask(np.zeros((16, 16), np.float32), 0.02)
    assert gpu_ctx.launch_count() > before


def test_async_frames_equal_sync_frames(gpu_ctx):
    """dfuse_kf_process_frame_async: frames enqueued back to back give the
    state and counts of the synchronous calls, bit for bit (stereo_frames is
    counted on the device); reset is stream-ordered too."""
    import torch

    spec = synth.small_spec(160, 120, frames=4)
    seq = synth.make_sequence(spec, 33, frames=4)
    cfg = RobustConfig(gn_iterations=3)
    geoms = [gpu_ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t,
                                                spec.camera()) for (q, t, _) in seq.frames]
    dev = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).cuda()
           for (_, _, I1) in seq.frames]
    torch.cuda.synchronize()
    a = api.Keyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    b = api.Keyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    for rep in range(2):
        for k in range(len(dev)):
            ra = a.process_frame(geoms[k], None, spec.search, cfg, "full",
                                 device_ptr=dev[k].data_ptr())
            b.process_frame_async(geoms[k], dev[k].data_ptr(), spec.search, cfg, "full")
        rb = b.last_result()
        assert (ra.observations, ra.inlier_count, ra.stereo_frames) == \
            (rb.observations, rb.inlier_count, rb.stereo_frames)
        sa, ma, _ = a.download()
        sb, mb, _ = b.download()
        assert sa.log_depth.tobytes() == sb.log_depth.tobytes()
        assert (sa.scale, sa.iteration) == (sb.scale, sb.iteration)
        assert ma.depth.tobytes() == mb.depth.tobytes()
        a.reset()
        b.reset()
    with pytest.raises(DfuseError):
        b.last_result()  # nothing enqueued since the last result
    a.close()
    b.close()


def test_session_c5_stress_matches_oracle(gpu_ctx, orc):
    """C5: 30 % textureless regions, Laplace priors, search range 0.1-20 m:
    the semi-dense map bit-exact and the fused state within tolerance for
    two tracked frames."""
    spec = synth.CONFIGS["C5"]
    seq = synth.make_sequence(spec, 41, frames=2)
    cfg = RobustConfig(gn_iterations=4)
    kf = api.Keyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    _, _, mask = kf.download()
    o_semi = SemiDenseMap.empty(spec.width, spec.height)
    for (q, t, I1) in seq.frames:
        g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
        before, _, _ = kf.download()
        res = kf.process_frame(g, I1, spec.search, cfg, "full")
        o_semi = orc.stereo_update(g, seq.I0, I1, mask, o_semi, spec.search).semi
        g_st, g_semi, _ = kf.download()
        assert g_semi.depth.tobytes() == o_semi.depth.tobytes()
        assert res.inlier_count == o_semi.inlier_count
        o_st, so = orc.optimize(before, o_semi, seq.pred, cfg, with_stats=True)
        assert rel_err(np.exp(g_st.log_depth), np.exp(o_st.log_depth)) < 1e-4
        assert rel_err(g_st.scale, o_st.scale) < 1e-4
        assert abs(res.stats.pcg_total - so.pcg_total) <= max(2, 0.02 * so.pcg_total)
    kf.close()


@pytest.mark.parametrize("name", ["S", "C2"])
def test_texture_gather_scan_is_bit_identical(orc, name):
    """The epipolar scan through the texture gather (dfuse_ctx_set_stereo_texture,
    default) and through plain loads give the same semi-dense map and fused
    state, bit for bit; the session uses the gather."""
    spec = synth.small_spec(160, 120, frames=3) if name == "S" else synth.CONFIGS["C2"]
    seq = synth.make_sequence(spec, 5, frames=3)
    cfg = RobustConfig(gn_iterations=spec.gn_iterations)
    out = {}
    for on in (True, False):
        ctx = api.Context(0)
        ctx.set_stereo_texture(on)
        kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
        obs = []
        for (q, t, I1) in seq.frames:
            g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
            obs.append(kf.process_frame(g, I1, spec.search, cfg, "full").observations)
        st, semi, _ = kf.download()
        out[on] = (obs, st.log_depth.tobytes(), semi.depth.tobytes(), semi.variance.tobytes(),
                   ctx.texture_launches())
        kf.close()
        ctx.close()
    assert out[True][4] == len(seq.frames)  # the gather path ran
    assert out[False][4] == 0
    assert out[True][:4] == out[False][:4]


def test_host_async_pipeline_equals_sync_frames(orc):
    """dfuse_kf_process_frame_host_async: host frames copied in on the copy
    stream, each frame's fused log-depth copied out while the next computes;
    every frame's output equals the synchronous path's download, bit for bit."""
    import torch

    spec = synth.CONFIGS["C2"]
    seq = synth.make_sequence(spec, 9, frames=5)
    cfg = RobustConfig(gn_iterations=spec.gn_iterations)
    ctx = api.Context(0)
    kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    geoms = [orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
             for (q, t, _) in seq.frames]
    ref = []
    for g, (_, _, I1) in zip(geoms, seq.frames):
        last_sync = kf.process_frame(g, I1, spec.search, cfg, "full")
        ref.append(kf.download()[0].log_depth.copy())
    kf.reset()
    pins = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).pin_memory()
            for (_, _, I1) in seq.frames]
    outs = [torch.empty((spec.height, spec.width), dtype=torch.float64).pin_memory()
            for _ in seq.frames]
    for g, p, o in zip(geoms, pins, outs):
        kf.process_frame_host_async(g, p.numpy(), spec.search, cfg, "full",
                                    log_depth_out=o.numpy())
    res = kf.last_result()
    for o, r in zip(outs, ref):
        assert o.numpy().tobytes() == r.tobytes()
    assert res.observations == last_sync.observations
    assert res.stereo_frames == len(seq.frames)
    kf.close()
    ctx.close()


@pytest.mark.parametrize("name,bands", [("C2", 0), ("S", 0), ("S", 3)])
def test_fp32_prediction_planes_are_bit_identical(orc, name, bands):
    """Float-exact prediction planes kept as float32 on the device
    (dfuse_ctx_set_fp32_predictions, default) give the same fused state, bit
    for bit, as the fp64 planes: the values are identical and the reciprocal
    variances are formed by the same division."""
    import ctypes as C

    spec = synth.small_spec(160, 120, frames=3) if name == "S" else synth.CONFIGS["C2"]
    seq = synth.make_sequence(spec, 13, frames=3)
    cfg = RobustConfig(gn_iterations=spec.gn_iterations)
    out = {}
    L = api.lib()
    L.dfuse_ctx_set_fp32_predictions.argtypes = [C.c_void_p, C.c_int]
    for on in (1, 0):
        ctx = api.Context(0)
        assert L.dfuse_ctx_set_fp32_predictions(ctx.handle, on) == 0
        if bands:
            kf = api.BandedKeyframe(ctx, spec.camera(), seq.I0, seq.pred, bands, 0.02)
        else:
            kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
        pcg = []
        for (q, t, I1) in seq.frames:
            g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
            pcg.append(kf.process_frame(g, I1, spec.search, cfg, "full").stats.pcg_total)
        st, semi, _ = kf.download()
        out[on] = (pcg, st.log_depth.tobytes(), st.scale, st.iteration, semi.depth.tobytes())
        kf.close()
        ctx.close()
    assert out[1] == out[0]
