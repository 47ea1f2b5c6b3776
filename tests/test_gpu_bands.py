"""GPU parity for the row-band keyframe (SURVEY 8(e), config C4's
decomposition): per-band planes with halo rows, per-band stereo, and the
optimiser over all bands with the two-level all-reduce. One band is the
streaming solver exactly (bit for bit); any band count matches the oracle
pipeline within the fusion tolerance, with the semi-dense map bit-exact."""
import numpy as np
import pytest

from paper_2207_12244_b200 import api, synth
from paper_2207_12244_b200._ffi import DfuseError, RobustConfig, SemiDenseMap, init_state
from helpers import rel_err

pytestmark = pytest.mark.gpu


def _geom(ctx, spec, q, t):
    return ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())


def test_one_band_is_the_streaming_session(gpu_ctx):
    spec = synth.small_spec(160, 120, frames=2)
    seq = synth.make_sequence(spec, 11, frames=2)
    cfg = RobustConfig(gn_iterations=4)
    gpu_ctx.set_solver_path("streaming")
    try:
        a = api.Keyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0.02)
        b = api.BandedKeyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 1, 0.02)
        for q, t, I1 in seq.frames:
            g = _geom(gpu_ctx, spec, q, t)
            ra = a.process_frame(g, I1, spec.search, cfg, "full")
            rb = b.process_frame(g, I1, spec.search, cfg, "full")
            assert (ra.observations, ra.inlier_count) == (rb.observations, rb.inlier_count)
            assert ra.stats.pcg_total == rb.stats.pcg_total
        sa, ma, ka = a.download()
        sb, mb, kb = b.download()
        assert np.array_equal(ka, kb)
        assert sa.log_depth.tobytes() == sb.log_depth.tobytes()
        assert sa.scale == sb.scale and sa.iteration == sb.iteration
        a.close()
        b.close()
    finally:
        gpu_ctx.set_solver_path("auto")


@pytest.mark.parametrize("name,bands,mode", [("S", 2, "full"), ("S", 3, "nopairwise"),
                                             ("S", 5, "lsscale"), ("C1", 4, "full"),
                                             ("C1", 8, "full")])
def test_bands_match_oracle_pipeline(gpu_ctx, orc, name, bands, mode):
    spec = synth.small_spec(160, 120, frames=3) if name == "S" else synth.CONFIGS["C1"]
    seq = synth.make_sequence(spec, 23, frames=3)
    cfg = RobustConfig(gn_iterations=spec.gn_iterations if name != "S" else 6)
    kf = api.BandedKeyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, bands, 0.02)
    st, semi, mask = kf.download()
    assert np.array_equal(mask, orc.texture_mask(seq.I0, 0.02))
    assert np.array_equal(st.log_depth, seq.pred.log_depth) and semi.inlier_count == 0
    o_semi = SemiDenseMap.empty(spec.width, spec.height)
    for q, t, I1 in seq.frames:
        g = _geom(gpu_ctx, spec, q, t)
        before, _, _ = kf.download()
        res = kf.process_frame(g, I1, spec.search, cfg, mode)
        r = orc.stereo_update(g, seq.I0, I1, mask, o_semi, spec.search)
        o_semi = r.semi
        assert res.observations == r.n_obs and res.inlier_count == o_semi.inlier_count
        g_st, g_semi, _ = kf.download()
        assert g_semi.depth.tobytes() == o_semi.depth.tobytes()
        assert g_semi.variance.tobytes() == o_semi.variance.tobytes()
        assert np.array_equal(g_semi.valid, o_semi.valid)
        try:
            o_st, so = orc.optimize(before, o_semi, seq.pred, cfg, mode, with_stats=True)
        except DfuseError as e:  # the reference diverges too: state unchanged (H10)
            assert e.code == "CgDivergence" and res.optimize_status == 20
            assert g_st.log_depth.tobytes() == before.log_depth.tobytes()
            continue
        assert res.optimize_status == 0
        assert g_st.iteration == o_st.iteration
        assert rel_err(np.exp(g_st.log_depth), np.exp(o_st.log_depth)) < 1e-4
        assert rel_err(g_st.scale, o_st.scale) < 1e-4
        assert abs(res.stats.pcg_total - so.pcg_total) <= max(2, 0.02 * so.pcg_total)
    kf.reset()
    st, semi, _ = kf.download()
    assert st.iteration == 0 and semi.inlier_count == 0
    kf.close()


def test_band_count_is_validated(gpu_ctx):
    spec = synth.small_spec(32, 8, frames=1)
    seq = synth.make_sequence(spec, 1, frames=1)
    with pytest.raises(Exception):
        api.BandedKeyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 9, 0.02)
    with pytest.raises(Exception):
        api.BandedKeyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0, 0.02)


def test_rank_form_single_process(gpu_ctx):
    """dfuse_bkf_create_rank with world 1 (no peers to connect): the same
    band, the same kernel with system-scope fences, the same bits as the
    single-launch form."""
    from paper_2207_12244_b200.bands_dist import DistributedBandedKeyframe

    spec = synth.small_spec(160, 120, frames=2)
    seq = synth.make_sequence(spec, 12, frames=2)
    cfg = RobustConfig(gn_iterations=4)
    a = api.BandedKeyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 1, 0.02)
    b = DistributedBandedKeyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0.02, world=1, rank=0)
    for q, t, I1 in seq.frames:
        g = _geom(gpu_ctx, spec, q, t)
        ra = a.process_frame(g, I1, spec.search, cfg, "full")
        rb = b.process_frame(g, I1, spec.search, cfg, "full")
        assert (ra.observations, ra.inlier_count) == (rb.observations, rb.inlier_count)
    sa, ma, _ = a.download()
    sb, mb, _ = b.download()
    assert sa.log_depth.tobytes() == sb.log_depth.tobytes()
    assert ma.depth.tobytes() == mb.depth.tobytes() and ma.inlier_count == mb.inlier_count
    a.close()
    b.close()
