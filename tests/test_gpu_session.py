"""GPU parity: the device-resident keyframe session (make_keyframe +
process_frame for tracked frames, pipeline.hpp:125-228) against the oracle
pipeline (stereo_update + optimize per frame)."""
import numpy as np
import pytest

from paper_2207_12244_b200 import api, synth
from paper_2207_12244_b200._ffi import RobustConfig, SemiDenseMap, init_state
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
