"""GPU parity for keyframe creation on the device:
make_keyframe from a DFPRED file (load_predictions + focal_adjust on the
device, pipeline.hpp:133-150) against the reference build's own
load_predictions / focal_adjust on the same bytes, the reference's corrupt-file
KATs (test_predictions.cpp:63-101) through the device path, and the cached
median_predicted_depth (pipeline.hpp:94-99) against the oracle."""
import ctypes as C
import struct

import numpy as np
import pytest

from paper_2207_12244_b200 import api, synth
from paper_2207_12244_b200._ffi import DfuseError, RobustConfig
from helpers import synth_oracle
from test_predictions_cpu import planes_of, ref_load, smooth_gt

pytestmark = pytest.mark.gpu


def _scene(name="S"):
    spec = synth.small_spec(96, 72, frames=1) if name == "S" else synth.CONFIGS[name]
    seq = synth.make_sequence(spec, 3, frames=1)
    return spec, seq


@pytest.mark.parametrize("name", ["S", "C1"])
def test_dfpred_keyframe_equals_plane_keyframe(gpu_ctx, name):
    """source_focal == fx: the DFPRED path is the plane path, bit for bit,
    through creation and one tracked frame."""
    spec, seq = _scene(name)
    cam = spec.camera()
    data = synth.to_dfpred(seq.pred, cam.fx)
    a = api.Keyframe(gpu_ctx, cam, seq.I0, seq.pred, 0.02)
    b = api.Keyframe(gpu_ctx, cam, seq.I0, None, 0.02, dfpred=data)
    sa, ma, ka = a.download()
    sb, mb, kb = b.download()
    assert np.array_equal(ka, kb)
    assert sa.log_depth.tobytes() == sb.log_depth.tobytes()
    q, t, I1 = seq.frames[0]
    g = gpu_ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, cam)
    ra = a.process_frame(g, I1, spec.search, RobustConfig(gn_iterations=2), "full")
    rb = b.process_frame(g, I1, spec.search, RobustConfig(gn_iterations=2), "full")
    assert ra.observations == rb.observations
    assert a.download()[0].log_depth.tobytes() == b.download()[0].log_depth.tobytes()
    a.close()
    b.close()


@pytest.mark.parametrize("source_focal", [262.5, 300.0, 1000.0])
def test_dfpred_focal_adjust_matches_reference(gpu_ctx, orc, ref, tmp_path, source_focal):
    spec, seq = _scene("S")
    cam = spec.camera()
    data = synth.to_dfpred(seq.pred, source_focal)
    path = tmp_path / "p.dfpred"
    path.write_bytes(data)
    h, w = seq.I0.shape
    rc, planes, f, _ = ref_load(ref, str(path), w, h)
    assert rc == 0
    ld = np.ascontiguousarray(planes[: w * h].copy())
    assert ref.lib.ref_focal_adjust(w, h, ld.ctypes.data_as(C.c_void_p), C.c_double(f),
                                    C.c_double(cam.fx)) == 0
    kf = api.Keyframe(gpu_ctx, cam, seq.I0, None, 0.02, dfpred=data)
    st, _, _ = kf.download()
    assert st.log_depth.ravel().tobytes() == ld.tobytes()  # init_state = adjusted predictions
    orc.lib.orc_median_predicted_depth.restype = C.c_double
    med = orc.lib.orc_median_predicted_depth(ld.ctypes.data_as(C.c_void_p), C.c_long(w * h))
    assert kf.median_depth() == med
    assert kf.median_depth() == med  # cached
    kf.close()


def test_dfpred_corrupt_file_kats(gpu_ctx):
    """test_predictions.cpp:63-101 through the device path"""
    p = synth_oracle(smooth_gt(8, 6), 0.1, 0.02, 3, 200.0)
    cam = synth.small_spec(8, 6).camera()
    I0 = np.zeros((6, 8), np.float32)
    good = synth.to_dfpred(p, 200.0)
    n = 8 * 6

    def create(data, camera=cam):
        return api.Keyframe(gpu_ctx, camera, I0, None, 0.02, dfpred=data)

    with pytest.raises(DfuseError) as e:
        create(b"XFPR" + good[4:])
    assert e.value.code == "BadMagic"
    off = 24 + n * 4 + 5 * 4
    with pytest.raises(DfuseError) as e:
        create(good[:off] + struct.pack("<f", 0.0) + good[off + 4:])
    assert e.value.code == "NonPositiveVariance"
    assert "log_depth_var" in str(e.value) and str(off) in str(e.value)
    for bad in (-1.0, float("inf"), float("nan")):  # v > 0 and finite, every variance channel
        o = 24 + 5 * n * 4 + 47 * 4
        with pytest.raises(DfuseError) as e:
            create(good[:o] + struct.pack("<f", bad) + good[o + 4:])
        assert e.value.code == "NonPositiveVariance" and "grad_y_var[47]" in str(e.value)
    with pytest.raises(DfuseError) as e:
        create(good[:24 + 3 * n * 4 + 10])
    assert e.value.code == "TruncatedFile" and "grad_x_var" in str(e.value)
    with pytest.raises(DfuseError) as e:  # pipeline.hpp:139-141
        create(good, synth.small_spec(10, 6).camera())
    assert e.value.code == "DimensionMismatch"


def test_median_depth_plane_keyframe(gpu_ctx, orc):
    spec, seq = _scene("C1")
    kf = api.Keyframe(gpu_ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    ld = np.ascontiguousarray(seq.pred.log_depth)
    orc.lib.orc_median_predicted_depth.restype = C.c_double
    assert kf.median_depth() == orc.lib.orc_median_predicted_depth(
        ld.ctypes.data_as(C.c_void_p), C.c_long(ld.size))
    kf.close()
