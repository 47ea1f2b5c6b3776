"""Diagnostics: per-frame stereo time and step statistics of the C2 sequence."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12244_b200 import api, synth  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig  # noqa: E402

ctx = api.context(0)
spec = synth.CONFIGS["C2"]
seq = synth.make_sequence(spec, 0)
kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
cfg = RobustConfig(cg_tol=0.0, cg_max_iters=5)
for rep in range(2):
    out = []
    for f, (q, t, I1) in enumerate(seq.frames):
        g = ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
        r = kf.process_frame(g, I1, spec.search, cfg, "full")
        out.append(f"{r.stereo_ms:.3f}/{r.observations}")
    kf.reset()
    print("frame stereo ms/obs:", " ".join(out))
