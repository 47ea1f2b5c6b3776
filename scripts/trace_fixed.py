"""Run with DFUSE_LIB=paper_2207_12244_b200/libdfuse_cuda_diag.so (make -C
paper_2207_12244_b200/csrc diag).
Diagnostics: per-phase trace (DFUSE_TRACE=1) of the C2 optimize in the
fixed-effort regime (10 GN x 5 PCG iterations)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12244_b200 import api, synth  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig  # noqa: E402

ctx = api.context(0)
spec = synth.CONFIGS["C2"]
seq = synth.make_sequence(spec, 0, frames=3)
kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
cfg = RobustConfig(cg_tol=0.0, cg_max_iters=5)
for f, (q, t, I1) in enumerate(seq.frames):
    g = ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
    r = kf.process_frame(g, I1, spec.search, cfg, "full")
    print(f"frame {f}: stereo {r.stereo_ms:.3f} ms optimise {r.optimise_ms:.3f} ms "
          f"pcg {r.stats.pcg_total} syncs {r.stats.grid_syncs}", file=sys.stderr)
