"""Run with DFUSE_LIB=paper_2207_12244_b200/libdfuse_cuda_diag.so (make -C
paper_2207_12244_b200/csrc diag).
Diagnostics: per-phase trace (DFUSE_TRACE=1, printed by the library on
stderr) of the C2 optimize for a few tracked frames on one solver path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12244_b200 import api, synth  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig  # noqa: E402

ctx = api.context(0)
ctx.set_solver_path(sys.argv[1] if len(sys.argv) > 1 else "auto")
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = synth.CONFIGS["C2"]
seq = synth.make_sequence(spec, 0)
kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
cfg = RobustConfig()
for f, (q, t, I1) in enumerate(seq.frames[:nf]):
    g = ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
    r = kf.process_frame(g, I1, spec.search, cfg, "full")
    print(f"frame {f}: optimise {r.optimise_ms:.3f} ms pcg {r.stats.pcg_total}", file=sys.stderr)
