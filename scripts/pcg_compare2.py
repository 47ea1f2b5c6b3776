"""Diagnostics: which part of the optimize() context slows the PCG loop."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_12244_b200 import api, synth  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig, SemiDenseMap, init_state  # noqa: E402

ctx = api.context(0)
gpu = ctx.api
spec = synth.CONFIGS["C2"]
seq = synth.make_sequence(spec, 0, frames=1)
mask = gpu.texture_mask(seq.I0, 0.02)
semi = SemiDenseMap.empty(spec.width, spec.height)
q, t, I1 = seq.frames[0]
g = gpu.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
semi = gpu.stereo_update(g, seq.I0, I1, mask, semi, spec.search).semi
st = init_state(seq.pred)
for label, cfg in [
    ("optimize gn=1 its=200", RobustConfig(gn_iterations=1, cg_tol=0.0, cg_max_iters=200)),
    ("optimize gn=1 its=200 no-scale", RobustConfig(gn_iterations=1, cg_tol=0.0, cg_max_iters=200,
                                                    estimate_scale=False)),
    ("optimize gn=1 its=200 nopairwise", RobustConfig(gn_iterations=1, cg_tol=0.0,
                                                      cg_max_iters=200)),
]:
    print(label, file=sys.stderr)
    gpu.optimize(st, semi, seq.pred, cfg, "nopairwise" if "nopair" in label else "full")
eq = gpu.assemble_normal_equations(st, semi, seq.pred)
print("standalone its=200", file=sys.stderr)
gpu.solve_depth_step(eq, RobustConfig(cg_tol=0.0, cg_max_iters=200))
