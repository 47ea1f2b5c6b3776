"""Profiling driver: one fixed-iteration PCG solve (dfuse_solve_depth_step)
on a 640x480 system, solver path from argv[1] (auto|resident2r|streaming). Used under ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests"))
from helpers import make_random_problem  # noqa: E402
from paper_2207_12244_b200 import api  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig  # noqa: E402

ctx = api.context(0)
ctx.set_solver_path(sys.argv[1] if len(sys.argv) > 1 else "auto")
st, semi, pred = make_random_problem(5, 640, 480)
eq = ctx.api.assemble_normal_equations(st, semi, pred)
cfg = RobustConfig(cg_tol=0.0, cg_max_iters=int(os.environ.get("PCG_ITERS", "100")))
for _ in range(2):
    d, its = ctx.api.solve_depth_step(eq, cfg)
print("iterations", its)
