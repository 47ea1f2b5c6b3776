"""Diagnostics: cost of one grid-wide all-reduce of the fusion solver
(dfuse_debug_sync_bench) per variant and grid size, and the per-iteration
cost of the PCG at C2 size on both data paths. Prints JSON lines."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12244_b200 import api  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests"))
from helpers import make_random_problem  # noqa: E402

ctx = api.context(0)
L = api.lib()
L.dfuse_debug_sync_bench.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_float)]
ms = C.c_float()
only = [int(a) for a in sys.argv[1:]]
for variant in only or (10, 11, 12, 2):
    for grid in (74, 148) if variant in (11, 12, 13, 14, 15, 16) else (32, 74, 148):
        t = {}
        L.dfuse_debug_sync_bench(ctx.handle, 50000, variant, grid, C.byref(ms))  # clock warm-up
        for n in (0, 20000):
            best = 1e9
            for _ in range(3):
                rc = L.dfuse_debug_sync_bench(ctx.handle, n, variant, grid, C.byref(ms))
                assert rc == 0, L.dfuse_last_error(ctx.handle)
                best = min(best, ms.value)
            t[n] = best
        print(json.dumps({"what": "allreduce", "variant": variant, "grid": grid,
                          "us_per_op": round((t[20000] - t[0]) * 1e3 / 20000, 3)}), flush=True)
if only:
    sys.exit(0)

# PCG per-iteration cost at 640x480 (fixed iteration counts)
st, semi, pred = make_random_problem(5, 640, 480)
gpu = ctx.api
eq = gpu.assemble_normal_equations(st, semi, pred)
for streaming in (False, True):
    ctx.set_solver_path(streaming)
    res = {}
    for its in (1, 201):
        cfg = RobustConfig(cg_tol=0.0, cg_max_iters=its)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            gpu.solve_depth_step(eq, cfg)
            best = min(best, time.perf_counter() - t0)
        res[its] = best
    print(json.dumps({"what": "pcg", "path": "streaming" if streaming else "resident",
                      "us_per_iter_wall": round((res[201] - res[1]) * 1e6 / 200, 3)}), flush=True)
ctx.set_solver_path(False)
