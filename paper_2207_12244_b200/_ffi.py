"""ctypes mirror of include/dfuse_cuda.h plus the Python-side API shape.

The function set declared in dfuse_cuda.h is exported by three libraries:
the product (``libdfuse_cuda.so``, ``dfuse_*`` with a leading context
argument) and the two test oracles (``orc_*`` / ``ref_*``, no context; see
oracle/dfuse_oracle.h). :class:`Bindings` marshals numpy arrays for any of
them, so the parity tests call the GPU path and the oracle through one API
that reads like the reference's own (fusion.hpp / semidense.hpp names,
argument meaning and error behaviour).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# errors: dfuse::Err (errors.hpp:8-42); C code = int(Err) + 1
ERR_NAMES = [
    "NonPositiveDepth", "BehindCamera", "OutOfBounds", "DegenerateBaseline", "NoMinimum",
    "ZeroBaselineStep", "DegenerateJacobian", "BorderPixel", "BadMagic", "DimensionMismatch",
    "NonPositiveVariance", "TruncatedFile", "NonPositiveFocal", "NonPositiveGroundTruth",
    "MissingFile", "MalformedLine", "NonUnitQuaternion", "BadImageFormat", "NonPositiveScale",
    "CgDivergence", "NoSemiDenseSupport", "NoValidGroundTruth", "MismatchedKeyframeSets",
    "IoError", "UnknownKey", "TypeError", "InvalidArgument",
]
ERR_CODE = {name: i + 1 for i, name in enumerate(ERR_NAMES)}
E_CUDA = 100


class DfuseError(RuntimeError):
    """Mirror of dfuse::Error (errors.hpp:79-88): one exception type, the
    failure class in ``.code`` (an Err name)."""

    def __init__(self, code: int, detail: str = ""):
        self.code_value = int(code)
        self.code = ERR_NAMES[code - 1] if 1 <= code <= len(ERR_NAMES) else (
            "Cuda" if code == E_CUDA else f"Unknown({code})")
        super().__init__(f"{self.code}: {detail}" if detail else self.code)


# EpipolarStatus (semidense.hpp:46-53)
EPI_OK, EPI_DEGENERATE_BASELINE, EPI_OUT_OF_BOUNDS, EPI_BEHIND_CAMERA, EPI_NO_MINIMUM, \
    EPI_DEGENERATE_JACOBIAN = range(6)
EPI_NOT_SEARCHED = -1
EPI_NAMES = ["Ok", "DegenerateBaseline", "OutOfBounds", "BehindCamera", "NoMinimum",
             "DegenerateJacobian"]

# FusionMode (fusion.hpp:33)
MODE_FULL, MODE_NOPAIRWISE, MODE_LSSCALE = 0, 1, 2
MODES = {"full": MODE_FULL, "nopairwise": MODE_NOPAIRWISE, "lsscale": MODE_LSSCALE}
STATS_MAX_GN = 512


# --------------------------------------------------------------------------
# C structs
class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class EpiGeom(C.Structure):
    _fields_ = [("R_10", C.c_double * 9), ("t_10", C.c_double * 3), ("t_01", C.c_double * 3),
                ("K", Intrinsics)]


class SearchCfgC(C.Structure):
    _fields_ = [("min_depth", C.c_double), ("max_depth", C.c_double),
                ("max_rms_error", C.c_double)]


class RobustCfgC(C.Structure):
    _fields_ = [("delta_semi", C.c_double), ("delta_net", C.c_double),
                ("delta_grad", C.c_double), ("cg_tol", C.c_double),
                ("gn_iterations", C.c_int32), ("cg_max_iters", C.c_int32),
                ("estimate_scale", C.c_int32), ("reserved", C.c_int32)]


class ObsC(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("depth", C.c_double),
                ("error5", C.c_double * 5), ("jacobian", C.c_double * 5),
                ("variance", C.c_double)]


OBS_DTYPE = np.dtype([("x", "f8"), ("y", "f8"), ("depth", "f8"), ("error5", "f8", 5),
                      ("jacobian", "f8", 5), ("variance", "f8")])
assert OBS_DTYPE.itemsize == C.sizeof(ObsC) == 112


class FusionInputsC(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("semi_depth", C.POINTER(C.c_double)), ("semi_variance", C.POINTER(C.c_double)),
                ("semi_valid", C.POINTER(C.c_uint8)), ("inlier_count", C.c_int32),
                ("reserved", C.c_int32), ("pred", C.POINTER(C.c_double) * 6)]


class SolverStatsC(C.Structure):
    _fields_ = [("gn_done", C.c_int32), ("pcg_total", C.c_int32), ("cost_evals", C.c_int32),
                ("grid_syncs", C.c_int32), ("pcg_iters", C.c_int32 * STATS_MAX_GN),
                ("scale_step", C.c_double * STATS_MAX_GN),
                ("depth_step", C.c_double * STATS_MAX_GN)]


class FrameResultC(C.Structure):
    _fields_ = [("observations", C.c_int32), ("inlier_count", C.c_int32),
                ("stereo_frames", C.c_int32), ("optimize_status", C.c_int32),
                ("stereo_ms", C.c_float), ("optimise_ms", C.c_float),
                ("stats", SolverStatsC), ("epipolar_steps", C.c_int64),
                ("solver_ppt", C.c_int32), ("reserved", C.c_int32)]


# --------------------------------------------------------------------------
# Python-side value types (names follow the reference)
@dataclass
class CameraIntrinsics:  # geometry.hpp:18-41
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def c(self) -> Intrinsics:
        return Intrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


@dataclass
class SearchConfig:  # semidense.hpp:66-73
    min_depth: float = 0.25
    max_depth: float = 50.0
    max_rms_error: float = 0.05

    def c(self) -> SearchCfgC:
        return SearchCfgC(self.min_depth, self.max_depth, self.max_rms_error)


@dataclass
class RobustConfig:  # fusion.hpp:23-31
    delta_semi: float = 0.3
    delta_net: float = 0.3
    delta_grad: float = 0.1
    gn_iterations: int = 10
    cg_tol: float = 1e-6
    cg_max_iters: int = 200
    estimate_scale: bool = True

    def c(self) -> RobustCfgC:
        return RobustCfgC(self.delta_semi, self.delta_net, self.delta_grad, self.cg_tol,
                          int(self.gn_iterations), int(self.cg_max_iters),
                          1 if self.estimate_scale else 0, 0)


@dataclass
class SemiDenseMap:  # semidense.hpp:21-31
    depth: np.ndarray
    variance: np.ndarray
    valid: np.ndarray
    inlier_count: int = 0

    @staticmethod
    def empty(width: int, height: int) -> "SemiDenseMap":
        return SemiDenseMap(np.zeros((height, width)), np.zeros((height, width)),
                            np.zeros((height, width), np.uint8), 0)

    def copy(self) -> "SemiDenseMap":
        return SemiDenseMap(self.depth.copy(), self.variance.copy(), self.valid.copy(),
                            int(self.inlier_count))


PRED_CHANNELS = ("log_depth", "log_depth_var", "grad_x", "grad_x_var", "grad_y", "grad_y_var")


@dataclass
class PredictionSet:  # predictions.hpp:18-29
    log_depth: np.ndarray
    log_depth_var: np.ndarray
    grad_x: np.ndarray
    grad_x_var: np.ndarray
    grad_y: np.ndarray
    grad_y_var: np.ndarray
    source_focal: float = 0.0

    def planes(self):
        return [np.ascontiguousarray(getattr(self, c), dtype=np.float64) for c in PRED_CHANNELS]

    def copy(self) -> "PredictionSet":
        return PredictionSet(*[p.copy() for p in self.planes()], source_focal=self.source_focal)


@dataclass
class FusionState:  # fusion.hpp:17-21
    log_depth: np.ndarray
    scale: float = 1.0
    iteration: int = 0

    def copy(self) -> "FusionState":
        return FusionState(self.log_depth.copy(), float(self.scale), int(self.iteration))


def init_state(pred: PredictionSet) -> FusionState:  # fusion.hpp:44-46
    return FusionState(np.array(pred.log_depth, dtype=np.float64, copy=True), 1.0, 0)


@dataclass
class NormalEquations:  # fusion.hpp:107-141
    diag: np.ndarray
    right: np.ndarray
    down: np.ndarray
    b: np.ndarray


@dataclass
class SolverStats:
    gn_done: int
    pcg_total: int
    cost_evals: int
    grid_syncs: int
    pcg_iters: list
    scale_step: list
    depth_step: list

    @staticmethod
    def from_c(s: SolverStatsC) -> "SolverStats":
        n = min(s.gn_done, STATS_MAX_GN)
        return SolverStats(s.gn_done, s.pcg_total, s.cost_evals, s.grid_syncs,
                           list(s.pcg_iters[:n]), list(s.scale_step[:n]), list(s.depth_step[:n]))


@dataclass
class StereoResult:
    semi: SemiDenseMap
    n_obs: int
    status: np.ndarray
    best: np.ndarray
    n_steps: np.ndarray
    obs: np.ndarray  # OBS_DTYPE records, raster order


# --------------------------------------------------------------------------
def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _mode(mode) -> int:
    if isinstance(mode, str):
        return MODES[mode]
    return int(mode)


class Bindings:
    """Reference-shaped API over one library exporting the dfuse_cuda.h
    function set under ``prefix`` (``dfuse_`` takes a context first)."""

    def __init__(self, lib: C.CDLL, prefix: str, ctx=None, name: str = ""):
        self.lib = lib
        self.prefix = prefix
        self.ctx = ctx
        self.name = name or prefix.rstrip("_")
        vp = C.c_void_p
        P = C.POINTER
        sig = {
            "make_epipolar_geometry": [P(C.c_double), P(C.c_double), P(C.c_double),
                                       P(C.c_double), P(Intrinsics), P(EpiGeom)],
            "texture_mask": [vp, C.c_int, C.c_int, C.c_double, vp],
            "search_depth": [P(EpiGeom), vp, vp, C.c_int, vp, vp, vp, P(SearchCfgC), vp, vp, vp,
                             vp],
            "update_semidense": [C.c_int, C.c_int, vp, vp, vp, P(C.c_int32), C.c_int, vp],
            "stereo_update": [P(EpiGeom), vp, vp, vp, P(SearchCfgC), vp, vp, vp, P(C.c_int32),
                              P(C.c_int32), vp, vp, vp, vp],
            "assemble_normal_equations": [P(FusionInputsC), vp, C.c_double, P(RobustCfgC),
                                          C.c_int, vp, vp, vp, vp],
            "total_cost": [P(FusionInputsC), vp, C.c_double, P(RobustCfgC), C.c_int,
                           P(C.c_double)],
            "cost_gradient": [P(FusionInputsC), vp, C.c_double, P(RobustCfgC), C.c_int,
                              P(C.c_double), vp, P(C.c_double)],
            "stencil_apply": [C.c_int, C.c_int, vp, vp, vp, vp, vp],
            "solve_depth_step": [C.c_int, C.c_int, vp, vp, vp, vp, P(RobustCfgC), vp,
                                 P(C.c_int32)],
            "solve_scale_step": [P(FusionInputsC), vp, C.c_double, P(RobustCfgC),
                                 P(C.c_double)],
            "optimize": [P(FusionInputsC), vp, P(C.c_double), P(C.c_int32), P(RobustCfgC),
                         C.c_int, P(SolverStatsC)],
        }
        self._fn = {}
        for name, args in sig.items():
            f = getattr(lib, prefix + name)
            f.restype = C.c_int
            if name == "make_epipolar_geometry":
                f.argtypes = args
            else:
                f.argtypes = ([vp] if ctx is not None else []) + args
            self._fn[name] = f

    # ---------------------------------------------------------------- utils
    def _call(self, name, *args):
        f = self._fn[name]
        rc = f(self.ctx, *args) if self.ctx is not None else f(*args)
        if rc != 0:
            detail = ""
            if self.ctx is not None and hasattr(self.lib, "dfuse_last_error"):
                self.lib.dfuse_last_error.restype = C.c_char_p
                self.lib.dfuse_last_error.argtypes = [C.c_void_p]
                msg = self.lib.dfuse_last_error(self.ctx)
                detail = msg.decode() if msg else ""
            raise DfuseError(rc, f"{self.prefix}{name}: {detail}")
        return rc

    @staticmethod
    def _inputs(semi: SemiDenseMap, pred: PredictionSet):
        h, w = np.shape(pred.log_depth)
        planes = pred.planes()
        for p in planes:
            if p.shape != (h, w):
                raise DfuseError(ERR_CODE["DimensionMismatch"], "fusion state vs predictions")
        sd, sv, svalid = _f64(semi.depth), _f64(semi.variance), _u8(semi.valid)
        if sd.shape != (h, w) or sv.shape != (h, w) or svalid.shape != (h, w):
            raise DfuseError(ERR_CODE["DimensionMismatch"], "fusion state vs semi-dense map")
        keep = [sd, sv, svalid] + planes
        arr = (C.POINTER(C.c_double) * 6)(*[_dptr(p) for p in planes])
        c = FusionInputsC(w, h, _dptr(sd), _dptr(sv), svalid.ctypes.data_as(C.POINTER(C.c_uint8)),
                          int(semi.inlier_count), 0, arr)
        return c, keep

    @staticmethod
    def _state(state: FusionState, pred: PredictionSet):
        ld = _f64(state.log_depth)
        if ld.shape != np.shape(pred.log_depth):
            raise DfuseError(ERR_CODE["DimensionMismatch"], "fusion state vs predictions")
        return ld

    # ----------------------------------------------------------- geometry
    def make_epipolar_geometry(self, q0, t0, q1, t1, K: CameraIntrinsics) -> EpiGeom:
        """semidense.hpp:101-106; poses as (quaternion w,x,y,z ; translation)."""
        a = [np.ascontiguousarray(v, dtype=np.float64) for v in (q0, t0, q1, t1)]
        g = EpiGeom()
        kc = K.c()
        f = self._fn["make_epipolar_geometry"]
        rc = f(*[_dptr(v) for v in a], C.byref(kc), C.byref(g))
        if rc:
            raise DfuseError(rc, "make_epipolar_geometry")
        return g

    # ----------------------------------------------------------- stereo
    def texture_mask(self, img, threshold: float) -> np.ndarray:
        """semidense.hpp:77-91"""
        img = _f32(img)
        h, w = img.shape
        mask = np.zeros((h, w), np.uint8)
        self._call("texture_mask", img.ctypes.data, w, h, float(threshold), mask.ctypes.data)
        return mask

    def search_depth(self, g: EpiGeom, I0, I1, px, prior=None, has_prior=None,
                     cfg: SearchConfig | None = None):
        """search_depth (semidense.hpp:277-379) over a list of pixels.
        Returns (status[n], obs[n] OBS_DTYPE, best[n], n_steps[n])."""
        cfg = cfg or SearchConfig()
        I0, I1 = _f32(I0), _f32(I1)
        px = _f64(np.reshape(px, (-1, 2)))
        n = px.shape[0]
        pr = None if prior is None else _f64(np.reshape(prior, (-1, 2)))
        hp = None if has_prior is None else _u8(has_prior)
        status = np.zeros(n, np.int32)
        obs = np.zeros(n, OBS_DTYPE)
        best = np.zeros(n, np.int32)
        nst = np.zeros(n, np.int32)
        c = cfg.c()
        self._call("search_depth", C.byref(g), I0.ctypes.data, I1.ctypes.data, n, px.ctypes.data,
                   None if pr is None else pr.ctypes.data, None if hp is None else hp.ctypes.data,
                   C.byref(c), status.ctypes.data, obs.ctypes.data, best.ctypes.data,
                   nst.ctypes.data)
        return status, obs, best, nst

    def update_semidense(self, semi: SemiDenseMap, obs) -> SemiDenseMap:
        """semidense.hpp:393-417 (value semantics: returns a new map)."""
        out = semi.copy()
        out.depth, out.variance, out.valid = _f64(out.depth), _f64(out.variance), _u8(out.valid)
        h, w = out.depth.shape
        obs = np.ascontiguousarray(obs, dtype=OBS_DTYPE)
        cnt = C.c_int32(int(out.inlier_count))
        self._call("update_semidense", w, h, out.depth.ctypes.data, out.variance.ctypes.data,
                   out.valid.ctypes.data, C.byref(cnt), len(obs), obs.ctypes.data)
        out.inlier_count = cnt.value
        return out

    def stereo_update(self, g: EpiGeom, I0, I1, mask, semi: SemiDenseMap,
                      cfg: SearchConfig | None = None, want_obs: bool = True) -> StereoResult:
        """stereo_scan + update_semidense (pipeline.hpp:157-190,207-212)."""
        cfg = cfg or SearchConfig()
        I0, I1, mask = _f32(I0), _f32(I1), _u8(mask)
        out = semi.copy()
        out.depth, out.variance, out.valid = _f64(out.depth), _f64(out.variance), _u8(out.valid)
        h, w = I0.shape
        cnt = C.c_int32(int(out.inlier_count))
        nobs = C.c_int32(0)
        status = np.zeros((h, w), np.int8)
        best = np.zeros((h, w), np.int32)
        nst = np.zeros((h, w), np.int32)
        obs = np.zeros(w * h if want_obs else 0, OBS_DTYPE)
        c = cfg.c()
        self._call("stereo_update", C.byref(g), I0.ctypes.data, I1.ctypes.data, mask.ctypes.data,
                   C.byref(c), out.depth.ctypes.data, out.variance.ctypes.data,
                   out.valid.ctypes.data, C.byref(cnt), C.byref(nobs), status.ctypes.data,
                   best.ctypes.data, nst.ctypes.data, obs.ctypes.data if want_obs else None)
        out.inlier_count = cnt.value
        return StereoResult(out, nobs.value, status, best, nst, obs[:nobs.value].copy())

    # ----------------------------------------------------------- fusion
    def assemble_normal_equations(self, state: FusionState, semi: SemiDenseMap,
                                  pred: PredictionSet, cfg: RobustConfig | None = None,
                                  mode="full") -> NormalEquations:
        """fusion.hpp:171-222"""
        cfg = cfg or RobustConfig()
        inp, keep = self._inputs(semi, pred)
        ld = self._state(state, pred)
        h, w = ld.shape
        eq = NormalEquations(*[np.zeros((h, w)) for _ in range(4)])
        c = cfg.c()
        self._call("assemble_normal_equations", C.byref(inp), ld.ctypes.data, float(state.scale),
                   C.byref(c), _mode(mode), eq.diag.ctypes.data, eq.right.ctypes.data,
                   eq.down.ctypes.data, eq.b.ctypes.data)
        return eq

    def total_cost(self, state, semi, pred, cfg=None, mode="full") -> float:
        """fusion.hpp:225-253"""
        cfg = cfg or RobustConfig()
        inp, keep = self._inputs(semi, pred)
        ld = self._state(state, pred)
        out = C.c_double(0)
        c = cfg.c()
        self._call("total_cost", C.byref(inp), ld.ctypes.data, float(state.scale), C.byref(c),
                   _mode(mode), C.byref(out))
        return out.value

    def cost_gradient(self, state, semi, pred, cfg=None, mode="full"):
        """fusion.hpp:263-308 -> (cost, wrt_log_depth, wrt_ln_scale)"""
        cfg = cfg or RobustConfig()
        inp, keep = self._inputs(semi, pred)
        ld = self._state(state, pred)
        g = np.zeros_like(ld)
        cost, gs = C.c_double(0), C.c_double(0)
        c = cfg.c()
        self._call("cost_gradient", C.byref(inp), ld.ctypes.data, float(state.scale), C.byref(c),
                   _mode(mode), C.byref(cost), g.ctypes.data, C.byref(gs))
        return cost.value, g, gs.value

    def stencil_apply(self, eq: NormalEquations, x) -> np.ndarray:
        """StencilMatrix::apply, fusion.hpp:120-135"""
        d, r, dn = _f64(eq.diag), _f64(eq.right), _f64(eq.down)
        h, w = d.shape
        x = _f64(np.reshape(x, (h, w)))
        y = np.zeros((h, w))
        self._call("stencil_apply", w, h, d.ctypes.data, r.ctypes.data, dn.ctypes.data,
                   x.ctypes.data, y.ctypes.data)
        return y

    def solve_depth_step(self, eq: NormalEquations, cfg: RobustConfig | None = None):
        """fusion.hpp:316-368 -> (delta, pcg_iterations)"""
        cfg = cfg or RobustConfig()
        d, r, dn, b = _f64(eq.diag), _f64(eq.right), _f64(eq.down), _f64(eq.b)
        h, w = d.shape
        x = np.zeros((h, w))
        its = C.c_int32(0)
        c = cfg.c()
        self._call("solve_depth_step", w, h, d.ctypes.data, r.ctypes.data, dn.ctypes.data,
                   b.ctypes.data, C.byref(c), x.ctypes.data, C.byref(its))
        return x, its.value

    def solve_scale_step(self, state, semi, cfg=None) -> float:
        """fusion.hpp:373-391 (the prediction planes are not read)"""
        cfg = cfg or RobustConfig()
        h, w = np.shape(state.log_depth)
        z = np.ones((h, w))
        dummy = PredictionSet(z, z, z, z, z, z)
        inp, keep = self._inputs(semi, dummy)
        ld = _f64(state.log_depth)
        out = C.c_double(0)
        c = cfg.c()
        self._call("solve_scale_step", C.byref(inp), ld.ctypes.data, float(state.scale),
                   C.byref(c), C.byref(out))
        return out.value

    def optimize(self, state: FusionState, semi: SemiDenseMap, pred: PredictionSet,
                 cfg: RobustConfig | None = None, mode="full", with_stats: bool = False):
        """fusion.hpp:402-454 -> new FusionState (and SolverStats)"""
        cfg = cfg or RobustConfig()
        inp, keep = self._inputs(semi, pred)
        ld = self._state(state, pred).copy()
        sc = C.c_double(float(state.scale))
        it = C.c_int32(int(state.iteration))
        stats = SolverStatsC()
        c = cfg.c()
        self._call("optimize", C.byref(inp), ld.ctypes.data, C.byref(sc), C.byref(it),
                   C.byref(c), _mode(mode), C.byref(stats))
        out = FusionState(ld, sc.value, it.value)
        if with_stats:
            return out, SolverStats.from_c(stats)
        return out
