"""Python mirror of the reference API, bound to the CUDA library.

``cuda()`` returns a :class:`Bindings` over ``libdfuse_cuda.so`` (the
``dfuse_*`` C-ABI of include/dfuse_cuda.h) with methods named like the
reference's functions: texture_mask, search_depth, update_semidense,
stereo_update (stereo_scan + update_semidense), assemble_normal_equations,
total_cost, cost_gradient, stencil_apply, solve_depth_step,
solve_scale_step, optimize. :class:`Keyframe` is the device-resident
session (make_keyframe + process_frame, pipeline.hpp:125-228).

There is no CPU fallback: if the library is missing or no sm_100 device is
visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._ffi import (Bindings, DfuseError, EpiGeom, FrameResultC, Intrinsics, PredictionSet,
                   RobustConfig, SearchConfig, SemiDenseMap, SolverStats, FusionState, _f32,
                   _f64, _mode)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFUSE_LIB") or os.path.join(HERE, "libdfuse_cuda.so")

_lib = None
_default = {}


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                               f"g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.dfuse_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.dfuse_ctx_create.restype = C.c_int
        L.dfuse_ctx_destroy.argtypes = [C.c_void_p]
        L.dfuse_last_error.argtypes = [C.c_void_p]
        L.dfuse_last_error.restype = C.c_char_p
        L.dfuse_ctx_set_solver_ctas.argtypes = [C.c_void_p, C.c_int]
        L.dfuse_ctx_launch_count.argtypes = [C.c_void_p]
        L.dfuse_ctx_launch_count.restype = C.c_int64
        L.dfuse_err_name.restype = C.c_char_p
        L.dfuse_ctx_stream.argtypes = [C.c_void_p]
        L.dfuse_ctx_stream.restype = C.c_void_p
        L.dfuse_kf_create.argtypes = [C.c_void_p, C.POINTER(Intrinsics), C.c_void_p,
                                      C.POINTER(C.c_void_p), C.c_double, C.POINTER(C.c_void_p)]
        L.dfuse_kf_destroy.argtypes = [C.c_void_p]
        L.dfuse_kf_reset.argtypes = [C.c_void_p]
        for name in ("dfuse_kf_process_frame", "dfuse_kf_process_frame_dev"):
            f = getattr(L, name)
            f.argtypes = [C.c_void_p, C.POINTER(EpiGeom), C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_int, C.POINTER(FrameResultC)]
        L.dfuse_kf_download.argtypes = [C.c_void_p] + [C.c_void_p] * 8
        L.dfuse_kf_process_frame_async.argtypes = [C.c_void_p, C.POINTER(EpiGeom), C.c_void_p,
                                                   C.c_void_p, C.c_void_p, C.c_int]
        L.dfuse_kf_last_result.argtypes = [C.c_void_p, C.POINTER(FrameResultC)]
        L.dfuse_kf_create_dfpred.argtypes = [C.c_void_p, C.POINTER(Intrinsics), C.c_void_p,
                                             C.c_char_p, C.c_size_t, C.c_double,
                                             C.POINTER(C.c_void_p)]
        L.dfuse_dfpred_header.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t,
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                          C.POINTER(C.c_double)]
        L.dfuse_kf_median_depth.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.dfuse_bkf_create.argtypes = [C.c_void_p, C.POINTER(Intrinsics), C.c_void_p,
                                       C.POINTER(C.c_void_p), C.c_double, C.c_int,
                                       C.POINTER(C.c_void_p)]
        L.dfuse_bkf_destroy.argtypes = [C.c_void_p]
        L.dfuse_bkf_reset.argtypes = [C.c_void_p]
        for name in ("dfuse_bkf_process_frame", "dfuse_bkf_process_frame_dev"):
            f = getattr(L, name)
            f.argtypes = [C.c_void_p, C.POINTER(EpiGeom), C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_int, C.POINTER(FrameResultC)]
        L.dfuse_bkf_download.argtypes = [C.c_void_p] + [C.c_void_p] * 8
        L.dfuse_score_depth.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 5
        L.dfuse_kf_score.argtypes = [C.c_void_p] + [C.c_void_p] * 3
        L.dfuse_kf_export_depth_u16.argtypes = [C.c_void_p, C.c_double, C.c_void_p]
        _lib = L
    return _lib


class Context:
    """One device + one stream (dfuse_ctx)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        rc = L.dfuse_ctx_create(int(device), C.byref(h))
        if rc != 0:
            raise DfuseError(rc, f"dfuse_ctx_create(device={device}): no usable sm_100 device")
        self.handle = h
        self.device = device
        self.api = Bindings(L, "dfuse_", h, "cuda")

    def set_solver_ctas(self, n: int) -> None:
        lib().dfuse_ctx_set_solver_ctas(self.handle, int(n))

    SOLVER_PATHS = {"auto": 0, "resident": 0, "streaming": 1, "resident2r": 2, "resident1r": 3}

    def set_solver_path(self, path) -> None:
        """"auto"/"resident" (or False): SM-resident pipelined PCG (one
        all-reduce per iteration, overlapped with the SpMV) when the raster
        fits on chip (default); "streaming" (or True): always the streaming
        PCG; "resident1r": SM-resident Chronopoulos-Gear PCG (one exposed
        all-reduce); "resident2r": SM-resident with the reference's direct
        p.q (two all-reduces per iteration)."""
        if isinstance(path, bool):
            path = "streaming" if path else "auto"
        L = lib()
        L.dfuse_ctx_set_solver_path.argtypes = [C.c_void_p, C.c_int]
        rc = L.dfuse_ctx_set_solver_path(self.handle, self.SOLVER_PATHS[path])
        if rc:
            raise DfuseError(rc, "dfuse_ctx_set_solver_path")

    def stream_handle(self) -> int:
        """cudaStream_t the library launches on (wrap with torch.cuda.ExternalStream)."""
        return int(lib().dfuse_ctx_stream(self.handle))

    def launch_count(self) -> int:
        return int(lib().dfuse_ctx_launch_count(self.handle))

    def set_stereo_texture(self, on: bool) -> None:
        """Epipolar scan reads the tracked frame through a texture gather
        (default) or plain loads; the results are bit-identical."""
        L = lib()
        L.dfuse_ctx_set_stereo_texture.argtypes = [C.c_void_p, C.c_int]
        rc = L.dfuse_ctx_set_stereo_texture(self.handle, 1 if on else 0)
        if rc:
            raise DfuseError(rc, "dfuse_ctx_set_stereo_texture")

    def texture_launches(self) -> int:
        L = lib()
        L.dfuse_ctx_texture_launches.argtypes = [C.c_void_p]
        L.dfuse_ctx_texture_launches.restype = C.c_int64
        return int(L.dfuse_ctx_texture_launches(self.handle))

    def close(self) -> None:
        if self.handle:
            lib().dfuse_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def cuda(device: int = 0) -> Bindings:
    """The reference-shaped API on the GPU (default context of `device`)."""
    return context(device).api


class KeyframeScoreC(C.Structure):  # dfuse_keyframe_score
    _fields_ = [("pct_within_10", C.c_double), ("n_evaluated", C.c_int32),
                ("median_abs_rel", C.c_double)]


def score_depth(ctx: "Context", est, gt_metres, gt_valid, est_valid=None) -> KeyframeScoreC:
    """pct_within_10 + median_abs_rel (eval.hpp:34-68) on the device."""
    est = _f64(est)
    gt = _f64(gt_metres)
    gv = np.ascontiguousarray(gt_valid, np.uint8)
    ev = None if est_valid is None else np.ascontiguousarray(est_valid, np.uint8)
    h, w = est.shape
    out = KeyframeScoreC()
    L = lib()
    rc = L.dfuse_score_depth(ctx.handle, w, h, est.ctypes.data,
                             None if ev is None else ev.ctypes.data, gt.ctypes.data,
                             gv.ctypes.data, C.byref(out))
    if rc != 0:
        raise DfuseError(rc, L.dfuse_last_error(ctx.handle).decode())
    return out


def dfpred_header(data: bytes):
    """load_predictions' header checks (predictions.hpp:72-95), host code in
    the library (no device needed) -> (width, height, source_focal)."""
    L = lib()
    w, h, f = C.c_int32(0), C.c_int32(0), C.c_double(0.0)
    rc = L.dfuse_dfpred_header(None, data, len(data), C.byref(w), C.byref(h), C.byref(f))
    if rc != 0:
        raise DfuseError(rc, "dfuse_dfpred_header")
    return w.value, h.value, f.value


class Keyframe:
    """Device-resident keyframe (dfuse_keyframe): make_keyframe on creation,
    process_frame per tracked frame, download() for the state."""

    def __init__(self, ctx: Context, camera, I0, pred: PredictionSet | None,
                 texture_threshold: float = 0.02, dfpred: bytes | None = None):
        """`pred`: the prediction planes (already focal-adjusted), or
        `dfpred`: the bytes of a DFPRED file (make_keyframe's
        load_predictions + focal_adjust to camera.fx, on the device)."""
        L = lib()
        self.ctx = ctx
        self._inflight = []  # host buffers of enqueued host-async frames
        self.W, self.H = camera.width, camera.height
        self._I0 = _f32(I0)
        kc = camera.c()
        h = C.c_void_p()
        if dfpred is not None:
            rc = L.dfuse_kf_create_dfpred(ctx.handle, C.byref(kc), self._I0.ctypes.data,
                                          bytes(dfpred), len(dfpred), float(texture_threshold),
                                          C.byref(h))
        else:
            self._planes = pred.planes()
            arr = (C.c_void_p * 6)(*[p.ctypes.data for p in self._planes])
            rc = L.dfuse_kf_create(ctx.handle, C.byref(kc), self._I0.ctypes.data, arr,
                                   float(texture_threshold), C.byref(h))
        if rc != 0:
            raise DfuseError(rc, L.dfuse_last_error(ctx.handle).decode())
        self.handle = h

    def score(self, gt_metres, gt_valid) -> KeyframeScoreC:
        """finalize_keyframe's score of the fused state (pipeline.hpp:232-247)"""
        gt = _f64(gt_metres)
        gv = np.ascontiguousarray(gt_valid, np.uint8)
        out = KeyframeScoreC()
        self._check(lib().dfuse_kf_score(self.handle, gt.ctypes.data, gv.ctypes.data,
                                         C.byref(out)), "dfuse_kf_score")
        return out

    def export_depth_u16(self, depth_scale: float = 5000.0) -> np.ndarray:
        """export_depth_image's 16-bit raster (eval.hpp:221-226)"""
        out = np.zeros((self.H, self.W), np.uint16)
        self._check(lib().dfuse_kf_export_depth_u16(self.handle, float(depth_scale),
                                                    out.ctypes.data), "dfuse_kf_export_depth_u16")
        return out

    def median_depth(self) -> float:
        """median_predicted_depth (pipeline.hpp:94-99), cached on the device"""
        v = C.c_double(0.0)
        self._check(lib().dfuse_kf_median_depth(self.handle, C.byref(v)), "dfuse_kf_median_depth")
        return v.value

    def _check(self, rc, what):
        if rc != 0:
            raise DfuseError(rc, f"{what}: " + lib().dfuse_last_error(self.ctx.handle).decode())

    def reset(self):
        self._check(lib().dfuse_kf_reset(self.handle), "dfuse_kf_reset")

    def process_frame(self, g: EpiGeom, I1, search: SearchConfig | None = None,
                      robust: RobustConfig | None = None, mode="full", device_ptr=None):
        """One tracked frame: stereo scan + semi-dense update + optimize.
        `I1` is a host image, or pass `device_ptr` (int) of a float32 device
        image. Returns the dfuse_frame_result struct."""
        search = search or SearchConfig()
        robust = robust or RobustConfig()
        sc, rc_ = search.c(), robust.c()
        res = FrameResultC()
        L = lib()
        if device_ptr is not None:
            rc = L.dfuse_kf_process_frame_dev(self.handle, C.byref(g), C.c_void_p(device_ptr),
                                              C.byref(sc), C.byref(rc_), _mode(mode),
                                              C.byref(res))
        else:
            img = _f32(I1)
            rc = L.dfuse_kf_process_frame(self.handle, C.byref(g), img.ctypes.data, C.byref(sc),
                                          C.byref(rc_), _mode(mode), C.byref(res))
        self._check(rc, "dfuse_kf_process_frame")
        return res

    def process_frame_async(self, g: EpiGeom, device_ptr: int,
                            search: SearchConfig | None = None,
                            robust: RobustConfig | None = None, mode="full") -> None:
        """process_frame for a device image, enqueued without waiting
        (dfuse_kf_process_frame_async); last_result() waits and returns the
        last enqueued frame's result."""
        search = search or SearchConfig()
        robust = robust or RobustConfig()
        self._sc, self._rc = search.c(), robust.c()  # alive until the call returns
        self._check(lib().dfuse_kf_process_frame_async(
            self.handle, C.byref(g), C.c_void_p(device_ptr), C.byref(self._sc),
            C.byref(self._rc), _mode(mode)), "dfuse_kf_process_frame_async")

    def process_frame_host_async(self, g: EpiGeom, I1_host: np.ndarray,
                                 search: SearchConfig | None = None,
                                 robust: RobustConfig | None = None, mode="full",
                                 log_depth_out: np.ndarray | None = None) -> None:
        """process_frame for a HOST image, pipelined
        (dfuse_kf_process_frame_host_async): the copy-in overlaps the previous
        frame's compute, and the fused log-depth lands in log_depth_out
        (float64 [H, W]) while the next frame computes. Pass pinned arrays
        (torch.empty(..).pin_memory().numpy()) and keep them untouched until
        last_result()."""
        search = search or SearchConfig()
        robust = robust or RobustConfig()
        P = self.W * self.H
        if not (isinstance(I1_host, np.ndarray) and I1_host.dtype == np.float32
                and I1_host.flags.c_contiguous and I1_host.size == P):
            raise DfuseError(27, f"process_frame_host_async: I1_host must be a C-contiguous "
                                 f"float32 array of {P} pixels")
        out = None
        if log_depth_out is not None:
            if not (isinstance(log_depth_out, np.ndarray) and log_depth_out.dtype == np.float64
                    and log_depth_out.flags.c_contiguous and log_depth_out.size == P
                    and log_depth_out.flags.writeable):
                raise DfuseError(27, f"process_frame_host_async: log_depth_out must be a "
                                     f"writeable C-contiguous float64 array of {P} pixels")
            out = C.c_void_p(log_depth_out.ctypes.data)
        self._sc, self._rc = search.c(), robust.c()
        # the copies run asynchronously: keep both buffers alive until
        # last_result() / reset() has waited for them
        self._inflight.append((I1_host, log_depth_out))
        L = lib()
        L.dfuse_kf_process_frame_host_async.argtypes = [
            C.c_void_p, C.POINTER(EpiGeom), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
            C.c_void_p]
        self._check(L.dfuse_kf_process_frame_host_async(
            self.handle, C.byref(g), C.c_void_p(I1_host.ctypes.data), C.byref(self._sc),
            C.byref(self._rc), _mode(mode), out), "dfuse_kf_process_frame_host_async")

    def last_result(self):
        res = FrameResultC()
        self._check(lib().dfuse_kf_last_result(self.handle, C.byref(res)), "dfuse_kf_last_result")
        self._inflight = []
        return res

    def download(self):
        """-> (FusionState, SemiDenseMap, mask)"""
        h, w = self.H, self.W
        ld = np.zeros((h, w))
        sd, sv = np.zeros((h, w)), np.zeros((h, w))
        valid = np.zeros((h, w), np.uint8)
        mask = np.zeros((h, w), np.uint8)
        scale = C.c_double(0)
        it = C.c_int32(0)
        cnt = C.c_int32(0)
        self._check(lib().dfuse_kf_download(self.handle, ld.ctypes.data, C.addressof(scale),
                                            C.addressof(it), sd.ctypes.data, sv.ctypes.data,
                                            valid.ctypes.data, C.addressof(cnt),
                                            mask.ctypes.data), "dfuse_kf_download")
        return (FusionState(ld, scale.value, it.value), SemiDenseMap(sd, sv, valid, cnt.value),
                mask)

    def close(self):
        if getattr(self, "handle", None):
            lib().dfuse_kf_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BandedKeyframe(Keyframe):
    """A keyframe split into row bands (dfuse_banded_keyframe):
    the same make_keyframe / process_frame / download as Keyframe, with the
    per-pixel state in per-band allocations that exchange halo rows and
    all-reduce through two levels, as across GPUs."""

    _P = "dfuse_bkf_"

    def __init__(self, ctx: Context, camera, I0, pred: PredictionSet, bands: int,
                 texture_threshold: float = 0.02):
        L = lib()
        self.ctx = ctx
        self.bands = bands
        self.W, self.H = camera.width, camera.height
        self._I0 = _f32(I0)
        self._planes = pred.planes()
        arr = (C.c_void_p * 6)(*[p.ctypes.data for p in self._planes])
        kc = camera.c()
        h = C.c_void_p()
        rc = L.dfuse_bkf_create(ctx.handle, C.byref(kc), self._I0.ctypes.data, arr,
                                float(texture_threshold), int(bands), C.byref(h))
        if rc != 0:
            raise DfuseError(rc, L.dfuse_last_error(ctx.handle).decode())
        self.handle = h

    def reset(self):
        self._check(lib().dfuse_bkf_reset(self.handle), "dfuse_bkf_reset")

    def process_frame_async(self, *a, **k):
        raise NotImplementedError("the row-band keyframe has no asynchronous frame call")

    def process_frame_host_async(self, *a, **k):
        raise NotImplementedError("the row-band keyframe has no pipelined host-frame call")

    def last_result(self):
        raise NotImplementedError("the row-band keyframe has no asynchronous frame call")

    def process_frame(self, g: EpiGeom, I1, search: SearchConfig | None = None,
                      robust: RobustConfig | None = None, mode="full", device_ptr=None):
        search = search or SearchConfig()
        robust = robust or RobustConfig()
        sc, rc_ = search.c(), robust.c()
        res = FrameResultC()
        L = lib()
        if device_ptr is not None:
            rc = L.dfuse_bkf_process_frame_dev(self.handle, C.byref(g), C.c_void_p(device_ptr),
                                               C.byref(sc), C.byref(rc_), _mode(mode),
                                               C.byref(res))
        else:
            img = _f32(I1)
            rc = L.dfuse_bkf_process_frame(self.handle, C.byref(g), img.ctypes.data,
                                           C.byref(sc), C.byref(rc_), _mode(mode), C.byref(res))
        self._check(rc, "dfuse_bkf_process_frame")
        return res

    def download(self):
        h, w = self.H, self.W
        ld = np.zeros((h, w))
        sd, sv = np.zeros((h, w)), np.zeros((h, w))
        valid = np.zeros((h, w), np.uint8)
        mask = np.zeros((h, w), np.uint8)
        scale = C.c_double(0)
        it = C.c_int32(0)
        cnt = C.c_int32(0)
        self._check(lib().dfuse_bkf_download(self.handle, ld.ctypes.data, C.addressof(scale),
                                             C.addressof(it), sd.ctypes.data, sv.ctypes.data,
                                             valid.ctypes.data, C.addressof(cnt),
                                             mask.ctypes.data), "dfuse_bkf_download")
        return (FusionState(ld, scale.value, it.value), SemiDenseMap(sd, sv, valid, cnt.value),
                mask)

    def close(self):
        if getattr(self, "handle", None):
            lib().dfuse_bkf_destroy(self.handle)
            self.handle = None
