"""One row band per GPU (SURVEY 8(e), config C4 across GPUs).

Each rank (one process per GPU, torch.distributed initialised) creates its
band with dfuse_bkf_create_rank, the ranks exchange their dfuse_band_peer
records (CUDA-IPC handle of the band allocation + its layout), and
dfuse_bkf_connect maps the peers' allocations: the neighbours' halo rows and
the level-2 all-reduce arrays are then NVLink peer memory, and the ranks'
persistent optimise kernels meet through them (no NCCL on the data path).
process_frame is called by every rank for the same frame; the per-rank
observation / inlier counts are summed here with one small all-reduce.

The exchange and the count reduction are host logic and run under gloo on
CPU in tests/test_dist_cpu.py; the single-GPU form of the same band layout
(all bands in one cooperative launch) is tested on the GPU in
tests/test_gpu_bands.py.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import api
from ._ffi import DfuseError, EpiGeom, FrameResultC, RobustConfig, SearchConfig, _f32, _mode


class BandPeer(C.Structure):  # dfuse_band_peer
    _fields_ = [("handle", C.c_char * 64), ("cpr", C.c_int32), ("y0", C.c_int32),
                ("y1", C.c_int32), ("width", C.c_int32)]


def exchange_peers(record: bytes, world: int) -> list[bytes]:
    """All ranks' peer records in rank order (all_gather_object)."""
    import torch.distributed as dist

    if world == 1:
        return [record]
    out = [None] * world
    dist.all_gather_object(out, record)
    return out


def sum_over_ranks(values, world: int):
    """Integer counts summed over ranks (each rank reports its band's)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return [int(v) for v in values]
    dev = "cpu"
    if dist.get_backend() == "nccl":
        dev = f"cuda:{torch.cuda.current_device()}"
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    return [int(v) for v in t.tolist()]


def _lib():
    L = api.lib()
    if not getattr(L, "_bands_dist", False):
        L.dfuse_bkf_create_rank.argtypes = [C.c_void_p, C.POINTER(api.Intrinsics), C.c_void_p,
                                            C.POINTER(C.c_void_p), C.c_double, C.c_int, C.c_int,
                                            C.POINTER(C.c_void_p)]
        L.dfuse_bkf_peer_info.argtypes = [C.c_void_p, C.POINTER(BandPeer)]
        L.dfuse_bkf_connect.argtypes = [C.c_void_p, C.POINTER(BandPeer)]
        L._bands_dist = True
    return L


class DistributedBandedKeyframe(api.BandedKeyframe):
    """This rank's band of a keyframe split across the process group."""

    def __init__(self, ctx: api.Context, camera, I0, pred, texture_threshold: float = 0.02,
                 world: int | None = None, rank: int | None = None):
        import torch.distributed as dist

        if world is None:
            world = dist.get_world_size() if dist.is_initialized() else 1
            rank = dist.get_rank() if dist.is_initialized() else 0
        L = _lib()
        self.ctx = ctx
        self.world, self.rank, self.bands = world, rank, world
        self.W, self.H = camera.width, camera.height
        self._I0 = _f32(I0)
        self._planes = pred.planes()
        arr = (C.c_void_p * 6)(*[p.ctypes.data for p in self._planes])
        kc = camera.c()
        h = C.c_void_p()
        rc = L.dfuse_bkf_create_rank(ctx.handle, C.byref(kc), self._I0.ctypes.data, arr,
                                     float(texture_threshold), int(world), int(rank), C.byref(h))
        if rc != 0:
            raise DfuseError(rc, L.dfuse_last_error(ctx.handle).decode())
        self.handle = h
        if world > 1:
            me = BandPeer()
            self._check(L.dfuse_bkf_peer_info(self.handle, C.byref(me)), "dfuse_bkf_peer_info")
            recs = exchange_peers(bytes(me), world)
            peers = (BandPeer * world)(*[BandPeer.from_buffer_copy(r) for r in recs])
            self._check(L.dfuse_bkf_connect(self.handle, peers), "dfuse_bkf_connect")

    def process_frame(self, g: EpiGeom, I1, search: SearchConfig | None = None,
                      robust: RobustConfig | None = None, mode="full", device_ptr=None):
        res = super().process_frame(g, I1, search, robust, mode, device_ptr)
        res.observations, res.inlier_count = sum_over_ranks(
            [res.observations, res.inlier_count], self.world)
        return res
