"""Worker of tests/test_gpu_bands_ipc.py (run under torch.distributed.run,
gloo): two processes on ONE GPU build the two row bands of one keyframe with
dfuse_bkf_create_rank, exchange dfuse_band_peer records (real CUDA-IPC
handles) through all_gather_object, map each other's band allocation with
dfuse_bkf_connect, and store their boundary rows into the neighbour's halo
rows from a kernel (the solver's halo_put stores over the peer mapping).
No cooperative solve runs: two persistent kernels that wait on each other
cannot share one GPU. Exit code 0 = every check passed."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch.distributed as dist

    from paper_2207_12244_b200 import api, shard, synth
    from paper_2207_12244_b200.bands_dist import BandPeer, DistributedBandedKeyframe

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    spec = synth.small_spec(160, 120, frames=1)
    seq = synth.make_sequence(spec, 3, frames=1)
    ctx = api.context(0)
    kf = DistributedBandedKeyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    L = api.lib()
    L.dfuse_bkf_debug_halo_put.argtypes = [C.c_void_p, C.c_int, C.c_double]
    L.dfuse_bkf_debug_halo_get.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    me = BandPeer()
    assert L.dfuse_bkf_peer_info(kf.handle, C.byref(me)) == 0
    y0, y1 = shard.row_bands(spec.height, world)[rank]
    checks = {"band_rows_match_shard": (me.y0, me.y1) == (y0, y1)}
    W = spec.width
    for plane in range(8):
        base = 1e6 * (plane + 1) + 1e5 * (rank + 1)
        assert L.dfuse_bkf_debug_halo_put(kf.handle, plane, base) == 0
        dist.barrier()  # every rank's stores are done (the put call synchronised)
        above, below = np.full(W, np.nan), np.full(W, np.nan)
        assert L.dfuse_bkf_debug_halo_get(kf.handle, plane, above.ctypes.data,
                                          below.ctypes.data) == 0
        if rank > 0:  # row y0 - 1 comes from rank - 1's last row
            exp = 1e6 * (plane + 1) + 1e5 * rank + ((y0 - 1) * W + np.arange(W))
            checks[f"plane{plane}_above"] = bool(np.array_equal(above, exp))
        if rank + 1 < world:  # row y1 comes from rank + 1's first row
            exp = 1e6 * (plane + 1) + 1e5 * (rank + 2) + (y1 * W + np.arange(W))
            checks[f"plane{plane}_below"] = bool(np.array_equal(below, exp))
        dist.barrier()
    print(json.dumps({"rank": rank, "checks": checks}), flush=True)
    kf.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if all(checks.values()) else 1)


if __name__ == "__main__":
    main()
