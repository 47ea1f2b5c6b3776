"""Where the e2e (host buffers) time goes vs device-resident frames: C2,
fixed-effort regime, wall clock over N frames of (a) device frames async,
(b) host frames pipelined without the log-depth copy-out, (c) with it."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12244_b200 import api, synth  # noqa: E402
import bench  # noqa: E402

spec = synth.CONFIGS["C2"]
seq = synth.make_sequence(spec, 1000)
cfg = bench.solver_cfg(spec, sys.argv[1] if len(sys.argv) > 1 else "fixed")
ctx = api.Context(0)
kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
geoms = [ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
         for (q, t, _) in seq.frames]
dev = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).cuda() for (_, _, I1) in seq.frames]
pin = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).pin_memory().numpy()
       for (_, _, I1) in seq.frames]
outs = [torch.empty((spec.height, spec.width), dtype=torch.float64).pin_memory().numpy()
        for _ in range(2)]
nF = len(seq.frames)
N = 200


def run(mode):
    kf.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(N):
        k = s % nF
        if k == 0 and s > 0:
            kf.reset()
        if mode == "dev":
            kf.process_frame_async(geoms[k], dev[k].data_ptr(), spec.search, cfg, "full")
        else:
            kf.process_frame_host_async(geoms[k], pin[k], spec.search, cfg, "full",
                                        log_depth_out=outs[s & 1] if mode == "host+out" else None)
    t1 = time.perf_counter()
    kf.last_result()
    t2 = time.perf_counter()
    print(f"{mode:9s}: {N / (t2 - t0):8.1f} updates/s  (host issue {1e6 * (t1 - t0) / N:.1f} us/frame)",
          flush=True)


def run_events(flush_mb=0):
    """device frames with events around each frame (as bench.py's timed
    region; a fill of flush_mb MiB between frames, outside the events):
    event sum vs wall clock"""
    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    fl = torch.empty(max(1, flush_mb) * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    kf.reset()
    torch.cuda.synchronize()
    ev = []
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        for s in range(N):
            k = s % nF
            if k == 0 and s > 0:
                kf.reset()
            if flush_mb:
                fl.fill_(float(s))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            kf.process_frame_async(geoms[k], dev[k].data_ptr(), spec.search, cfg, "full")
            e1.record(stream)
            ev.append((e0, e1))
    kf.last_result()
    t2 = time.perf_counter()
    inside = sum(a.elapsed_time(b) for a, b in ev)
    span = ev[0][0].elapsed_time(ev[-1][1])
    print(f"flush {flush_mb:4d} MiB events: inside {1e3 * inside / N:.1f} us/frame, first-to-last {1e3 * span / N:.1f} "
          f"us/frame, wall {1e6 * (t2 - t0) / N:.1f} us/frame", flush=True)


for mb in [0, 8, 64, 160, 512, 0]:
    run_events(mb)
samp = bench.ClockSampler(0)
samp.start()
for m in ["dev", "host", "host+out", "dev", "host+out"]:
    run(m)
print("clocks", samp.stop())
