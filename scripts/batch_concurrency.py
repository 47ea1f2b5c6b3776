#!/usr/bin/env python3
"""Experiment: K independent 640x480 keyframes on ONE GPU, each in its own
context (own stream, own solver CTAs), frames enqueued round-robin with
process_frame_async. Prints updates/s per (K, path, ctas) setting.

usage: python scripts/batch_concurrency.py [--frames 40] [--regime defaults]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12244_b200 import api, synth  # noqa: E402
import bench  # noqa: E402


def run(K, path, ctas, n, regime, seqs):
    spec = synth.CONFIGS["C2"]
    cfg = bench.solver_cfg(spec, regime)
    kfs = []
    for k in range(K):
        ctx = api.Context(0)
        ctx.set_solver_path(path)
        if ctas:
            ctx.set_solver_ctas(ctas)
        seq = seqs[k]
        kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
        geoms = [ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
                 for (q, t, _) in seq.frames]
        frames = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).cuda()
                  for (_, _, I1) in seq.frames]
        kfs.append((ctx, kf, geoms, frames))
    nF = len(seqs[0].frames)

    def go(steps):
        for s in range(steps):
            for (ctx, kf, geoms, frames) in kfs:
                j = s % nF
                if j == 0 and s > 0:
                    kf.reset()
                kf.process_frame_async(geoms[j], frames[j].data_ptr(), spec.search, cfg, "full")
        for (_, kf, _, _) in kfs:
            kf.last_result()
        torch.cuda.synchronize()

    go(nF)
    for (_, kf, _, _) in kfs:
        kf.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    go(n)
    dt = time.perf_counter() - t0
    out = K * n / dt
    for (ctx, kf, _, _) in kfs:
        kf.close()
        ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=40)
    ap.add_argument("--regime", default="defaults")
    ap.add_argument("--sets", default="1:auto:0,1:streaming:0,2:streaming:74,3:streaming:49,"
                                      "4:streaming:37")
    a = ap.parse_args()
    spec = synth.CONFIGS["C2"]
    seqs = [synth.make_sequence(spec, 1000 * k) for k in range(8)]
    for s in a.sets.split(","):
        K, path, ctas = s.split(":")
        v = run(int(K), path, int(ctas), a.frames, a.regime, seqs)
        print(f"K={K} path={path} ctas={ctas} regime={a.regime}: {v:.1f} updates/s", flush=True)


if __name__ == "__main__":
    main()
