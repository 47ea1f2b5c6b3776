#!/usr/bin/env python3
"""Benchmark: fused keyframe updates/s at 640x480 (BASELINE.json metric).

One step = one fused keyframe update on a tracked frame (pipeline.hpp:205-226):
stereo_scan + update_semidense + optimize, on the device-resident keyframe
session (dfuse_kf_process_frame*). Workload = BASELINE config C2 (640x480,
fx=fy=525, 10 tracked frames per keyframe, reference solver defaults: 10 GN
iterations, PCG tol 1e-6 / max 200), seeded synthetic scene (the paper's
datasets are not available; see paper_2207_12244_b200/synth.py). After the
10th tracked frame the keyframe is reset on the device (inside the timed
step) and the sequence repeats.

  value   device-timed (CUDA events on the library's stream), input frames
          already resident in HBM, L2 flushed before every step (a 512 MiB
          write outside the timed events)
  e2e     the same metric through the C-ABI with HOST buffers
          (dfuse_kf_process_frame_host_async): every step copies its tracked
          frame in from pinned host memory and its fused log-depth map out to
          pinned host memory (copy stream, overlapped with the neighbouring
          frames' compute); wall clock from the first call to last_result()
  roofline  k_fusion (the dominant kernel): algorithmic bytes of the executed
          sweeps (SURVEY.md 8(d) byte model) / its device time, vs the measured
          HBM copy bandwidth in MEASURED_PEAKS.json
  cpu_baseline  the reference's own code (oracle/_ref) on the host cores

--impl reference times the reference's CPU implementation (oracle/_ref,
OpenMP on all host threads) on the same workload and prints the same line.
Multi-GPU (torchrun): every rank runs its own independent keyframe
(weak scaling, no data-path collective); value = total updates / max time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused keyframe updates/sec (Mpix/s) at 640x480; solver HBM GB/s vs peak"
UNIT = "updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--regime", default="defaults", choices=["defaults", "fixed"],
                    help="defaults: reference solver settings; fixed: cg_tol=0, 5 PCG/GN")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--solver-ctas", type=int, default=0,
                    help="persistent CTAs of the fusion solver (0 = the library's choice)")
    ap.add_argument("--bands", type=int, default=0,
                    help="row bands of one keyframe (C4 form); under torchrun with --config C4 "
                         "each rank computes one band (strong scaling)")
    ap.add_argument("--frames", type=int, default=0,
                    help="tracked frames to generate (default: the config's)")
    ap.add_argument("--solver-path", default="auto",
                    choices=["auto", "resident", "resident1r", "resident2r", "streaming"],
                    help="PCG data path (dfuse_ctx_set_solver_path); auto is the product default")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel`
    from the committed ncu capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return int(json.load(f)[kernel]["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


# FP64 issue rate of this GPU, measured (scripts/micro/fp64_rate.cu): 58 DFMA
# lane-operations per SM per clock, x 148 SMs x 1.965 GHz
FP64_PEAK_GOPS = round(58 * 148 * 1.965, 1)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if len(s) >= 8 and s[0].replace('.', '').isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 8 and s[1].replace('.', '').isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) < 8:
                continue
            for k, n in enumerate(names):
                if s[4 + k].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def solver_cfg(spec, regime):
    from paper_2207_12244_b200._ffi import RobustConfig

    if regime == "fixed":
        return RobustConfig(gn_iterations=spec.gn_iterations, cg_tol=0.0, cg_max_iters=5)
    return RobustConfig(gn_iterations=spec.gn_iterations)


def fusion_bytes_per_px(stats) -> float:
    """SURVEY.md 8(d) byte model over the EXECUTED sweeps of one optimize()."""
    total = 0.0
    for k in range(min(stats.gn_done, 512)):
        s_step, d_step, n_cg = stats.scale_step[k], stats.depth_step[k], stats.pcg_iters[k]
        if s_step >= 0:  # scale block ran: 3 rounds + c0 + trials
            trials = 6 if s_step == 0 else int(round(-np.log2(s_step))) + 1
            total += 3 * 25 + 49 + 49 * trials
        if n_cg >= 0:  # depth block: assemble + c0 + PCG init + PCG + trials + accept
            trials = 6 if d_step == 0 else int(round(-np.log2(d_step))) + 1
            total += 81 + 49 + 32 + 112 * n_cg + 57 * trials + (8 if d_step > 0 else 0)
    return total


# --------------------------------------------------------------------------
def run_reference(args, spec, seq):
    """The reference's CPU implementation (oracle/_ref, OpenMP) on the same
    workload; each step = one process_frame on a tracked frame."""
    import ctypes as C

    import oracle
    from paper_2207_12244_b200._ffi import FusionInputsC, SemiDenseMap, _dptr

    ref = oracle.reference()
    L = ref.lib
    L.ref_process_frame.restype = C.c_int
    threads = L.ref_omp_max_threads()
    cfg = solver_cfg(spec, args.regime)
    mask = ref.texture_mask(seq.I0, 0.02)
    geoms = [ref.make_epipolar_geometry(np.array([1.0, 0, 0, 0]), np.zeros(3), q, t,
                                        spec.camera()) for (q, t, _) in seq.frames]
    planes = seq.pred.planes()
    P = spec.width * spec.height

    def fresh():
        semi = SemiDenseMap.empty(spec.width, spec.height)
        return semi, seq.pred.log_depth.copy(), C.c_double(1.0), C.c_int32(0), C.c_int32(0)

    state = list(fresh())
    frame_idx = [0]

    def step():
        semi, ld, scale, it, cnt = state
        if frame_idx[0] % len(seq.frames) == 0 and frame_idx[0] > 0:
            state[:] = fresh()
            semi, ld, scale, it, cnt = state
        k = frame_idx[0] % len(seq.frames)
        frame_idx[0] += 1
        inp = FusionInputsC(spec.width, spec.height, None, None, None, 0, 0,
                            (C.POINTER(C.c_double) * 6)(*[_dptr(p) for p in planes]))
        nobs = C.c_int32(0)
        sms, oms = C.c_double(0), C.c_double(0)
        sc, rc_ = spec.search.c(), cfg.c()
        I1 = np.ascontiguousarray(seq.frames[k][2], np.float32)
        rc = L.ref_process_frame(C.byref(geoms[k]), C.c_void_p(seq.I0.ctypes.data),
                                 C.c_void_p(I1.ctypes.data), C.c_void_p(mask.ctypes.data),
                                 C.byref(sc), C.byref(inp), C.c_void_p(semi.depth.ctypes.data),
                                 C.c_void_p(semi.variance.ctypes.data),
                                 C.c_void_p(semi.valid.ctypes.data), C.byref(cnt),
                                 C.c_void_p(ld.ctypes.data), C.byref(scale), C.byref(it),
                                 C.byref(rc_), 0, C.byref(nobs), C.byref(sms), C.byref(oms))
        return rc

    for _ in range(min(args.warmup, 3)):
        step()
    # bounded sample: the K timed steps, or as many as fit in the budget
    budget = getattr(args, "budget_s", 120.0)
    t0 = time.perf_counter()
    done = 0
    while done < args.steps:
        step()
        done += 1
        if time.perf_counter() - t0 > budget:
            break
    dt = time.perf_counter() - t0
    args.steps_done = done
    value = done / dt
    return value, dt * 1e3 / done, threads


def cpu_baseline(spec, seq, regime, budget_s=20.0):
    """Bounded sample of the same workload on the reference build."""
    class A:
        pass

    a = A()
    a.regime = regime
    a.warmup = 0
    # one update first to size the sample
    a.steps = 1
    v1, ms1, threads = run_reference(a, spec, seq)
    n = max(1, min(len(seq.frames) - 1, int(budget_s * 1e3 / max(ms1, 1.0))))
    a.steps = n
    v, ms, threads = run_reference(a, spec, seq)
    return {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n} tracked-frame updates of {spec.name} (first frames of the seeded "
                      f"sequence; reference headers + OpenMP, {threads} threads)"}


# --------------------------------------------------------------------------
def main():
    args = parse()
    ws, rank, local = dist_env()
    from paper_2207_12244_b200 import synth

    spec = synth.CONFIGS[args.config]
    if args.impl == "reference":
        if rank != 0:
            return
        seq = synth.make_sequence(spec, args.seed)
        value, ms, threads = run_reference(args, spec, seq)
        line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded Perlin-textured planes, BASELINE C2)",
                "impl": "reference",
                "config": {"workload": f"{spec.name}: {spec.width}x{spec.height}, "
                                       f"{spec.frames} tracked frames/keyframe, solver "
                                       f"{args.regime}", "regime": args.regime},
                "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                                 "kind": "reference",
                                 "sample": f"{args.steps_done} of the {args.steps} requested "
                                           f"updates (120 s budget) after "
                                           f"{min(args.warmup, 3)} warm-up"},
                "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    if ws > 1:
        import torch.distributed as dist

        # one rank per GPU; with fewer GPUs than ranks (validating the
        # multi-rank path of independent keyframe streams on one GPU) the
        # ranks share devices -- they never wait on one another
        shared = torch.cuda.device_count() < ws
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if shared:  # NCCL needs one device per rank
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local
    red_dev = (f"cuda:{device}" if ws > 1 and torch.distributed.get_backend() == "nccl"
               else "cpu")  # device of the max-over-ranks reductions
    from paper_2207_12244_b200 import api
    from paper_2207_12244_b200._ffi import SemiDenseMap

    # C4 under torchrun: ONE keyframe split into row bands across the ranks
    # (strong scaling); otherwise every rank runs its own keyframe stream
    # (C2/C3 form, weak scaling)
    split = args.config == "C4" and ws > 1
    seq = synth.make_sequence(spec, args.seed + (0 if split else 1000 * rank),
                              frames=args.frames or None)
    cfg = solver_cfg(spec, args.regime)
    ctx = api.context(device)
    ctx.set_solver_path(args.solver_path)
    if args.solver_ctas:
        ctx.set_solver_ctas(args.solver_ctas)
    if split:
        from paper_2207_12244_b200.bands_dist import DistributedBandedKeyframe

        kf = DistributedBandedKeyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    elif args.bands > 0:
        kf = api.BandedKeyframe(ctx, spec.camera(), seq.I0, seq.pred, args.bands, 0.02)
    else:
        kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
    download = (api.lib().dfuse_bkf_download if isinstance(kf, api.BandedKeyframe)
                else api.lib().dfuse_kf_download)
    jobs = 1 if split else ws  # keyframe updates per step, whole job
    geoms = [ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
             for (q, t, _) in seq.frames]
    dev_frames = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).cuda(device)
                  for (_, _, I1) in seq.frames]
    torch.cuda.synchronize(device)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=torch.device("cuda", device))
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")
    nF = len(seq.frames)
    P = spec.width * spec.height

    counter = [0]

    def step(dev=True, host_images=None):
        k = counter[0] % nF
        if k == 0 and counter[0] > 0:
            kf.reset()
        counter[0] += 1
        if dev:
            return kf.process_frame(geoms[k], None, spec.search, cfg, "full",
                                    device_ptr=dev_frames[k].data_ptr())
        return kf.process_frame(geoms[k], host_images[k], spec.search, cfg, "full")

    for _ in range(max(3, args.warmup)):
        step()
    # ---------------- per-frame statistics: one synchronous pass over the
    # keyframe's frames (the computation is deterministic, so the timed pass
    # below repeats exactly these frames)
    kf.reset()
    counter[0] = 0
    stats_pass = [step() for _ in range(nF)]
    # ---------------- device-timed region: frames enqueued back to back
    # (process_frame_async where the keyframe has it; the row-band form is
    # synchronous), per-step CUDA events on the library's stream
    use_async = hasattr(kf, "process_frame_async") and not isinstance(kf, api.BandedKeyframe)

    def step_async():
        k = counter[0] % nF
        if k == 0 and counter[0] > 0:
            kf.reset()
        counter[0] += 1
        kf.process_frame_async(geoms[k], dev_frames[k].data_ptr(), spec.search, cfg, "full")

    kf.reset()
    counter[0] = 0
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(device)
    launches0 = ctx.launch_count()
    sampler = ClockSampler(device)
    sampler.start()
    events = []
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush.fill_(float(counter[0]))  # evict L2 (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if use_async:
                step_async()
            else:
                step()
            e1.record(stream)
            events.append((e0, e1))
        if use_async:
            kf.last_result()
    torch.cuda.synchronize(device)
    clocks = sampler.stop()
    launches = ctx.launch_count() - launches0
    step_ms = [e0.elapsed_time(e1) for e0, e1 in events]
    fusion_ms = [r.optimise_ms for r in stats_pass]
    stereo_ms = [r.stereo_ms for r in stats_pass]
    fusion_bytes = [fusion_bytes_per_px(r.stats) * P for r in stats_pass]
    pcg = [r.stats.pcg_total for r in stats_pass]
    steps_ep = [r.epipolar_steps for r in stats_pass]
    obs = [r.observations for r in stats_pass]
    total_ms = float(np.sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=red_dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = jobs * args.steps / (total_ms / 1e3)

    # ---------------- end-to-end through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        import ctypes as C

        # inputs and the result in pinned host memory (DMA copies, no staging)
        pinned = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).pin_memory()
                  for (_, _, I1) in seq.frames]
        host_imgs = [p.numpy() for p in pinned]
        out_pinned = torch.empty((spec.height, spec.width), dtype=torch.float64).pin_memory()
        out_ld = out_pinned.numpy()
        kf.reset()
        counter[0] = 0
        # the pipelined host-buffer call where the keyframe has it: frame n's
        # copy-in overlaps frame n-1's compute, its log-depth is copied out
        # while frame n+1 computes (two pinned result slots, alternating)
        host_async = hasattr(kf, "process_frame_host_async") and not isinstance(
            kf, api.BandedKeyframe)
        outs = [out_ld, torch.empty((spec.height, spec.width),
                                    dtype=torch.float64).pin_memory().numpy()]
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        if host_async:
            for s_ in range(args.steps):
                k = counter[0] % nF
                if k == 0 and counter[0] > 0:
                    kf.reset()
                counter[0] += 1
                kf.process_frame_host_async(geoms[k], host_imgs[k], spec.search, cfg, "full",
                                            log_depth_out=outs[s_ & 1])
            kf.last_result()
        else:
            for _ in range(args.steps):
                step(dev=False, host_images=host_imgs)
                download(kf.handle, out_ld.ctypes.data, None, None, None, None, None, None, None)
        dt = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([dt], device=red_dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": round(jobs * args.steps / dt, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(P * 4),
               "d2h_bytes_per_step": int(P * 8 + C.sizeof(api.FrameResultC))}

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    peak, peak_kind = peaks()
    fus_s = np.array(fusion_ms) / 1e3
    achieved = float(np.sum(fusion_bytes) / np.sum(fus_s) / 1e9)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if split else "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded Perlin-textured planes; BASELINE {spec.name} "
                "shapes/distributions)",
        "config": {"workload": f"{spec.name}: {spec.width}x{spec.height} keyframe, {nF} tracked "
                               f"frames (reset after the last), solver {args.regime}",
                   "regime": args.regime, "solver_path": args.solver_path,
                   "gn_iterations": cfg.gn_iterations,
                   "cg_tol": cfg.cg_tol, "cg_max_iters": cfg.cg_max_iters,
                   "parallelism": (f"row bands x{ws} (one keyframe; halo rows and the "
                                   "band-level all-reduce over NVLink peer memory)") if split
                   else (f"replicas x{ws} (independent keyframes)"
                         + (f", {args.bands} row bands each" if args.bands else "")),
                   "l2": "flushed before every step (512 MiB write)"},
        "mpix_per_s": round(value * P / 1e6, 4),
        "stage_ms": {"stereo": round(float(np.mean(stereo_ms)), 4),
                     "optimise": round(float(np.mean(fusion_ms)), 4),
                     "source": "one synchronous pass over the keyframe's frames"},
        "submission": "async (frames enqueued back to back)" if use_async else "synchronous",
        "pcg_iters_per_update": round(float(np.mean(pcg)), 2),
        "observations_per_update": round(float(np.mean(obs)), 1),
        "roofline": {"kernel": "k_fusion", "bound": "hbm", "achieved": round(achieved, 2),
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_traffic("k_fusion"),
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, one launch)",
                     "bytes_per_update": float(np.mean(fusion_bytes)),
                     "note": "achieved = SURVEY 8(d) streaming byte model (351 + 112 n_cg B/px "
                             "per GN step, executed counts) / k_fusion device time; the "
                             "SM-resident solver moves only `traffic` DRAM bytes per launch, so "
                             "frac > 1 = faster than a streaming solver at full HBM bandwidth"},
        "stereo_roofline": {
            "kernel": "k_stereo", "bound": "fp64", "unit": "GFP64op/s",
            "achieved": round(165.0 * float(np.sum(steps_ep)) / (np.sum(stereo_ms) / 1e3) / 1e9, 1),
            "peak": FP64_PEAK_GOPS,
            "frac": round(165.0 * float(np.sum(steps_ep)) / (np.sum(stereo_ms) / 1e3) / 1e9
                          / FP64_PEAK_GOPS, 4),
            "epipolar_steps_per_update": round(float(np.mean(steps_ep)), 1),
            "model": "165 FP64 operations per epipolar step (SURVEY 8(a) a6; 11 IEEE divisions "
                     "counted as one operation each) / stereo stage time",
            "peak_source": "scripts/micro/fp64_rate.cu on B200: 58 DFMA lane-ops per SM per "
                           "clock x 148 SMs x 1965 MHz (operations, not FLOP)"},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
    }
    if not args.no_cpu_baseline and ws == 1:
        try:
            line["cpu_baseline"] = cpu_baseline(spec, seq, args.regime)
        except Exception as exc:  # the baseline never gates the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
