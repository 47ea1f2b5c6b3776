#!/usr/bin/env python3
"""Benchmark: fused keyframe updates/s at 640x480 (BASELINE.json metric).

One step = one fused keyframe update on a tracked frame (pipeline.hpp:205-226):
stereo_scan + update_semidense + optimize, on the device-resident keyframe
session (dfuse_kf_process_frame*). Default workload = BASELINE config C2
(640x480, fx=fy=525, 10 tracked frames per keyframe, reference solver
defaults: 10 GN iterations, PCG tol 1e-6 / max 200), seeded synthetic scene
(the paper's datasets are not available; see paper_2207_12244_b200/synth.py).
A keyframe is reset on the device before its first tracked frame (inside the
timed step), so K steps walk the keyframe's 10 frames over and over.

  --config C3   the batch of 64 independent keyframes (3-8 planes or boxes),
                keyframe k on rank k mod N (shard.keyframes_for_rank); each
                rank's K steps walk its keyframes in order, 10 frames each
  --config C4   the 3840x2160 keyframe; under torchrun one row band per rank

Reported (one JSON line on rank 0):
  value     device-timed (CUDA events on the library's stream), input frames
            resident in HBM, L2 flushed before every step (512 MiB write
            outside the events)
  e2e       the same metric through the C-ABI with HOST buffers
            (dfuse_kf_process_frame_host_async): every step copies its
            tracked frame in from pinned host memory and its fused log-depth
            map out to pinned host memory; wall clock from the first call to
            last_result(); the host pipeline is warmed up before the clock
  fixed_effort  the same measurements at the north-star's fixed effort
            (cg_tol = 0, 5 PCG iterations per GN iteration), same run
  roofline  k_fusion: with the SM-resident PCG (C1/C2/C3/C5) the solver
            moves ~25 MB of DRAM per optimize and is bound by the latency of
            its one grid all-reduce per PCG iteration: achieved = PCG
            iterations per ms (from the two regimes' optimise times), peak =
            1 / the all-reduce time measured in this run; the SURVEY 8(d)
            HBM byte model is kept beside it (hbm_model). With the streaming
            PCG (C4) the roofline is the HBM byte model against the measured
            copy bandwidth.
  self_check  the final device state of the timed passes hashed against the
            synchronous pass over the same frames, and (cpu_baseline leg)
            the reference's state after its sample frames against ours
  cpu_baseline  the reference's own code (oracle/_ref) on the host cores

--impl reference times the reference's CPU implementation (oracle/_ref,
OpenMP on all host threads) on the same workload and prints the same line
with the same config dict.

Multi-GPU: under torchrun every rank runs its own keyframes (C2: one
independent keyframe stream per rank; C3: keyframe k on rank k mod N) --
weak scaling, no data-path collective; value = all ranks' updates / the max
over ranks of the device time. `--gpus N` without torchrun relaunches itself
under torch.distributed.run with N ranks (fails if fewer GPUs are visible).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
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
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--regime", default="defaults", choices=["defaults", "fixed"],
                    help="defaults: reference solver settings; fixed: cg_tol=0, 5 PCG/GN")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--keyframes", type=int, default=0,
                    help="C3 batch size (default: the config's 64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fixed", action="store_true",
                    help="skip the fixed-effort sub-measurement")
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


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: relaunch under
    torch.distributed.run with N ranks, one GPU each."""
    import torch

    visible = torch.cuda.device_count()
    if visible < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {visible} GPU(s) visible", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def ncu_record(kernel):
    """The committed ncu facts of `kernel` (profiles/ncu_traffic.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return dict(json.load(f)[kernel])
    except (OSError, KeyError, ValueError):
        return {}


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
# workload
def keyframe_ids(args, spec, ws, rank):
    """The keyframes this rank owns: C3 -> k mod N over the batch; otherwise
    one keyframe stream per rank (C2/C1/C5), or one shared keyframe (C4 split)."""
    from paper_2207_12244_b200 import shard

    if spec.name == "C3":
        n = args.keyframes or spec.keyframes
        return shard.keyframes_for_rank(n, ws, rank)
    return [rank]


def keyframe_seed(args, spec, k, split):
    if spec.name == "C3":
        return args.seed + k
    return args.seed + (0 if split else 1000 * k)


def _make_seq(job):
    from paper_2207_12244_b200 import synth

    name, seed, frames = job
    return synth.make_sequence(synth.CONFIGS[name], seed, frames=frames)


def make_sequences(spec, seeds, frames, ws):
    """Seeded sequences, generated in parallel processes when there are
    several (C3): ~5 s of numpy per 640x480 sequence."""
    jobs = [(spec.name, s, frames) for s in seeds]
    if len(jobs) <= 1:
        return [_make_seq(j) for j in jobs]
    import concurrent.futures as cf
    import multiprocessing as mp

    workers = max(1, min(len(jobs), (os.cpu_count() or 2) // max(1, ws)))
    with cf.ProcessPoolExecutor(workers, mp_context=mp.get_context("fork")) as ex:
        return list(ex.map(_make_seq, jobs))


def config_dict(args, spec, cfg, ws, split, n_keyframes):
    """The workload description printed by BOTH arms (same dict)."""
    if spec.name == "C3":
        par = (f"keyframe batch of {n_keyframes}: keyframe k on rank k mod {ws} "
               "(no data-path collective)")
    elif split:
        par = (f"row bands x{ws} (one keyframe; halo rows and the band-level all-reduce over "
               "NVLink peer memory)")
    else:
        par = f"independent keyframe streams x{ws}" + (
            f", {args.bands} row bands each" if args.bands else "")
    return {"workload": f"{spec.name}: {spec.width}x{spec.height} keyframe(s), {spec.frames} "
                        f"tracked frames each (keyframe reset before its first frame), solver "
                        f"{args.regime}",
            "regime": args.regime, "gn_iterations": cfg.gn_iterations, "cg_tol": cfg.cg_tol,
            "cg_max_iters": cfg.cg_max_iters, "keyframes": n_keyframes, "seed": args.seed,
            "parallelism": par, "l2": "flushed before every device-timed step (512 MiB write)"}


def state_arrays(kf):
    st, semi, _ = kf.download()
    return st, semi


def state_hash(st, semi) -> str:
    h = hashlib.sha1()
    for a in (st.log_depth, semi.depth, semi.variance, semi.valid):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.float64(st.scale).tobytes())
    h.update(np.int64(st.iteration).tobytes())
    h.update(np.int64(semi.inlier_count).tobytes())
    return h.hexdigest()


# --------------------------------------------------------------------------
def run_reference(args, spec, seq, steps, warmup, budget_s=120.0, keep_state_after=None):
    """The reference's CPU implementation (oracle/_ref, OpenMP) on the same
    workload; each step = one process_frame on a tracked frame (the keyframe
    reset before its first frame). Returns (updates/s, ms/step, threads,
    steps done, state after `keep_state_after` steps or None)."""
    import ctypes as C

    import oracle
    from paper_2207_12244_b200._ffi import FusionInputsC, SemiDenseMap, _dptr

    ref = oracle.reference()
    L = ref.lib
    L.ref_process_frame.restype = C.c_int
    # all the host threads this process may use (torchrun sets OMP_NUM_THREADS=1)
    L.ref_omp_set_threads(len(os.sched_getaffinity(0)))
    threads = L.ref_omp_max_threads()
    cfg = solver_cfg(spec, args.regime)
    mask = ref.texture_mask(seq.I0, 0.02)
    geoms = [ref.make_epipolar_geometry(np.array([1.0, 0, 0, 0]), np.zeros(3), q, t,
                                        spec.camera()) for (q, t, _) in seq.frames]
    planes = seq.pred.planes()
    nF = len(seq.frames)

    def fresh():
        semi = SemiDenseMap.empty(spec.width, spec.height)
        return semi, seq.pred.log_depth.copy(), C.c_double(1.0), C.c_int32(0), C.c_int32(0)

    state = list(fresh())
    frame_idx = [0]

    def step():
        k = frame_idx[0] % nF
        if k == 0:
            state[:] = fresh()
        semi, ld, scale, it, cnt = state
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

    for _ in range(warmup):
        step()
    frame_idx[0] = 0
    t0 = time.perf_counter()
    done = 0
    snap = None
    while done < steps:
        step()
        done += 1
        if keep_state_after is not None and done == keep_state_after:
            semi, ld, scale, it, cnt = state
            snap = (ld.copy(), semi.depth.copy(), semi.variance.copy(), semi.valid.copy(),
                    scale.value, it.value, cnt.value)
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, dt * 1e3 / done, threads, done, snap


def cpu_baseline(args, spec, seq, snapshots, budget_s=20.0):
    """Bounded sample of the same workload on the reference build, plus a
    parity check of its state against ours after the same frames."""
    _, ms1, _, _, _ = run_reference(args, spec, seq, 1, 0)
    n = max(1, min(len(seq.frames), int(budget_s * 1e3 / max(ms1, 1.0))))
    v, ms, threads, done, snap = run_reference(args, spec, seq, n, 0, keep_state_after=n)
    out = {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "reference",
           "sample": f"the first {done} tracked-frame updates of {spec.name} keyframe 0 "
                     f"(reference headers + OpenMP, {threads} threads)"}
    if snap is not None and done - 1 < len(snapshots):
        ours_st, ours_semi = snapshots[done - 1]
        ld, sd, sv, sval, scale, it, cnt = snap
        rel = float(np.max(np.abs(np.exp(ours_st.log_depth) - np.exp(ld)) / np.exp(ld)))
        out["parity_vs_ours"] = {
            "frames": done,
            "semi_map_bit_exact": bool(ours_semi.depth.tobytes() == sd.tobytes()
                                       and ours_semi.variance.tobytes() == sv.tobytes()
                                       and ours_semi.valid.tobytes() == sval.tobytes()),
            "inlier_count_equal": bool(ours_semi.inlier_count == cnt),
            "max_rel_depth": rel, "scale_rel": abs(ours_st.scale - scale) / abs(scale),
            "iteration_equal": bool(ours_st.iteration == it),
            "tolerance": "semi map bit-exact; exp(log_depth) and scale within 1e-4 rel",
            "ok": bool(ours_semi.depth.tobytes() == sd.tobytes() and rel <= 1e-4
                       and abs(ours_st.scale - scale) <= 1e-4 * abs(scale))}
    return out


# --------------------------------------------------------------------------
class Stream:
    """One keyframe of this rank with its tracked frames (device + pinned host)."""

    def __init__(self, kid, seq, kf, geoms, dev_frames):
        self.kid, self.seq, self.kf, self.geoms, self.dev = kid, seq, kf, geoms, dev_frames
        self.host = None


def schedule(n_streams, nF, steps):
    """step s -> (stream, frame): each stream's frames in order, streams in turn"""
    return [((s // nF) % n_streams, s % nF) for s in range(steps)]


def measure(ctx, streams, cfg, args, device, ws, red_dev, flush, cstream, snapshot_stream0,
            clocks_out=None):
    """Device-timed and end-to-end passes of `args.steps` steps at solver
    settings `cfg`, plus a synchronous statistics pass over the same frames."""
    import torch

    from paper_2207_12244_b200 import api

    nF = len(streams[0].geoms)
    sched = schedule(len(streams), nF, args.steps)
    used = sorted({j for j, _ in sched})
    search = streams[0].seq.spec.search
    banded = isinstance(streams[0].kf, api.BandedKeyframe)
    use_async = not banded

    def frame_sync(st, k):
        return st.kf.process_frame(st.geoms[k], None, search, cfg, "full",
                                   device_ptr=st.dev[k].data_ptr())

    # ---- warm-up (untimed), then the statistics pass: every used keyframe's
    # frames once, synchronously (the computation is deterministic, so the
    # timed passes repeat exactly these frames)
    for w in range(max(3, args.warmup)):
        st = streams[used[0]]
        if w % nF == 0:
            st.kf.reset()
        frame_sync(st, w % nF)
    last_j, last_k = sched[-1]
    per_frame = []  # results in schedule order of the first pass over the used streams
    snapshots, final_hash = [], None
    for j in used:
        st = streams[j]
        st.kf.reset()
        for k in range(nF):
            per_frame.append(frame_sync(st, k))
            if j == 0 and snapshot_stream0:
                snapshots.append(state_arrays(st.kf))
            if j == last_j and k == last_k:
                final_hash = state_hash(*state_arrays(st.kf))
    # results of the scheduled steps (for stage times / counts)
    res_of = {(j, k): per_frame[used.index(j) * nF + k] for j in used for k in range(nF)}
    sched_res = [res_of[s] for s in sched]

    # ---- device-timed region: frames enqueued back to back, per-step CUDA
    # events on the library's stream, L2 flushed before every step
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(device)
    launches0 = ctx.launch_count()
    sampler = ClockSampler(device) if clocks_out is not None else None
    if sampler:
        sampler.start()
    events = []
    with torch.cuda.stream(cstream):
        for (j, k) in sched:
            st = streams[j]
            flush.fill_(float(k))  # evict L2 (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(cstream)
            if k == 0:
                st.kf.reset()
            if use_async:
                st.kf.process_frame_async(st.geoms[k], st.dev[k].data_ptr(), search, cfg, "full")
            else:
                frame_sync(st, k)
            e1.record(cstream)
            events.append((e0, e1))
        if use_async:
            for j in used:
                streams[j].kf.last_result()
    torch.cuda.synchronize(device)
    if sampler:
        clocks_out.update(sampler.stop())
    launches = ctx.launch_count() - launches0
    step_ms = [e0.elapsed_time(e1) for e0, e1 in events]
    total_ms = float(np.sum(step_ms))
    dev_hash = state_hash(*state_arrays(streams[last_j].kf))
    if ws > 1:
        t = torch.tensor([total_ms], device=red_dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())

    # ---- end to end through the C-ABI with host buffers
    e2e, e2e_hash = None, None
    if not args.no_e2e:
        import ctypes as C

        P = streams[0].seq.spec.width * streams[0].seq.spec.height
        H, W = streams[0].seq.spec.height, streams[0].seq.spec.width
        for j in used:
            st = streams[j]
            if st.host is None:  # inputs and results in pinned host memory
                st.host = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).pin_memory()
                           .numpy() for (_, _, I1) in st.seq.frames]
                st.outs = [torch.empty((H, W), dtype=torch.float64).pin_memory().numpy()
                           for _ in range(2)]  # result slots, alternating
        host_async = use_async

        def e2e_step(s_, j, k):
            st = streams[j]
            if k == 0:
                st.kf.reset()
            if host_async:
                st.kf.process_frame_host_async(st.geoms[k], st.host[k], search, cfg, "full",
                                               log_depth_out=st.outs[s_ & 1])
            else:
                st.kf.process_frame(st.geoms[k], st.host[k], search, cfg, "full")
                api.lib().dfuse_bkf_download(st.kf.handle, st.outs[0].ctypes.data, None, None,
                                             None, None, None, None, None)

        # warm-up: the host pipeline of every used keyframe is built on its
        # first call (device slots, copy streams, events, texture objects)
        for j in used:
            e2e_step(0, j, 0)
            if host_async:
                streams[j].kf.last_result()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for s_, (j, k) in enumerate(sched):
            e2e_step(s_, j, k)
        if host_async:
            for j in used:
                streams[j].kf.last_result()
        dt = time.perf_counter() - t0
        e2e_hash = state_hash(*state_arrays(streams[last_j].kf))
        if ws > 1:
            t = torch.tensor([dt], device=red_dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        jobs = ws if not banded or args.bands else 1
        e2e = {"value": round(jobs * args.steps / dt, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(P * 4),
               "d2h_bytes_per_step": int(P * 8 + C.sizeof(api.FrameResultC))}
    return {"total_ms": total_ms, "step_ms": step_ms, "launches": launches, "sched_res": sched_res,
            "snapshots": snapshots, "e2e": e2e,
            "self_check": {"reference": "synchronous pass over the same frames",
                           "device_timed_state_equal": dev_hash == final_hash,
                           "e2e_state_equal": None if e2e_hash is None else e2e_hash == final_hash,
                           "state": "log-depth, semi-dense map, scale, iteration, inliers "
                                    f"of keyframe {streams[last_j].kid} after frame {last_k}"}}


def allreduce_floor_us(ctx):
    """Device time of one grid all-reduce of the fusion solver (the LL
    all-to-all it runs once per PCG iteration), on the solver's grid."""
    import ctypes as C

    from paper_2207_12244_b200 import api

    L = api.lib()
    L.dfuse_debug_sync_bench.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(C.c_float)]
    ms = C.c_float(0)
    L.dfuse_debug_sync_bench(ctx.handle, 2000, 10, 0, C.byref(ms))  # warm-up
    n = 20000
    rc = L.dfuse_debug_sync_bench(ctx.handle, n, 10, 0, C.byref(ms))
    return None if rc else 1e3 * ms.value / n


def summarize(m, P, jobs, args):
    res = m["sched_res"]
    fusion_ms = [r.optimise_ms for r in res]
    stereo_ms = [r.stereo_ms for r in res]
    fusion_bytes = [fusion_bytes_per_px(r.stats) * P for r in res]
    pcg = [r.stats.pcg_total for r in res]
    steps_ep = [r.epipolar_steps for r in res]
    value = jobs * args.steps / (m["total_ms"] / 1e3)
    achieved = float(np.sum(fusion_bytes) / (np.sum(fusion_ms) / 1e3) / 1e9)
    return {"value": value, "fusion_ms": float(np.mean(fusion_ms)),
            "stereo_ms": float(np.mean(stereo_ms)), "pcg": float(np.mean(pcg)),
            "hbm_achieved": achieved, "bytes_per_update": float(np.mean(fusion_bytes)),
            "steps_ep": float(np.mean(steps_ep)), "stereo_ms_sum": float(np.sum(stereo_ms)),
            "steps_ep_sum": float(np.sum(steps_ep)),
            "obs": float(np.mean([r.observations for r in res])),
            "ppt": int(res[-1].solver_ppt)}


# --------------------------------------------------------------------------
def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "ours" and ws == 1 and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    from paper_2207_12244_b200 import synth

    spec = synth.CONFIGS[args.config]
    split = args.config == "C4" and ws > 1
    kids = keyframe_ids(args, spec, ws, rank)
    n_kf_total = (args.keyframes or spec.keyframes) if spec.name == "C3" else (1 if split else ws)
    cfg = solver_cfg(spec, args.regime)

    if args.impl == "reference":
        if rank != 0:
            return
        seq = synth.make_sequence(spec, keyframe_seed(args, spec, kids[0], split),
                                  frames=args.frames or None)
        value, ms, threads, done, _ = run_reference(args, spec, seq, args.steps,
                                                    min(args.warmup, 3))
        line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
                "higher_is_better": True, "scaling": "strong" if split else "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": f"synthetic (seeded Perlin-textured scenes; BASELINE {spec.name} "
                        "shapes/distributions)",
                "impl": "reference",
                "config": config_dict(args, spec, cfg, ws if ws > 1 else args.gpus, split,
                                      n_kf_total),
                "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                                 "kind": "reference",
                                 "sample": f"{done} of the {args.steps} requested updates "
                                           f"(120 s budget) of keyframe 0, after "
                                           f"{min(args.warmup, 3)} warm-up"},
                "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    # sequences first (forked workers; CUDA not initialised yet)
    nF_cfg = args.frames or spec.frames
    n_used = min(len(kids), max(1, math.ceil(args.steps / nF_cfg)))
    seqs = make_sequences(spec, [keyframe_seed(args, spec, k, split) for k in kids[:n_used]],
                          args.frames or None, ws)

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

    ctx = api.context(device)
    ctx.set_solver_path(args.solver_path)
    if args.solver_ctas:
        ctx.set_solver_ctas(args.solver_ctas)
    streams = []
    for kid, seq in zip(kids, seqs):
        if split:
            from paper_2207_12244_b200.bands_dist import DistributedBandedKeyframe

            kf = DistributedBandedKeyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
        elif args.bands > 0:
            kf = api.BandedKeyframe(ctx, spec.camera(), seq.I0, seq.pred, args.bands, 0.02)
        else:
            kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
        geoms = [ctx.api.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t,
                                                spec.camera()) for (q, t, _) in seq.frames]
        dev = [torch.from_numpy(np.ascontiguousarray(I1, np.float32)).cuda(device)
               for (_, _, I1) in seq.frames]
        streams.append(Stream(kid, seq, kf, geoms, dev))
    torch.cuda.synchronize(device)
    cstream = torch.cuda.ExternalStream(ctx.stream_handle(), device=torch.device("cuda", device))
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")
    P = spec.width * spec.height
    jobs = 1 if split else ws  # keyframe updates per step, whole job

    # (the reference takes minutes per 4K update: no C4 CPU leg in the default run)
    want_cpu = not args.no_cpu_baseline and ws == 1 and spec.name != "C4"
    clocks = {}
    m = measure(ctx, streams, cfg, args, device, ws, red_dev, flush, cstream, want_cpu, clocks)
    s = summarize(m, P, jobs, args)
    fixed = None
    if args.regime == "defaults" and not args.no_fixed:
        cfg_f = solver_cfg(spec, "fixed")
        mf = measure(ctx, streams, cfg_f, args, device, ws, red_dev, flush, cstream, False)
        sf = summarize(mf, P, jobs, args)
        fixed = (cfg_f, mf, sf)
    # the all-reduce floor, only where the latency roofline uses it
    ar_us = allreduce_floor_us(ctx) if s["ppt"] > 0 and fixed is not None else None

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    peak, peak_kind = peaks()
    ncu_f = ncu_record("k_fusion")

    def hbm_roofline(sx):
        return {"kernel": "k_fusion", "bound": "hbm", "achieved": round(sx["hbm_achieved"], 2),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(sx["hbm_achieved"] / peak, 4),
                "traffic": ncu_f.get("dram_bytes_per_launch") if sx["ppt"] > 0 else None,
                "bytes_per_update": sx["bytes_per_update"],
                "model": "SURVEY 8(d) streaming byte model (351 + 112 n_cg B/px per GN step, "
                         "executed counts) / k_fusion device time"}

    if s["ppt"] > 0:
        # SM-resident PCG: on-chip; latency of the per-iteration grid all-reduce
        t_iter = None
        if fixed is not None and s["pcg"] > fixed[2]["pcg"] + 1:
            t_iter = 1e3 * (s["fusion_ms"] - fixed[2]["fusion_ms"]) / (s["pcg"] - fixed[2]["pcg"])
        roof = {"kernel": "k_fusion", "bound": "latency",
                "unit": "PCG iterations/ms",
                "achieved": round(1e3 / t_iter, 2) if t_iter else None,
                "peak": round(1e3 / ar_us, 2) if ar_us else None,
                "frac": round(ar_us / t_iter, 4) if (t_iter and ar_us) else None,
                "us_per_pcg_iteration": round(t_iter, 3) if t_iter else None,
                "allreduce_us": round(ar_us, 3) if ar_us else None,
                "method": "us per PCG iteration = (optimise ms at defaults - at fixed effort) / "
                          "(PCG iterations at defaults - at fixed effort), same frames, same GN "
                          "count; peak = one grid all-reduce (LL all-to-all over the solver's "
                          "CTAs, dfuse_debug_sync_bench) -- the one serial exchange per "
                          "iteration of the pipelined PCG",
                "traffic": ncu_f.get("dram_bytes_per_launch"),
                "smem_wavefronts_per_sm_clk": ncu_f.get("smem_wavefronts_per_sm_clk"),
                "ncu_source": ncu_f.get("source"),
                "hbm_model": hbm_roofline(s)}
    else:
        roof = hbm_roofline(s)

    line = {
        "metric": METRIC, "value": round(s["value"], 4), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(m["total_ms"] / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if split else "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded Perlin-textured scenes; BASELINE {spec.name} "
                "shapes/distributions)",
        "config": config_dict(args, spec, cfg, ws, split, n_kf_total),
        "mpix_per_s": round(s["value"] * P / 1e6, 4),
        "stage_ms": {"stereo": round(s["stereo_ms"], 4), "optimise": round(s["fusion_ms"], 4),
                     "source": "synchronous pass over the same frames"},
        "submission": ("async (frames enqueued back to back)" if not isinstance(
            streams[0].kf, api.BandedKeyframe) else "synchronous"),
        "solver_path": "SM-resident PCG (%d px/thread)" % s["ppt"] if s["ppt"] else "streaming PCG",
        "pcg_iters_per_update": round(s["pcg"], 2),
        "observations_per_update": round(s["obs"], 1),
        "roofline": roof,
        "stereo_roofline": {
            "kernel": "k_stereo", "bound": "fp64", "unit": "GFP64op/s",
            "achieved": round(165.0 * s["steps_ep_sum"] / (s["stereo_ms_sum"] / 1e3) / 1e9, 1),
            "peak": FP64_PEAK_GOPS,
            "frac": round(165.0 * s["steps_ep_sum"] / (s["stereo_ms_sum"] / 1e3) / 1e9
                          / FP64_PEAK_GOPS, 4),
            "epipolar_steps_per_update": round(s["steps_ep"], 1),
            "model": "165 FP64 operations per epipolar step (SURVEY 8(a) a6; 11 IEEE divisions "
                     "counted as one operation each) / stereo stage time",
            "peak_source": "scripts/micro/fp64_rate.cu on B200: 58 DFMA lane-ops per SM per "
                           "clock x 148 SMs x 1965 MHz (operations, not FLOP)"},
        "gpu_launches": int(m["launches"]),
        "clocks": clocks,
        "e2e": m["e2e"],
        "self_check": m["self_check"],
    }
    if fixed is not None:
        cfg_f, mf, sf = fixed
        line["fixed_effort"] = {
            "regime": f"cg_tol = 0, cg_max_iters = {cfg_f.cg_max_iters} "
                      f"({cfg_f.gn_iterations} GN iterations)",
            "value": round(sf["value"], 4), "unit": UNIT,
            "ms_per_step": round(mf["total_ms"] / args.steps, 4),
            "e2e": mf["e2e"], "pcg_iters_per_update": round(sf["pcg"], 2),
            "stage_ms": {"stereo": round(sf["stereo_ms"], 4),
                         "optimise": round(sf["fusion_ms"], 4)},
            "roofline_hbm_model": hbm_roofline(sf),
            "gpu_launches": int(mf["launches"]), "self_check": mf["self_check"]}
    if want_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(args, spec, streams[0].seq, m["snapshots"])
        except Exception as exc:  # the baseline never gates the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
