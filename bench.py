#!/usr/bin/env python
"""Benchmark of the SLIM-VDB per-frame integration hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = one frame of the BASELINE workload integrated into the map
(BASELINE.json configs[1] by default: closed-set 64x1024 LiDAR, identity
rotations, through Mapper.integrate -> svx_integrate).  Prints ONE JSON line.

ours:
  value     points integrated/s with inputs resident in HBM; per-step CUDA
            events on the launching stream; L2 flushed (256 MiB write, then
            a 256 MiB read so the flush's write-back stays outside the step)
            between steps outside the events; max over ranks.  With N > 1
            (torchrun) the map is sharded by leaf ownership: every rank gets
            the same frames, marches its slice, and rows go to their owners by
            NCCL all-to-all (paper_2512_12945_b200/sharded.py; strong scaling).
  e2e       same metric through the public API from pinned HOST buffers:
            H2D of points+labels and D2H of the frame report inside each step.
  roofline  dominant stage (per-stage CUDA events inside libsvx) against the
            measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline  the CPU oracle port (oracle/, OpenMP, all host threads) on a
            bounded sample of the same frames (rank 0, N=1 only).
reference:
  times the reference's own CPU implementation (semvox built in
  baseline/_ref, native backend, all host threads; else the oracle port) on
  the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "points integrated/sec"
UNIT = "points/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--depth", action="store_true",
                    help="camera configs (1, 3, 5): feed depth rasters through integrate_depth "
                         "(back-projection on the GPU) instead of point clouds")
    ap.add_argument("--tsdf-dtype", default="float64")
    ap.add_argument("--update-mode", default="auto", choices=["auto", "segments", "slots", "leaves"],
                    help="row grouping of closed-set frames (Mapper.set_update_mode)")
    ap.add_argument("--async-frames", type=int, default=2,
                    help="frames Mapper.integrate may leave in flight (0 = synchronous)")
    ap.add_argument("--cpu-frames", type=int, default=0, help="oracle sample frames (0=auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-frames", type=int, default=5,
                    help="extra frames run eagerly with per-stage events (roofline attribution)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# -- clocks during the timed region -------------------------------------------------

class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        reasons = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# -- byte model (fixed fp32 state layout) ----------------------------

def frame_bytes(used, touched, kind, C=0, D=0):
    """bytes_frame = N_used*(12+P) + 2*U*S."""
    if kind == "closed":
        P, S = 4, 8 + 4 * C
    elif kind == "open":
        P, S = 4 * D, 8 + 8 * D
    else:
        P, S = 0, 8
    return used * (12 + P) + 2 * touched * S


def stage_bytes(stage, rep, kind, C, D, tsdf_elem, mode="segments"):
    """Algorithmic bytes one launch of a stage must move.
    Voxel state is counted at the SURVEY 8(d) fp32 model (S = 8 + 4C closed,
    8 + 8D open), read + write; hash probes, claims and frame scratch beyond
    the rows and slots are overhead, not counted."""
    n, used, R, U = rep.points_in, rep.points_used, rep.band_hits, rep.touched_voxels
    P = 4 if kind == "closed" else (4 * D if kind == "open" else 0)
    S = 8 + (4 * C if kind == "closed" else (8 * D if kind == "open" else 0))
    if mode == "leaves":   # rows {key 8, point 4} -> {leaf|rank 8, slot|point 4} -> bins of 4 B
        return {
            "walk": n * (12 + P) + used * 32 + R * 12,
            "resolve": R * 12 + R * 12,
            "seg": 0,   # per listed leaf only (counted as overhead)
            "scatter": R * 12 + R * 4,
            "update": 2 * U * S + R * 4,
            "update_b": 0,
        }[stage]
    if mode == "slots":   # slot mode: rows {key 8, point 4, d 8, label 4}, slots {point, label, d} 16 B
        return {
            "walk": n * (12 + P) + R * 24,
            "resolve": R * 24 + R * 16 + U * 8,
            "update": 2 * U * S + R * 16 + U * 8,
            "update_b": 0, "seg": 0, "scatter": 0,
        }[stage]
    return {
        # read points (+labels/features), write the ray table and one 8-byte key per row
        "walk": n * (12 + P) + used * 32 + R * 8,
        # per row: key in, voxel id out, one count; per voxel: leaf lookup, slot, key
        "resolve": R * (8 + 4 + 4) + U * (16 + 4 + 8 + 4),
        "seg": U * 8,
        # per row: voxel id + count in; single-row voxels also ray + label + state
        "scatter": R * (4 + 4 + 4) + U * (32 + 2 * S),
        # multi-row voxels: rows, rays, labels, and state (upper bound: all
        # voxels); open-set: the frame's feature array once (SURVEY 8(d):
        # N_used * 4D) -- a row's re-read of its point's features (~9 per point)
        # is the implementation's cost, not algorithmic bytes
        "update": 2 * U * S + R * (4 + 32 + (4 if kind == "closed" else 0)) + (used * 4 * D if kind == "open" else 0),
        "update_b": 0,
    }[stage]


def measured_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(stage):
    """dram bytes per launch from the committed ncu summary, if any."""
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(stage)
    except Exception:
        return None


# -- workloads -----------------------------------------------------------------------

def load_scenes():
    """paper_2512_12945_b200/scenes.py as a standalone module: it needs only
    numpy and torch, and importing it this way does not import the package
    (whose __init__ loads libsvx.so) -- the reference arm must not map the
    engine's library."""
    import importlib.util

    name = "_svx_bench_scenes"
    if name in sys.modules:
        return sys.modules[name]
    path = os.path.join(REPO, "paper_2512_12945_b200", "scenes.py")
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def make_frames(cfg, count, device, start=0):
    scenes = load_scenes()
    wl = scenes.workload(cfg, device=device)
    frames = [wl.make_frame((start + i) % wl.n_frames) for i in range(count)]
    return wl, frames


def config_dict(args, wl, world):
    """The workload description, identical in both arms (the driver compares
    them); how each arm runs it goes in top-level keys."""
    kw = wl.mapper_kwargs
    return {
        "workload": wl.name, "points_per_frame": wl.points_per_frame,
        "voxel_size": kw["voxel_size"], "truncation": kw["truncation"],
        "max_range": kw.get("max_range"),
        "num_classes": kw.get("num_classes") or None, "feature_dim": kw.get("feature_dim") or None,
        "tsdf_dtype": args.tsdf_dtype,
        "input": "depth rasters" if args.depth else "point clouds",
        "parallelism": f"leaf-shard{world}" if world > 1 else "single",
        "frames_timed": f"{args.warmup}..{args.warmup + args.steps - 1}",
    }


def sem_kind_of(kw):
    return "closed" if kw.get("num_classes") else ("open" if kw.get("feature_dim") else None)


def run_oracle_sample(wl, frames, threads):
    """Time the CPU oracle port on host copies of the frames."""
    from oracle.oracle import OracleMap

    om = OracleMap(**wl.mapper_kwargs, threads=threads)
    used, secs = 0, 0.0
    kind = sem_kind_of(wl.mapper_kwargs)
    for f in frames:
        pts = f.points.cpu().numpy()
        lab = f.labels.cpu().numpy() if f.labels is not None else None
        feat = f.features.cpu().numpy() if f.features is not None else None
        t0 = time.perf_counter()
        r = om.integrate(pts, f.pose, labels=lab if kind == "closed" else None,
                         features=feat if kind == "open" else None)
        secs += time.perf_counter() - t0
        used += r.points_used
    return used, secs


# -- our arm ------------------------------------------------------------------------

def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    from paper_2512_12945_b200 import Mapper, _lib
    from paper_2512_12945_b200.sharded import DistTransport, ShardedMapper

    K, W = args.steps, args.warmup
    # N > 1: one map sharded by leaf ownership; every rank gets the same frame
    # stream, marches its slice and exchanges rows over NCCL (strong scaling:
    # the work per frame is fixed).  Stage profiling covers the 1-GPU path.
    sharded = world > 1
    P = 0 if sharded else args.profile_frames
    wl, frames = make_frames(args.config, W + K + P, dev)
    kw = dict(wl.mapper_kwargs, tsdf_dtype=args.tsdf_dtype, device=local)
    kind = sem_kind_of(kw)
    C = kw.get("num_classes", 0)
    D = kw.get("feature_dim", 0)
    tsdf_elem = 8 if args.tsdf_dtype == "float64" else 4
    # L2 flush between steps: write a 256 MiB buffer (> the 126 MB L2), then
    # read a second one so the written lines are written back before the
    # step starts (otherwise the step pays the flush's own write-back).
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=dev)

    def l2_flush():
        flush.zero_()
        flush_rd.sum()

    def integrate(m, f, host=None):
        if host is not None:
            pts, lab, feat = host
        else:
            pts, lab, feat = f.points, f.labels, f.features
        if args.depth:   # pts = depth raster, lab/feat = payload raster
            pay = lab if kind == "closed" else feat
            if host is None:
                h, w = f.camera["height"], f.camera["width"]
                pts = f.depth
                pay = f.labels.reshape(h, w) if kind == "closed" else f.features.reshape(h, w, -1)
            return m.integrate_depth(pts, pay, f.camera, pose=f.pose)
        extra = {"reduce_report": False} if sharded else {}
        return m.integrate(pts, f.pose, labels=lab if kind == "closed" else None,
                           features=feat if kind == "open" else None, **extra)

    def new_map():
        if sharded:
            return ShardedMapper(**kw, rank=rank, world=world, transport=DistTransport())
        mm = Mapper(**kw, async_frames=args.async_frames)
        mm.set_update_mode(args.update_mode)
        return mm

    # ---- device-resident pass ------------------------------------------------------
    m = new_map()
    for f in frames[:W]:
        integrate(m, f)
    # pool headroom for the timed frames, so no growth copy lands inside them
    st = m.engine_stats()
    per_frame = max(1, st["active_voxels"] // max(W, 1))
    m.reserve(st["active_voxels"] + 2 * per_frame * (K + P),
              st["leaf_count"] * (1 + 2 * (K + P) // max(W, 1)))
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K)]
    reps, stage_hist = [], []
    launches0 = _lib.kernel_launches()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(K):
            l2_flush()
            evs[i][0].record(stream)
            reps.append(integrate(m, frames[W + i]))
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    launches = _lib.kernel_launches() - launches0
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    used = sum(r.points_used for r in reps)   # whole frames (global counts) in both modes
    touched = sum(r.touched_voxels for r in reps)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    tv = torch.tensor([touched], dtype=torch.float64, device=dev)
    if sharded:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(tv)   # each voxel is owned by one rank
    total_ms_max, touched_all = float(t.item()), float(tv.item())
    value = used / (total_ms_max / 1e3)

    # ---- per-stage device times: a separate eager pass over P further frames -------
    m.set_profiling(True)
    prof_reps = []
    for f in frames[W + K:W + K + P]:
        l2_flush()
        prof_reps.append(integrate(m, f))
        stage_hist.append(m.stage_times())
    m.set_profiling(False)
    if not stage_hist:
        stage_hist, prof_reps = [{s: 0.0 for s in _lib.STAGES}], reps[-1:]

    # ---- roofline of the dominant stage -------------------------------------------
    stages = list(_lib.STAGES)
    mean_stage = {s: statistics.mean(h[s] for h in stage_hist) for s in stages}
    dom = max(_lib.KERNEL_STAGES, key=lambda s: mean_stage[s])
    est = m.engine_stats() if not sharded else {}
    slots = est.get("frames_slot_mode", 0) > 0
    leaves = est.get("frames_leaf_mode", 0) > 0
    dom_ms = mean_stage[dom]
    umode = "leaves" if leaves else ("slots" if slots else "segments")
    if umode == "segments" and dom in ("update", "update_b"):
        # segment mode: the byte model covers both update kernels together
        # (K5 short/long or open, then K5b long / huge), so they are timed together
        dom, dom_ms = "update", mean_stage["update"] + mean_stage["update_b"]
    dom_bytes = statistics.mean(stage_bytes(dom, r, kind, C, D, tsdf_elem, umode) for r in prof_reps)
    peak, peak_src = measured_peak()
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    fb = frame_bytes(used / K, touched_all / K, kind, C, D)   # mean frame, global counts
    frame_gbs = fb / (total_ms_max / K / 1e3) / 1e9
    traffic = ncu_traffic(umode + ":" + dom)

    # ---- e2e pass: host pinned buffers through the public API ---------------------------
    e2e = None
    if not args.no_e2e:
        host = []
        for f in frames:
            src_pts = f.depth if args.depth else f.points
            pts = torch.empty(src_pts.shape, dtype=src_pts.dtype, pin_memory=True)
            pts.copy_(src_pts)
            lab = feat = None
            if f.labels is not None:
                src = f.labels.reshape(f.depth.shape) if args.depth else f.labels
                lab = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
                lab.copy_(src)
            if f.features is not None:
                src = (f.features.reshape(f.depth.shape[0], f.depth.shape[1], -1) if args.depth
                       else f.features)
                feat = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
                feat.copy_(src)
            host.append((pts.numpy(), lab.numpy() if lab is not None else None,
                         feat.numpy() if feat is not None else None))
        m2 = new_map()
        for f, h in zip(frames[:W], host[:W]):
            integrate(m2, f, h)
        st = m2.engine_stats()
        m2.reserve(st["active_voxels"] + 2 * per_frame * K,
                   st["leaf_count"] * (1 + 2 * K // max(W, 1)))
        dstream = torch.cuda.default_stream()
        e_ms, e_used, h2d, d2h = 0.0, 0, 0, 0
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for i in range(K):
            l2_flush()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(dstream)
            r = integrate(m2, frames[W + i], host[W + i])
            e_used += r.points_used   # the frame's report, read back from the device
            b.record(dstream)
            b.synchronize()
            e_ms += a.elapsed_time(b)
            io = m2.engine_stats() if not sharded else None   # bytes the library moved
            h2d += io["last_h2d_bytes"] if io else sum(x.nbytes for x in host[W + i] if x is not None)
            d2h += io["last_d2h_bytes"] if io else 0
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": e_used / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d // K), "d2h_bytes_per_step": int(d2h // K),
               "ms_per_step": float(te.item()) / K}
        del m2

    # ---- CPU baseline (rank 0, N=1) ---------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nf = args.cpu_frames or min(K + W, 30 if kind == "closed" else 4)
        threads = host_threads()
        cused, csecs = run_oracle_sample(wl, frames[:nf], threads)
        cpu = {"value": cused / csecs, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"frames 0..{nf - 1} of {wl.name} through the C oracle "
                         f"(oracle/svx_oracle.c, OpenMP x{threads}, {cpu_model()}), "
                         f"{csecs:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": total_ms_max / K, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_dict(args, wl, world),
            "api": ("ShardedMapper.integrate -> svx_shard_{march,plan,pack,apply} + NCCL "
                    "all-to-all" if sharded else
                    ("Mapper.integrate_depth -> svx_integrate_depth (depth rasters, "
                     "back-projection on the GPU)" if args.depth else
                     "Mapper.integrate -> svx_integrate")),
            "l2": "flushed between steps (256 MiB write + 256 MiB read, outside step events)",
            "ms_per_frame_p50": statistics.median(step_ms),
            "points_used_per_frame": used / K,
            "touched_voxels_per_frame": touched_all / K,
            "band_rows_per_frame": statistics.mean(r.band_hits for r in reps),
            "roofline": ({"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                          "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                          "peak_source": peak_src,
                          "bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms,
                          "timing": "kernel span inside the frame graph (%globaltimer, FrameParams.kspan)",
                          "update_mode": umode}
                         if not sharded else
                         {"bound": "hbm", "kernel": "whole frame (per-rank peak x ranks)",
                          "achieved": frame_gbs, "peak": peak * world, "unit": "GB/s",
                          "frac": frame_gbs / (peak * world), "traffic": None,
                          "peak_source": peak_src}),
            "frame_roofline": {"bytes_per_frame": fb, "achieved": frame_gbs, "unit": "GB/s",
                               "frac": frame_gbs / (peak * world),
                               "model": "N_used*(12+P) + 2*U*S, fp32 state (SURVEY 8d)"},
            "stages_ms": {s: round(mean_stage[s], 4) for s in stages},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if sharded:
            import torch.distributed as dist

            line["nccl"] = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                            "version": ".".join(map(str, torch.cuda.nccl.version()))}
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


# -- reference arm ------------------------------------------------------------------------

def load_reference():
    ref = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "semvox")):
        sys.path.insert(0, ref)
        try:
            import semvox  # noqa: F401
            from semvox.backend import NATIVE_AVAILABLE

            return semvox, NATIVE_AVAILABLE
        except Exception:
            sys.path.remove(ref)
    return None, False


def _ref_frame_inputs(semvox, args, f, kind, i):
    """One frame as the reference's own API takes it: a semvox.Frame from the
    sensor points (or, with --depth, semvox.ingest.project_depth of the depth
    raster, ingest.py:285-322)."""
    import numpy as np

    if args.depth:
        from semvox.config import CameraConfig
        from semvox.ingest import project_depth

        cam = CameraConfig(**{k: f.camera[k] for k in ("fx", "fy", "cx", "cy", "width", "height",
                                                        "depth_scale", "stride")})
        h, w = f.camera["height"], f.camera["width"]
        pay = (f.labels.cpu().numpy().reshape(h, w) if kind == "closed"
               else f.features.cpu().numpy().reshape(h, w, -1))
        return lambda: project_depth(f.depth.cpu().numpy(), pay, cam, pose=f.pose, frame_id=i)
    pts = f.points.cpu().numpy()
    lab = f.labels.cpu().numpy() if kind == "closed" else None
    feat = f.features.cpu().numpy() if kind == "open" else None
    return lambda: semvox.Frame(points=pts, pose=f.pose, labels=lab, features=feat, frame_id=i)


def _ref_run(semvox, native, kw, kind, args, frames, threads, stages=None):
    """integrate_frame (evalbench.py:409-413) per frame on fresh grids; wall
    time per frame (Frame construction + integrate_frame, as the reference's
    own benchmark times it).  `stages`: collect the backend's stage timers."""
    fusion = semvox.FusionConfig(voxel_size=kw["voxel_size"], truncation=kw["truncation"],
                                 max_range=kw["max_range"])
    closed = semvox.ClosedSetConfig(num_classes=kw["num_classes"]) if kind == "closed" else None
    open_set = semvox.OpenSetConfig(feature_dim=kw["feature_dim"]) if kind == "open" else None
    tsdf, sem = semvox.make_grids(fusion, closed=closed, open_set=open_set,
                                  backend="native" if native else "python")
    be = tsdf.backend
    orig = be.integrate_points
    if stages is not None:
        # pass-through wrapper: keeps the t_*_ms timers integrate_points
        # returns (_core.pyx:705-857), which IntegrationReport drops
        def traced(*a, **k):
            out = orig(*a, **k)
            stages.append({n: out[n] for n in out if n.startswith("t_")})
            return out

        be.integrate_points = traced
    times, used = [], []
    try:
        for i, f in enumerate(frames):
            mk = _ref_frame_inputs(semvox, args, f, kind, i)
            t0 = time.perf_counter()
            r = semvox.integrate_frame(tsdf, sem, mk(), fusion, threads=threads)
            times.append(time.perf_counter() - t0)
            used.append(r.points_used)
    finally:
        be.integrate_points = orig
    return times, used


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import torch

    K, W = args.steps, args.warmup
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    wl, frames = make_frames(args.config, W + K, dev)
    kw = wl.mapper_kwargs
    kind = sem_kind_of(kw)
    threads = host_threads()
    semvox, native = load_reference()
    extra = {}
    if semvox is not None:
        stages = []
        times, used_l = _ref_run(semvox, native, kw, kind, args, frames, threads, stages)
        secs, used = sum(times[W:]), sum(used_l[W:])
        # single-thread number and the allocation split
        n1 = min(len(frames), W + K, 6 if kind == "closed" else 2)
        t1, u1 = _ref_run(semvox, native, kw, kind, args, frames[:n1], 1)
        steady1 = t1[1:] if n1 > 1 else t1
        st_mean = {k: statistics.mean(s[k] for s in stages[W:] if k in s)
                   for k in (stages[W] if len(stages) > W else {})}
        extra = {
            "ms_per_frame_first": times[0] * 1e3,
            "ms_per_frame_steady": secs * 1e3 / K,
            "allocation_note": "frame 0 allocates the map's first leaves (allocation-heavy); "
                               "timed frames are steady state (warm-up frames allocate first)",
            "stage_ms": {k: round(v, 3) for k, v in st_mean.items()},
            "stage_ms_source": "integrate_points' own t_*_ms timers (_core.pyx:705-857), "
                               "mean over the timed frames",
            "threads_1": {"value": sum(u1[1:] if n1 > 1 else u1) / sum(steady1), "unit": UNIT,
                          "ms_per_frame": statistics.mean(steady1) * 1e3,
                          "sample": f"frames 1..{n1 - 1} after frame 0, threads=1"},
        }
        what = (f"semvox (reference) {'native Cython/C++ OpenMP' if native else 'numpy'} backend "
                f"from baseline/_ref, integrate_frame per frame, threads={threads}, {cpu_model()}")
        kind_s = "reference"
    else:
        from oracle.oracle import OracleMap

        om = OracleMap(**kw, threads=threads)
        used, secs = 0, 0.0
        for i, f in enumerate(frames):
            t0 = time.perf_counter()
            r = om.integrate(f.points.cpu().numpy(), f.pose,
                             labels=f.labels.cpu().numpy() if kind == "closed" else None,
                             features=f.features.cpu().numpy() if kind == "open" else None)
            dt = time.perf_counter() - t0
            if i >= W:
                secs += dt
                used += r.points_used
        what = f"oracle port (oracle/svx_oracle.c) OpenMP x{threads}, {cpu_model()}"
        kind_s = "port"
    value = used / secs
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(world, args.gpus),
        "steps": K, "warmup": W,
        "ms_per_step": secs * 1e3 / K, "higher_is_better": True,
        "scaling": "strong" if max(world, args.gpus) > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": config_dict(args, wl, max(world, args.gpus)),
        "api": "semvox.Frame + semvox.integrate_frame (reference CPU path)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind_s,
                         "sample": what},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    print(json.dumps(line))


def spawn_ranks(args):
    """`bench.py --gpus N` without a torchrun environment: launch N ranks
    (one process per GPU, NCCL) through torch.distributed.run and pass their
    output through; rank 0 prints the JSON line.  Fails loudly when fewer
    than N GPUs are visible (ranks never share a GPU)."""
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
                         f"found {have}; not running (would otherwise report n_gpus=1)\n")
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":   # rank 0 alone runs the reference
            run_reference(args)
            return
        spawn_ranks(args)
    world = dist_env()[0]
    if args.impl == "ours" and world != max(args.gpus, 1):
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
