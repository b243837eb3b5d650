"""Per-stage device times of one update mode on a BASELINE config (profiling
spans), e.g.  python tools/mode_diag.py --config 2 --mode leaves --frames 8"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--mode", default="leaves")
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--async-frames", type=int, default=0)
    ap.add_argument("--watchdog", type=float, default=0.0, help="dump the Python stack and exit after this many s")
    args = ap.parse_args()
    t_start = time.perf_counter()
    if args.watchdog > 0:
        import faulthandler

        faulthandler.dump_traceback_later(args.watchdog, exit=True)
    import torch

    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(args.config, device="cuda")
    m = Mapper(**wl.mapper_kwargs, async_frames=args.async_frames)
    m.set_update_mode(args.mode)
    m.set_profiling(True)
    for i in range(args.frames):
        f = wl.make_frame(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = m.integrate(f.points, f.pose, labels=f.labels, features=f.features)
        r.points_used
        dt = (time.perf_counter() - t0) * 1e3
        st = m.stage_times()
        fc = m.frame_counters()
        print(f"frame {i} wall {dt:.3f} ms rows {r.band_hits} touched {r.touched_voxels} "
              + " ".join(f"{k} {v * 1e3:.1f}" for k, v in st.items()) + f" {fc}", flush=True)
    print(f"t={time.perf_counter() - t_start:.1f}s", flush=True)
    print(m.engine_stats(), flush=True)
    print(f"t={time.perf_counter() - t_start:.1f}s", flush=True)


def pipeline(config=2, frames=30, mode="auto", async_frames=2, flush=False, reserve=True):
    """Frames back to back (asynchronous), events around the whole run:
    the device time per frame including graph launch gaps."""
    import torch

    from paper_2512_12945_b200 import Mapper, scenes

    wl = scenes.workload(config, device="cuda")
    fr = [wl.make_frame(i) for i in range(frames)]
    m = Mapper(**wl.mapper_kwargs, async_frames=async_frames)
    m.set_update_mode(mode)
    for f in fr[:5]:
        m.integrate(f.points, f.pose, labels=f.labels, features=f.features)
    st = m.engine_stats()
    if reserve:
        m.reserve(st["active_voxels"] * 4, st["leaf_count"] * 4)
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    reps = []
    host = 0.0
    for f in fr[5:]:
        if flush:
            buf.zero_()
        t0 = time.perf_counter()
        reps.append(m.integrate(f.points, f.pose, labels=f.labels, features=f.features))
        host += time.perf_counter() - t0
    b.record()
    b.synchronize()
    n = len(fr) - 5
    used = sum(r.points_used for r in reps)
    ms = a.elapsed_time(b)
    st = m.engine_stats()
    print(f"pipeline mode={mode} async={async_frames} flush={flush} reserve={reserve}: {1e3 * ms / n:.1f} us/frame "
          f"{used / (ms / 1e3) / 1e6:.0f} M points/s; host {1e6 * host / n:.1f} us/call; "
          f"reruns {st['async_reruns']} vcap {st['voxel_capacity']} bcap {st['block_capacity']}")


if __name__ == "__main__":
    if "--pipeline" in sys.argv:
        cfg = int(os.environ.get("DIAG_CONFIG", "2"))
        for af in ([int(a) for a in sys.argv[sys.argv.index("--pipeline") + 1].split(",")]
                   if len(sys.argv) > sys.argv.index("--pipeline") + 1 else (0, 1, 2, 3, 4)):
            pipeline(config=cfg, mode="auto", async_frames=af, reserve=True)
    else:
        main()
