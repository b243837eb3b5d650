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


if __name__ == "__main__":
    main()
