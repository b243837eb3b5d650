import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2512_12945_b200 import Mapper, scenes
wl = scenes.workload(3, device="cuda")
m = Mapper(**wl.mapper_kwargs)
fr = [wl.make_frame(i) for i in range(8)]
for i, f in enumerate(fr):
    h, w = f.camera["height"], f.camera["width"]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = m.integrate_depth(f.depth, f.features.reshape(h, w, -1), f.camera, pose=f.pose)
    torch.cuda.synchronize(); print("frame", i, "wall ms", round((time.perf_counter()-t0)*1e3, 2), "kernel_ms", round(r.kernel_ms, 2), "touched", r.touched_voxels, "stats", m.engine_stats()["voxel_capacity"], flush=True)
