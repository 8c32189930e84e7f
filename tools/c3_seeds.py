"""Per-seed C3 latency (device span of tabi_pack, inputs in HBM) -- the
distribution behind the bench line's p50 / p99.

    python tools/c3_seeds.py [--rho 1.5] [--reps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import chartgen  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rho", type=float, default=1.5)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
ctx = Context(0, max_charts=4096, max_vertices=1 << 17, max_atlas_side=4096)
allt = []
for seed in range(8):
    cs = chartgen.config3(seed, rho=a.rho)
    xy, st = torch.from_numpy(cs.xy).cuda(), torch.from_numpy(cs.start).cuda()
    ts = []
    for i in range(a.reps + 3):
        _, _, info = ctx.pack(xy, st, spec_of(cs))
        if i >= 3:
            ts.append(info.device_ms)
    allt += ts
    print(f"seed {seed} m {info.scale_index} launches {info.gpu_launches} median {np.median(ts):.4f} ms",
          flush=True)
print(f"rho {a.rho}: p50 {np.percentile(allt, 50):.4f} p99 {np.percentile(allt, 99):.4f} "
      f"mean {np.mean(allt):.4f} ms")
