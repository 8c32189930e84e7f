"""Minimal driver for ncu: W warm-up packs then one pack of the bench workload.

    python tools/profile_once.py [--workload C3] [--rho 0.5] [--warmup 3]
Each pack launches 8 kernels (proxy, sort, prep, profile tiles, profile large, offsets, pack, select).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
ap.add_argument("--rho", type=float, default=0.5)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
cs, _ = bench.workload(a.workload, 0, a.rho)
ctx = Context(0, max_charts=max(cs.n_charts, 1024), max_vertices=cs.n_vertices + 16,
              max_atlas_side=max(cs.atlas_w, cs.atlas_h))
xy = torch.from_numpy(cs.xy).cuda()
st = torch.from_numpy(cs.start).cuda()
for _ in range(a.warmup + 1):
    s, _, info = ctx.pack(xy, st, spec_of(cs))
torch.cuda.synchronize()
print("m", info.scale_index, "launches/pack", info.gpu_launches)
