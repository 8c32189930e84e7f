"""Where the host-pointer batch's extra time goes: tabi_pack_many on C5 from
pinned host memory vs device pointers -- library device span, outer stream
events and wall clock per call.

    python tools/e2e_probe.py [--reps 5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_07782_b200 import PLACEMENT_DTYPE, Context, concat_chart_sets, spec_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
sets = bench.c5_sets(list(range(512)))
xy, cst, abase, res = concat_chart_sets(sets)
N = int(abase[-1])
ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=4096)
spec = spec_of(sets[0])
s = torch.cuda.Stream()
xy_d, cst_d = torch.from_numpy(xy).cuda(), torch.from_numpy(cst).cuda()
xy_p = torch.from_numpy(xy).pin_memory().numpy()
cst_p = torch.from_numpy(cst).pin_memory().numpy()
out_p = torch.empty(N * 32, dtype=torch.uint8).pin_memory().numpy().view(PLACEMENT_DTYPE)
modes = {"device": lambda: ctx.pack_many(xy_d, cst_d, abase, spec, res_xy=res, stream=s.cuda_stream),
         "pinned": lambda: ctx.pack_many(xy_p, cst_p, abase, spec, res_xy=res, out=out_p,
                                         stream=s.cuda_stream)}
for name, f in modes.items():
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    dev, ev, wall = [], [], []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        bi = f()[4]
        e1.record(s)
        torch.cuda.synchronize()
        wall.append(1e3 * (time.perf_counter() - t0))
        ev.append(e0.elapsed_time(e1))
        dev.append(bi.device_ms)
    st = np.zeros(4)
    if os.environ.get("TABI_TIMING") == "1":
        st = np.array(bi.stage_ms[:4])
    print(f"{name:7s} stages {np.round(st, 3)} chunks={os.environ.get('TABI_UPLOAD_CHUNKS', '8')} library {np.median(dev):.3f} ms  "
          f"outer events {np.median(ev):.3f} ms  wall {np.median(wall):.3f} ms", flush=True)
