"""Minimal driver for ncu: W warm-up calls then one call of the bench workload.

    python tools/profile_once.py [--workload C5|C3|C2|C4|...] [--rho 1.5] [--warmup 3] [--atlases 512]
C5: one tabi_pack_many of the batch (4 kernels: reset, proxies, sort+slots,
pack queue); single-pack workloads: one tabi_pack (reset, proxy, sort+prep,
fused wave, select; with TABI_GRAPH=0, see below).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_07782_b200 import Context, concat_chart_sets, spec_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C5")
ap.add_argument("--rho", type=float, default=1.5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--atlases", type=int, default=512)
a = ap.parse_args()
if a.workload == "C5":
    sets = bench.c5_sets(list(range(a.atlases)))
    xy, cst, abase, res = concat_chart_sets(sets)
    ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=4096)
    xy_d, cst_d = torch.from_numpy(xy).cuda(), torch.from_numpy(cst).cuda()
    for _ in range(a.warmup + 1):
        st, pl, infos, ast, bi = ctx.pack_many(xy_d, cst_d, abase, spec_of(sets[0]), res_xy=res)
    torch.cuda.synchronize()
    print("atlases", len(sets), "evaluated", bi.candidates_evaluated, "launches/pack", bi.gpu_launches)
else:
    # ncu cannot profile the kernel nodes of a graph that holds a conditional
    # node (the device-side wave loop): the host-driven loop enqueues the same
    # kernels one by one
    os.environ["TABI_GRAPH"] = "0"
    cs, _ = bench.workload(a.workload, 0, a.rho)
    ctx = Context(0, max_charts=max(cs.n_charts, 1024), max_vertices=cs.n_vertices + 16,
                  max_atlas_side=max(cs.atlas_w, cs.atlas_h))
    xy = torch.from_numpy(cs.xy).cuda()
    st = torch.from_numpy(cs.start).cuda()
    for _ in range(a.warmup + 1):
        s, _, info = ctx.pack(xy, st, spec_of(cs, **bench.WORKLOAD_SPEC.get(a.workload, {})))
    torch.cuda.synchronize()
    print("m", info.scale_index, "launches/pack", info.gpu_launches)
