"""Quick probe of the batch pipeline (tabi_pack_many) on C5: per-stage device
times (TABI_TIMING) and the batch kernel's phase cycles.

    python tools/many_probe.py [--atlases 512] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_07782_b200 import Context, concat_chart_sets, spec_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--atlases", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
sets = bench.c5_sets(list(range(a.atlases)))
xy, cst, abase, res = concat_chart_sets(sets)
ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=4096)
xy_d, cst_d = torch.from_numpy(xy).cuda(), torch.from_numpy(cst).cuda()
spec = spec_of(sets[0])
os.environ["TABI_TIMING"] = "0"
for _ in range(2):
    ctx.pack_many(xy_d, cst_d, abase, spec, res_xy=res)
os.environ["TABI_TIMING"] = "1"
for _ in range(a.reps):
    st, pl, infos, ast, bi = ctx.pack_many(xy_d, cst_d, abase, spec, res_xy=res)
    cyc = list(bi.cycles)
    tot = sum(cyc) or 1
    print(f"device {bi.device_ms:.3f} ms  stages " + " ".join(f"{v:.3f}" for v in bi.stage_ms) +
          f"  items {bi.candidates_evaluated}  cycles raster/pairs/pack " +
          " / ".join(f"{100.0 * c / tot:.1f}%" for c in cyc) +
          f"  per item us {tot / bi.candidates_evaluated / 1965.0:.1f}"
          f"  tail {bi.tail_ms:.3f} ms  busy {100 * bi.busy_frac:.1f}%", flush=True)
