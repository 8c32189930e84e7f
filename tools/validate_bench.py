"""Time tabi_validate (N3) on device-resident inputs for the C2/C3/C4 packs:
host-call latency (median of 20, the call synchronizes internally) and texels
checked per second.  Needs a CUDA device."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import chartgen  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402


def main():
    ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=16384)
    for cs in (chartgen.config2(0), chartgen.config3(0), chartgen.config4(0)):
        _, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs))
        xy = torch.from_numpy(cs.xy).cuda()
        st = torch.from_numpy(cs.start).cuda()
        pd = torch.from_numpy(pl.view(np.uint8).copy()).cuda()
        m = ctx.validate(xy, st, pd, cs.atlas_w, cs.atlas_h, gutter=cs.gutter)
        ts = []
        for _ in range(20):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m = ctx.validate(xy, st, pd, cs.atlas_w, cs.atlas_h, gutter=cs.gutter)
            ts.append((time.perf_counter() - t0) * 1e3)
        ms = statistics.median(ts)
        print(json.dumps(dict(workload=cs.name, n=cs.n_charts, atlas=cs.atlas_w, ms=round(ms, 3),
                              atlas_texels_per_s=cs.atlas_w * cs.atlas_h / ms * 1e3,
                              covered=m["covered"], occupancy=round(m["occupancy"], 4),
                              l2_stretch=m["l2_stretch"], overlap=m["overlap"],
                              gutter=m["gutter"], oob=m["oob"], launches=m["gpu_launches"])))
    ctx.close()


if __name__ == "__main__":
    main()
