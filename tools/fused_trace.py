"""Fused-kernel timeline + K4 row phases on the bench workloads (GPU box):
python tools/fused_trace.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import chartgen  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402

os.environ["TABI_TIMING"] = "1"
ctx = Context(0, max_charts=25000, max_vertices=1 << 21, max_atlas_side=16384)
us = lambda v: round(v / 1000, 1)  # noqa: E731
for name, cs in (("C3", chartgen.config3(0, rho=0.5)), ("C2", chartgen.config2(0)),
                 ("C4", chartgen.config4(0, t_opt_bp=0))):
    for f in ("1", "0"):
        os.environ["TABI_FUSED"] = f
        for _ in range(3):
            st, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs))
        tr = ctx.trace()
        cands = ctx.candidates(cs.scale_count)
        ev = cands["evaluated"] != 0
        rows = int(cands["rows"][ev].sum())
        ph = {k: us(v) for k, v in tr.pop("phases").items()}
        print(name, "fused" if f == "1" else "split", "m", info.scale_index,
              "stages_us", [round(x * 1000) for x in info.stage_ms[:7]],
              {k: (us(v) if k in ("raster_end", "pack_end", "pack_wait", "raster_wait") else v)
               for k, v in tr.items()},
              "rows(sum over evaluated)", rows, "packers", int(ev.sum()),
              "phase_us(sum)", ph, "ns/row", {k: round(v * 1000 / max(rows, 1)) for k, v in ph.items()},
              flush=True)
