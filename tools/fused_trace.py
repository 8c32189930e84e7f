"""Fused-kernel timeline + K4 row phases on the bench workloads (GPU box).

    TABI_NVCC_EXTRA=-DTABI_PHASE_TRACE python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)"
    python tools/fused_trace.py

Row phases are SM cycles in the library (only in a -DTABI_PHASE_TRACE build);
printed here as ns per row at the B200's 1965 MHz boost clock.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import chartgen  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402

MHZ = float(os.environ.get("SM_MHZ", "1965"))
os.environ["TABI_TIMING"] = "1"
ctx = Context(0, max_charts=25000, max_vertices=1 << 21, max_atlas_side=16384)
us = lambda v: round(v / 1000, 1)  # noqa: E731
only = os.environ.get("TRACE_MODES", "1,0").split(",")
SETS = {"C3": lambda: chartgen.config3(0, rho=0.5), "C3r15": lambda: chartgen.config3(0, rho=1.5),
        "C2": lambda: chartgen.config2(0), "C4": lambda: chartgen.config4(0, t_opt_bp=0)}
for name in os.environ.get("TRACE_SETS", "C3,C2,C4").split(","):
    cs = SETS[name]()
    for f in only:
        os.environ["TABI_FUSED"] = f
        for _ in range(3):
            st, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs))
        tr = ctx.trace()
        cands = ctx.candidates(cs.scale_count)
        ev = cands["evaluated"] != 0
        rows = int(cands["rows"][ev].sum())
        ph = tr.pop("phases")
        rp = tr.pop("raster_phases")
        fr = tr.pop("first_row_ns")
        tiles = max(tr.get("tiles", 0), 1)
        alg1_passes = tr.pop("alg1_passes", 0)
        print(name, "fused" if f == "1" else "split", "m", info.scale_index,
              "stages_us", [round(x * 1000) for x in info.stage_ms[:7]],
              {k: (us(v) if k in ("raster_end", "pack_end", "pack_wait", "raster_wait") else v)
               for k, v in tr.items()},
              "rows", rows, "ns/row", {k: round(v / MHZ * 1000 / max(rows, 1)) for k, v in ph.items()},
              "raster ns/tile", {k: round(v / MHZ * 1000 / tiles) for k, v in rp.items()},
              "first row us", {k: round(v / 1000, 1) for k, v in fr.items()},
              "alg1 passes (slot 0)", alg1_passes,
              flush=True)
