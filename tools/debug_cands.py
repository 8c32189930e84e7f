"""Print GPU vs oracle per-candidate outcomes for one case (debug aid).

    python tools/debug_cands.py <chartgen expr> [t_opt_bp] [TABI_WAVE]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import chartgen  # noqa: E402,F401
import oracle  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402

cs = eval("chartgen." + sys.argv[1])
t = int(sys.argv[2]) if len(sys.argv) > 2 else cs.t_opt_bp
if len(sys.argv) > 3:
    os.environ["TABI_WAVE"] = sys.argv[3]
ctx = Context(0, max_charts=max(cs.n_charts, 1024), max_vertices=cs.n_vertices + 16)
st, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs, t_opt_bp=t))
sto, plo, infoo, co = oracle.pack(cs, with_cands=True, t_opt_bp=t)
gc = ctx.candidates(cs.scale_count)
print("gpu", st, info.scale_index, info.l2_stretch, "oracle", sto, infoo.scale_index, infoo.l2_stretch)
for m in range(cs.scale_count, 0, -1):
    g = gc[m - 1]
    o = co[m - 1]
    if not g["evaluated"]:
        continue
    fields = ("success", "score", "rows", "prefix_rows", "p", "switched_at")
    gv = tuple(int(g[f]) for f in fields)
    ov = tuple(int(getattr(o, f)) for f in fields)
    print(m, "OK " if gv == ov else "BAD", "gpu", gv, "oracle", ov)
