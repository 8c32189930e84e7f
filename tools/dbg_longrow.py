"""Candidate records GPU vs oracle for the long-row case (GPU box)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import chartgen  # noqa: E402
import oracle  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402
oracle.build()
rng = np.random.default_rng(3)
polys = []
N = int(os.environ.get("N", "3000"))
for _ in range(N):
    a, b = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    polys.append([(0, 0), (a, 0), (a, b), (0, b)])
cs = chartgen.from_polygons(polys, int(os.environ.get("W", "16384")), 64)
ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=16384)
M = int(os.environ.get("M", "64"))
st, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs, scale_count=M))
sto, plo, io, co = oracle.pack(cs, with_cands=True, scale_count=M)
gc = ctx.candidates(M)
print("winner gpu", info.scale_index, "oracle", io.scale_index, "rows", info.rows, io.rows)
for m in range(M, 0, -1):
    if not gc["evaluated"][m - 1]:
        continue
    o = co[m - 1]
    g = {f: int(gc[f][m - 1]) for f in ("success", "score", "rows", "knees_found", "knee_rows")}
    oo = {f: int(getattr(o, f)) for f in ("success", "score", "rows", "knees_found", "knee_rows")}
    if g != oo:
        print(m, "gpu", g, "oracle", oo)
for f in ("tx", "ty", "mirror_x"):
    d = np.nonzero(pl[f] != plo[f])[0]
    print(f, "mismatches", len(d), d[:10], pl[f][d[:5]], plo[f][d[:5]])
