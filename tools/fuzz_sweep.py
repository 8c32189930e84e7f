"""Wide random parity sweep on the GPU box: the first N cases of
tests/test_gpu_fuzz.py (seeded random specs, families, flags) packed by the
CUDA path and the oracle, placements compared byte for byte; prints the
mismatching cases.

    python tools/fuzz_sweep.py [N=160] [case|edge|large]
"""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np
import importlib.util
spec = importlib.util.spec_from_file_location("fz", "tests/test_gpu_fuzz.py")
fz = importlib.util.module_from_spec(spec); spec.loader.exec_module(fz)
import oracle
from paper_2602_07782_b200 import Context, spec_of
ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=16384)
bad = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 160):
    kind = sys.argv[2] if len(sys.argv) > 2 else "case"
    cs, kw = {"case": fz.case, "edge": fz.edge_case, "large": fz.large_case}[kind](i)
    st_o, pl_o, info_o, _ = oracle.pack(cs, with_cands=True, **kw)
    st_g, pl_g, info_g = ctx.pack(cs.xy, cs.start, spec_of(cs, **kw))
    same = st_o == st_g and (st_o != 0 or pl_g.tobytes() == np.ascontiguousarray(pl_o).tobytes())
    if not same:
        bad.append((i, cs.n_charts, kw, info_o.scale_index, info_g.scale_index, info_o.prefix_rows))
print("mismatches", len(bad))
for b in bad: print(b)
