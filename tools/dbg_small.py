"""Localize a failure: pack small cases one by one, fused and split (GPU box)."""
import os
import sys
import faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(60, exit=True)
import chartgen  # noqa: E402
from paper_2602_07782_b200 import Context, spec_of  # noqa: E402
mode = os.environ.get("TABI_FUSED", "1")
ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=16384)
cases = [chartgen.config1a(s) for s in range(3)] + [chartgen.small_case(s, n=48) for s in range(2)] + \
        [chartgen.config2(0), chartgen.config3(0)]
for cs in cases:
    print(mode, cs.name, end=" ", flush=True)
    st, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs), raise_on_error=False)
    print(st, info.scale_index, info.rows, ctx.last_error(), flush=True)
    if st == 3:
        break
