"""Ablation table on the GPU path (P:1052 and the ablation
table after): mean L2 stretch and median pack time per mode over a
seeded corpus of the paper's workload families.  Prints one JSON line per
mode and a markdown table.  Needs a CUDA device."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import chartgen  # noqa: E402
from paper_2602_07782_b200 import ABLATIONS, Context, spec_of  # noqa: E402


def corpus():
    out = [chartgen.config2(s) for s in range(8)]
    out += [chartgen.small_case(s, n=400, family="uv", side=1024, rho=0.9) for s in range(4)]
    out += [chartgen.config3(s, rho=r) for s in range(2) for r in (0.5, 2.0)]
    out += [chartgen.generate("lightmap", 2500, 2048, 2048, s, rho=0.8, name=f"lm-{s}")
            for s in range(2)]
    return out


def main():
    ctx = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=16384)
    rows = {}
    cs_all = corpus()
    for name, kw in ABLATIONS.items():
        st_all, ts = [], []
        for cs in cs_all:
            spec = spec_of(cs, **kw)
            ctx.pack(cs.xy, cs.start, spec)  # warm (graph capture)
            times = []
            for _ in range(5):
                t0 = time.perf_counter()
                _, _, info = ctx.pack(cs.xy, cs.start, spec)
                times.append((time.perf_counter() - t0) * 1e3)
            st_all.append(info.l2_stretch)
            ts.append(statistics.median(times))
        rows[name] = dict(mode=name, mean_stretch=sum(st_all) / len(st_all),
                          median_ms=statistics.median(ts), n=len(cs_all))
        print(json.dumps(rows[name]))
    print("| mode | mean L2 stretch | median host-call ms | paper (P:1052) |")
    print("|---|---|---|---|")
    paper = {"tabi": 2.16, "tight_only": 2.33, "balanced_only": 2.27, "chameleon": 2.48}
    for name, r in rows.items():
        print(f"| {name} | {r['mean_stretch']:.4f} | {r['median_ms']:.3f} | {paper[name]} |")
    ctx.close()


if __name__ == "__main__":
    main()
