"""Print an ncu launch list (gpu__time_duration.sum CSV) as a table with shares.

    python tools/launch_table.py gpurun_out/launches_C3.csv
"""
import csv
import sys


def main():
    lines = open(sys.argv[1]).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, vi, gi, ui = (h.index(x) for x in ("Kernel Name", "Metric Value", "Grid Size", "Metric Unit"))
    recs = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
        recs.append((r[ki].split("(")[0].split("::")[-1], r[gi], v * scale))
    tot = sum(t for _, _, t in recs)
    for name, grid, t in recs:
        print(f"{name:24s} grid={grid:>14s} {t:9.1f} us  {100 * t / tot:5.1f}%")
    print(f"{'total':24s} {'':19s} {tot:9.1f} us")


if __name__ == "__main__":
    main()
