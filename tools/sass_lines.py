"""Attribute an ncu SASS-level profile to CUDA source lines (run here, no GPU).

    python tools/sass_lines.py gpurun_out/prof_X.ncu-rep <kernel_substring> <file.cu> [N]

Extracts the cubin of <file.cu> from the in-tree libtabi.so (must be the same
build the report was taken with), disassembles the kernel with line info
(`nvdisasm -g`), maps each profiled SASS instruction to its source line by
offset, and prints the N source lines with the most executed warp
instructions and warp-stall samples.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, kname, cu = sys.argv[1], sys.argv[2], sys.argv[3]
    topn = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kname}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    h = rows[hi]
    ia, ie, ws = h.index("Address"), h.index("Instructions Executed"), h.index(
        "Warp Stall Sampling (All Samples)")
    prof = [(int(r[ia], 16), float(r[ie] or 0), float(r[ws] or 0)) for r in rows[hi + 1:] if r and r[ia].startswith("0x")]
    # optional per-line stall reasons / shared-memory excess (REASONS=1)
    rcols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    xcol = h.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in h else None
    extra = {int(r[ia], 16): ([float(r[i] or 0) for i, _ in rcols],
                              float(r[xcol] or 0) if xcol is not None else 0.0)
             for r in rows[hi + 1:] if r and r[ia].startswith("0x")}
    base = min(a for a, _, _ in prof)
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2602_07782_b200", "libtabi.so")],
                   cwd=tmp, capture_output=True)
    stem = os.path.basename(cu).replace(".cu", "")
    cub = [f for f in os.listdir(tmp) if f.startswith(stem + ".")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                         text=True).stdout
    # locate the kernel's function body
    fn = None
    line = None
    off2line = {}
    src = open(os.path.join(ROOT, "paper_2602_07782_b200", "csrc", os.path.basename(cu))).read().splitlines()
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        if fn is None or (os.environ.get("MANGLED", kname)) not in fn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and line:
            off2line[int(m.group(1), 16)] = line
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    tot = [0.0, 0.0]
    for a, n, s in prof:
        key = off2line.get(a - base, ("?", 0))
        agg[key][0] += n
        agg[key][1] += s
        tot[0] += n
        tot[1] += s
    print(f"total warp instructions {tot[0]:.0f}, stall samples {tot[1]:.0f}, mapped lines {len(agg)}")
    # optional phase buckets over line ranges of <file.cu>: PHASES="name:lo-hi,..."
    if os.environ.get("PHASES"):
        ph = []
        for item in os.environ["PHASES"].split(","):
            name, rng = item.split(":")
            fn = os.path.basename(cu)
            if "@" in rng:  # name:file@lo-hi
                fn, rng = rng.split("@")
            lo, hi = map(int, rng.split("-"))
            ph.append((name, fn, lo, hi))
        bk = collections.defaultdict(lambda: [0.0, 0.0])
        for (f, l), (n, s) in agg.items():
            nm = next((name for name, fn, lo, hi in ph if fn == f and lo <= l <= hi), "other:" + f)
            bk[nm][0] += n
            bk[nm][1] += s
        for nm, (n, s) in sorted(bk.items(), key=lambda kv: -kv[1][0]):
            print(f"  phase {nm:24s} {n / tot[0] * 100:5.1f}% inst {s / max(tot[1], 1) * 100:5.1f}% stall")
    if os.environ.get("REASONS"):
        lr = collections.defaultdict(lambda: [[0.0] * len(rcols), 0.0])
        for a, _, _ in prof:
            key = off2line.get(a - base, ("?", 0))
            v, x = extra[a]
            acc = lr[key]
            acc[0] = [p + q for p, q in zip(acc[0], v)]
            acc[1] += x
        for (f, l), (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:topn]:
            v, x = lr[(f, l)]
            top = sorted(((val, c) for val, (_, c) in zip(v, rcols) if val > 0), reverse=True)[:3]
            print(f"{s:6.0f} samples  {f}:{l}  smem-excess {x:.0f}  " +
                  ", ".join(f"{c[6:]} {val:.0f}" for val, c in top))
        return
    for (f, l), (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:topn]:
        fp = os.path.join(ROOT, "paper_2602_07782_b200", "csrc", f)
        lines = src if f == os.path.basename(cu) else (
            open(fp).read().splitlines() if os.path.exists(fp) else [])
        text = lines[l - 1].strip()[:80] if 0 < l <= len(lines) else ""
        print(f"{n / tot[0] * 100:5.1f}% inst {s / max(tot[1], 1) * 100:5.1f}% stall  {f}:{l}  {text}")


if __name__ == "__main__":
    main()
