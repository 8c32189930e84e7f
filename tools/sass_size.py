"""Static SASS size of one kernel by source file / line range (no GPU).

    python tools/sass_size.py <kernel_substring> <file.cu> [PHASES-style ranges]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
kname, cu = sys.argv[1], sys.argv[2]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2602_07782_b200", "libtabi.so")],
               cwd=tmp, capture_output=True)
stem = os.path.basename(cu).replace(".cu", "")
cub = [f for f in os.listdir(tmp) if f.startswith(stem + ".")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
fn = None
line = ("?", 0)
cnt = collections.Counter()
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        fn = m.group(1)
        continue
    if fn is None or kname not in fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        cnt[line] += 1
tot = sum(cnt.values())
print("instructions", tot, "bytes", tot * 16)
ph = []
for item in (sys.argv[3].split(",") if len(sys.argv) > 3 else []):
    name, rng = item.split(":")
    fnm = os.path.basename(cu)
    if "@" in rng:
        fnm, rng = rng.split("@")
    lo, hi = map(int, rng.split("-"))
    ph.append((name, fnm, lo, hi))
bk = collections.Counter()
for (f, l), n in cnt.items():
    bk[next((nm for nm, fnm, lo, hi in ph if fnm == f and lo <= l <= hi), "other:" + f)] += n
for nm, n in bk.most_common(30):
    print(f"  {nm:28s} {n:7d} instr  {100.0 * n / tot:5.1f}%")
