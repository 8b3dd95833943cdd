"""Warp-stall reasons summed over a source-line range of one kernel, from an ncu report (read here):
   python tools/ncu_stalls.py <report> <kernel-regex> <mangled-substring> <file.cuh> <first> <last>
(the in-tree .so must be the one the report was taken with)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kre, fn, src, lo, hi = sys.argv[1:7]
lo, hi = int(lo), int(hi)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Address")
d = [r for r in rows if len(r) == len(h) and r[0].startswith("0x")]
base = int(d[0][0], 16)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2506_22033_b200", "libsampler_b200.so")],
               cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
line_of, infn, loc = {}, False, None
for l in sass.splitlines():
    if l.startswith("//----") and ".text." in l:
        infn = fn in l
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        loc = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and loc:
        line_of[int(m.group(1), 16)] = loc
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
ie = h.index("Instructions Executed")
S, tot_all, ins = collections.Counter(), 0.0, 0.0
for r in d:
    loc = line_of.get(int(r[0], 16) - base, ("?", 0))
    v = sum(float(r[i] or 0) for i in cols)
    tot_all += v
    if loc[0] == src and lo <= loc[1] <= hi:
        ins += float(r[ie] or 0)
        for i in cols:
            S[h[i]] += float(r[i] or 0)
t = sum(S.values())
print(f"lines {src}:{lo}-{hi}: {t:.0f} samples = {100 * t / max(tot_all, 1):.1f}% of the kernel; {ins:.0f} warp instructions")
for k, v in S.most_common(10):
    print(f"  {k:28s} {100 * v / max(t, 1):5.1f}%")
