"""Warp-stall samples and executed instructions per CUDA source line, from an ncu report's SASS page
and the line table of the library's cubin (nvdisasm -g), read here without a GPU:
   python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> <mangled-function-substring> [top]
(the .so must be the one the report was taken with)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kre, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
by_inst = len(sys.argv) > 5 and sys.argv[5] == 'inst'

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Address")
d = [r for r in rows if len(r) == len(h) and r[0].startswith("0x")]
ws, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(d[0][0], 16)

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2506_22033_b200", "libsampler_b200.so")],
               cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
line_of = {}
cur, infn, loc = None, False, None
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

f = lambda x: float(x or 0)
S, I = collections.Counter(), collections.Counter()
for r in d:
    loc = line_of.get(int(r[0], 16) - base, ("?", 0))
    S[loc] += f(r[ws])
    I[loc] += f(r[ie])
tot = sum(S.values())
srcs = {}
print("samples", tot)
for loc, v in (I if by_inst else S).most_common(top):
    v = S[loc]
    path = os.path.join(ROOT, "paper_2506_22033_b200", "csrc", loc[0])
    if loc[0] not in srcs and os.path.exists(path):
        srcs[loc[0]] = open(path).read().splitlines()
    txt = srcs.get(loc[0], [""] * (loc[1] + 1))[loc[1] - 1].strip() if loc[1] else ""
    print("%5.1f%% %10d  %s:%d  %s" % (100 * v / tot, I[loc], loc[0], loc[1], txt[:90]))
