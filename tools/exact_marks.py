"""Summarise EXPROF lines (tools/exact_marks.sh): per mark, microseconds since mark 1 of the row's
leader CTA, for the last sample() call."""
import collections
import re
import sys

txt = open(sys.argv[1]).read().split("---")
blk = [b for b in txt if "EXPROF" in b][-1]
t = collections.defaultdict(dict)
for m in re.finditer(r"EXPROF r(\d+) c(\d+) m(\d+) (\d+)", blk):
    r, c, k, v = map(int, m.groups())
    t[(r, c)].setdefault(k, []).append(v)
for (r, c), d in sorted(t.items()):
    t0 = d[1][0]
    print(f"row {r} cta {c}: " + "  ".join(f"m{k}:{(v[-1] - t0) / 1000:.1f}" if k < 23 else f"m{k}:{v[-1]}" + (f"x{len(v)}" if len(v) > 1 else "")
                                          for k, v in sorted(d.items())))
