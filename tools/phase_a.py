"""Per-kernel device times of the c3 step under SAMPLER_DBG switches (development tool).
   python tools/phase_a.py  -> one JSON line per switch value (run in fresh processes)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import torch
    from tools.kbench import c3_bench
    r = c3_bench()
    print(json.dumps({"dbg": os.environ.get("SAMPLER_DBG", "0"), "stagger": os.environ.get("SAMPLER_STAGGER"), **r}))
else:
    for d in sys.argv[1:] or ["0", "1", "2", "4", "7"]:
        dd, _, stg = d.partition(":")
        env = dict(os.environ, SAMPLER_DBG=dd, SAMPLER_STAGGER=stg or "0")
        out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-500:], flush=True)
