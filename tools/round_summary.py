"""Copy one tools/round_r02.sh session (gpurun_out/<tag>/) into profiles/ (read here, no GPU):
   python tools/round_summary.py gpurun_out/<tag> <round-tag>
writes profiles/bench_<round>_<cfg>.json for every bench line, bench_ref_<round>_c3.json,
configs_<round>.txt (one line per config: step, raw-launch step, rows/s, dominant kernel, its
roofline fraction, every kernel's time, e2e), launches_<round>_{c3,c2}.{csv,txt} (per-kernel mean /
min / share of the ncu launch list), clocks_<round>.csv, box_<round>.txt, and runs
tools/ncu_summary.py on the full captures (ncu_<round>_{c3,c2}.txt)."""
import collections
import csv
import glob
import io
import json
import os
import shutil
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, rnd = sys.argv[1], sys.argv[2]
P = os.path.join(ROOT, "profiles")


def last_json(path):
    for l in reversed(open(path).read().strip().splitlines()):
        if l.startswith("{"):
            return json.loads(l)
    raise ValueError(path)


lines = [f"# round {rnd} ({src}, one B200 box, graph-replayed bench.py lines; rotation >= 2x L2 for every config)"]
order = ["c3", "c1", "c2", "c4"] + [f"c5_b{b}" for b in (1, 2, 4, 8, 16, 32)] + \
    ["c3_vocab1_p2p", "c3_vocab1_nccl", "c2_vocab1_p2p"]
for name in order:
    f = os.path.join(src, f"bench_{name}.json")
    if not os.path.exists(f):
        continue
    d = last_json(f)
    open(os.path.join(P, f"bench_{rnd}_{name}.json"), "w").write(json.dumps(d) + "\n")
    ro = d["roofline"]
    kt = {k: round(v, 1) for k, v in (ro.get("kernel_times_us") or {}).items()}
    lines.append(f"{d['config']['workload']:4s} {d['config']['parallelism']:22s} B={d['config']['B']:<5d} step_us={d['ms_per_step'] * 1e3:8.2f} "
                 f"raw_launch_us={d.get('ms_per_step_raw_launch', float('nan')) * 1e3:8.2f} rows/s={d['value']:.3g} "
                 f"dominant={ro['kernel']} frac={ro['frac']:.3f} kernels_us={kt} e2e_rows/s={d['e2e']['value']:.3g} "
                 f"sm_mhz={d['clocks']['sm_mhz']} reasons={d['clocks']['reasons']}")
open(os.path.join(P, f"configs_{rnd}.txt"), "w").write("\n".join(lines) + "\n")
if os.path.exists(os.path.join(src, "bench_ref.json")):
    open(os.path.join(P, f"bench_ref_{rnd}_c3.json"), "w").write(json.dumps(last_json(os.path.join(src, "bench_ref.json"))) + "\n")
for f, dst in (("smi.txt", f"box_{rnd}.txt"), ("clocks.csv", f"clocks_{rnd}.csv"), ("parity.json", f"parity_{rnd}.json"),
               ("parity_sharded4.json", f"parity_{rnd}_sharded4.json")):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(P, dst))
for cfg in ("c3", "c2"):
    lf = os.path.join(src, f"launches_{cfg}.csv")
    if not os.path.exists(lf):
        continue
    shutil.copy(lf, os.path.join(P, f"launches_{rnd}_{cfg}.csv"))
    rows = list(csv.reader(io.StringIO("".join(l for l in open(lf) if l.startswith('"')))))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    t = collections.defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            t[r[ki]].append(v / 1000.0 if r[ui] in ("ns", "nsecond") else v)
    tot = sum(sum(v) for v in t.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised), {src}"]
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[:50]:50s} n={len(v):4d} mean_us={statistics.mean(v):9.2f} min_us={min(v):9.2f} share={sum(v) / tot:.3f}")
    open(os.path.join(P, f"launches_{rnd}_{cfg}.txt"), "w").write("\n".join(out) + "\n")
    rep = os.path.join(src, f"full_{cfg}.ncu-rep")
    if os.path.exists(rep):
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, cfg, rnd], check=False)
print(open(os.path.join(P, f"configs_{rnd}.txt")).read())
