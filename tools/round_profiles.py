"""Copy one tools/gpu_round.sh session into profiles/ (read here, no GPU):
   python tools/round_profiles.py gpurun_out/<tag> <round-tag> [config]
writes profiles/{bench,bench_ref}_<round>_<cfg>.json, launches_<round>_<cfg>.{csv,txt} (per-kernel
mean / min / share of the ncu launch list), clocks_<round>_<cfg>.txt (nvidia-smi samples taken
during the bench), box_<round>.txt, and runs tools/ncu_summary.py on the full capture."""
import collections
import csv
import os
import shutil
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, rnd = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "c3"
P = os.path.join(ROOT, "profiles")


def last_line(path):
    return open(path).read().strip().splitlines()[-1] + "\n"


open(os.path.join(P, f"bench_{rnd}_{cfg}.json"), "w").write(last_line(os.path.join(src, "bench.json")))
open(os.path.join(P, f"bench_ref_{rnd}_{cfg}.json"), "w").write(last_line(os.path.join(src, "bench_ref.json")))
shutil.copy(os.path.join(src, "smi.txt"), os.path.join(P, f"box_{rnd}.txt"))

# launch list: gpu__time_duration per launch, grouped by kernel name
lines = [l for l in open(os.path.join(src, "launches.csv")) if l.startswith('"')]
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(P, f"launches_{rnd}_{cfg}.csv"))
per = collections.defaultdict(list)
for r in csv.DictReader(lines):
    if r["Metric Name"] == "gpu__time_duration.sum":
        per[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]) / 1e3)
tot = sum(sum(v) for v in per.values())
with open(os.path.join(P, f"launches_{rnd}_{cfg}.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised), {src}\n")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        f.write("%-50s n=%4d mean_us=%9.2f min_us=%9.2f share=%.3f\n" % (k, len(v), statistics.mean(v), min(v), sum(v) / tot))

# clocks sampled during the bench
rows = [r for r in csv.reader(open(os.path.join(src, "clocks.csv"))) if r and r[0].strip().isdigit()]
mhz = [float(r[1].split()[0]) for r in rows]
load = [m for m, r in zip(mhz, rows) if float(r[3].split()[0]) > 150] or mhz
reasons = {name: sorted({r[i].strip() for r in rows}) for i, name in
           ((5, "hw_slowdown"), (6, "hw_thermal"), (7, "sw_thermal"), (8, "sw_power_cap"))}
with open(os.path.join(P, f"clocks_{rnd}_{cfg}.txt"), "w") as f:
    f.write("nvidia-smi -lms 200 during python bench.py (%s): samples=%d sm_mhz min=%.0f median(under load)=%.0f max=%.0f "
            "power_w max=%.0f active_reasons=%s %s\n" % (src, len(rows), min(mhz), statistics.median(load), max(mhz),
                                                       max(float(r[3].split()[0]) for r in rows),
                                                       sorted({r[4].strip() for r in rows}), reasons))

rep = os.path.join(src, "full.ncu-rep")
if os.path.exists(rep):
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, cfg, rnd], check=True)
print(open(os.path.join(P, f"launches_{rnd}_{cfg}.txt")).read() + open(os.path.join(P, f"clocks_{rnd}_{cfg}.txt")).read())
