"""Summarise an ncu --set full report (read here, no GPU) into profiles/:
   python tools/ncu_summary.py gpurun_out/<tag>/full.ncu-rep <config> <round-tag>
writes profiles/ncu_<round-tag>_<config>.txt (key metrics per kernel) and updates
profiles/ncu_traffic.json {config_kernel: dram bytes read+write per launch} (and {config: stream_kernel's})."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, cfg, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out, traffic = [], {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        out.append(name)
        vals = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"  {k} = {r[i]} {units[i]}")
                vals[k] = (r[i], units[i])
        rd = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * SCALE.get(vals["dram__bytes_read.sum"][1], 1)
        wr = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * SCALE.get(vals["dram__bytes_write.sum"][1], 1)
        out.append(f"  dram read+write per launch = {rd + wr:.0f} bytes")
        traffic.setdefault(name.split()[-1].split("<")[0], rd + wr)
    path = os.path.join(root, "profiles", f"ncu_{tag}_{cfg}.txt")
    open(path, "w").write(f"# ncu --set full --clock-control none, {rep}\n" + "\n".join(out) + "\n")
    tj = os.path.join(root, "profiles", "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    for k, v in traffic.items():  # per (config, kernel); bench.py reports the dominant kernel's
        d[f"{cfg}_{k}"] = v
    if "stream_kernel" in traffic:
        d[cfg] = traffic["stream_kernel"]
    json.dump(d, open(tj, "w"), indent=1)
    print(open(path).read())


if __name__ == "__main__":
    main()
