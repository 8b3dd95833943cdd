"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count/mean/min (us)."""
import collections
import csv
import sys


def summarise(path):
    hdr = None
    data = collections.defaultdict(list)
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d.get("Metric Unit"), 1e-3)
                data[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in data.values())
    out = []
    for k, v in data.items():
        out.append(f"{k:50s} n={len(v):4d} mean_us={sum(v) / len(v):9.2f} min_us={min(v):9.2f} share={sum(v) / tot:.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
