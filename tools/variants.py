"""A/B timing of tuning-constant variants of the library on one box.

Build here:   python tools/variants.py build NAME=-DSMP_KCW=28,-DSMP_KNS=3 ...
              (variants land in .variants/NAME.so; 'base' = the default constants)
Run on box:   python tools/variants.py run ROUNDS   (swaps each .so into place, runs the c3 bench,
              alternating variants; prints ms_per_step and the per-kernel times)."""
import json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VD = os.path.join(ROOT, ".variants")  # git-ignored; travels to the box

if sys.argv[1] == "build":
    from paper_2506_22033_b200 import build as b
    os.makedirs(VD, exist_ok=True)
    for spec in ["base="] + sys.argv[2:]:
        name, flags = spec.split("=", 1)
        b.build(force=True, out=os.path.join(VD, name + ".so"), extra=[f for f in flags.split(",") if f])
        print("built", name)
else:
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    lib = os.path.join(ROOT, "paper_2506_22033_b200", "libsampler_b200.so")
    names = sorted(f[:-3] for f in os.listdir(VD) if f.endswith(".so"))
    for r in range(rounds):
        for n in names:
            shutil.copy(os.path.join(VD, n + ".so"), lib)
            out = subprocess.run([sys.executable, "bench.py", "--steps", "1000", "--warmup", "20", "--no-cpu-baseline",
                                  "--e2e-steps", "3"], cwd=ROOT, capture_output=True, text=True, timeout=300).stdout
            d = json.loads(out.strip().splitlines()[-1])
            print(r, n, round(d["ms_per_step"] * 1e3, 2), {k: round(v, 2) for k, v in d["roofline"]["kernel_times_us"].items()}, flush=True)
