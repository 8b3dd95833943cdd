"""Runs tools/ubench_esum.cu: elements per clock per SM of the exp-sum inner-loop variants."""
import ctypes, os, subprocess, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "gpurun_out", "libubench_esum.so")
os.makedirs(os.path.dirname(so), exist_ok=True)
subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                "-fPIC", "-o", so, os.path.join(ROOT, "tools", "ubench_esum.cu")], check=True)
lib = ctypes.CDLL(so)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(nsm * 1024, device="cuda")
clk = 1.965e9
for v, u in [(0, 1), (0, 2), (0, 4), (1, 1), (1, 2), (1, 4), (2, 2), (3, 2), (4, 2), (4, 4)]:
    for thr in (256, 512, 1024):
        ms = ctypes.c_float()
        iters = 200
        rc = lib.run_esum(v, u, thr, nsm, iters, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
        elems = nsm * iters * 2048 * 8
        print(f"V{v} unroll{u} threads{thr:5d}: {elems / (ms.value * 1e-3) / nsm / clk:6.2f} elem/clk/SM  rc={rc}")
