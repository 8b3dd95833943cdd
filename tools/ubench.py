"""Run tools/ubench.cu microbenchmarks (build first; see the .cu header)."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libubench.so")


def build():
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
           "-fPIC", "-o", SO, os.path.join(HERE, "ubench.cu")]
    subprocess.check_call(cmd)


def main():
    if not os.path.exists(SO):
        build()
    lib = ctypes.CDLL(SO)
    lib.ub_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_int, ctypes.c_void_p]
    n = 256 * 152064
    xs = [(2 * torch.randn(n, device="cuda")).to(torch.bfloat16) for _ in range(5)]
    out = torch.zeros(4096, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    for kind, grids in ((0, (296,)), (1, (296, 592, 1184, 2368))):
        for mode in range(4):
            for grid in grids:
                for i in range(5):
                    lib.ub_run(kind, mode, xs[i].data_ptr(), n * 2, out.data_ptr(), grid, st)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                iters = 50
                for i in range(iters):
                    lib.ub_run(kind, mode, xs[i % 5].data_ptr(), n * 2, out.data_ptr(), grid, st)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / iters * 1000
                res[f"{'tma' if kind == 0 else 'ldg'}_m{mode}_g{grid}"] = (round(us, 2), round(n * 2 / us / 1e3, 1))
    lib.ub_gen.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    for cfg, grids in ((0, (148,)), (1, (148,)), (2, (148, 296)), (3, (148, 296)), (4, (148,)), (5, (296, 592, 888))):
        for grid in grids:
            for i in range(5):
                lib.ub_gen(cfg, xs[i].data_ptr(), n * 2, out.data_ptr(), grid, st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(50):
                lib.ub_gen(cfg, xs[i % 5].data_ptr(), n * 2, out.data_ptr(), grid, st)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 50 * 1000
            res[f"gen{cfg}_g{grid}"] = (round(us, 2), round(n * 2 / us / 1e3, 1))
    lib.ub_xu.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    for kind in (0, 1):
        grid, iters = 148 * 4, 2000
        lib.ub_xu(kind, out.data_ptr(), grid, iters, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.ub_xu(kind, out.data_ptr(), grid, iters, st)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000
        n_exp = grid * 512 * iters * 8
        res[f"xu{kind}"] = (round(us, 1), "exp/clk/SM @1965MHz", round(n_exp / (us * 1e-6) / 148 / 1.965e9, 2))
    lib.ub_chain.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    for kind in range(5):
        iters = 20000
        lib.ub_chain(kind, out.data_ptr(), iters, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.ub_chain(kind, out.data_ptr(), iters, st)
        e1.record()
        torch.cuda.synchronize()
        ns = e0.elapsed_time(e1) * 1e6 / iters
        res[f"chain{kind}_ns_per_link"] = round(ns, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
