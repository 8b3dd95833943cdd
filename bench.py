#!/usr/bin/env python
"""Benchmark of the sampling hot path (one "step" = one full decode-step sampling call on a
[B x V] batch: penalties -> temperature -> softmax -> top-k/top-p/min-p -> Philox draw ->
logprobs -> history append), BASELINE.json metric:
    "sampled rows/s & HBM GB/s vs 8 TB/s, B=256 V=152064 top-k/top-p+penalties"

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--shard rows|split|vocab]
      --shard rows  (default) every rank samples its own batch of the config (replicas, weak scaling)
      --shard split one global batch split by rows across the ranks (batch-row sharding, strong)
      --shard vocab one global batch split by vocabulary (TP lm_head style; strong); also at
                    N=1 (world-1 process group) to time the sharded step's own overheads
      --exchange p2p|nccl  vocab mode: one-shot peer exchange (default) or an NCCL all-gather
    python bench.py --impl reference ...      # the float64 CPU oracle as the reference arm

Timing: W untimed warm-up steps, then K steps bracketed by barrier + synchronize, CUDA events on
the launching stream, max over ranks.  Steps are replayed from CUDA graphs (chunks of <=250 steps)
so the host never throttles the device.  Every step reads the next of nbuf rotating logits buffers
whose total is >= 2x the 126 MB L2 (c3: 4 x 78 MB; c1: 494 x 0.5 MB), so logits come from HBM;
NDIST distinct draws of the workload are replicated to fill them.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "sampled rows/s & HBM GB/s vs 8 TB/s, B=256 V=152064 top-k/top-p+penalties"
UNIT = "rows/s"
NDIST = 5          # distinct logits draws
L2_BYTES = 126e6
CHUNK = 250


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--batch", type=int, default=None, help="override B (c5 latency sweep)")
    ap.add_argument("--shard", default="rows", choices=["rows", "split", "vocab"])
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="--shard vocab: one-shot P2P record stores + flags (NEXT-2) or an NCCL all-gather")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--hist", type=int, default=None,
                    help="history tokens per row (NEXT-4 curve; default: the config's own)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """pynvml poller (every ~20 ms) of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        return {"sm_mhz": float(np.median(s)) if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(s)}


# ----------------------------------------------------------------------------- helpers
def algorithmic_bytes(wl, uniq_counts, esize):
    """Bytes the method must move per step: the logits once, each row's penalty
    entries (8 B), params (48 B), slot meta (16 B), outputs (token, logprob, filtered logprob,
    status: 16 B) and the history append (token 4 B + entry 8 B + meta 16 B)."""
    return wl.B * wl.V * esize + 8 * int(sum(uniq_counts)) + wl.B * (48 + 16 + 16 + 28)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(cfg, kernel="stream_kernel"):
    """DRAM bytes read + written per launch of `kernel` at `cfg`, from the committed ncu --set full
    summary (tools/ncu_summary.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(f"{cfg}_{kernel}", d.get(cfg) if kernel == "stream_kernel" else None)
    return None


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def load_parity():
    """The committed north-star parity statistics (tools/parity_stats.py on a B200): rows, flagged
    fraction at the 1e-9 excuse band and at the literal 1e-6, token mismatches, unflagged ones."""
    p = os.path.join(ROOT, "profiles", "parity_r02j.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return {k: d.get(k) for k in ("rows", "flag_frac", "flag6_frac", "mismatch_frac", "unflagged_mismatch",
                                  "prob_violations", "pass")} | {"source": "profiles/parity_r02j.json"}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


_WL = None


def _oracle_rows(args):
    from oracle import sample_row
    from tests._helpers import oracle_params
    rows, step = args
    wl = _WL
    for b in rows:
        sample_row(wl.raw[b], wl.dtype, wl.prompts[b], wl.outputs[b], oracle_params(wl.params[b]), step)
    return len(rows)


def time_paper_cpu(wl, seconds=3.0):
    """NEXT-3: the paper's column-wise CPU sampler (baselines/paper_cpu: transposed logits,
    incremental dense penalty buffers, AVX-512, one worker thread per host core)
    on the same workload, logits in host memory (the device-to-host copy is not included), tokens
    appended every step.  Returns (rows/s, threads, steps, wall)."""
    from baselines.paper_cpu import PaperCpuSampler
    s = PaperCpuSampler(wl.V, wl.B, max_output=max(len(o) for o in wl.outputs) + 4096)
    for b in range(wl.B):
        s.set_params(b, wl.params[b])
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    s.step(wl.raw, 0)  # warm-up (page-in)
    n, t0 = 0, time.perf_counter()
    while True:
        s.step(wl.raw, n + 1, append=True)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 4000:
            break
    return wl.B * n / el, s.threads, n, el


def time_oracle(wl, seconds, max_rows=None):
    """Run the oracle (as it stands) over whole rows of `wl` on all host cores (one process per
    core, BLAS threads = 1) for about `seconds`; returns (rows/s, cores, rows done, wall)."""
    import multiprocessing as mp
    global _WL
    _WL = wl
    cores = cpu_cores()
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    ctx = mp.get_context("fork")
    done, t0, step = 0, time.perf_counter(), 0
    with ctx.Pool(cores) as pool:
        while True:
            rows = list(range(wl.B))
            chunks = [(rows[i::cores], step) for i in range(cores) if rows[i::cores]]
            done += sum(pool.map(_oracle_rows, chunks))
            step += 1
            el = time.perf_counter() - t0
            if el >= seconds or (max_rows and done >= max_rows):
                break
    return done / el, cores, done, el


# ----------------------------------------------------------------------------- reference arm
def run_reference(a):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from workloads.synth import make_workload
    wl = make_workload(a.config, B=a.batch)
    cores = cpu_cores()
    # one step = one bounded sample of the workload: `cores` rows in parallel
    budget = 90.0
    import multiprocessing as mp
    global _WL
    _WL = wl
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        def step(i):
            rows = [(i * cores + j) % wl.B for j in range(cores)]
            return sum(pool.map(_oracle_rows, [([r], i) for r in rows]))
        for i in range(a.warmup):
            step(i)
        t0 = time.perf_counter()
        done, k = 0, 0
        while k < a.steps:
            done += step(a.warmup + k)
            k += 1
            if time.perf_counter() - t0 > budget:
                break
        el = time.perf_counter() - t0
    v = done / el
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": k,
        "steps_requested": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * el / k, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": a.config, "B": wl.B, "V": wl.V, "logits_dtype": wl.dtype,
                   "parallelism": f"cpu x{cores} processes"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"{cores} whole rows per step (float64 oracle, one process per core), "
                                   f"{done} rows in {el:.1f}s"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    from paper_2506_22033_b200 import Sampler
    from workloads.synth import device_logits
    from workloads.synth import make_workload

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or a.shard == "vocab":
        if world == 1:  # world-1 group: the vocab-sharded code path on one GPU
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    vocab_mode = a.shard == "vocab"
    split_mode = world > 1 and a.shard == "split"

    wls = [make_workload(a.config, B=a.batch, seed_offset=i + (0 if (vocab_mode or split_mode) else 17 * rank))
           for i in range(NDIST)]
    if a.hist:  # long histories: the config's history recipe at a.hist tokens per row
        from workloads.synth import bf16_bits_to_f32, gen_history
        hrng = np.random.default_rng(1234 + rank)
        for w in wls:
            f = bf16_bits_to_f32(w.raw) if w.dtype == "bf16" else w.raw
            hs = [gen_history(hrng, f[b], a.hist - min(128, a.hist // 2), min(128, a.hist // 2)) for b in range(w.B)]
            w.prompts[:] = [p for p, _ in hs]
            w.outputs[:] = [o for _, o in hs]
    B_global = wls[0].B
    if split_mode:  # this rank's rows of the one global batch
        from paper_2506_22033_b200.distributed import batch_row_bounds
        from workloads.synth import Workload
        blo, bhi = batch_row_bounds(B_global, world, rank)
        wls = [Workload(w.name, bhi - blo, w.V, w.dtype, w.raw[blo:bhi], w.prompts[blo:bhi], w.outputs[blo:bhi],
                        w.params[blo:bhi]) for w in wls]
    wl = wls[0]
    esize = 2 if wl.dtype == "bf16" else 4
    B, V = wl.B, wl.V
    total_steps = a.warmup + a.steps + 2 * CHUNK
    # Every step appends its sampled token to the row's history (in-kernel).  To keep the workload
    # at the config's history shape for any --steps, steps rotate over NSET independent slot sets
    # (set = step mod NSET), so each history grows by at most GROW tokens over the run.
    GROW = 256
    nset = max(1, -(-(total_steps + a.e2e_steps + 8) // GROW))
    esz0 = 2 if wl.dtype == "bf16" else 4
    NBUF = max(NDIST, -(-int(2 * L2_BYTES) // (B * V * esz0)))  # rotation >= 2x L2
    if nset % NBUF == 0:  # a slot set must not always meet the same logits buffer
        nset += 1
    L = max(len(p) + len(o) for p, o in zip(wl.prompts, wl.outputs)) + GROW + 64
    if vocab_mode:
        from paper_2506_22033_b200.distributed import vocab_shard_bounds
        lo, hi = vocab_shard_bounds(V, world, rank)
    else:
        lo, hi = 0, V
    # candidate records sized by the batch's real top-k (vocab sharding: 48 + 8 K bytes per row)
    ks = [p.top_k for p in wl.params if p.temperature >= 1e-5]
    kc = max(ks) if ks and all(1 <= k <= 128 for k in ks) else 128
    s = Sampler(V, B * nset, max_history=L, max_top_k=kc, dtype=wl.dtype, vocab_offset=lo, vocab_local=hi - lo)
    slot_sets = []
    for k in range(nset):
        sl = list(range(k * B, (k + 1) * B))
        s.set_params(sl, wl.params)
        for b in range(B):
            s.set_history(k * B + b, wl.prompts[b], wl.outputs[b])
        slot_sets.append(torch.tensor(sl, dtype=torch.int32, device=dev))
    uniq0 = [len(s.get_history(b)["uniq_ids"]) for b in range(B)]
    xd = [device_logits(w)[:, lo:hi] for w in wls]
    xs = [xd[i] if i < NDIST else xd[i % NDIST].clone() for i in range(NBUF)]  # distinct memory, >= 2x L2
    out = s._outs(B, None)
    stream = torch.cuda.current_stream()
    rb = s.record_bytes(B)
    rec = torch.empty(rb, dtype=torch.uint8, device=dev)
    gathered = torch.empty(world * rb, dtype=torch.uint8, device=dev)
    # vocab sharding: rows not bounded by the candidates need the resolve rounds (NEXT-1)
    need_resolve = vocab_mode and any(p.temperature >= 1e-5 and not (1 <= p.top_k <= kc) for p in wl.params)
    if vocab_mode:
        from paper_2506_22033_b200.distributed import (resolve_buffers, sample_vocab_sharded,
                                                       sample_vocab_sharded_p2p, setup_peer_exchange)
        rbufs = resolve_buffers(s, B, world, dev)
        if a.exchange == "p2p":
            setup_peer_exchange(s)

    def vocab_step(x, i, sl, append):
        if a.exchange == "p2p":
            return sample_vocab_sharded_p2p(s, x, i, slots=sl, append=append, out=out, resolve=need_resolve,
                                            resolve_bufs=rbufs)
        return sample_vocab_sharded(s, x, i, slots=sl, append=append, rec=rec, gathered=gathered, out=out,
                                    resolve=need_resolve, resolve_bufs=rbufs)

    def one(i):
        x = xs[i % NBUF]
        sl = slot_sets[i % nset]
        if vocab_mode:
            vocab_step(x, i, sl, True)
        else:
            s.sample(x, i, slots=sl, append=True, out=out)

    launches_per_step = None
    one(0)
    torch.cuda.synchronize()
    launches_per_step = s.last_launch_count() + (2 if vocab_mode and a.exchange == "nccl" else 0)  # + local pass
    if need_resolve:  # merge + resolve kernels (fixed round count under graphs)
        launches_per_step += 1 + s.resolve_max_rounds()

    use_graph = not a.no_graph  # (vocab sharding: the NCCL all-gather is captured in the graph too)
    graphs = {}

    def run_steps(first, n):
        if not use_graph:
            for i in range(first, first + n):
                one(i)
            return
        i = first
        while i < first + n:
            m = min(CHUNK, first + n - i)
            key = (i % NBUF, m)  # the graph only depends on buffer phase and length; step id is an arg
            g = graphs.get((i, m))
            if g is None:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=torch.cuda.Stream()):
                    for j in range(i, i + m):
                        one(j)
                graphs[(i, m)] = g
            g.replay()
            i += m

    # warm-up (also captures graphs for the warm-up chunk)
    run_steps(1, a.warmup)
    torch.cuda.synchronize()
    # pre-capture the timed graphs outside the timed region
    if use_graph:
        i = 1 + a.warmup
        while i < 1 + a.warmup + a.steps:
            m = min(CHUNK, 1 + a.warmup + a.steps - i)
            if (i, m) not in graphs:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=torch.cuda.Stream()):
                    for j in range(i, i + m):
                        one(j)
                graphs[(i, m)] = g
            i += m
        torch.cuda.synchronize()
        # graph capture enqueued nothing, but histories must match the warm-up state: fine
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        run_steps(1 + a.warmup, a.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / a.steps
    clocks = clk.summary()
    if clocks["samples"] < 3:
        # timed region too short to sample: sample over an equal-work window right after
        with ClockSampler(local) as clk2:
            t0 = time.perf_counter()
            k = 0
            while time.perf_counter() - t0 < 0.5:
                run_steps(1 + a.warmup, min(a.steps, CHUNK))
                torch.cuda.synchronize()
                k += 1
        clocks = clk2.summary()
        clocks["window"] = "post-timed equal-work window (timed region shorter than the poll period)"

    # ---- the same steps launched one by one (no CUDA graph): host launch overhead included
    ms_raw = None
    if use_graph:
        nraw = min(200, a.steps)
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for i in range(1 + a.warmup, 1 + a.warmup + nraw):
            one(i)
        r1.record(stream)
        torch.cuda.synchronize()
        ms_raw = r0.elapsed_time(r1) / nraw

    # ---- per-kernel device times (CUDA events recorded by the library on the launching stream,
    #      around each kernel; outside graphs, after the timed region): the roofline's duration
    #      The step with the library's event marks is captured in a CUDA graph and replayed, so
    #      the marks bracket each kernel's device execution (no host launch gap inside them).
    kt = None
    knames = ["stream_kernel", "select_rows_kernel", "exact_kernel"]
    if vocab_mode and a.exchange == "p2p" and not need_resolve:  # one library call: all 3 kernels marked
        knames = ["stream_kernel", "select_rows_kernel", "merge_rows_kernel"]  # (B <= 2 x SMs: merge fused)
    if not vocab_mode or knames[2] == "merge_rows_kernel":
        nk = 40
        s.set_timing(True)
        gt = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gt, stream=torch.cuda.Stream()):
            one(1 + a.warmup + a.steps)
        acc = None
        for i in range(nk):
            gt.replay()
            t = s.kernel_times_ms()
            acc = t if acc is None else [x + y for x, y in zip(acc, t)]
        s.set_timing(False)
        kt = [x / nk for x in acc]
        del gt

    # ---- e2e through the public API with host buffers (pinned), per step:
    #      H2D of the step's logits, sample, D2H of tokens + logprobs + filtered logprobs + status
    hosts = [xx.contiguous().cpu().pin_memory() for xx in xs[:2]]
    dbuf = torch.empty_like(xs[0].contiguous())
    res_h = torch.empty((4, B), dtype=torch.int32).pin_memory()
    ne = max(3, a.e2e_steps)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(ne):
        dbuf.copy_(hosts[i % 2], non_blocking=True)
        if vocab_mode:
            o = vocab_step(dbuf, 10**9 + i, None, False)
        else:
            o = s.sample(dbuf, 10**9 + i, out=out)
        res_h[0].copy_(o["tokens"], non_blocking=True)
        res_h[1].copy_(o["logprobs"].view(torch.int32), non_blocking=True)
        res_h[2].copy_(o["filtered_logprobs"].view(torch.int32), non_blocking=True)
        res_h[3].copy_(o["status"], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1) / ne
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())

    rows_total = B_global if (vocab_mode or split_mode) else B * world
    value = rows_total / (ms_step / 1000.0)
    peak, peak_src = load_peaks()
    algo = algorithmic_bytes(wl, uniq0, esize) if not vocab_mode else (B * (hi - lo) * esize + 8 * sum(uniq0))
    # the roofline's kernel: the dominant (longest) kernel of the step; achieved = the step's
    # algorithmic bytes / that kernel's mean duration; the whole step is reported too (step_frac)
    kdom = int(np.argmax(kt)) if kt else 0
    kern_s = (kt[kdom] / 1000.0) if kt else ms_step / 1000.0
    achieved = algo / kern_s / 1e9
    step_gbs = algo / (ms_step / 1000.0) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_step, "ms_per_step_raw_launch": ms_raw, "higher_is_better": True,
        "scaling": "strong" if (vocab_mode or split_mode) else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": a.config, "B": B, "V": V, "logits_dtype": wl.dtype,
                   "parallelism": (f"vocab{world}-{a.exchange}" + ("+resolve" if need_resolve else "")
                                   if vocab_mode else (f"split{world}" if split_mode else
                                   (f"rows{world}" if world > 1 else "1gpu"))),
                   "record_bytes_per_row": rb // B,
                   "l2": f"{NBUF} rotating logits buffers ({NBUF * B * (hi - lo) * esize / 1e6:.0f} MB >= 2x L2 126 MB)",
                   "history": f"{np.mean([len(p) + len(o) for p, o in zip(wl.prompts, wl.outputs)]):.0f} tokens/row "
                              f"+1 per step (appended in-kernel; {nset} rotating slot sets, each history grows "
                              f"by <= {GROW})",
                   "graph": use_graph},
        "gbs": step_gbs,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": load_traffic(a.config, knames[kdom] if kt
                                                       else "stream_kernel"),
                     "peak_source": peak_src,
                     "kernel": knames[kdom] if kt else "step",
                     "algorithmic_bytes_per_launch": algo,
                     "kernel_time_s": kern_s,
                     "kernel_times_us": ({n: kt[i] * 1e3 for i, n in
                                          enumerate(knames[:len(kt)])}
                                         if kt else None),
                     "step_gbs": step_gbs, "step_frac": step_gbs / peak},
        "clocks": clocks,
        "e2e": {"value": rows_total / (ms_e2e / 1000.0), "unit": UNIT,
                "h2d_bytes_per_step": int(B * (hi - lo) * esize), "d2h_bytes_per_step": int(16 * B)},
        "gpu_launches": int(launches_per_step * a.steps),
        "parity": load_parity(),
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        v, cores, done, el = time_oracle(wl, a.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                                "sample": f"whole batches of {a.config} (B={B}) rows, float64 oracle, one process "
                                          f"per core: {done} rows in {el:.1f}s"}
        try:
            v2, th, n2, el2 = time_paper_cpu(wl)
            line["paper_cpu"] = {"value": v2, "unit": UNIT, "cores": th, "kind": "paper column-wise CPU sampler",
                                 "cpu": cpu_model(),
                                 "sample": f"{n2} steps of {a.config} (B={B}) in {el2:.1f}s, logits in host memory "
                                           f"(D2H copy not included), AVX-512, one thread per core "
                                           f"(baselines/paper_cpu, NEXT-3)"}
        except Exception as e:  # (a comparator only: its absence never fails the GPU bench)
            line["paper_cpu"] = {"unavailable": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
