#!/usr/bin/env python
"""bench.py -- STEP eigenpairs/sec fp64 of the B200 MRRR solver (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config random_20000]

A "step" is one full MRRR solve (all SURVEY §8(a) rows: norms/split, root
RRR, root bisection, classification, representation tree, singleton
RQC/twisted vectors, output) of the workload through the C ABI
``mrrr_stemr`` with device-resident inputs and preallocated outputs.  The
default workload is BASELINE.json configs[1]: random tridiagonal, n=20000,
d, e iid U(-1,1) (numpy default_rng(0)), all eigenpairs, fp64.

``value`` = eigenpairs/s over the K timed steps (CUDA events on the solve
stream, L2 flushed before each step by writing a 256 MiB buffer, outside the
events; max over ranks).  ``e2e`` = the same metric through
``mrrr_stemr_host`` with pinned HOST buffers: d, e copied in and w, Z copied
out inside the timed region.  ``roofline`` = the dominant kernel's
algorithmic fp64 flop rate against the FP64 ALU peak.
``cpu_baseline`` = the sequential C oracle timed on a bounded sample on the
host cores (test infrastructure; the only other use of oracle/ here is
``--impl reference``).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1205_2107_b200 import workloads as W  # noqa: E402

EPS = 2.0 ** -52
# FP64 ALU peak: 148 SMs x 64 FP64 FMA lanes x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# algorithmic work model, in FP64-pipe slots
R_RQC = 3                   # twisted factorizations per eigenpair (yardstick)
W_DIV = 1.708e13 / 1.2945e12  # measured DFMA/s / IEEE DDIV/s (profiles/r01_microbench_fp64.json)
HBM_GBS = 6554.6            # MEASURED_PEAKS.json hbm_gbs (Z write bound)
RTOL_C = 2.0 ** -20
METRIC = "STEP eigenpairs/sec fp64 (n=20k, all pairs) at 1/2/4/8 B200; % of roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="random_20000")
    ap.add_argument("--collective", default="torch", choices=["torch", "nccl"],
                    help="N>1: the protocol's all-gathers through the torch.distributed NCCL group "
                         "(mrrr_stemr_dist + callback) or issued by the library on its own ncclComm_t (mrrr_stemr_nccl)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-pairs", type=int, default=0,
                    help="oracle sample size in eigenpairs (0: auto ~15 s)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------------------
# work model (implementation independent)
def bisection_steps(d, e, w):
    """B_j = max(1, ceil(log2(spdiam / (rtol_c |lambda_j - sigma0|)))) with the
    root shift just left of the Gershgorin interval."""
    r = np.abs(d).copy() * 0
    if len(e):
        r[:-1] += np.abs(e)
        r[1:] += np.abs(e)
    gl, gu = float(np.min(d - r)), float(np.max(d + r))
    spd = gu - gl
    tn = float(np.max(np.abs(d) + r))
    sigma0 = gl - 4 * EPS * tn
    x = spd / (RTOL_C * np.maximum(np.abs(np.asarray(w) - sigma0), 1e-300))
    return np.maximum(1, np.ceil(np.log2(x)))


class Clocks:
    """nvidia-smi sampler over the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_bench_{os.getpid()}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons, pw = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "power_w_max": max(pw) if pw else None, "reasons": sorted(reasons)}


# --------------------------------------------------------------------------
def cpu_oracle_sample(d, e, pairs: int):
    """Oracle on a bounded sample of the workload: the INDEX range of `pairs`
    eigenpairs centred in the spectrum (same matrix), single host thread."""
    import oracle  # test infrastructure (bench cpu_baseline leg only)
    oracle.build()
    n = len(d)
    pairs = max(1, min(pairs, n))
    il = (n - pairs) // 2 + 1
    iu = il + pairs - 1
    t0 = time.perf_counter()
    w, Z = oracle.stemr(d, e, il=il, iu=iu)
    dt = time.perf_counter() - t0
    return pairs / dt, dt, f"oracle_stemr INDEX il..iu={il}..{iu} ({pairs} pairs, with vectors) of the same n={n} matrix"


def _oracle_window(job):
    """One host process of the sharded baseline: the oracle on one index window."""
    cfg, il, iu = job
    import oracle  # test infrastructure (bench cpu_baseline / reference legs only)
    oracle.build()
    d, e, _ = W.make(cfg)
    t0 = time.perf_counter()
    oracle.stemr(d, e, il=il, iu=iu)
    return time.perf_counter() - t0


def cpu_oracle_sharded(cfg, n, k, seconds=12.0, cores=None):
    """The oracle as it stands on ALL host cores: `cores` independent
    processes, each solving one index window of the same matrix (SURVEY §8(d)
    "sharded": the paper's static division of eigenpairs over processes,
    P:L1139-1146), windows spread through the spectrum so that they sample
    its clusters; each window is sized for ~`seconds` of single-core work.
    Returns (pairs/s over the slowest process, cores, sample text, seconds)."""
    import multiprocessing as mpr
    import oracle
    oracle.build()  # once, before the processes start
    cores = cores or os.cpu_count() or 1
    per = auto_pairs(n, seconds)
    per = max(10, min(per, k // cores if k >= cores else 1))
    jobs = []
    for c in range(cores):
        mid = int((c + 0.5) * k / cores)
        il = max(1, min(k - per + 1, mid - per // 2 + 1))
        jobs.append((cfg, il, il + per - 1))
    with mpr.get_context("spawn").Pool(cores) as pool:
        times = pool.map(_oracle_window, jobs)
    tot = per * cores
    return (tot / max(times), cores,
            f"oracle_stemr on {cores} host processes, each one INDEX window of {per} pairs (with vectors) of the "
            f"same n={n} matrix, windows centred at ({'...'.join(str(j[1]) for j in (jobs[0], jobs[-1]))}) spread "
            f"through the spectrum; rate = {tot} pairs / slowest process", max(times))


def auto_pairs(n, seconds=15.0):
    # ~`seconds` of single-thread oracle work (measured ~0.6 us per pair per element)
    return int(max(50, min(n, seconds / (0.6e-6 * n))))


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    d, e, rng = W.make(args.config)
    n = len(d)
    k = n if rng is None else rng[1] - rng[0] + 1
    # each step: a bounded sample on every host core (~3 s of work per core
    # per step, so that warmup + steps end within a few minutes)
    steps_total = args.warmup + args.steps
    vals = []
    for i in range(steps_total):
        v, cores, desc, dt = cpu_oracle_sharded(args.config, n, k, seconds=3.0)
        if i >= args.warmup:
            vals.append((v, dt))
    value = statistics.median(v for v, _ in vals)
    line = {"metric": METRIC, "value": value, "unit": "eigenpairs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.mean(dt for _, dt in vals),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "n": n, "k": k},
            "cpu_baseline": {"value": value, "unit": "eigenpairs/s", "cores": cores,
                             "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "eigenpairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: launch N ranks, one per GPU,
    through torch.distributed.run on this node (rendezvous on 127.0.0.1), and
    pass their output through (rank 0 prints the JSON line)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import paper_1205_2107_b200 as P
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    d, e, rng = W.make(args.config)
    n = len(d)
    k = n if rng is None else rng[1] - rng[0] + 1
    kw = {} if rng is None else {"il": rng[0], "iu": rng[1]}
    dt_ = torch.tensor(d, device=dev)
    et_ = torch.tensor(e, device=dev)
    w = torch.empty(k, dtype=torch.float64, device=dev)
    Z = torch.empty((k, n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    cb = None
    comm = None
    if world > 1 and args.collective == "nccl":
        comm = P.NcclComm(dev)  # ncclUniqueId broadcast through the default process group
    elif world > 1:
        cb = P.mrrr.torch_allgather()  # the protocol's all-gathers on the torch NCCL group

    def step():
        if comm is not None:
            wa, Zl, _ = P.stemr_nccl(dt_, et_, comm, stream=stream, **kw)
            return wa, Zl
        if world > 1:
            wa, Zl, _ = P.stemr_dist(dt_, et_, rank=rank, nranks=world, allgather=cb, stream=stream, **kw)
            return wa, Zl
        return P.stemr(dt_, et_, w=w, Z=Z, stream=stream, **kw)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stats = []
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clk = Clocks(dev.index or 0)
    clk.start()
    time.sleep(1.0)  # let the sampler start before the timed region (host-side orchestration)
    step()           # and bring the clocks back up after the pause (untimed)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.random_(0, 255)  # L2 flush outside the events
        evs[i][0].record(stream)
        wk = step()[0]  # (keep no view of Z: e2e below frees it)
        evs[i][1].record(stream)
        stats.append(P.last_stats())
        hist_last = P.rqc_histogram()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = clk.stop()
    ms = [a.elapsed_time(b) for a, b in evs]
    tot_ms = sum(ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    m = wk.shape[0]
    # whole job: the m eigenpairs of a step are computed once across the ranks
    value = m * args.steps / (tot_ms / 1e3)

    # ---------------- roofline (SURVEY §8(d) work model)
    # FP64-pipe slots: a bisection step costs 2 + w_div per element, a
    # twisted factorization + solve 10 + 2 w_div, the final scale 1; R = 3
    # factorizations per eigenpair is the fixed yardstick.  Reported as
    # TFLOP/s with one slot = one DFMA = 2 flops (peak 37.2 TFLOP/s).
    w_host = wk.double().cpu().numpy()
    kv = statistics.mean(s["ms_k_vectors"] for s in stats)
    kb = statistics.mean(s["ms_k_root_bisect"] for s in stats)
    B = bisection_steps(d, e, w_host)
    slots_bis = float(np.sum(B)) * (2 + W_DIV) * n
    # The roofline UNIT is the whole step: the path's kernels run
    # concurrently on up to ten streams (the tree on a high-priority stream, the
    # vector pieces on eight side streams), so no single kernel's launch
    # duration is a share of the step (summed piece durations
    # were 1.8x the step).  achieved = the work model's FP64-pipe slots per
    # step (x2 flop) over the step time; frac = T_roof / T_step with T_roof =
    # max(W_slots / P64, 8 n m / BW).  The model
    # charges every IEEE division the paper's recurrences perform at w_div
    # slots; the kernels' projective sweeps execute none, so this is model
    # work per second (the BASELINE metric's "% of roofline"), and the
    # hardware view is the per-kernel table below: ncu-measured executed
    # FP64 instructions of each kernel against the FP64 peak (profiles/r02).
    w_slots = (float(np.sum(B)) * (2 + W_DIV) + m * (R_RQC * (10 + 2 * W_DIV) + 1)) * n
    t_alu = w_slots / (FP64_PEAK_TFLOPS * 1e12 / 2)
    t_z = 8.0 * n * m / (HBM_GBS * 1e9)
    t_roof = max(t_alu, t_z)
    t_step = tot_ms / args.steps / 1e3
    kernels, traffic, ksrc, hw_slots = None, None, None, None
    kt = os.path.join(ROOT, "profiles", "r02", f"kernel_table_{args.config}.json")
    if os.path.exists(kt):
        try:
            kj = json.load(open(kt))
            ksrc = os.path.relpath(kt, ROOT)
            kernels = {k: {"launches": round(v["launches"], 1), "ncu_ms": round(v["ms"], 3),
                           "fp64_slots_executed": v["fp64_slots"],
                           "hw_fp64_frac": round(v["hw_fp64_frac"], 4) if v["hw_fp64_frac"] else None,
                           "dram_bytes": v["dram_bytes"]}
                       for k, v in list(kj["kernels"].items())[:8]}
            traffic = sum(v["dram_bytes"] for v in kj["kernels"].values())
            hw_slots = sum(v["fp64_slots"] for v in kj["kernels"].values())
        except Exception:
            kernels = None
    roof = {"bound": "alu", "kernel": "whole step (all SURVEY §8(a) rows; kernels overlap on up to ten streams)",
            "achieved": 2 * w_slots / t_step / 1e12, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": t_roof / t_step, "traffic": traffic,
            "algorithmic_bytes": 8.0 * n * m, "t_roof_ms": 1e3 * t_roof, "t_alu_ms": 1e3 * t_alu,
            "t_z_ms": 1e3 * t_z, "w_slots": w_slots, "w_div": W_DIV, "kernel_share_of_step": 1.0,
            "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 1.965 GHz = 1.861e13 slots/s, x2 flop "
                           "(guide unit counts; microbenchmark 1.708e13 DFMA/s, profiles/r01_microbench_fp64.json); "
                           "BW = MEASURED_PEAKS.json hbm_gbs",
            "note": "achieved/frac are the work model's FP64-pipe slots (IEEE division = w_div slots, as the "
                    "paper's recurrences need) per second: model work/s, not executed instructions; "
                    "`kernels` gives each kernel's executed FP64 instructions (ncu) against the peak",
            "kernels_source": ksrc, "kernels": kernels,
            # the hardware view of the whole step: FP64-pipe slots the kernels
            # EXECUTED in one solve (ncu: DFMA + DMUL + DADD, all kernels) per
            # step time, against the FP64 peak
            "hw_fp64_slots_per_solve": hw_slots,
            "hw_step_fp64_frac": (hw_slots / t_step / (FP64_PEAK_TFLOPS * 1e12 / 2)) if hw_slots else None,
            "vector_kernels_event_ms": kv, "root_bisect_event_ms": kb,
            "root_bisect_model_work_tflops": 2 * slots_bis / (kb / 1e3) / 1e12 if kb else None}

    # ---------------- end to end through the host-buffer C ABI
    e2e = None
    if not args.no_e2e and world > 1:
        # end to end on N GPUs: pinned host d, e -> device, sharded solve, this
        # rank's Z columns and all w -> pinned host
        dh = torch.tensor(d).pin_memory()
        eh = torch.tensor(e).pin_memory()
        wh = torch.empty(k, dtype=torch.float64).pin_memory()
        Zh = torch.empty((P.mrrr.dist_capacity(k, world), n), dtype=torch.float64).pin_memory()
        ml = [0]
        torch.distributed.barrier()
        e_ms = []
        for i in range(args.steps):
            flush.random_(0, 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dt_.copy_(dh, non_blocking=True)
            et_.copy_(eh, non_blocking=True)
            wa, Zl = step()
            wh[:wa.shape[0]].copy_(wa, non_blocking=True)
            if Zl is not None and Zl.shape[1]:
                Zh[:Zl.shape[1]].copy_(Zl.T, non_blocking=True)
                ml[0] = Zl.shape[1]
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        etot = sum(e_ms)
        t = torch.tensor([etot], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        etot = float(t.item())
        e2e = {"value": m * args.steps / (etot / 1e3), "unit": "eigenpairs/s",
               "h2d_bytes_per_step": 8 * (2 * n - 1), "d2h_bytes_per_step": 8 * m + 8 * n * ml[0],
               "ms_per_step": etot / args.steps, "note": "d2h per rank: all w + own Z columns"}
    if not args.no_e2e and world == 1:
        # the host entry allocates its own device buffers: release the
        # device-resident ones first (Z is 80 GB at n = 1e5)
        del Z, w
        torch.cuda.empty_cache()
        P.trim_workspace()
        dh = torch.tensor(d).pin_memory()
        eh = torch.tensor(e).pin_memory()
        wh = torch.empty(k, dtype=torch.float64).pin_memory()
        Zh = torch.empty((k, n), dtype=torch.float64).pin_memory()
        P.stemr_host(dh, eh, w=wh, Z=Zh, stream=stream, **kw)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e_ms = []
        for i in range(args.steps):
            flush.random_(0, 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            P.stemr_host(dh, eh, w=wh, Z=Zh, stream=stream, **kw)
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        etot = sum(e_ms)
        if world > 1:
            t = torch.tensor([etot], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            etot = float(t.item())
        e2e = {"value": m * args.steps / (etot / 1e3), "unit": "eigenpairs/s",
               "h2d_bytes_per_step": 8 * (2 * n - 1), "d2h_bytes_per_step": 8 * m + 8 * n * m,
               "ms_per_step": etot / args.steps, "z_copies_per_step": P.last_stats()["z_copies"]}

    # ---------------- CPU oracle on a bounded sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, desc, dt = cpu_oracle_sharded(args.config, n, k, seconds=12.0)
        cpu = {"value": v, "unit": "eigenpairs/s", "cores": cores, "kind": "oracle", "sample": desc,
               "seconds": dt}
        if args.cpu_pairs:  # single-core reference point on request
            v1, dt1, desc1 = cpu_oracle_sample(d, e, args.cpu_pairs)
            cpu["single_core"] = {"value": v1, "sample": desc1, "seconds": dt1}

    s0 = stats[-1]
    rqc_hist = hist_last  # eigenpairs by twisted factorizations of their RQC (mrrr_get_rqc_histogram)
    launches = sum(int(s["kernel_launches"]) for s in stats)
    line = {"metric": METRIC, "value": value, "unit": "eigenpairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "step_ms": [round(x, 3) for x in ms],
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n": n, "k": k, "range": "all" if rng is None else
                       f"index {rng[0]}..{rng[1]}", "l2": "flushed (256 MiB write) before each step",
                       "parallelism": f"eigen-index shards x{world} (all-gather of w)" if world > 1
                       else "single"},
            "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks,
            "phases_ms": {"root": s0["ms_root"], "tree": s0["ms_tree"], "vectors": s0["ms_vectors"],
                          "total": s0["ms_total"]},
            "tree": {"nodes": s0["nodes"], "levels": s0["levels"], "rqc_iters": s0["rqc_iters"],
                     "rqc_fallbacks": s0["rqc_fallbacks"], "safe_resweeps": s0["safe_resweeps"],
                     "vec_items": s0["vec_items"], "vec_nudges": s0["vec_nudges"],
                     "rqc_hist": rqc_hist},
            "memory": {"pool_bytes": s0["pool_bytes"], "workspace_bytes": s0["workspace_bytes"],
                       "z_bytes": 8 * n * m if world == 1 else None,
                       "note": "device workspace the library holds (all of it, child RRR pools included) "
                               "beside the caller's w and Z"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
