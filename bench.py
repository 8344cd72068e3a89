#!/usr/bin/env python
"""Benchmark: batched TabuCol moves/s on BASELINE config 1.

Workload ("c2", BASELINE.json configs[1]): Erdos-Renyi G(500, 0.5) (seed 1,
62,289 edges), k = 48, D = 8192 individuals with uniform random initial
colourings (Stream.derive(1, TAG_INIT, i)), 50,000 TabuCol iterations per
individual per step, stream keys stream_key(1, TAG_LS, step, i).  Validation
mode: the reference's SplitMix64 streams, bit-exact trajectories.

One step = one `improve_population`-equivalent pass over the whole population
(D fixed, sharded evenly over ranks = strong scaling), plus, for N > 1, the
NCCL all-gather of every rank's best colourings (uint8) and best conflicts --
the per-generation elite exchange.

Metric: moves/s = sum(iters_used) over all individuals / max-over-ranks device
time (CUDA events, launching stream).  Inputs are resident in HBM in the timed
region; L2 is flushed (256 MB write) between timed steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the CPU restatement of the reference kernel
(oracle/, C + OpenMP on every host core) on a bounded sample of the same
workload: the reference itself is numba (Python) and cannot be installed on
the GPU box ("Reference arm").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time


ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (seed, n, p_edge, k, D, depth)
    "c2": (1, 500, 0.5, 48, 8192, 50000),   # BASELINE configs[1] (the metric's config)
    "c1": (1, 125, 0.5, 18, 64, 10000),     # configs[0], CPU-runnable
    "c3": (1, 1000, 0.5, 83, 16384, 100000),
}
METRIC = "TabuCol moves/sec (whole box) G(500,0.5) k=48 D=8192 at 1/2/4/8 GPU; x CPU ref"


def algorithmic_bytes(k, sum_c, sum_deg):
    """per iteration 2k*C (gamma rows) + 2(k-1)*C (tabu stamps)
    + 8*deg(v*) (read+write gamma[u,a], gamma[u,b]); element sizes 2 B."""
    return 2 * k * sum_c + 2 * (k - 1) * sum_c + 8 * sum_deg


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""
        return False

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(",") for r in self.out.strip().splitlines() if r.strip()]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
                for nm, val in zip(names, r[4:8]):
                    if val.strip() == "Active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(wl, start, count):
    from paper_2109_05948_b200.graph import rand_graph
    from paper_2109_05948_b200.init import random_col_assigns

    seed, n, pe, k, D, depth = WORKLOADS[wl]
    g = rand_graph(seed, n, pe)
    A = random_col_assigns(n, k, count, seed, start=start)
    return g, A


def cpu_sample(wl, threads, n_ind, depth=None):
    """Time the CPU restatement of `_tabucol_batch` on the first n_ind
    individuals of the same population (full depth unless given)."""
    from oracle import oracle
    from paper_2109_05948_b200.rng import TAG_LS, stream_keys

    seed, n, pe, k, D, dep = WORKLOADS[wl]
    depth = depth or dep
    g, A = make_inputs(wl, 0, n_ind)
    keys = stream_keys(seed, TAG_LS, 0, n_ind)
    oracle.tabucol_batch(g, A[:1].copy(), k, keys[:1], 10, threads=threads)  # warm-up
    t0 = time.perf_counter()
    out = oracle.tabucol_batch(g, A.copy(), k, keys, depth, threads=threads)
    dt = time.perf_counter() - t0
    moves = int(out["iters_used"].sum())
    return moves / dt, moves, dt


def run_reference(args):
    """--impl reference: the CPU restatement on all host cores (rank 0 only)."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle

    oracle.build()
    cores = os.cpu_count() or 1
    seed, n, pe, k, D, depth = WORKLOADS[args.workload]
    n_ind = max(64, 2 * cores)
    vals = []
    for s in range(args.warmup + args.steps):
        v, moves, dt = cpu_sample(args.workload, cores, n_ind, depth=args.ref_depth)
        if s >= args.warmup:
            vals.append((v, moves, dt))
    value = statistics.median(v for v, _, _ in vals)
    ms = 1e3 * statistics.mean(dt for _, _, dt in vals)
    sample = (f"{n_ind} of {D} individuals x {args.ref_depth or depth} iterations per step "
              f"(C restatement of _tabucol_batch, OpenMP, {cores} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "moves/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: G({n},{pe}) k={k} D={D} depth={depth}",
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": "moves/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "moves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2109_05948_b200 import _native as N
    from paper_2109_05948_b200 import device as Dv
    from paper_2109_05948_b200 import localsearch as LS
    from paper_2109_05948_b200.rng import TAG_LS, stream_keys

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    seed, n, pe, k, D, depth = WORKLOADS[args.workload]
    if args.pop:
        D = args.pop
    if args.depth:
        depth = args.depth
    lo, hi = (D * rank) // world, (D * (rank + 1)) // world
    g, A = make_inputs(args.workload, lo, hi - lo)
    dg = Dv.DeviceGraph(g, dev)
    a0 = torch.from_numpy(A).to(dev)
    flags = N.FLAG_DIAG | (N.FLAG_PRODUCTION if args.rng == "philox" else 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def keys_for(step):
        return Dv.keys_to_tensor(stream_keys(seed, TAG_LS, step, hi - lo, start=lo), dev)

    gathered = None
    if world > 1:
        gathered = torch.empty((D // world * world, n), dtype=torch.uint8, device=dev)

    def step(s, ev=None):
        a = a0.clone()
        keys = keys_for(s)
        if ev:
            ev[0].record(stream)
        out = Dv.tabucol_batch(dg, a, k, keys, depth, flags=flags, counters=True)
        if ev:
            ev[1].record(stream)
        if world > 1:  # per-generation elite exchange over NVLink
            best8 = out["best_assigns"].to(torch.uint8)
            dist.all_gather_into_tensor(gathered, best8[: D // world])
            fit = torch.empty(world * (hi - lo), dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(fit, out["best_conflicts"])
        if ev:
            ev[2].record(stream)
        return out

    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    moves = 0
    sum_c = sum_deg = 0
    kern_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (not in the events)
            out = step(args.warmup + s, evs[s])
            moves += int(out["iters_used"].sum().item())
            ctr = out["counters"].sum(dim=0).tolist()
            sum_c += ctr[0]
            sum_deg += ctr[1]
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[2]) for e in evs]
    kern_ms = [e[0].elapsed_time(e[1]) for e in evs]
    coll_ms = [e[1].elapsed_time(e[2]) for e in evs]
    t_local = sum(step_ms) / 1e3
    stats = torch.tensor([t_local, float(moves), float(sum_c), float(sum_deg)], dtype=torch.float64,
                         device=dev)
    if world > 1:
        tmax = stats[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tot = stats[1:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        t_max, moves_all, sumc_all, sumdeg_all = tmax.item(), *tot.tolist()
    else:
        t_max, moves_all, sumc_all, sumdeg_all = t_local, float(moves), float(sum_c), float(sum_deg)
    value = moves_all / t_max

    # ---- e2e: the public API with host buffers (H2D + D2H inside the timed region)
    e2e = None
    if rank == 0 and not args.no_e2e:
        pin = torch.empty((hi - lo, n), dtype=torch.int32).pin_memory()
        host_keys = stream_keys(seed, TAG_LS, 999, hi - lo, start=lo)
        e2e_moves, e2e_t = 0, 0.0
        reps = max(1, min(args.steps, 3))
        for r in range(reps + 1):
            pin.numpy()[:] = A
            t0 = time.perf_counter()
            res = LS._run_tabucol_batch(g, pin.numpy(), k, host_keys, depth, rng=args.rng)
            dt = time.perf_counter() - t0
            if r > 0:  # first call warms the host path
                e2e_moves += int(res["iters_used"].sum())
                e2e_t += dt
        h2d = A.nbytes + host_keys.nbytes + g.adj_indptr.nbytes + g.adj_indices.nbytes + 8 * g.m
        d2h = 2 * A.nbytes + 4 * 8 * (hi - lo)
        e2e = {"value": e2e_moves / e2e_t * (world if world > 1 else 1), "unit": "moves/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "paper_2109_05948_b200.localsearch._run_tabucol_batch -> mcb_tabucol_batch_host",
               "note": "rank-0 shard through the host-buffer C-ABI call, scaled by n_gpus"
               if world > 1 else "whole population through the host-buffer C-ABI call"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline (dominant kernel: tabucol, shared-memory bound)
    alg_bytes_total = algorithmic_bytes(k, sumc_all, sumdeg_all) / world  # rank 0's share
    kern_s = sum(kern_ms) / 1e3
    achieved = alg_bytes_total / kern_s / 1e9  # GB/s per GPU
    gbs = C_double = None
    import ctypes

    desc = ctypes.create_string_buffer(256)
    N.check(N.lib().mcb_tabucol_describe(n, k, hi - lo, desc, 256))
    kernel_desc = desc.value.decode()
    gbs, pms = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().mcb_probe_smem_bandwidth(ctypes.byref(gbs), ctypes.byref(pms)))
    smem_peak = gbs.value
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass

    # ---- CPU baseline: the oracle on this host, rank 0 at N = 1 only, bounded sample
    cpu = None
    if not args.no_cpu and world == 1:
        cores = os.cpu_count() or 1
        n_ind = max(64, 2 * cores)
        v, m_, dt = cpu_sample(args.workload, cores, n_ind, depth=args.ref_depth)
        cpu = {"value": v, "unit": "moves/s", "cores": cores, "kind": "port",
               "sample": f"{n_ind} individuals x {args.ref_depth or WORKLOADS[args.workload][5]} "
                         f"iterations of the same population, {dt:.1f} s wall "
                         "(C restatement of _tabucol_batch, OpenMP)"}

    clocks = clk.summary()
    traffic, traffic_src = ncu_traffic(D // world)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "moves/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: G({n},{pe}) seed {seed}, m={g.m}, k={k}, "
                               f"D={D}, {depth} iterations/individual/step",
                   "mode": "validation (SplitMix64, bit-exact)" if args.rng == "splitmix"
                   else "production (Philox)",
                   "parallelism": f"population sharded {D // world}/GPU" + (
                       ", NCCL all_gather of elites per step" if world > 1 else ""),
                   "l2": "flushed (256 MB write) between timed steps"},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                     "frac": achieved / smem_peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": kernel_desc,
                     "peak_source": "measured: mcb_probe_smem_bandwidth (LDS.128 stream, all SMs)",
                     "alg_bytes_per_launch": alg_bytes_total / args.steps,
                     "latency_bound": ncu_latency_evidence(),
                     "kernel_ms_per_launch": 1e3 * kern_s / args.steps,
                     "hbm_peak_gbs": peaks.get("hbm_gbs")},
        "cpu_baseline": cpu,
        "e2e": e2e,
        # per step: adjacency bitset build + the TabuCol kernel (the CTA-kernel
        # fallback pass launches only for individuals whose tables overflow)
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
        "collective_ms_per_step": statistics.mean(coll_ms) if world > 1 else 0.0,
        "mean_C": sumc_all / moves_all, "mean_deg": sumdeg_all / moves_all,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _ncu_capture():
    """The newest committed `ncu --set full` capture of the TabuCol kernel."""
    prof = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    for name in ("r01d_tabucol_warp_ncu_raw.csv", "r01c_tabucol_warp_ncu_raw.csv"):
        if os.path.exists(os.path.join(prof, name)):
            return os.path.join(prof, name)
    return os.path.join(prof, "missing.csv")


def ncu_latency_evidence():
    """Issue-slot use and warp availability of the TabuCol kernel from the same
    committed `ncu --set full` capture: the kernel is latency-bound, which is
    why roofline.frac is low (profiles/r01d_summary.md)."""
    path = _ncu_capture()
    try:
        import csv

        rows = list(csv.reader(open(path)))
        h, v = rows[0], rows[2]
        g = lambda m: round(float(v[h.index(m)]), 3)  # noqa: E731
        return {"issue_slots_busy_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active_per_sm": g("sm__warps_active.avg.per_cycle_active"),
                "warps_eligible_per_scheduler": g("smsp__warps_eligible.avg.per_cycle_active"),
                "source": "profiles/" + os.path.basename(path)}
    except (OSError, ValueError, KeyError, IndexError):
        return None


def ncu_traffic(individuals):
    """DRAM bytes (read + write) of one launch of the TabuCol kernel from the
    committed `ncu --set full` capture (profiles/r01c_tabucol_warp_ncu_raw.csv:
    one wave of 1184 individuals x 50k iterations, same kernel variant), scaled
    to this launch's individuals; (None, reason) when the capture is absent."""
    path = _ncu_capture()
    try:
        import csv

        rows = list(csv.reader(open(path)))
        h, u, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = sum(float(v[h.index(m)]) * scale[u[h.index(m)]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return tot * individuals / 1184.0, ("ncu --set full of the same kernel variant (profiles/" + os.path.basename(path)
                                            + ", D=1184), dram read+write scaled per individual; the state stays on chip")
    except (OSError, ValueError, KeyError, IndexError):
        return None, "no ncu capture in profiles/"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--rng", default="splitmix", choices=["splitmix", "philox"])
    ap.add_argument("--pop", type=int, default=0, help="override D (testing)")
    ap.add_argument("--depth", type=int, default=0, help="override depth (testing)")
    ap.add_argument("--ref-depth", type=int, default=0, help="CPU sample depth override")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
