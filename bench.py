#!/usr/bin/env python
"""Benchmark: batched TabuCol moves/s on BASELINE config 1.

Headline workload ("c2", BASELINE.json configs[1]): Erdos-Renyi G(500, 0.5)
(seed 1, 62,289 edges), k = 48, D = 8192 individuals with uniform random
initial colourings (Stream.derive(1, TAG_INIT, i)), 50,000 TabuCol iterations
per individual per step, stream keys stream_key(1, TAG_LS, step, i).
Validation mode: the reference's SplitMix64 streams, bit-exact trajectories.

One step = one `improve_population`-equivalent pass over the whole population
(D fixed, sharded evenly over ranks = strong scaling) plus, for N > 1, the NCCL
all-gather of every rank's best colourings (uint8) and best conflicts -- the
per-generation elite exchange.  Metric: moves/s = sum(iters_used) over all
individuals / max-over-ranks device time (CUDA events on the launching
stream).  Inputs are resident in HBM in the timed region; L2 is flushed (256 MB
write) between timed steps.  `e2e` is the same metric through the public
host-buffer API (`localsearch._run_tabucol_batch`), copies included, timed on
every rank at once (max over ranks).

The other named configs are measured after the headline, one timed step each
at a bounded depth (stated in their `config`), under "workloads": c3 (G(1000,
.5) k=83 D=16384), c4 (weighted, `_run_wvcp_batch`, G(500,.5) w<=100 k=60
D=8192) and c5 (G(2000,.5) k=150 D=2048); `--workload cN` makes any of them
the headline at full depth.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one per GPU; refused when fewer GPUs are
visible).  `--dry-run` runs the same sharding / all-gather on CPU ranks (gloo)
with the C restatement of the kernel, for tests without a GPU.

`--impl reference` times the reference itself -- the numba package installed
from /root/reference into baseline/_ref (`_run_tabucol_batch`,
`mc/localsearch.py:556`) -- on the host cores, rank 0 only; when that install
is absent it falls back to the C restatement (oracle/, kind "port").
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name: kind, seed, n, edge p, wmax, k, D, depth, rounds
WORKLOADS = {
    "c1": ("col", 1, 125, 0.5, 1, 18, 64, 10000, 1),        # configs[0], CPU-runnable
    "c2": ("col", 1, 500, 0.5, 1, 48, 8192, 50000, 1),      # configs[1]: the metric's config
    "c3": ("col", 1, 1000, 0.5, 1, 83, 16384, 100000, 1),   # configs[2]
    "c4": ("wvcp", 1, 500, 0.5, 100, 60, 8192, 5000, 10),   # configs[3]: 10 rounds x 5000
    "c5": ("col", 1, 2000, 0.5, 1, 150, 2048, 200000, 1),   # configs[4]
}
# bounded depth of the extra workloads in a default run (iterations, or
# iterations x rounds for WVCP); --workload cN runs any of them at full depth
EXTRA_DEPTH = {"c3": (10000, 1), "c4": (5000, 2), "c5": (5000, 1), "c2p": (10000, 1)}
# "<config>p": the config in production mode (Philox4x32-10 tie-break and
# tenure draws: statistically equivalent to the reference, not bit-identical;
# tests/test_production_stats_gpu.py)
METRIC = "TabuCol moves/sec (whole box) G(500,0.5) k=48 D=8192 at 1/2/4/8 GPU; x CPU ref"
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def algorithmic_bytes(k, sum_c, sum_deg):
    """per iteration 2k*C (gamma rows) + 2(k-1)*C (tabu stamps)
    + 8*deg(v*) (read+write gamma[u,a], gamma[u,b]); element sizes 2 B."""
    return 2 * k * sum_c + 2 * (k - 1) * sum_c + 8 * sum_deg


def wvcp_bytes_per_iter(n, k, mean_deg, nranks):
    """2kn (full gamma scan) + 2n (vertex tabu stamps) +
    8 deg(v*) + 4 nranks (two class-count rows)."""
    return 2 * k * n + 2 * n + 8 * mean_deg + 4 * nranks


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.out = ""

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


def make_graph(wl):
    from paper_2109_05948_b200.graph import rand_graph

    kind, seed, n, pe, wmax, k, D, depth, rounds = WORKLOADS[wl]
    return rand_graph(seed, n, pe, wmax=wmax)


def make_inputs(wl, start, count):
    from paper_2109_05948_b200.init import random_col_assigns

    kind, seed, n, pe, wmax, k, D, depth, rounds = WORKLOADS[wl]
    return make_graph(wl), random_col_assigns(n, k, count, seed, start=start)


def shard(D, world, rank):
    """Contiguous shard of rank `rank`, and the padded shard size every rank
    uses for the all-gathers (ceil(D / world))."""
    lo, hi = (D * rank) // world, (D * (rank + 1)) // world
    return lo, hi, -(-D // world)


# ---------------------------------------------------------------------------
# the reference (numba) and the C restatement on the host cores
# ---------------------------------------------------------------------------
def reference_module():
    """`memcolor.localsearch` from baseline/_ref (the unmodified reference
    installed by pip), or None when it is not installed / numba is missing."""
    if not os.path.isdir(os.path.join(REF_PATH, "memcolor")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "mcb_numba_cache"))
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        import numba  # noqa: F401
        from memcolor import localsearch as RL
    except Exception:  # noqa: BLE001 -- any import failure means "unavailable"
        return None
    return RL


def cpu_time(wl, n_ind, depth, rounds, threads, impl):
    """Moves/s of the CPU path on the first n_ind individuals of the workload
    at the given depth: impl "reference" (numba, baseline/_ref) or "port" (the
    C restatement, oracle/).  Returns (moves/s, moves, seconds)."""
    from paper_2109_05948_b200.localsearch import default_wvcp_phi0
    from paper_2109_05948_b200.rng import TAG_LS, stream_keys

    kind, seed, n, pe, wmax, k, D, _, _ = WORKLOADS[wl]
    g, A = make_inputs(wl, 0, n_ind)
    keys = stream_keys(seed, TAG_LS, 0, n_ind)
    phi0 = default_wvcp_phi0(g, k)
    if impl == "reference":
        import numba

        RL = reference_module()
        numba.set_num_threads(threads)
        if kind == "col":
            run = lambda a, ky, d: RL._run_tabucol_batch(g, a, k, ky, d)  # noqa: E731
        else:
            run = lambda a, ky, d: RL._run_wvcp_batch(g, a, k, ky, d, rounds, True, phi0)  # noqa: E731
    else:
        from oracle import oracle

        if kind == "col":
            run = lambda a, ky, d: oracle.tabucol_batch(g, a, k, ky, d, threads=threads)  # noqa: E731
        else:
            run = lambda a, ky, d: oracle.wvcp_batch(g, a, k, ky, d, rounds, True, phi0, threads=threads)  # noqa: E731
    run(A[:1].copy(), keys[:1], 10)  # JIT / warm-up
    t0 = time.perf_counter()
    out = run(A.copy(), keys, depth)
    dt = time.perf_counter() - t0
    moves = int(out["iters_used"].sum()) if kind == "col" else n_ind * depth * rounds
    return moves / dt, moves, dt


def cpu_baseline(wl, depth, rounds, full=True):
    """The reference on this host (kind "reference"; the C port if the
    reference is not installed): D_cpu = max(64, 8 x cores) individuals at the
    given depth on every core, plus a 1-thread figure."""
    cores = os.cpu_count() or 1
    impl = "reference" if reference_module() is not None else "port"
    kind = WORKLOADS[wl][0]
    if full:
        n_ind = max(64, 8 * cores)
        n_one = 8
    else:  # the extra workloads: a small sample
        n_ind = 16
        n_one = 0
    v, moves, dt = cpu_time(wl, n_ind, depth, rounds, cores, impl)
    res = {"value": v, "unit": "moves/s", "cores": cores, "kind": impl, "cpu_model": cpu_model(),
           "sample": f"{n_ind} individuals x {depth}{' x ' + str(rounds) + ' rounds' if kind == 'wvcp' else ''} "
                     f"iterations of the same population, {dt:.1f} s wall on {cores} threads "
                     + ("(numba reference from baseline/_ref, " + ("_run_tabucol_batch)" if kind == "col"
                                                                   else "_run_wvcp_batch)")
                        if impl == "reference" else "(C restatement of the reference kernel, OpenMP)")}
    if n_one:
        v1, _, dt1 = cpu_time(wl, n_one, depth, rounds, 1, impl)
        res["value_1thread"] = v1
        res["sample_1thread"] = f"{n_one} individuals x {depth} iterations, {dt1:.1f} s wall, 1 thread"
    return res


def run_reference(args):
    """--impl reference: the reference's own CPU path, rank 0 only."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    kind, seed, n, pe, wmax, k, D, depth, rounds = WORKLOADS[args.workload]
    depth = args.ref_depth or depth
    cores = os.cpu_count() or 1
    impl = "reference" if reference_module() is not None else "port"
    if impl == "port":
        from oracle import oracle

        oracle.build()
    n_ind = max(64, 8 * cores)
    vals = []
    for s in range(args.warmup + args.steps):
        if s < args.warmup and s > 0:
            continue  # one untimed warm-up call is enough for the JIT
        v, moves, dt = cpu_time(args.workload, n_ind, depth, rounds, cores, impl)
        if s >= args.warmup:
            vals.append((v, moves, dt))
    value = statistics.median(v for v, _, _ in vals)
    ms = 1e3 * statistics.mean(dt for _, _, dt in vals)
    sample = (f"{n_ind} of {D} individuals x {depth} iterations per step "
              + ("(numba reference from baseline/_ref, _run_tabucol_batch, " if impl == "reference"
                 else "(C restatement of _tabucol_batch, OpenMP, ") + f"{cores} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "moves/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": workload_config(args.workload, depth, world),
        "cpu_baseline": {"value": value, "unit": "moves/s", "cores": cores, "kind": impl,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "moves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(wl, depth, world, rounds=None):
    prod = wl.endswith("p")
    if prod:
        wl = wl[:-1]
    kind, seed, n, pe, wmax, k, D, dep, rnd = WORKLOADS[wl]
    rounds = rounds or rnd
    w = f"{wl}: G({n},{pe}) seed {seed}" + (f", weights 1..{wmax}" if wmax > 1 else "") + f", k={k}, D={D}, "
    w += (f"{rounds} rounds x {depth} iterations/individual/step (iterated WVCP tabu)" if kind == "wvcp"
          else f"{depth} iterations/individual/step")
    return {"workload": w,
            "mode": ("production (Philox4x32-10 draws, statistically equivalent, not bit-identical)" if prod
                     else "validation (SplitMix64, bit-exact)"),
            "parallelism": f"population sharded {-(-D // world)}/GPU" + (
                ", NCCL all_gather of elites per step" if world > 1 else ""),
            "l2": "flushed (256 MB write) between timed steps"}


# ---------------------------------------------------------------------------
# CPU dry run of the multi-rank path (gloo, the C restatement per shard)
# ---------------------------------------------------------------------------
def run_dry(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2109_05948_b200.rng import TAG_LS, stream_keys

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    kind, seed, n, pe, wmax, k, D, depth, rounds = WORKLOADS["c1"]
    D, depth = args.pop or 24, args.depth or 2000
    lo, hi, pad = shard(D, world, rank)
    g, A = make_inputs("c1", lo, hi - lo)
    keys = stream_keys(seed, TAG_LS, 0, hi - lo, start=lo)
    t0 = time.perf_counter()
    out = oracle.tabucol_batch(g, A.copy(), k, keys, depth, threads=1)
    dt = time.perf_counter() - t0
    best = np.zeros((pad, n), dtype=np.int32)
    best[: hi - lo] = out["best_assigns"]
    fit = np.full(pad, -1, dtype=np.int64)
    fit[: hi - lo] = out["best_conflicts"]
    stats = torch.tensor([dt, float(out["iters_used"].sum())], dtype=torch.float64)
    if world > 1:
        gb = [torch.empty((pad, n), dtype=torch.int32) for _ in range(world)]
        gf = [torch.empty(pad, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gb, torch.from_numpy(best))
        dist.all_gather(gf, torch.from_numpy(fit))
        tmax = stats[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tot = stats[1:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        rows = [gb[r][: shard(D, world, r)[1] - shard(D, world, r)[0]] for r in range(world)]
        fits = [gf[r][: shard(D, world, r)[1] - shard(D, world, r)[0]] for r in range(world)]
        allb, allf = torch.cat(rows).numpy(), torch.cat(fits).numpy()
        t_max, moves = tmax.item(), tot.item()
    else:
        allb, allf, t_max, moves = best[: hi - lo], fit[: hi - lo], dt, stats[1].item()
    if rank == 0:
        h = hashlib.sha256(np.ascontiguousarray(allb).tobytes() + np.ascontiguousarray(allf).tobytes())
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "value": moves / t_max,
                          "unit": "moves/s", "moves": moves, "D": D, "depth": depth,
                          "digest": h.hexdigest()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2109_05948_b200 import _native as N
    from paper_2109_05948_b200 import device as Dv
    from paper_2109_05948_b200 import localsearch as LS
    from paper_2109_05948_b200.rng import TAG_LS, stream_keys

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # communicator init lines (NVLS / NVLink use) visible, on stderr: rank 0's
        # stdout carries exactly one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload
    kind, seed, n, pe, wmax, k, D, depth, rounds = WORKLOADS[wl]
    if kind != "col":
        raise SystemExit("the headline workload must be a TabuCol config (c1, c2, c3, c5); c4 runs as an extra")
    if args.pop:
        D = args.pop
    if args.depth:
        depth = args.depth
    lo, hi, pad = shard(D, world, rank)
    g, A = make_inputs(wl, lo, hi - lo)
    dg = Dv.DeviceGraph(g, dev)
    a0 = torch.from_numpy(A).to(dev)
    flags = N.FLAG_DIAG | (N.FLAG_PRODUCTION if args.rng == "philox" else 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    g_best = torch.empty((world * pad, n), dtype=torch.uint8, device=dev) if world > 1 else None
    g_fit = torch.empty(world * pad, dtype=torch.int64, device=dev) if world > 1 else None
    best8 = torch.zeros((pad, n), dtype=torch.uint8, device=dev)
    fit = torch.full((pad,), -1, dtype=torch.int64, device=dev)

    def keys_for(step):
        return Dv.keys_to_tensor(stream_keys(seed, TAG_LS, step, hi - lo, start=lo), dev)

    def step(s, ev=None):
        a = a0.clone()
        keys = keys_for(s)
        if ev:
            ev[0].record(stream)
        out = Dv.tabucol_batch(dg, a, k, keys, depth, flags=flags, counters=True)
        if ev:
            ev[1].record(stream)
        if world > 1:  # per-generation elite exchange over NVLink (padded shards)
            best8[: hi - lo].copy_(out["best_assigns"])
            fit[: hi - lo].copy_(out["best_conflicts"])
            dist.all_gather_into_tensor(g_best, best8)
            dist.all_gather_into_tensor(g_fit, fit)
        if ev:
            ev[2].record(stream)
        return out

    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    moves = sum_c = sum_deg = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
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

    def reduce_max_sum(tmax_v, sums):
        if world == 1:
            return tmax_v, list(sums)
        t = torch.tensor([tmax_v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        u = torch.tensor(list(sums), dtype=torch.float64, device=dev)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        return t.item(), u.tolist()

    t_max, (moves_all, sumc_all, sumdeg_all) = reduce_max_sum(t_local, [moves, sum_c, sum_deg])
    value = moves_all / t_max
    coll_max, _ = reduce_max_sum(statistics.mean(coll_ms) if world > 1 else 0.0, [])

    # ---- e2e: the public API with host buffers on every rank at once
    e2e = None
    if not args.no_e2e:
        pin = torch.empty((hi - lo, n), dtype=torch.int32).pin_memory()
        host_keys = stream_keys(seed, TAG_LS, 999, hi - lo, start=lo)
        pin.numpy()[:] = A
        LS._run_tabucol_batch(g, pin.numpy(), k, host_keys, min(depth, 100))  # warms the host path
        reps = max(1, min(args.steps, 3))
        e2e_t, e2e_moves = 0.0, 0
        for r in range(reps):
            pin.numpy()[:] = A
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            res = LS._run_tabucol_batch(g, pin.numpy(), k, host_keys, depth, rng=args.rng)
            dt = time.perf_counter() - t0
            dtm, (mv,) = reduce_max_sum(dt, [int(res["iters_used"].sum())])
            e2e_t += dtm
            e2e_moves += mv
        h2d = A.nbytes + host_keys.nbytes + g.adj_indptr.nbytes + g.adj_indices.nbytes + 8 * g.m
        d2h = 2 * A.nbytes + 4 * 8 * (hi - lo)
        e2e = {"value": e2e_moves / e2e_t, "unit": "moves/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "api": "paper_2109_05948_b200.localsearch._run_tabucol_batch -> mcb_tabucol_batch_host",
               "note": ("every rank's shard through the host-buffer C-ABI call, max wall time over ranks"
                        if world > 1 else "whole population through the host-buffer C-ABI call")
               + "; bytes per rank"}

    # ---- the other named configs, one timed step each (bounded depth)
    extras = {}
    if not args.no_extra and wl == "c2" and not args.pop and not args.depth:
        for x in args.extra.split(","):
            if x:
                extras[x] = run_extra(x, world, rank, dev, flush, reduce_max_sum)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline (dominant kernel: TabuCol, shared-memory bound)
    import ctypes

    alg_bytes = algorithmic_bytes(k, sumc_all, sumdeg_all) / world  # one rank's share per launch set
    kern_s = sum(kern_ms) / 1e3
    achieved = alg_bytes / kern_s / 1e9
    desc = ctypes.create_string_buffer(256)
    N.check(N.lib().mcb_tabucol_describe(n, k, hi - lo, desc, 256))
    gbs, pms = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().mcb_probe_smem_bandwidth(ctypes.byref(gbs), ctypes.byref(pms)))
    smem_peak = gbs.value
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass

    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(wl, args.ref_depth or depth, 1)
        if reference_module() is not None:
            try:  # the C restatement beside it, same sample
                v, _, dtp = cpu_time(wl, max(64, 8 * (os.cpu_count() or 1)), args.ref_depth or depth, 1,
                                     os.cpu_count() or 1, "port")
                cpu["port_value"] = v
            except Exception:  # noqa: BLE001
                pass

    clocks = clk.summary()
    traffic, traffic_src = ncu_traffic(-(-D // world))
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
        # the same config object as the reference arm's (D only when --pop overrides it)
        "config": workload_config(wl, depth, world) | ({"D": D} if D != WORKLOADS[wl][6] else {}),
        "roofline": {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                     "frac": achieved / smem_peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": desc.value.decode(),
                     "peak_source": "measured: mcb_probe_smem_bandwidth (LDS.128 stream, all SMs)",
                     "alg_bytes_per_launch": alg_bytes / args.steps,
                     "latency_bound": ncu_latency_evidence(),
                     "kernel_ms_per_launch": 1e3 * kern_s / args.steps,
                     "hbm_peak_gbs": peaks.get("hbm_gbs")},
        "cpu_baseline": cpu,
        "e2e": e2e,
        # per step: adjacency bitset build + the TabuCol kernel (the fallback
        # passes launch only for individuals whose tables overflow)
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
        "collective_ms_per_step": coll_max,
        "mean_C": sumc_all / moves_all, "mean_deg": sumdeg_all / moves_all,
    }
    if extras:
        line["workloads"] = extras
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_extra(wl, world, rank, dev, flush, reduce_max_sum):
    """One timed step of another named config (bounded depth), sharded like the
    headline; roofline and a small reference sample on rank 0 at N = 1."""
    import ctypes

    import torch

    from paper_2109_05948_b200 import _native as N
    from paper_2109_05948_b200 import device as Dv
    from paper_2109_05948_b200.localsearch import default_wvcp_phi0
    from paper_2109_05948_b200.rng import TAG_LS, stream_keys

    depth, rounds = EXTRA_DEPTH[wl]
    prod = wl.endswith("p")
    base = wl[:-1] if prod else wl
    kind, seed, n, pe, wmax, k, D, full_depth, full_rounds = WORKLOADS[base]
    lo, hi, pad = shard(D, world, rank)
    g, A = make_inputs(base, lo, hi - lo)
    dg = Dv.DeviceGraph(g, dev)
    a0 = torch.from_numpy(A).to(dev)
    keys = Dv.keys_to_tensor(stream_keys(seed, TAG_LS, 0, hi - lo, start=lo), dev)
    phi0 = default_wvcp_phi0(g, k)
    stream = torch.cuda.current_stream()

    def once(d, ev=None):
        a = a0.clone()
        if ev:
            ev[0].record(stream)
        if kind == "col":
            out = Dv.tabucol_batch(dg, a, k, keys, d, flags=N.FLAG_DIAG | (N.FLAG_PRODUCTION if prod else 0),
                                   counters=True)
        else:
            out = Dv.wvcp_batch(dg, a, k, keys, d, rounds, True, phi0,
                                flags=N.FLAG_DIAG | (N.FLAG_PRODUCTION if prod else 0))
        if ev:
            ev[1].record(stream)
        return out

    once(min(depth, 200))
    torch.cuda.synchronize()
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    out = once(depth, ev)
    torch.cuda.synchronize()
    dt = ev[0].elapsed_time(ev[1]) / 1e3
    if kind == "col":
        c = out["counters"].sum(dim=0).tolist()
        mv = float(out["iters_used"].sum().item())
        sums = [mv, c[0], c[1]]
    else:
        mv = float((hi - lo) * depth * rounds)
        sums = [mv, 0.0, 0.0]
    t_max, (mv_all, sc, sd) = reduce_max_sum(dt, sums)
    res = {"value": mv_all / t_max, "unit": "moves/s", "ms": 1e3 * t_max, "moves": mv_all,
           "config": workload_config(wl, depth, world, rounds) | {
               "note": f"bounded depth; the config asks {full_rounds} rounds x {full_depth}" if kind == "wvcp"
               else f"bounded depth from random colourings; the config asks {full_depth}"}}
    if rank != 0:
        return res
    if kind == "col":
        desc = ctypes.create_string_buffer(256)
        N.check(N.lib().mcb_tabucol_describe(n, k, hi - lo, desc, 256))
        alg = algorithmic_bytes(k, sc, sd) / world
        in_l2 = "gamma in L2" in desc.value.decode()
        gbs, pms = ctypes.c_double(), ctypes.c_double()
        if in_l2:
            N.check(N.lib().mcb_probe_l2_bandwidth(ctypes.byref(gbs), ctypes.byref(pms)))
        else:
            N.check(N.lib().mcb_probe_smem_bandwidth(ctypes.byref(gbs), ctypes.byref(pms)))
        ach = alg / dt / 1e9
        res["roofline"] = {"bound": "l2" if in_l2 else "smem", "achieved": ach, "peak": gbs.value,
                           "unit": "GB/s", "frac": ach / gbs.value, "kernel": desc.value.decode(),
                           "peak_source": "measured: mcb_probe_" + ("l2" if in_l2 else "smem") + "_bandwidth",
                           "mean_C": sc / mv_all, "mean_deg": sd / mv_all}
    else:
        mean_deg = 2.0 * g.m / n
        per = wvcp_bytes_per_iter(n, k, mean_deg, len(g.weight_values))
        ach = per * mv / dt / 1e9
        gbs, pms = ctypes.c_double(), ctypes.c_double()
        N.check(N.lib().mcb_probe_smem_bandwidth(ctypes.byref(gbs), ctypes.byref(pms)))
        res["roofline"] = {"bound": "smem", "achieved": ach, "peak": gbs.value, "unit": "GB/s",
                           "frac": ach / gbs.value, "kernel": "wvcp_kernel (CTA per individual)",
                           "bytes_per_iter": per, "note": "deg(v*) taken as the mean degree 2m/n"}
    if world == 1:
        try:
            res["cpu_baseline"] = cpu_baseline(base, depth, rounds, full=False)
            if prod:
                res["cpu_baseline"]["note"] = "the reference's own (validation) mode on the same config"
        except Exception as e:  # noqa: BLE001
            res["cpu_baseline"] = {"error": str(e)[:200]}
    return res


def _ncu_capture():
    """The newest committed `ncu --set full` capture of the TabuCol kernel."""
    prof = os.path.join(ROOT, "profiles")
    for name in ("r02_tabucol_ncu_raw.csv", "r01d_tabucol_warp_ncu_raw.csv"):
        if os.path.exists(os.path.join(prof, name)):
            return os.path.join(prof, name)
    return os.path.join(prof, "missing.csv")


def ncu_latency_evidence():
    """Issue-slot use and warp availability of the TabuCol kernel from the
    committed `ncu --set full` capture."""
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
    """DRAM bytes (read + write) of one launch from the committed capture,
    scaled to this launch's individuals; (None, reason) without a capture."""
    path = _ncu_capture()
    try:
        import csv

        rows = list(csv.reader(open(path)))
        h, u, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = sum(float(v[h.index(m)]) * scale[u[h.index(m)]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        n_cap = 1184.0
        return tot * individuals / n_cap, ("ncu --set full of the TabuCol kernel (profiles/" + os.path.basename(path)
                                           + ", 1184 individuals), dram read+write scaled per individual")
    except (OSError, ValueError, KeyError, IndexError):
        return None, "no ncu capture in profiles/"


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--extra", default="c3,c4,c5,c2p",
                    help="other configs measured after the headline (a trailing p: production mode)")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--rng", default="splitmix", choices=["splitmix", "philox"])
    ap.add_argument("--pop", type=int, default=0, help="override D (testing)")
    ap.add_argument("--depth", type=int, default=0, help="override depth (testing)")
    ap.add_argument("--ref-depth", type=int, default=0, help="CPU sample depth override")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="CPU ranks (gloo) + the C restatement")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")

    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torchrun
        if not args.dry_run:
            import torch

            have = torch.cuda.device_count()
            if have < args.gpus:
                print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}),
                      flush=True)
                raise SystemExit(2)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
