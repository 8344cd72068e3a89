"""Device-resident generation of the memetic loop.

One generation of `mc/engine.py:_generation_loop` (:203-316) without the
surrogate (the reference's ablation setting, `use_surrogate=False`,
`mc/crossover.py:103-131`), for k-colouring (`run_col_fixed_k`, :346-368) and
weighted colouring (`run_wvcp`, :321-343), with every array kept in HBM
between the operators:

    init        init_col_population / init_wvcp_population (greedy, on the GPU)
    LS          improve_population -> TabuCol / iterated WVCP tabu   (:205-214)
    distances   pairwise_distances(pop, improved)                    (:287-289)
    pool        update_population(pop, improved, fitness, ...)      (:290)
    matching    match_parents(pop, K)                                (:294)
    offspring   build_offspring_batch + uniform selection           (:295-301)

Same keys as the reference: LS `stream_key(seed, TAG_LS, t, i)`, GPX
`stream_key(seed, TAG_CROSS, t, i K + j)`, selection
`Stream.derive(seed, TAG_SELECT, t, i).below(K)`.  The state after every
generation is bit-identical to the reference's (tests/test_engine_gpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as Dv
from .population import min_spacing
from .rng import TAG_CROSS, TAG_LS, TAG_SELECT, stream_keys


def _stream():
    return torch.cuda.current_stream().cuda_stream


@dataclass
class ColState:
    """Population (assigns, fitness, distance matrix) and the offspring that
    the next generation's local search starts from -- all device tensors."""

    pop_assigns: torch.Tensor  # int32 [p, n]
    pop_fitness: torch.Tensor  # int64 [p]
    pop_dist: torch.Tensor  # int32 [p, p]
    offspring: torch.Tensor  # int32 [p, n]
    k: int
    generation: int = 0
    best_score: int = 2 ** 62
    mode: str = "col"

    @property
    def p(self):
        return self.pop_assigns.shape[0]

    @property
    def n(self):
        return self.pop_assigns.shape[1]


def init_state(dg, init_assigns, k):
    """`Population.from_colorings` of the initial colourings (`mc/population.py:47-56`)
    with their conflict counts as fitness; the first offspring are the same
    colourings (`mc/engine.py:199`)."""
    a = torch.as_tensor(np.ascontiguousarray(init_assigns, dtype=np.int32)).to(dg.device)
    p = a.shape[0]
    _, within = Dv.pairwise(a[:0], a, k)
    # conflicts of each colouring from scratch: edges with equal colours
    fit = (a[:, dg.eu.long()] == a[:, dg.ev.long()]).sum(dim=1).to(torch.int64)
    st = ColState(pop_assigns=a.clone(), pop_fitness=fit, pop_dist=within, offspring=a.clone(), k=k)
    st.best_score = int(fit.min().item()) if p else 2 ** 62
    return st


INF_SCORE = 2 ** 62


def wvcp_scores(dg, assigns, k):
    """`wvcp_score` (`mc/coloring.py:53-67`) of every row: the sum over
    nonempty classes of the class's largest weight."""
    p = assigns.shape[0]
    w = dg.weights.unsqueeze(0).expand(p, -1)
    mx = torch.zeros((p, k), dtype=torch.int64, device=assigns.device)
    mx.scatter_reduce_(1, assigns.long(), w, reduce="amax", include_self=True)
    return mx.sum(dim=1)


def init_state_wvcp(dg, g, p, seed):
    """`run_wvcp`'s start (`mc/engine.py:330-335`): p randomized greedy
    colourings built on the GPU (`init_wvcp_population`, `mc/init.py:57-64`),
    palette k = the most colours any of them opened, fitness = score."""
    from .init import greedy_wvcp_assigns, stream_keys_init

    a, used = greedy_wvcp_assigns(g, stream_keys_init(seed, p), device=True)
    k = int(used.max().item())
    fit = wvcp_scores(dg, a, k)
    st = ColState(pop_assigns=a.clone(), pop_fitness=fit, pop_dist=Dv.pairwise(a[:0], a, k)[1],
                  offspring=a.clone(), k=k, mode="wvcp")
    st.best_score = int(fit.min().item())
    return st


def col_generation(dg, st, *, seed, depth, K, ms=None, timings=None):
    """k-colouring generation (kept name); see `generation`."""
    return generation(dg, st, seed=seed, depth=depth, K=K, ms=ms, timings=timings)


def _all_gather_blocks(pad, group):
    """Equal-size blocks of every rank, concatenated in rank order: NCCL
    all-gather into one tensor; other backends (gloo, e.g. the world-2 test
    on one GPU) through host staging."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    short = pad.dtype == torch.int16  # neither torch's NCCL nor gloo group takes int16: move its bytes
    wire = pad.view(torch.uint8) if short else pad
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world * wire.shape[0],) + tuple(wire.shape[1:]), dtype=wire.dtype, device=wire.device)
        dist.all_gather_into_tensor(buf, wire, group=group)
    else:
        host = wire.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        buf = torch.cat(parts, 0).to(pad.device)
    return buf.view(torch.int16) if short else buf


def _gather_rows(local, total, world, rank, group):
    """Rows [lo_r, hi_r) of every rank -> the whole (total, ...) tensor on this
    device (all-gather of equal-size padded blocks)."""
    import torch.distributed as dist

    from .shard import shard_range

    if not dist.is_initialized():
        return local.contiguous()
    cap = -(-total // world)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    buf = _all_gather_blocks(pad, group)
    parts = []
    for r in range(world):
        lo, hi = shard_range(total, world, r)
        parts.append(buf[r * cap: r * cap + (hi - lo)])
    return torch.cat(parts, 0).contiguous()


def generation(dg, st, *, seed, depth, K, ms=None, timings=None, max_rounds=10, phi0=None, net=None,
               epochs=1, batch_size=64, group=None, force_shard=False):
    """Advance `st` by one generation in place; returns the LS outputs.

    With a surrogate ``net`` (`surrogate.SurrogateNet`; the reference's
    `use_surrogate=True`): after the LS it trains on (LS start points,
    realized best scores) when at least two are finite, with
    `Stream.derive(seed, TAG_TRAIN, t)` (`mc/engine.py:263-281`), and every
    individual keeps the candidate with the lowest prediction
    (`mc/crossover.py:114-118`) instead of a uniform draw.

    WVCP (`st.mode == "wvcp"`): `improve_population(..., WVCP, ...)`
    (`mc/localsearch.py:642-662`) -- phi0 = (k / 2n) max weight, schedule on,
    `max_rounds` rounds of `depth`; an individual that never reached a legal
    colouring keeps its start with fitness INF_SCORE.

    Multi-GPU (`group`, one process per GPU, NCCL): every rank
    holds the whole population; the LS runs on this rank's individuals
    [lo, hi) with their global stream keys, the improved colourings and
    fitness are all-gathered, the distance job space is split and each rank's
    results all-gathered as compact int16 vectors (`mcb_pairwise_jobs`,
    expanded by `mcb_pairwise_scatter`), the pool update / matching / surrogate training
    run replicated (deterministic), GPX and selection run on this rank's rows
    and the offspring are all-gathered -- the same results on every rank as
    one process (`shard.col_generation_sharded` is the host-level twin, tested
    at world size 2)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 or (force_shard and dist.is_initialized()) else 0
    if world > 1 or force_shard:
        return _generation_sharded(dg, st, seed=seed, depth=depth, K=K, ms=ms, max_rounds=max_rounds, phi0=phi0,
                                   net=net, epochs=epochs, batch_size=batch_size, group=group, world=world,
                                   rank=rank, timings=timings)
    p, n, k, t = st.p, st.n, st.k, st.generation
    dev = st.pop_assigns.device
    ms = min_spacing(n) if ms is None else ms
    marks = []  # (stage ending here, event)

    def mark(name):
        if timings is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))

    mark(None)
    keys = Dv.keys_to_tensor(stream_keys(seed, TAG_LS, t, p), dev)
    if st.mode == "wvcp":
        if phi0 is None:
            phi0 = (k / (2.0 * n)) * dg.max_weight
        ls = Dv.wvcp_batch(dg, st.offspring.clone(), k, keys, depth, max_rounds, True, phi0)
        legal = ls["best_scores"] < INF_SCORE
        improved = torch.where(legal[:, None], ls["best_assigns"], st.offspring).contiguous()
        imp_fit = torch.where(legal, ls["best_scores"], torch.full_like(ls["best_scores"], INF_SCORE))
        ls["best_assigns"], ls["best_scores"] = improved, imp_fit
    else:
        ls = Dv.tabucol_batch(dg, st.offspring.clone(), k, keys, depth)
        improved, imp_fit = ls["best_assigns"], ls["best_conflicts"]
    st.best_score = min(st.best_score, int(imp_fit.min().item()))
    mark("ls")
    if net is not None:
        from .rng import TAG_TRAIN, Stream

        mask = imp_fit < INF_SCORE
        if int(mask.sum().item()) >= 2:
            net.train_generation(st.offspring[mask], imp_fit[mask].double().cpu().numpy(), k, epochs, batch_size,
                                 Stream.derive(seed, TAG_TRAIN, t))
        mark("surrogate_train")
    cross, within = Dv.pairwise(st.pop_assigns, improved, k)
    mark("distances")
    adm = torch.empty(p, dtype=torch.int32, device=dev)
    rule = torch.empty(p, dtype=torch.uint8, device=dev)
    new_dist = torch.empty((p, p), dtype=torch.int32, device=dev)
    new_assigns = torch.empty((p, n), dtype=torch.int32, device=dev)
    new_fit = torch.empty(p, dtype=torch.int64, device=dev)
    P = N.ptr
    N.check(N.lib().mcb_update_population(
        P(st.pop_dist), P(cross), P(within), P(st.pop_fitness), P(imp_fit), p, p, int(ms),
        P(st.pop_assigns), P(improved), n, P(adm), P(rule), P(new_dist), P(new_assigns), P(new_fit),
        _stream()))
    st.pop_assigns, st.pop_fitness, st.pop_dist = new_assigns, new_fit, new_dist
    mark("update_population")
    matches = torch.empty((p, K), dtype=torch.int64, device=dev)
    N.check(N.lib().mcb_match_parents(P(st.pop_dist), p, int(K), n, P(matches), _stream()))
    mark("match_parents")
    ck = Dv.keys_to_tensor(stream_keys(seed, TAG_CROSS, t, p * K), dev)
    cands = Dv.gpx_batch(st.pop_assigns, matches, k, ck)
    mark("gpx")
    if net is not None:
        pred = net.predict_assigns_device(cands.reshape(p * K, n), k).reshape(p, K)
        sel = pred.argmin(dim=1)
    else:
        # uniform selection: Stream.derive(seed, TAG_SELECT, t, i).below(K) = stream_value(key, 0) % K
        sk = Dv.keys_to_tensor(stream_keys(seed, TAG_SELECT, t, p), dev)
        sv = torch.empty(p, dtype=torch.int64, device=dev)
        zeros = torch.zeros(p, dtype=torch.int64, device=dev)
        N.check(N.lib().mcb_stream_values(P(sk), P(zeros), P(sv), p, _stream()))
        hi, lo = (sv >> 32) & 0xFFFFFFFF, sv & 0xFFFFFFFF  # unsigned 64-bit value mod K in int64
        sel = ((hi % K) * ((1 << 32) % K) + lo % K) % K
    st.offspring = cands[torch.arange(p, device=dev), sel].contiguous()
    mark("surrogate_select" if net is not None else "select")
    st.generation = t + 1
    if timings is not None:
        torch.cuda.synchronize()
        for (_, e0), (name, e1) in zip(marks[:-1], marks[1:]):
            timings[name] = timings.get(name, 0.0) + e0.elapsed_time(e1) / 1e3
    return ls


def _generation_sharded(dg, st, *, seed, depth, K, ms, max_rounds, phi0, net, epochs, batch_size, group, world,
                        rank, timings=None):
    import torch.distributed as dist

    from .shard import shard_range

    p, n, k, t = st.p, st.n, st.k, st.generation
    dev = st.pop_assigns.device
    ms = min_spacing(n) if ms is None else ms
    marks = []

    def mark(name):
        if timings is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))

    mark(None)
    lo, hi = shard_range(p, world, rank)
    keys = Dv.keys_to_tensor(stream_keys(seed, TAG_LS, t, hi - lo, start=lo), dev)
    start = st.offspring[lo:hi].clone()
    if st.mode == "wvcp":
        if phi0 is None:
            phi0 = (k / (2.0 * n)) * dg.max_weight
        ls = Dv.wvcp_batch(dg, start.clone(), k, keys, depth, max_rounds, True, phi0)
        legal = ls["best_scores"] < INF_SCORE
        imp_loc = torch.where(legal[:, None], ls["best_assigns"], start).contiguous()
        fit_loc = torch.where(legal, ls["best_scores"], torch.full_like(ls["best_scores"], INF_SCORE))
        end_fit_loc = ls["end_scores"]
    else:
        ls = Dv.tabucol_batch(dg, start.clone(), k, keys, depth)
        imp_loc, fit_loc = ls["best_assigns"], ls["best_conflicts"]
        end_fit_loc = ls["end_conflicts"]
    mark("ls")
    # elites: the improved colourings (uint8 over NVLink) and their fitness
    as8 = (lambda a: a.to(torch.uint8)) if k <= 256 else (lambda a: a)  # noqa: E731
    improved = _gather_rows(as8(imp_loc), p, world, rank, group).to(torch.int32)
    imp_fit = _gather_rows(fit_loc.contiguous(), p, world, rank, group)
    mark("elite_allgather")
    st.best_score = min(st.best_score, int(imp_fit.min().item()))
    if net is not None:
        from .rng import TAG_TRAIN, Stream

        mask = imp_fit < INF_SCORE
        if int(mask.sum().item()) >= 2:
            net.train_generation(st.offspring[mask], imp_fit[mask].double().cpu().numpy(), k, epochs, batch_size,
                                 Stream.derive(seed, TAG_TRAIN, t))
        mark("surrogate_train")
    # distances: this rank's slice of the reference's job space as compact
    # int16 results, all-gathered, then expanded into cross / within
    total = p * p + p * (p - 1) // 2
    jlo, jhi = shard_range(total, world, rank)
    jobs = Dv.pairwise_jobs(st.pop_assigns, improved, k, jlo, jhi)
    mark("distances")
    if dist.is_initialized():
        jobs = _gather_rows(jobs, total, world, rank, group)
    mark("distance_allgather")
    cross, within = Dv.pairwise_scatter(jobs, p, p, dev)
    # pool update and matching: replicated, identical on every rank
    adm = torch.empty(p, dtype=torch.int32, device=dev)
    rule = torch.empty(p, dtype=torch.uint8, device=dev)
    new_dist = torch.empty((p, p), dtype=torch.int32, device=dev)
    new_assigns = torch.empty((p, n), dtype=torch.int32, device=dev)
    new_fit = torch.empty(p, dtype=torch.int64, device=dev)
    P = N.ptr
    N.check(N.lib().mcb_update_population(
        P(st.pop_dist), P(cross), P(within), P(st.pop_fitness), P(imp_fit), p, p, int(ms),
        P(st.pop_assigns), P(improved), n, P(adm), P(rule), P(new_dist), P(new_assigns), P(new_fit),
        _stream()))
    st.pop_assigns, st.pop_fitness, st.pop_dist = new_assigns, new_fit, new_dist
    mark("update_population")
    matches = torch.empty((p, K), dtype=torch.int64, device=dev)
    N.check(N.lib().mcb_match_parents(P(st.pop_dist), p, int(K), n, P(matches), _stream()))
    mark("match_parents")
    # GPX and selection on this rank's rows, then the offspring all-gathered
    ck = Dv.keys_to_tensor(stream_keys(seed, TAG_CROSS, t, (hi - lo) * K, start=lo * K), dev)
    cands = Dv.gpx_rows(st.pop_assigns, matches[lo:hi].contiguous(), lo, k, ck)
    rows = hi - lo
    if net is not None:
        sel = net.predict_assigns_device(cands.reshape(rows * K, n), k).reshape(rows, K).argmin(dim=1)
    else:
        sk = Dv.keys_to_tensor(stream_keys(seed, TAG_SELECT, t, rows, start=lo), dev)
        sv = torch.empty(rows, dtype=torch.int64, device=dev)
        zeros = torch.zeros(rows, dtype=torch.int64, device=dev)
        N.check(N.lib().mcb_stream_values(P(sk), P(zeros), P(sv), rows, _stream()))
        hi32, lo32 = (sv >> 32) & 0xFFFFFFFF, sv & 0xFFFFFFFF
        sel = ((hi32 % K) * ((1 << 32) % K) + lo32 % K) % K
    off_loc = cands[torch.arange(rows, device=dev), sel].contiguous()
    mark("gpx_select")
    st.offspring = _gather_rows(as8(off_loc), p, world, rank, group).to(torch.int32)
    mark("offspring_allgather")
    st.generation = t + 1
    # the LS outputs of the whole population (every entry gathered)
    out = {"best_assigns": improved,
           "end_assigns": _gather_rows(as8(ls["end_assigns"]), p, world, rank, group).to(torch.int32),
           "diag": _gather_rows(ls["diag"].contiguous(), p, world, rank, group)}
    if st.mode == "wvcp":
        out["best_scores"] = imp_fit
        out["end_scores"] = _gather_rows(end_fit_loc.contiguous(), p, world, rank, group)
        out["end_conflicts"] = _gather_rows(ls["end_conflicts"].contiguous(), p, world, rank, group)
        out["phi_used"] = _gather_rows(ls["phi_used"].contiguous(), p, world, rank, group)
    else:
        out["best_conflicts"] = imp_fit
        out["end_conflicts"] = _gather_rows(end_fit_loc.contiguous(), p, world, rank, group)
        out["iters_used"] = _gather_rows(ls["iters_used"].contiguous(), p, world, rank, group)
    if timings is not None:
        torch.cuda.synchronize()
        for (_, e0), (name, e1) in zip(marks[:-1], marks[1:]):
            timings[name] = timings.get(name, 0.0) + e0.elapsed_time(e1) / 1e3
    return out
