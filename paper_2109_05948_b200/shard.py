"""Population sharding across the GPUs of one box.

One process per GPU (torchrun), `torch.distributed` for the plumbing.  The
individuals are independent -- each owns its stream key
`stream_key(seed, TAG_LS, generation, i)` keyed by its GLOBAL index i
(`localsearch.py:636-639`) -- so rank r simply runs the contiguous shard
[lo_r, hi_r) and results are bit-identical for any number of ranks.  The one
exchange step per generation is an all-gather of the improved colourings
(uint8, n bytes per individual) and fitness (int64), which gives every rank
the whole population for the next operator:

* local search: shard by individual, then all-gather the elites;
* pairwise distances: shard the reference's linear job space
  [0, p*q + q(q-1)/2) (`distance.py:94-113`) into contiguous ranges; every
  rank's results travel as one compact int16 vector of its job range
  (distances are <= n), all-gathered and expanded into cross / within --
  3 p q / 2 bytes per generation instead of all-reducing two int32 matrices;
* GPX: shard by individual i (rows of `matches`); parents are read from the
  replicated population; then all-gather the offspring rows.

The compute callables are injectable so the host-side logic is testable on
CPU with the `gloo` backend (tests/test_shard.py runs it with world size 2 and
the CPU oracle as the compute); production passes the CUDA operators and the
`nccl` backend.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .rng import TAG_CROSS, TAG_LS, TAG_SELECT, stream_keys, stream_values


def shard_range(total, world, rank):
    """Contiguous, balanced [lo, hi) of `total` units for `rank`."""
    lo = (total * rank) // world
    hi = (total * (rank + 1)) // world
    return lo, hi


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _all_gather_rows(local, total_rows, group, device):
    """All-gather variable-sized row blocks (contiguous shards) into one array."""
    world, rank = _world(group)
    if world == 1:
        return local
    local = np.ascontiguousarray(local)
    if local.dtype == np.int16 and dist.get_backend(group) == "gloo":
        # gloo has no int16: move the same bytes as (rows, 2) uint8
        return _all_gather_rows(local.view(np.uint8).reshape(-1, 2), total_rows, group, device).reshape(-1).view(
            np.int16)
    t = torch.as_tensor(local).to(device)
    shapes = [shard_range(total_rows, world, r) for r in range(world)]
    maxrows = max(hi - lo for lo, hi in shapes)
    pad = torch.zeros((maxrows,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
    pad[: t.shape[0]] = t
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    parts = [o[: hi - lo] for o, (lo, hi) in zip(out, shapes)]
    return torch.cat(parts, 0).cpu().numpy()


def improve_col_sharded(g, assigns, k, master_seed, generation, depth, ls_fn, group=None,
                        device="cpu"):
    """TabuCol over the whole population, this rank running its shard.

    `ls_fn(g, assigns_shard, k, keys_shard, depth) -> dict` is the batched
    operator (`localsearch._run_tabucol_batch` on the GPU; the oracle in the
    CPU tests).  Returns the gathered dict with best_assigns (int32, whole
    population), best_conflicts, end_conflicts, iters_used.
    """
    world, rank = _world(group)
    p = assigns.shape[0]
    lo, hi = shard_range(p, world, rank)
    keys = stream_keys(master_seed, TAG_LS, generation, hi - lo, start=lo)
    out = ls_fn(g, np.array(assigns[lo:hi], dtype=np.int32, copy=True), k, keys, depth)
    best8 = out["best_assigns"].astype(np.uint8 if k <= 256 else np.int32)
    fit = np.stack([out["best_conflicts"], out["end_conflicts"], out["iters_used"]], 1)
    best_all = _all_gather_rows(best8, p, group, device).astype(np.int32)
    fit_all = _all_gather_rows(fit.astype(np.int64), p, group, device)
    return {"best_assigns": best_all, "best_conflicts": fit_all[:, 0],
            "end_conflicts": fit_all[:, 1], "iters_used": fit_all[:, 2]}


def pairwise_sharded(pop, off, k, pair_fn, group=None, device="cpu"):
    """`pairwise_distances` with the job space split over ranks.

    `pair_fn(pop, off, k, job_begin, job_end) -> (cross, within)` computes the
    given job range (zeros elsewhere), e.g. `distance.pairwise_raw`; the
    range's distances are exchanged as int16 job vectors.
    """
    world, rank = _world(group)
    p, q = pop.shape[0], off.shape[0]
    pq = p * q
    total = pq + q * (q - 1) // 2
    lo, hi = shard_range(total, world, rank)
    cross, within = pair_fn(pop, off, k, lo, hi)
    if world == 1:
        return cross, within
    iu, ju = np.triu_indices(q, 1)  # the within jobs in the reference's order (:103-113)
    wl, wh = max(lo - pq, 0), max(hi - pq, 0)
    vec = np.concatenate([np.asarray(cross).reshape(-1)[min(lo, pq):min(hi, pq)],
                          np.asarray(within)[iu[wl:wh], ju[wl:wh]]]).astype(np.int16)
    allv = _all_gather_rows(vec, total, group, device).astype(np.int32)
    cross = allv[:pq].reshape(p, q).copy()
    within = np.zeros((q, q), dtype=np.int32)
    within[iu, ju] = allv[pq:]
    within[ju, iu] = allv[pq:]
    return cross, within


def offspring_sharded(pop, matches, k, master_seed, generation, gpx_fn, group=None, device="cpu"):
    """`build_offspring_batch` with individuals split over ranks.

    `gpx_fn(pop, matches_rows, k, keys_rows, row_offset) -> int32[rows, K, n]`
    builds the offspring of rows [lo, hi) (parents from the full `pop`).
    """
    world, rank = _world(group)
    p, K = matches.shape
    lo, hi = shard_range(p, world, rank)
    keys = stream_keys(master_seed, TAG_CROSS, generation, (hi - lo) * K, start=lo * K)
    out = gpx_fn(pop, matches[lo:hi], k, keys, lo)
    return _all_gather_rows(out.astype(np.int32), p, group, device)


def col_generation_sharded(g, pop_assigns, pop_fitness, pop_dist, offspring, k, master_seed, generation, depth,
                           K, ms, ops, group=None, device="cpu"):
    """One k-colouring generation of `mc/engine.py:_generation_loop` (:203-316,
    uniform selection) with the population split over the ranks.

    Sharded: the local search (by individual), the distance job space, GPX
    (by individual).  Replicated on every rank (deterministic, so every rank
    holds the same population afterwards): `update_population`,
    `match_parents`, the `TAG_SELECT` draws.  `ops` maps "ls", "pair", "gpx"
    to the callables of `improve_col_sharded` / `pairwise_sharded` /
    `offspring_sharded`, "update" to `(pdist, pop_fit, pop_assigns, improved,
    improved_fit, cross, within, ms) -> (admitted, by_rule, new_dist,
    new_assigns, new_fit)` and "match" to `(dist, K) -> int64[p, K]`.
    Returns (pop_assigns, pop_fitness, pop_dist, offspring, improved) as numpy.
    """
    ls = improve_col_sharded(g, offspring, k, master_seed, generation, depth, ops["ls"], group, device)
    improved, imp_fit = ls["best_assigns"], ls["best_conflicts"].astype(np.int64)
    cross, within = pairwise_sharded(pop_assigns, improved, k, ops["pair"], group, device)
    _, _, new_dist, new_assigns, new_fit = ops["update"](pop_dist, pop_fitness, pop_assigns, improved, imp_fit,
                                                         cross, within, ms)
    matches = ops["match"](new_dist, K)
    cands = offspring_sharded(new_assigns, matches, k, master_seed, generation, ops["gpx"], group, device)
    p = new_assigns.shape[0]
    # Stream.derive(seed, TAG_SELECT, t, i).below(K) = stream_value(key, 0) % K
    sel = stream_values(stream_keys(master_seed, TAG_SELECT, generation, p), np.zeros(p, np.uint64)) % np.uint64(K)
    off = cands[np.arange(p), sel.astype(np.int64)]
    return new_assigns, new_fit, new_dist, np.ascontiguousarray(off), improved

