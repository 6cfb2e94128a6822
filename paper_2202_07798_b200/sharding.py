"""Multi-GPU sharding of independent models.

Every (series, kind, restart) model is independent, so N GPUs need no
data-path collective: one process per GPU trains a disjoint shard chosen by
LPT (longest-processing-time first) on a cost estimate, and the results are
gathered once at the end in the caller's original task order (so the output
never depends on N).  Host plumbing only; the training itself is the same
batched device call on each rank.
"""

from __future__ import annotations

import heapq
from typing import Sequence

import numpy as np


def task_cost(n_train: int, kind: str, *, epochs: int = 300, batch: int = 10, d: int = 1,
              h: int = 1, max_epochs: int = 1000) -> float:
    """Sequential-work estimate: PNN ~ E * ceil(n/B) Adam steps; BR ~ n P^2 per
    epoch times the epoch cap."""
    if kind == "pnn":
        return float(epochs) * -(-int(n_train) // int(batch)) * batch
    P = h * (d + 2) + 1
    return float(n_train) * P * P * max_epochs / 50.0


def lpt_assign(costs: Sequence[float], world: int) -> list:
    """Indices per rank; each task exactly once, greedy largest-first onto the
    least-loaded rank (ties -> lowest rank), each shard in ascending order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    shards: list = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(s) for s in shards]


def merge_ordered(parts: Sequence[tuple], total: int) -> list:
    """parts = [(indices, results), ...] from every rank -> results in the
    original task order.  Raises if a task is missing or duplicated."""
    out: list = [None] * total
    seen = np.zeros(total, dtype=bool)
    for idx, res in parts:
        if len(idx) != len(res):
            raise ValueError("indices / results length mismatch")
        for i, r in zip(idx, res):
            if seen[i]:
                raise ValueError(f"task {i} returned twice")
            seen[i] = True
            out[i] = r
    if not seen.all():
        raise ValueError(f"{int((~seen).sum())} tasks missing from the gather")
    return out


def gather_ordered(local_idx: Sequence[int], local_results: Sequence, total: int, group=None) -> list:
    """All-gather every rank's (indices, results) as Python objects (the one
    collective, at the end) and merge them in task order on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    objs: list = [None] * world
    dist.all_gather_object(objs, (list(local_idx), list(local_results)), group=group)
    return merge_ordered(objs, total)


def train_many_distributed(pairs: Sequence[tuple], config, *, group=None, **kw) -> list:
    """experiment.train_many across the ranks of ``group``: LPT shard, train
    the local shard on this rank's GPU, gather SeriesResults in order."""
    import torch.distributed as dist

    from . import experiment

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    hidden_of = kw.get("br_hidden_of")
    costs = []
    for pair in pairs:  # (series, kind) or (series, kind, SplitSpec) as train_many takes
        series, kind = pair[0], pair[1]
        sp = pair[2] if len(pair) > 2 else config.split_spec()
        n = len(series) * (sp.fraction if sp.mode.value == "random" else 0.5)
        h = hidden_of(series) if hidden_of is not None else config.br_hidden
        costs.append(task_cost(n, kind, epochs=config.pnn_epochs, batch=config.pnn_batch_size,
                               d=series.arity, h=h, max_epochs=config.br_max_epochs))
    shards = lpt_assign(costs, world)
    mine = shards[rank]
    local = experiment.train_many([pairs[i] for i in mine], config, **kw).results if mine else []
    return gather_ordered(mine, local, len(pairs), group)
