"""Multi-rank host logic on CPU: LPT sharding and the ordered gather, with a
real world_size-2 gloo process group (127.0.0.1)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_07798_b200 import sharding


def test_lpt_partitions_every_task_once_and_balances():
    rng = np.random.default_rng(0)
    costs = rng.pareto(1.5, size=1000) + 1.0
    for world in (1, 2, 3, 8):
        shards = sharding.lpt_assign(costs, world)
        flat = np.sort(np.concatenate([np.asarray(s, dtype=int) for s in shards]))
        assert np.array_equal(flat, np.arange(1000))
        loads = [costs[s].sum() for s in shards]
        # LPT bound: max load <= 4/3 OPT (+ one task); OPT >= mean and >= max task
        opt = max(np.mean(loads), costs.max())
        assert max(loads) <= 4.0 / 3.0 * opt + costs.max()


def test_merge_ordered_detects_gaps_and_duplicates():
    parts = [([0, 2], ["a", "c"]), ([1], ["b"])]
    assert sharding.merge_ordered(parts, 3) == ["a", "b", "c"]
    with pytest.raises(ValueError):
        sharding.merge_ordered([([0], ["a"])], 2)
    with pytest.raises(ValueError):
        sharding.merge_ordered([([0], ["a"]), ([0], ["b"])], 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, costs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shards = sharding.lpt_assign(costs, world)
        mine = shards[rank]
        local = [("result", i, rank) for i in mine]  # stand-in for SeriesResults
        full = sharding.gather_ordered(mine, local, len(costs))
        q.put((rank, [(r[1], r[2]) for r in full]))
    finally:
        dist.destroy_process_group()


def test_gather_ordered_world_size_2_gloo():
    costs = list(np.random.default_rng(3).uniform(1, 100, size=37))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, costs, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = sharding.lpt_assign(costs, 2)
    owner = {i: r for r, s in enumerate(shards) for i in s}
    for rank in (0, 1):
        got = out[rank]
        assert [g[0] for g in got] == list(range(len(costs)))  # original order
        assert all(g[1] == owner[g[0]] for g in got)           # produced by its owner
    assert out[0] == out[1]


def _dist_worker(rank, world, port, q):
    """Runs sharding.train_many_distributed's real shard -> train -> gather
    path with experiment.train_many replaced by a CPU mock (no GPU here)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_07798_b200 import experiment, synth
        from paper_2202_07798_b200.experiment import BatchOutput, ExperimentConfig, SeriesResult
        from paper_2202_07798_b200.traces import BbSeries, SplitMode, SplitSpec

        seen = []

        def mock_train_many(pairs, config, **kw):
            seen.extend((p[0].key, p[1], p[2].fraction if len(p) > 2 else None) for p in pairs)
            hid = kw.get("br_hidden_of")
            return BatchOutput([SeriesResult(p[0].key, p[1], n_train=hid(p[0]) if hid else -1,
                                             mse=float(rank)) for p in pairs])

        experiment.train_many = mock_train_many
        series = [BbSeries(k, X, y) for k, X, y in synth.app20()[:7]]
        specs = [SplitSpec(SplitMode.RANDOM, f, 1) for f in (0.3, 0.7)]
        pairs = [(s, k, sp) for s in series for k in ("pnn", "brbpnn") for sp in specs]
        cfg = ExperimentConfig(split_mode=SplitMode.RANDOM)
        out = sharding.train_many_distributed(pairs, cfg, br_hidden_of=lambda s: 3 + s.key[2])
        q.put((rank, [(r.key, r.kind, r.n_train, r.mse) for r in out], seen,
               [(p[0].key, p[1], p[2].fraction) for p in pairs]))
    finally:
        dist.destroy_process_group()


def test_train_many_distributed_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, res, seen, pairs = q.get(timeout=180)
        out[rank] = (res, seen, pairs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res0, seen0, pairs = out[0]
    res1, seen1, _ = out[1]
    assert res0 == res1                                   # every rank holds the full, ordered result
    assert [(r[0], r[1]) for r in res0] == [(p[0], p[1]) for p in pairs]
    assert sorted(seen0 + seen1) == sorted(pairs)         # each task trained exactly once
    assert seen0 and seen1                                # both ranks got work
    owner = {t: 0 for t in seen0} | {t: 1 for t in seen1}
    for r, p in zip(res0, pairs):
        assert r[3] == float(owner[p])                    # result produced by the owning rank
        assert r[2] == 3 + p[0][2]                        # br_hidden_of reached the local call
