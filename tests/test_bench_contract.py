"""bench.py's JSON-line contract on the CPU-only reference arm.

`--impl reference` times the oracle port on the host cores; it
must print exactly one JSON line with the keys the driver reads, and under
torchrun with world_size 2 only rank 0 prints.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--workload", "app20", "--steps", "1", "--warmup", "0",
        "--cpu-sample", "4"]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _json_lines(out: str) -> list:
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _check(line: dict, n: int) -> None:
    assert KEYS <= set(line)
    assert line["impl"] == "reference" and line["n_gpus"] == n
    assert line["metric"] == "models trained/sec" and line["unit"] == "models/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["config"]["workload"] == "app20"
    assert line["cpu_baseline"]["kind"] in ("port", "reference")
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check(lines[0], 1)


def test_reference_arm_world_size_2_rank0_only():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        "29633", "bench.py", "--gpus", "2", *ARGS], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check(lines[0], 2)


def test_strong_scaling_shards_cover_every_unit_once():
    """bench.py --scaling strong: the fixed (series, restart) unit list is
    LPT-sharded over the ranks; every unit lands on exactly one rank and the
    per-rank cost loads are balanced."""
    import numpy as np

    sys.path.insert(0, ROOT)
    import bench
    from paper_2202_07798_b200 import sharding

    series, spec, kw = bench.workload_series("suite16")
    for world in (1, 2, 3, 8):
        shards = [bench.shard_units(series, spec, kw, 4, world, r)[0] for r in range(world)]
        allu = np.concatenate(shards)
        assert len(allu) == len(series) * 4
        assert len({tuple(u) for u in allu.tolist()}) == len(allu)
        cost = {}
        for (i, r) in allu.tolist():
            s = series[i]
            h = kw["br_hidden"](s.key)
            cost[(i, r)] = sum(sharding.task_cost(len(s) * 0.7, k, d=s.arity, h=h) for k in ("pnn", "brbpnn"))
        loads = [sum(cost[tuple(u)] for u in sh.tolist()) for sh in shards]
        assert max(loads) <= min(loads) + max(cost.values()) + 1e-6  # LPT bound
