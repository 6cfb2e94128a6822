"""Benchmark: models trained/sec for BB-ML's PNN + BR-BPNN on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload suite16]
                    [--restarts R] [--precision 64|32] [--scaling weak|strong]
                    [--impl ours|reference]

One step = train every model of the workload from scratch (PNN and BR-BPNN,
one fused kernel call each, concurrently), predict every model's test rows
and compute every model's test MSE / Pearson / Spearman on the device.
The headline arithmetic is FP64 (the reference's and the drop-in's);
``--precision 32`` runs the PNN fits in FP32 (BR-BPNN is FP64 always).

``value``: device-timed steps with the prepared inputs resident in HBM.
``e2e``: the public path a user runs, every step: raw series rows (host) ->
batched split + normalise + task tables (``batch.build_workload``) -> pinned
staging -> H2D -> train / predict / metrics -> D2H of weights, statuses and
per-model metrics.
Multi-GPU (torchrun, one process per GPU):
  weak   (default) every rank trains its own restarts of the workload;
  strong  the fixed unit list (series x restarts) is LPT-sharded over the
          ranks and every step ends with an all-gather of every model's
          status / metrics / weights in task order (sharding.py) — the only
          collective.  Time = max over ranks.
``--impl reference`` (and ``cpu_baseline``) time the CPU oracle port
(oracle/bbml_oracle.py, bit-identical to the reference on its golden
vectors) on the host cores: every task of restart 0 of the workload through
a process pool, plus the serial and GIL-thread (the reference's
``run_experiment(workers=...)``) modes.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = ("suite16", "app20", "sweep", "wide")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="suite16", choices=WORKLOADS)
    ap.add_argument("--restarts", type=int, default=None)
    ap.add_argument("--precision", type=int, default=64, choices=(32, 64))
    ap.add_argument("--scaling", default="weak", choices=("weak", "strong"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="CPU legs: a stratified subset of this many tasks instead of all (tests)")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


# restarts per GPU (weak) or in total (strong): suite16 32 (fills one GPU),
# sweep 16 (SURVEY §8d cfg 4), wide 7 (140 CTA-per-model fits on 148 SMs)
DEFAULT_RESTARTS = {"suite16": 32, "app20": 1, "sweep": 16, "wide": 7}

# BR-BPNN tasks at or above this hidden size are timed on the CPU for
# CPU_EPOCH_SAMPLE epochs and scaled per epoch (a full h = 64 fit takes
# minutes of CPU time); SURVEY §8d "time a sample and extrapolate"
CPU_WIDE_HIDDEN = 32
CPU_EPOCH_SAMPLE = 3


def workload_series(name: str):
    from paper_2202_07798_b200 import synth
    from paper_2202_07798_b200.traces import BbSeries, SplitMode, SplitSpec

    if name == "suite16":
        raw = synth.suite16(seed=0)
        spec = SplitSpec(SplitMode.RANDOM, 0.7, 0)
        kw = dict(br_hidden=lambda key: synth.suite16_hidden(key[0]))
    elif name == "app20":
        raw = synth.app20()
        spec = SplitSpec(SplitMode.HIGH_LOW, 0.7, 0)
        kw = {}
    elif name == "sweep":
        raw = synth.sweep(500, seed=0)
        spec = SplitSpec(SplitMode.HIGH_LOW, 0.7, 0)
        kw = {}
    else:  # wide BR-BPNN (P = 64 (d+2) + 1 = 257 at d = 2)
        raw = synth.app20(axis=tuple(range(1, 65)))
        spec = SplitSpec(SplitMode.HIGH_LOW, 0.7, 0)
        kw = dict(kinds=("brbpnn",), br_hidden=64)
    series = [BbSeries(k, X, y) for k, X, y in raw]
    return series, spec, kw


def pnn_flops(n, d, h, epochs, batch):
    """SURVEY §8d algorithmic FLOPs of one PNN model (FMA = 2)."""
    P = h * (d + 2) + 1
    steps = -(-n // batch)
    return epochs * (n * (4 * h * d + 10 * h + 14) + steps * 13 * P)


def lm_flops(n, d, h, epochs, trials):
    """SURVEY §8d algorithmic FLOPs of one BR-BPNN model given its epochs and
    LM trials: per epoch one J/J'J/J'r pass + the tridiagonal eigen-solve,
    per trial one damped solve + trial objective."""
    P = h * (d + 2) + 1
    per_epoch = n * (P * (P + 1) + 2 * P + 3 * h * d + 10 * h + 1) + 4 * P ** 3 / 3
    per_trial = P ** 3 / 3 + 2 * P ** 2 + n * (2 * h * d + 7 * h + 4)
    return epochs * per_epoch + trials * per_trial


def sample_clocks(stop_path):
    """nvidia-smi clocks during the timed region (started before, killed after)."""
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        return subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                 "-lms", "100"], stdout=open(stop_path, "w"), stderr=subprocess.DEVNULL)
    except FileNotFoundError:
        return None


def summarize_clocks(path, gpu_index):
    sm, mx, reasons = [], 0.0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    try:
        for line in open(path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or f[0] != str(gpu_index):
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
    except OSError:
        pass
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
            "reasons": sorted(reasons), "samples": len(sm)}


def measure_fma_peak(torch, precision):
    from paper_2202_07798_b200._lib import check, lib

    so = lib()
    scratch = torch.empty(16, dtype=torch.float64, device="cuda")
    blocks, iters = 148 * 8, 4096
    s = torch.cuda.current_stream()
    for _ in range(2):
        check(so.bbml_fma_peak(precision, blocks, iters, scratch.data_ptr(), s.cuda_stream), "fma")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(5):
        e0.record(s)
        check(so.bbml_fma_peak(precision, blocks, iters, scratch.data_ptr(), s.cuda_stream), "fma")
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, blocks * 256 * 8 * iters * 2 / (ms * 1e-3) / 1e12)
    return best


# ---------------------------------------------------------------------------
# CPU side (oracle port) — the checker / baseline only
# ---------------------------------------------------------------------------

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cpu_task(job):
    """(seconds, sampled) for one model on one core; wide BR fits are timed
    for CPU_EPOCH_SAMPLE epochs and scaled to the epochs the device ran."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import bbml_oracle as O

    key, X, y, kind, mode, frac, base, br_hidden, full_epochs = job
    sampled = kind == "brbpnn" and br_hidden >= CPU_WIDE_HIDDEN
    t0 = time.perf_counter()
    r = O.train_one(key, X, y, kind, mode=mode, fraction=frac, base_seed=base, br_hidden=br_hidden,
                    br_max_epochs=CPU_EPOCH_SAMPLE if sampled else 1000)
    dt = time.perf_counter() - t0
    if sampled and r.epochs_run:
        dt *= full_epochs / r.epochs_run
    return dt, sampled


def _cpu_worker_init():
    # one BLAS thread per worker process: the pool provides the parallelism
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)


def cpu_jobs(series, spec, wl_kw, full_epochs=1000):
    """Every (series, kind) task of restart 0 (run seed 0), longest first."""
    kinds = wl_kw.get("kinds", ("pnn", "brbpnn"))
    bh = wl_kw.get("br_hidden", 1)
    jobs = []
    for s in series:
        for kind in kinds:
            h = (bh(s.key) if callable(bh) else bh) if kind == "brbpnn" else 1
            cost = len(s) * (300.0 if kind == "pnn" else 20.0 * h * h)
            jobs.append((cost, (s.key, s.X, s.y, kind, spec.mode.value, spec.fraction, 0, h, full_epochs)))
    jobs.sort(key=lambda j: -j[0])
    return [j for _, j in jobs]


def run_cpu(series, spec, wl_kw, cores, full_epochs=1000, sample=None):
    """The reference algorithm (oracle port) on the host: every task of
    restart 0 through a process pool of ``cores`` workers (the best CPU mode;
    wall clock), the serial rate from the same per-task seconds, and the
    reference's own GIL-thread fan-out (``run_experiment(workers=cores)``,
    experiment.py:397-401) on a stratified 48-task subset."""
    from concurrent.futures import ProcessPoolExecutor, ThreadPoolExecutor

    jobs = cpu_jobs(series, spec, wl_kw, full_epochs)
    if sample:
        jobs = jobs[::max(1, len(jobs) // sample)][:sample]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=cores, initializer=_cpu_worker_init) as pool:
        res = list(pool.map(_cpu_task, jobs, chunksize=1))
    wall = time.perf_counter() - t0
    secs = [r[0] for r in res]
    sampled = any(r[1] for r in res)
    n = len(jobs)
    sub = jobs[::max(1, n // 48)][:min(48, n)]
    _cpu_worker_init()
    t1 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as tp:
        tres = list(tp.map(_cpu_task, sub))
    twall = time.perf_counter() - t1
    out = {
        "n": n, "wall_s": wall, "cpu_s": sum(secs),
        # sampled wide fits have no real wall clock: ideal pool over the scaled seconds
        "pool_models_per_s": (cores * n / sum(secs)) if sampled else n / wall,
        "ideal_pool_models_per_s": cores * n / sum(secs),
        "serial_models_per_s": n / sum(secs),
        "threads_models_per_s": len(sub) / (twall if not any(r[1] for r in tres) else sum(r[0] for r in tres)),
        "threads_tasks": len(sub),
        "cpu_model": cpu_model(), "cores": cores, "sampled": sampled, "subset": bool(sample),
    }
    return out


def cpu_sample_text(r, workload):
    s = (f"{'all ' if not r.get('subset') else 'a stratified subset of '}{r['n']} tasks of "
         f"{workload} restart 0 (run seed 0), oracle/bbml_oracle.py "
         f"(bit-identical to the reference), process pool of {r['cores']} workers "
         f"(1 BLAS thread each), longest first: wall {r['wall_s']:.1f} s, {r['cpu_s']:.1f} CPU-s; "
         f"serial {r['serial_models_per_s']:.2f} models/s (sum of per-task seconds); "
         f"reference GIL-thread mode (workers={r['cores']}) {r['threads_models_per_s']:.2f} models/s "
         f"on {r['threads_tasks']} stratified tasks; CPU {r['cpu_model']}")
    if r["sampled"]:
        s += (f"; BR-BPNN h>={CPU_WIDE_HIDDEN} fits timed for {CPU_EPOCH_SAMPLE} epochs and scaled "
              "to the device's epochs (value = ideal pool over the scaled seconds)")
    return s


def reference_arm(args, world, rank):
    if rank != 0:
        return
    series, spec, kw = workload_series(args.workload)
    restarts = args.restarts or DEFAULT_RESTARTS[args.workload]
    cores = os.cpu_count() or 1
    r = run_cpu(series, spec, kw, cores, sample=args.cpu_sample)
    v = r["pool_models_per_s"]
    line = {
        "metric": "models trained/sec", "value": v, "unit": "models/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": 1, "warmup": 0, "ms_per_step": 1e3 * r["wall_s"],
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.workload, "restarts_per_gpu": restarts, "split": spec.mode.value,
                   "sample": "restart 0 (the other restarts are the same shapes under other seeds)",
                   "steps_note": "one pass over every task of restart 0 is the CPU arm's step; "
                                 f"--steps {args.steps} --warmup {args.warmup} are not repeated "
                                 "so the arm ends within minutes"},
        "cpu_baseline": {"value": v, "unit": "models/s", "cores": cores, "kind": "port",
                         "sample": cpu_sample_text(r, args.workload),
                         "serial": r["serial_models_per_s"], "threads": r["threads_models_per_s"],
                         "ideal_pool": r["ideal_pool_models_per_s"], "cpu_model": r["cpu_model"]},
        "e2e": {"value": v, "unit": "models/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    out = json.dumps(line)
    print(out, flush=True)
    if args.json_out:
        with open(args.json_out, "w") as fh:
            fh.write(out + "\n")


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def shard_units(series, spec, kw, restarts, world, rank):
    """Strong scaling: the fixed (series, restart) unit list, LPT-sharded by
    cost (sharding.lpt_assign); returns (units of this rank, all shards)."""
    from paper_2202_07798_b200 import sharding

    bh = kw.get("br_hidden", 1)
    kinds = kw.get("kinds", ("pnn", "brbpnn"))
    frac = spec.fraction if spec.mode.value == "random" else 0.5
    units, costs = [], []
    for r in range(restarts):
        for i, s in enumerate(series):
            h = bh(s.key) if callable(bh) else bh
            c = sum(sharding.task_cost(len(s) * frac, k, d=s.arity, h=h) for k in kinds)
            units.append((i, r))
            costs.append(c)
    shards = sharding.lpt_assign(costs, world)
    units = np.array(units, dtype=np.int64)
    return units[shards[rank]], [units[s] for s in shards]


class Gather:
    """Strong-scaling result gather (the one collective): every rank's
    per-model status (raw bytes), metrics (4 doubles) and weights, padded to
    the largest shard, all-gathered over NCCL into rank-ordered buffers."""

    def __init__(self, torch, dist, dev, world):
        self.torch, self.dist, self.dev, self.world = torch, dist, dev, world
        sizes = torch.tensor([dev.status.numel(), dev.metrics.numel(), dev.weights.numel()],
                             dtype=torch.int64, device="cuda")
        allsz = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(allsz, sizes)
        self.max = torch.stack(allsz).max(0).values.tolist()
        self.bufs = [torch.zeros(m, dtype=t, device="cuda") for m, t in
                     zip(self.max, (torch.uint8, torch.float64, torch.float64))]
        self.out = [torch.zeros(world * m, dtype=t, device="cuda") for m, t in
                    zip(self.max, (torch.uint8, torch.float64, torch.float64))]

    def __call__(self):
        for src, buf, out in zip((self.dev.status, self.dev.metrics, self.dev.weights), self.bufs, self.out):
            buf[:src.numel()].copy_(src)
            self.dist.all_gather_into_tensor(out, buf)
        return 3

    @property
    def bytes(self) -> int:
        return sum(b.numel() * b.element_size() for b in self.out)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, world, rank)

    import torch
    import torch.distributed as dist

    from paper_2202_07798_b200 import batch, prep
    from paper_2202_07798_b200._lib import STATUS

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    series, spec, kw = workload_series(args.workload)
    restarts = args.restarts or DEFAULT_RESTARTS[args.workload]
    if args.scaling == "strong":
        units, shards = shard_units(series, spec, kw, restarts, world, rank)
        build_kw = dict(units=units)
        total_models_all = sum(len(s) for s in shards) * len(kw.get("kinds", ("pnn", "brbpnn")))
    else:
        build_kw = dict(restarts=list(range(rank * restarts, (rank + 1) * restarts)))
        total_models_all = None

    def build():
        # the public e2e path starts from the raw series rows
        return batch.build_workload(series, spec, precision=args.precision,
                                    table=prep.SeriesTable.from_series(series), **build_kw, **kw)

    wl = build()
    dev = batch.DeviceWorkload(wl)
    gather = Gather(torch, dist, dev, world) if (world > 1 and args.scaling == "strong") else None
    torch.cuda.synchronize()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(args.warmup):
        dev.step()
        if gather:
            gather()
    torch.cuda.synchronize()
    st = dev.fetch()["status"]
    n_bad = int((st["code"] != 0).sum())

    clock_path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
    os.makedirs(os.path.dirname(clock_path), exist_ok=True)
    clk = sample_clocks(clock_path) if rank == 0 else None
    time.sleep(0.3 if clk else 0)

    # device-timed region: K steps, L2 flushed between steps (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(float(k))
        a, b = ev[k]
        a.record(s)
        launches += dev.step()
        if gather:
            gather()
        b.record(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[1]) for e in ev]
    total_s = sum(step_ms) / 1e3

    # clock sampling covers the device-timed region; stopped before the e2e
    # loop (an nvidia-smi query holds the driver and stalls host CUDA calls)
    if clk:
        clk.terminate()
        clk.wait()

    # end-to-end: raw series -> batched prep -> pinned -> H2D -> step -> D2H
    e2e_times, prep_times = [], []
    for k in range(args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        wl_k = build()
        t1 = time.perf_counter()
        dev.refresh(wl_k)
        dev.step()
        if gather:
            gather()
        dev.fetch(predictions=False)  # weights, status, per-model metrics
        e2e_times.append(time.perf_counter() - t0)
        prep_times.append(t1 - t0)

    from paper_2202_07798_b200._lib import check, lib, ptr

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = []
        for _ in range(2):
            flush.fill_(1.0)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            reps.append(e0.elapsed_time(e1))
        return float(np.mean(reps))

    # each training call timed alone on its launching stream (CUDA events)
    pnn_ms = lm_ms = None
    if len(wl.pnn):
        pnn_ms = timed(lambda: check(lib().bbml_pnn_train(
            ptr(dev.pnn_tab), len(dev.pnn_tab), ptr(dev.X), ptr(dev.y), wl.train.stride,
            ptr(dev.weights), None, ptr(dev.status), wl.precision, s.cuda_stream), "pnn"))
    if len(wl.lm):
        off = 8 * int(wl.P_pnn.sum())
        lm_ms = timed(lambda: check(lib().bbml_lm_train(
            ptr(dev.lm_tab), len(dev.lm_tab), ptr(dev.X), ptr(dev.y), wl.train.stride,
            ptr(dev.weights) + off, None, ptr(dev.status) + STATUS.itemsize * len(wl.pnn),
            s.cuda_stream), "lm"))
    st_all = dev.fetch()["status"]
    peak32 = measure_fma_peak(torch, 32)
    peak64 = measure_fma_peak(torch, 64)

    t = torch.tensor([total_s, sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_s, e2e_step = float(t[0]), float(t[1])  # e2e: mean step, max over ranks
    models_per_step = total_models_all if total_models_all is not None else wl.n_models * world
    value = models_per_step * args.steps / total_s
    e2e_value = models_per_step / e2e_step

    if rank == 0:
        peak_p = peak32 if args.precision == 32 else peak64
        pnn_fl = sum(pnn_flops(int(r["n"]), int(r["d"]), int(r["h"]), int(r["epochs"]), int(r["batch"]))
                     for r in wl.pnn)
        st_lm = st_all[len(wl.pnn):]
        lm_fl = sum(lm_flops(int(r["n"]), int(r["d"]), int(r["h"]), int(e), int(tr))
                    for r, e, tr in zip(wl.lm, st_lm["epochs"], st_lm["trials"]))
        rl = {}
        if pnn_ms:
            a = pnn_fl / (pnn_ms * 1e-3) / 1e12
            kname = "pnn_f64_kernel" if args.precision == 64 else "pnn_lat_kernel"
            rl["pnn"] = {"bound": f"fp{args.precision}-pipe", "kernel": f"{kname} (bbml_pnn_train)",
                         "achieved": a, "peak": peak_p, "unit": "TFLOP/s", "frac": a / peak_p,
                         "kernel_ms": pnn_ms, "algorithmic_flops": pnn_fl, "traffic": None}
        if lm_ms:
            a = lm_fl / (lm_ms * 1e-3) / 1e12
            Pl = wl.lm["h"] * (wl.lm["d"] + 2) + 1
            kn = " + ".join(k for k, m in (("lm_warp_kernel", (Pl <= 32).any()),
                                           ("lm_wide_kernel", (Pl > 32).any())) if m)
            rl["lm"] = {"bound": "fp64-pipe", "kernel": f"{kn} (bbml_lm_train)",
                        "achieved": a, "peak": peak64, "unit": "TFLOP/s", "frac": a / peak64,
                        "kernel_ms": lm_ms, "algorithmic_flops": lm_fl, "traffic": None}
        try:  # DRAM bytes per launch of each kernel from the committed ncu captures
            with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as fh:
                traffic = json.load(fh)
        except (OSError, ValueError):
            traffic = {}
        for kk, v in rl.items():
            tr = traffic.get(f"{kk}_fp{args.precision}" if kk == "pnn" else kk)
            if tr and tr.get("workload") == args.workload:
                v["traffic"] = tr["bytes_per_launch"]
                v["traffic_source"] = tr["report"]
        dom = max(rl, key=lambda k: rl[k]["kernel_ms"]) if rl else None
        roof = dict(rl[dom]) if dom else {}
        roof["peak_source"] = ("measured: bbml_fma_peak FMA-pipe microbenchmark on this GPU "
                               "(MEASURED_PEAKS.json has only HBM / bf16-GEMM peaks)")
        roof["other"] = {k: v for k, v in rl.items() if k != dom}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            wide_ep = (float(st_lm["epochs"][wl.lm["h"] >= CPU_WIDE_HIDDEN].mean())
                       if len(wl.lm) and (wl.lm["h"] >= CPU_WIDE_HIDDEN).any() else 1000.0)
            r = run_cpu(series, spec, kw, cores, wide_ep, sample=args.cpu_sample)
            cpu = {"value": r["pool_models_per_s"], "unit": "models/s", "cores": cores, "kind": "port",
                   "sample": cpu_sample_text(r, args.workload), "serial": r["serial_models_per_s"],
                   "threads": r["threads_models_per_s"], "ideal_pool": r["ideal_pool_models_per_s"],
                   "cpu_model": r["cpu_model"]}
        tb = dev.table_bytes
        line = {
            "metric": "models trained/sec", "value": value, "unit": "models/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32" if args.precision == 32 else "f64",
            "data": "synthetic",
            "config": {"workload": args.workload,
                       ("restarts_per_gpu" if args.scaling == "weak" else "restarts_total"): restarts,
                       "models_per_gpu": wl.n_models, "models_per_step": models_per_step,
                       "pnn_models": len(wl.pnn), "br_models": len(wl.lm),
                       "pnn_precision": f"fp{args.precision}", "br_precision": "fp64",
                       "l2": "flushed (256 MiB write) between steps", "split": spec.mode.value},
            "e2e": {"value": e2e_value, "unit": "models/s",
                    "h2d_bytes_per_step": dev.h2d_bytes + tb,
                    "d2h_bytes_per_step": dev.d2h_bytes_for(False),
                    "prep_ms_per_step": 1e3 * float(np.mean(prep_times)),
                    "result": "trained weights + status + per-model test MSE / Pearson / "
                              "Spearman (bbml_metrics); inputs re-split / normalised / packed "
                              "from the raw series rows every step (prep.py)"
                              + ("; + NCCL all-gather of every shard's results" if gather else "")},
            "roofline": roof,
            "gpu_launches": launches,
            "models_failed": n_bad,
            "workload_stats": {
                "lm_epochs_mean": float(st_lm["epochs"].mean()) if len(wl.lm) else None,
                "lm_trials_mean": float(st_lm["trials"].mean()) if len(wl.lm) else None,
                "pnn_max_sequential_steps": int((wl.pnn["epochs"] * -(-wl.pnn["n"] // wl.pnn["batch"])).max())
                if len(wl.pnn) else None},
            "clocks": summarize_clocks(clock_path, local),
            "cpu_baseline": cpu,
            "step_ms": step_ms,
            "e2e_step_ms": [1e3 * x for x in e2e_times],
        }
        if gather:
            line["e2e"]["gather_bytes_per_step"] = gather.bytes
        out = json.dumps(line)
        print(out, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as fh:
                fh.write(out + "\n")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
