"""Benchmark: models trained/sec for BB-ML's PNN + BR-BPNN on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload suite16]
                    [--restarts R] [--precision 32|64] [--impl ours|reference]

One step = train every model of the workload from scratch (PNN and BR-BPNN,
one fused kernel each, concurrently), predict every model's test rows and
compute every model's test MSE / Pearson / Spearman on the device.
Inputs (CSR-packed, normalised training/test rows) are resident in HBM for
`value`; `e2e` times the public batched call (batch.fit_predict path) with
H2D from pinned host buffers and D2H of weights / status / per-model test
metrics (computed on the device from the predictions) each step.
Multi-GPU (torchrun): every rank trains its own restarts of the workload
(weak scaling, no data-path collective); time = max over ranks.
`--impl reference` times the CPU oracle port (numpy restatement of the
reference, bit-identical to it) on the host cores with a process pool.
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
    ap.add_argument("--precision", type=int, default=32, choices=(32, 64))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


# restarts per GPU: suite16 32 (fills the GPU), sweep 16 (SURVEY §8d cfg 4), wide 7
# (140 CTA-per-model BR-BPNN fits on 148 SMs)
DEFAULT_RESTARTS = {"suite16": 32, "app20": 1, "sweep": 16, "wide": 7}

# BR-BPNN tasks at or above this hidden size are timed on the CPU for
# CPU_EPOCH_SAMPLE epochs and extrapolated per epoch (a full h = 64 fit takes
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
# CPU side (oracle port) — the checker/baseline only
# ---------------------------------------------------------------------------

def _cpu_task(args):
    """Seconds for one model on one core; wide BR fits are timed for
    CPU_EPOCH_SAMPLE epochs and scaled to `full_epochs` epochs."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import bbml_oracle as O

    key, X, y, kind, mode, frac, base, br_hidden, full_epochs = args
    sampled = kind == "brbpnn" and br_hidden >= CPU_WIDE_HIDDEN
    t0 = time.perf_counter()
    r = O.train_one(key, X, y, kind, mode=mode, fraction=frac, base_seed=base, br_hidden=br_hidden,
                    br_max_epochs=CPU_EPOCH_SAMPLE if sampled else 1000)
    dt = time.perf_counter() - t0
    if sampled and r.epochs_run:
        dt *= full_epochs / r.epochs_run
    return dt


def cpu_sample_tasks(series, spec, wl_kw, restarts, sample, full_epochs=1000):
    """Stratified sample: tasks ordered by a cost estimate, one pick per
    equal-count stratum (median of the stratum)."""
    kinds = wl_kw.get("kinds", ("pnn", "brbpnn"))
    bh = wl_kw.get("br_hidden", 1)
    tasks = []
    for s in series:
        n = len(s) * spec.fraction if spec.mode.value == "random" else len(s) * 0.5
        for kind in kinds:
            h = bh(s.key) if callable(bh) else bh
            cost = n * (300.0 if kind == "pnn" else 20.0 * h * h)
            tasks.append((cost, s, kind, h))
    tasks.sort(key=lambda t: t[0])
    S = min(sample, len(tasks))
    picks = [tasks[int((i + 0.5) * len(tasks) / S)] for i in range(S)]
    return [(s.key, s.X, s.y, kind, spec.mode.value, spec.fraction, r % max(restarts, 1), h,
             full_epochs) for i, (_, s, kind, h) in enumerate(picks) for r in (i,)]


def _cpu_worker_init():
    # one BLAS thread per worker process: the pool provides the parallelism
    # (numpy is already imported in the parent, so the env var alone is too late)
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)


def run_cpu(series, spec, wl_kw, restarts, sample, cores, full_epochs=1000):
    from concurrent.futures import ProcessPoolExecutor

    jobs = cpu_sample_tasks(series, spec, wl_kw, restarts, sample, full_epochs)
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=cores, initializer=_cpu_worker_init) as pool:
        secs = list(pool.map(_cpu_task, jobs, chunksize=1))
    wall = time.perf_counter() - t0
    # ideal-pool throughput: every core busy, mean per-model time of the
    # stratified sample (favourable to the CPU: ignores the straggler tail)
    wide = any(j[3] == "brbpnn" and j[7] >= CPU_WIDE_HIDDEN for j in jobs)
    return {"models_per_s": cores * len(jobs) / sum(secs), "wall_s": wall, "n": len(jobs),
            "mean_model_s": sum(secs) / len(jobs),
            "note": (f"; BR-BPNN h>={CPU_WIDE_HIDDEN} fits timed for {CPU_EPOCH_SAMPLE} epochs and "
                     f"scaled to {full_epochs:.0f} epochs" if wide else "")}


def reference_arm(args, world, rank):
    if rank != 0:
        return
    series, spec, kw = workload_series(args.workload)
    restarts = args.restarts or DEFAULT_RESTARTS[args.workload]
    cores = os.cpu_count() or 1
    sample = args.cpu_sample or max(32, 4 * cores)
    vals = []
    for i in range(args.warmup + args.steps):
        r = run_cpu(series, spec, kw, restarts, sample, cores)
        if i >= args.warmup:
            vals.append(r)
    v = float(np.mean([r["models_per_s"] for r in vals]))
    line = {
        "metric": "models trained/sec", "value": v, "unit": "models/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean([r["wall_s"] for r in vals])),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.workload, "restarts": restarts},
        "cpu_baseline": {"value": v, "unit": "models/s", "cores": cores, "kind": "port",
                         "sample": f"{vals[0]['n']} stratified tasks/step (one median pick per "
                                   f"equal-count cost stratum) of the {args.workload} workload; "
                                   "ideal-pool throughput = cores / mean per-model seconds; "
                                   "oracle/bbml_oracle.py (bit-identical to the reference)"
                                   + vals[0]["note"]},
        "e2e": {"value": v, "unit": "models/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, world, rank)

    import torch
    import torch.distributed as dist

    from paper_2202_07798_b200 import batch
    from paper_2202_07798_b200._lib import STATUS

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    series, spec, kw = workload_series(args.workload)
    restarts = args.restarts or DEFAULT_RESTARTS[args.workload]
    my_restarts = list(range(rank * restarts, (rank + 1) * restarts))
    wl = batch.build_workload(series, spec, restarts=my_restarts, precision=args.precision, **kw)
    dev = batch.DeviceWorkload(wl)
    torch.cuda.synchronize()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(args.warmup):
        dev.step()
    torch.cuda.synchronize()
    st = dev.fetch()["status"]
    n_bad = int((st["code"] != 0).sum())

    clock_path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
    os.makedirs(os.path.dirname(clock_path), exist_ok=True)
    clk = sample_clocks(clock_path) if rank == 0 else None
    time.sleep(0.3 if clk else 0)

    # device-timed region: K steps, L2 flushed between steps (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(float(k))
        a, b, c, d_ = ev[k]
        a.record(s)
        launches += dev.step_timed(b, c) if hasattr(dev, "step_timed") else dev.step()
        d_.record(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[3]) for e in ev]
    total_s = sum(step_ms) / 1e3

    # clock sampling covers the device-timed region; stopped before the e2e loop
    # (an nvidia-smi query holds the driver and stalls host-side CUDA calls)
    if clk:
        clk.terminate()
        clk.wait()

    # end-to-end: public batched call with pinned host inputs, H2D + D2H every step
    e2e_times = []
    for k in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch.fit_predict(wl, dev, predictions=False)  # result: weights, status, metrics
        e2e_times.append(time.perf_counter() - t0)

    # dominant kernel (PNN train) timed alone on its stream for the roofline
    # each training kernel timed alone on its launching stream (CUDA events)
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
    models_per_step = wl.n_models * world
    value = models_per_step * args.steps / total_s
    e2e_value = models_per_step / e2e_step

    if rank == 0:
        peak_p = peak32 if args.precision == 32 else peak64
        pnn_fl = sum(pnn_flops(int(r["n"]), int(r["d"]), int(r["h"]), int(r["epochs"]), int(r["batch"]))
                     for r in wl.pnn)
        st_lm = st_all[len(wl.pnn):]
        lm_fl = sum(lm_flops(int(r["n"]), int(r["d"]), int(r["h"]), int(e), int(t))
                    for r, e, t in zip(wl.lm, st_lm["epochs"], st_lm["trials"]))
        rl = {}
        if pnn_ms:
            a = pnn_fl / (pnn_ms * 1e-3) / 1e12
            rl["pnn"] = {"bound": f"fp{args.precision}-pipe", "kernel": "pnn_lat_kernel (bbml_pnn_train)",
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
        try:  # DRAM bytes per launch of the dominant kernel from the committed ncu capture
            with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as fh:
                traffic = json.load(fh)
        except (OSError, ValueError):
            traffic = {}
        for v in rl.values():
            name = v["kernel"].split(" ")[0]
            if name in traffic:
                v["traffic"] = traffic[name]["bytes_per_launch"]
                v["traffic_source"] = f'{traffic[name]["report"]} ({traffic[name]["launch"]})'
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
            r = run_cpu(series, spec, kw, restarts, args.cpu_sample or max(32, 4 * cores), cores,
                        wide_ep)
            cpu = {"value": r["models_per_s"], "unit": "models/s", "cores": cores, "kind": "port",
                   "sample": f"{r['n']} stratified tasks (median pick per equal-count cost stratum) "
                             f"of {args.workload}; ideal-pool throughput = cores / mean per-model "
                             f"seconds ({r['mean_model_s']:.3f} s); wall {r['wall_s']:.1f} s"
                             + r["note"]}
        line = {
            "metric": "models trained/sec", "value": value, "unit": "models/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.precision == 32 else "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "restarts_per_gpu": restarts,
                       "models_per_gpu": wl.n_models, "pnn_models": len(wl.pnn),
                       "br_models": len(wl.lm), "pnn_precision": f"fp{args.precision}",
                       "br_precision": "fp64", "l2": "flushed (256 MiB write) between steps",
                       "split": spec.mode.value},
            "e2e": {"value": e2e_value, "unit": "models/s", "h2d_bytes_per_step": dev.h2d_bytes,
                    "d2h_bytes_per_step": dev.d2h_bytes_for(False),
                    "result": "trained weights + status + per-model test MSE / Pearson / "
                              "Spearman (bbml_metrics)"},
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
            "e2e_step_ms": [1e3 * t for t in e2e_times],
        }
        out = json.dumps(line)
        print(out, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as fh:
                fh.write(out + "\n")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
