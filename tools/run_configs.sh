#!/bin/bash
# bench lines for every BASELINE config workload (one box); logs into gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py --workload app20 > gpurun_out/bench_app20.log 2> gpurun_out/bench_app20.err; echo app20=$?
timeout 1200 python bench.py --workload sweep --steps 3 --warmup 3 > gpurun_out/bench_sweep.log 2> gpurun_out/bench_sweep.err; echo sweep=$?
timeout 1500 python bench.py --workload wide --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_wide.log 2> gpurun_out/bench_wide.err; echo wide=$?
for f in app20 sweep wide; do tail -1 gpurun_out/bench_$f.log | cut -c1-700; done
