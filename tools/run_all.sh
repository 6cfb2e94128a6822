#!/bin/bash
# round-end evidence: bench lines for every config + launch list (one box)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_suite16.log 2> gpurun_out/bench_suite16.err; echo suite16=$?
timeout 900 python bench.py --impl reference > gpurun_out/ref_suite16.log 2> gpurun_out/ref_suite16.err; echo ref=$?
timeout 900 python bench.py --workload app20 > gpurun_out/bench_app20.log 2> gpurun_out/bench_app20.err; echo app20=$?
timeout 1200 python bench.py --workload sweep --steps 3 --warmup 3 > gpurun_out/bench_sweep.log 2> gpurun_out/bench_sweep.err; echo sweep=$?
timeout 1500 python bench.py --workload wide --steps 3 --warmup 3 > gpurun_out/bench_wide.log 2> gpurun_out/bench_wide.err; echo wide=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --restarts 4 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
for f in suite16 app20 sweep wide; do tail -1 gpurun_out/bench_$f.log | cut -c1-300; done
tail -1 gpurun_out/ref_suite16.log | cut -c1-300
