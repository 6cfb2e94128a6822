#!/bin/bash
# round-end evidence: bench lines for every config (one box)
mkdir -p gpurun_out/all; O=gpurun_out/all; rm -f $O/*
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench_suite16.log 2> $O/bench_suite16.err; echo suite16=$?
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_suite16.log 2> $O/ref_suite16.err; echo ref=$?
timeout 900 python bench.py --precision 32 --no-cpu-baseline > $O/bench_suite16_fp32.log 2> $O/bench_suite16_fp32.err; echo suite16_fp32=$?
timeout 900 python bench.py --workload app20 > $O/bench_app20.log 2> $O/bench_app20.err; echo app20=$?
timeout 1500 python bench.py --workload sweep --steps 3 --warmup 3 > $O/bench_sweep.log 2> $O/bench_sweep.err; echo sweep=$?
timeout 1500 python bench.py --workload sweep --scaling strong --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_sweep_strong.log 2> $O/bench_sweep_strong.err; echo sweep_strong=$?
timeout 1800 python bench.py --workload wide --steps 3 --warmup 3 > $O/bench_wide.log 2> $O/bench_wide.err; echo wide=$?
for f in $O/bench_*.log $O/ref_suite16.log; do echo $f; tail -1 $f | cut -c1-400; done
