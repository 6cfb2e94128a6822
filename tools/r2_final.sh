# round-2 final evidence: bench lines for every config + launch list + DRAM traffic + ncu of the top kernels
set -x
O=gpurun_out/final; mkdir -p $O; rm -rf $O/*
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest=$?
timeout 900 python -m pytest tests/test_bench_parity.py -m gpu -q -s > $O/bench_parity.log 2>&1; echo bench_parity=$?
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench_suite16.log 2> $O/bench_suite16.err; echo suite16=$?
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_suite16.log 2> $O/ref_suite16.err; echo ref=$?
timeout 900 python bench.py --precision 32 --no-cpu-baseline > $O/bench_suite16_fp32.log 2> $O/bench_suite16_fp32.err; echo fp32=$?
timeout 900 python bench.py --workload app20 > $O/bench_app20.log 2> $O/bench_app20.err; echo app20=$?
timeout 1500 python bench.py --workload sweep --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_sweep.log 2> $O/bench_sweep.err; echo sweep=$?
timeout 1500 python bench.py --workload sweep --scaling strong --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_sweep_strong.log 2> $O/bench_sweep_strong.err; echo sweep_strong=$?
timeout 1800 python bench.py --workload wide --steps 3 --warmup 3 > $O/bench_wide.log 2> $O/bench_wide.err; echo wide=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/launches.log 2>&1; echo launches=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"pnn_|lm_" --csv --log-file $O/traffic.csv python tools/prof.py --precision 64 --restarts 32 --reps 1 > $O/traffic.log 2>&1; echo traffic=$?
cap() { name=$1; shift; timeout 900 ncu --set full --clock-control none --import-source on -c 1 "$@" > $O/ncu_$name.log 2>&1; echo $name=$?; python tools/ncu_summary.py $O/$name.ncu-rep "$name" > $O/$name.md 2>&1; python tools/ncu_lines.py $O/$name.ncu-rep 40 > $O/$name.lines 2>&1; rm -f $O/$name.ncu-rep; }
cap pnn_f64_long -k regex:pnn_f64_kernel -o $O/pnn_f64_long python tools/prof.py --precision 64 --kind pnn --app pathfinder --epochs 10 --reps 1
cap pnn_f64_short -k regex:pnn_f64_kernel_shared -o $O/pnn_f64_short python tools/prof.py --precision 64 --kind pnn --not-app 2mm,doitgen,gemm,pathfinder --restarts 32 --epochs 30 --reps 1
cap lm_h1 -k regex:lm_warp_kernel -o $O/lm_h1 python tools/prof.py --kind br --app atax,bicg,syrk,covariance --restarts 32 --reps 1
cap lm_warp32 -k regex:lm_warp_kernel -o $O/lm_warp32 python tools/prof.py --precision 64 --kind br --app gramschmit --restarts 32 --reps 1
