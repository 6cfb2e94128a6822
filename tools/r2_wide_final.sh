# wide (cfg 5) evidence: bench line + one ncu --set full capture of lm_wide_kernel_once (3 epochs)
O=gpurun_out/widef; mkdir -p $O; rm -rf $O/*
timeout 1800 python bench.py --workload wide --steps 3 --warmup 3 > $O/bench_wide.log 2> $O/bench_wide.err; echo wide=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lm_wide -c 1 -o $O/lm_wide python tools/prof.py --workload wide --kind br --br-epochs 3 --restarts 7 --reps 1 > $O/ncu.log 2>&1; echo ncu=$?
python tools/ncu_summary.py $O/lm_wide.ncu-rep lm_wide > $O/lm_wide.md 2>&1
python tools/ncu_lines.py $O/lm_wide.ncu-rep 60 > $O/lm_wide.lines 2>&1
rm -f $O/lm_wide.ncu-rep
