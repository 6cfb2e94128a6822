mkdir -p gpurun_out/r2q; rm -f gpurun_out/r2q/*
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2q/pytest.log 2>&1; echo pytest=$?
timeout 1800 python bench.py --workload wide --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2q/wide.log 2>&1; echo wide=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lm_wide --csv --log-file gpurun_out/r2q/wide_traffic.csv python tools/prof.py --workload wide --kind br --restarts 7 --br-epochs 40 --reps 1 > /dev/null 2>&1; echo traffic=$?
