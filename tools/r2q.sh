mkdir -p gpurun_out/r2q; rm -f gpurun_out/r2q/*
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2q/pytest.log 2>&1; echo pytest=$?
timeout 1800 python bench.py --workload wide --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2q/wide.log 2>&1; echo wide=$?
PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py > gpurun_out/r2q/mix.log 2>&1
