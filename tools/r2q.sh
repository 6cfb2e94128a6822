mkdir -p gpurun_out/r2q; rm -f gpurun_out/r2q/*
timeout 1800 python bench.py --workload wide --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2q/wide.log 2>&1; echo wide=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "wide or init" > gpurun_out/r2q/pytest.log 2>&1; echo pytest=$?
