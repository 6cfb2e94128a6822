mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2h/pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/r2h/bench64.log 2> gpurun_out/r2h/bench64.err; echo b64=$?
timeout 900 python bench.py --precision 32 --no-cpu-baseline > gpurun_out/r2h/bench32.log 2> gpurun_out/r2h/bench32.err; echo b32=$?
timeout 900 python bench.py --workload sweep --scaling strong --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2h/sweep_strong.log 2> gpurun_out/r2h/sweep_strong.err; echo sweep=$?
