mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --precision 64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a/bench64.log 2>&1; echo b64=$?
PREC=64 STEPMIX_CASES=3 timeout 600 python tools/step_mix.py > gpurun_out/r2a/mix64.log 2>&1; echo mix=$?
lscpu | head -20 > gpurun_out/r2a/lscpu.txt
