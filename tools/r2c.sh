mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2c/pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/prof.py --app pathfinder --kind pnn --precision 64 --epochs 20 > gpurun_out/r2c/pf64.log 2>&1; echo pf=$?
timeout 300 python tools/prof.py --app bicg --kind pnn --precision 64 --epochs 20 --restarts 8 > gpurun_out/r2c/bicg64.log 2>&1; echo bicg=$?
PREC=64 STEPMIX_CASES=3 timeout 600 python tools/step_mix.py > gpurun_out/r2c/mix64.log 2>&1; echo mix=$?
