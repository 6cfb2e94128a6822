mkdir -p gpurun_out/r2t; rm -f gpurun_out/r2t/*
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2t/pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/prof.py --app pathfinder --kind pnn --precision 64 --epochs 20 > gpurun_out/r2t/pf64.log 2>&1
timeout 300 python tools/prof.py --app bicg --kind pnn --precision 64 --epochs 20 --restarts 8 > gpurun_out/r2t/bicg64.log 2>&1
for rep in 1 2; do PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2t/mix.log 2>&1; done
