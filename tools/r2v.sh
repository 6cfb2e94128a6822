mkdir -p gpurun_out/r2v; rm -f gpurun_out/r2v/*
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2v/pytest.log 2>&1; echo pytest=$?
timeout 900 python tools/artifacts_time.py > gpurun_out/r2v/artifacts.log 2>&1; echo art=$?
