mkdir -p gpurun_out/r2l; rm -f gpurun_out/r2l/*
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2l/pytest.log 2>&1; echo pytest=$?
