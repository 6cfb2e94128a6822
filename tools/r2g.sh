mkdir -p gpurun_out/r2g
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2g/pytest.log 2>&1; echo pytest=$?
