# A/B of two LM builds (ab/head.so vs ab/new.so): hidden-1 LM call + suite16 FP64 step mix, then the GPU tests
mkdir -p gpurun_out/q3; rm -f gpurun_out/q3/*
for rep in 1 2; do for lib in ab/head.so ab/new.so; do
  echo "== $lib" >> gpurun_out/q3/ab.log
  BBML_LIB=$lib timeout 300 python tools/prof.py --precision 64 --kind br --app atax,bicg,syrk,covariance --restarts 32 >> gpurun_out/q3/ab.log 2>&1
  BBML_LIB=$lib PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/q3/ab.log 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/q3/pytest.log 2>&1; echo pytest=$?
timeout 900 python -m pytest tests/test_bench_parity.py -m gpu -q -s > gpurun_out/q3/bench_parity.log 2>&1
