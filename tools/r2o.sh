mkdir -p gpurun_out/r2o; rm -f gpurun_out/r2o/*
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2o/pytest.log 2>&1; echo pytest=$?
for lib in paper_2202_07798_b200/libbbml.so ab/lm_minb6.so ab/lm_minb8.so; do
  echo "== $lib" >> gpurun_out/r2o/ab.log
  BBML_LIB=$lib timeout 300 python tools/prof.py --precision 64 --kind br --app gramschmit --restarts 32 >> gpurun_out/r2o/ab.log 2>&1
  BBML_LIB=$lib PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2o/ab.log 2>&1
done
