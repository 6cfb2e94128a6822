mkdir -p gpurun_out/r2o; rm -f gpurun_out/r2o/*
for rep in 1 2; do
for lib in paper_2202_07798_b200/libbbml.so ab/lm_h1minb5.so ab/lm_h1minb4.so; do
  echo "== $lib" >> gpurun_out/r2o/ab.log
  BBML_LIB=$lib PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2o/ab.log 2>&1
done; done
