mkdir -p gpurun_out/r2u; rm -f gpurun_out/r2u/*
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2u/pytest.log 2>&1; echo pytest=$?
for rep in 1 2; do for lib in ab/head.so paper_2202_07798_b200/libbbml.so; do
  echo "== $lib" >> gpurun_out/r2u/ab.log
  BBML_LIB=$lib PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2u/ab.log 2>&1
done; done
for lib in ab/head.so paper_2202_07798_b200/libbbml.so; do
  echo "== wide $lib" >> gpurun_out/r2u/ab.log
  BBML_LIB=$lib timeout 600 python tools/prof.py --workload wide --kind br --restarts 7 --br-epochs 100 >> gpurun_out/r2u/ab.log 2>&1
done
