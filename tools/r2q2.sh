# A/B of two PNN builds (ab/head.so vs ab/new.so: pathfinder chain + suite16 FP64 step mix), phase clocks from ab_prof/pnnprof.so, then the GPU tests
mkdir -p gpurun_out/q2; rm -f gpurun_out/q2/*
BBML_LIB=ab_prof/pnnprof.so timeout 300 python tools/prof.py --precision 64 --kind pnn --app pathfinder --restarts 8 --epochs 10 --reps 1 > gpurun_out/q2/prof.log 2>&1
for lib in ab/head.so ab/new.so; do
  echo "== $lib" >> gpurun_out/q2/ab.log
  BBML_LIB=$lib timeout 300 python tools/prof.py --precision 64 --kind pnn --app pathfinder --restarts 8 --epochs 10 >> gpurun_out/q2/ab.log 2>&1
  BBML_LIB=$lib PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/q2/ab.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/q2/pytest.log 2>&1; echo pytest=$?
