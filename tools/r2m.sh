mkdir -p gpurun_out/r2m; rm -f gpurun_out/r2m/*
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2m/pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/prof.py --app bicg --kind pnn --precision 64 --epochs 20 --restarts 8 > gpurun_out/r2m/bicg64.log 2>&1
timeout 300 python tools/prof.py --app pathfinder --kind pnn --precision 64 --epochs 20 > gpurun_out/r2m/pf64.log 2>&1
BBML_F64_LONG_NPW=1 timeout 300 python tools/prof.py --app pathfinder --kind pnn --precision 64 --epochs 20 > gpurun_out/r2m/pf64_npw1.log 2>&1
for cfg in "4 4" "1 4" "2 4" "1 3"; do
  set -- $cfg
  echo "== F64_LONG_NPW=$1 SHORT_MINB=$2" >> gpurun_out/r2m/ab.log
  BBML_F64_LONG_NPW=$1 BBML_F64_SHORT_MINB=$2 PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2m/ab.log 2>&1
done
for npw in 4 2 1; do
  echo "== FP32 PNN_NPW=$npw" >> gpurun_out/r2m/ab.log
  BBML_PNN_NPW=$npw PREC=32 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2m/ab.log 2>&1
done
