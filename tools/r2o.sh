mkdir -p gpurun_out/r2o; rm -f gpurun_out/r2o/*
BBML_F64_LONG_NPW=1 timeout 300 python tools/prof.py --app pathfinder --kind pnn --precision 64 --epochs 20 > gpurun_out/r2o/pf_p1.log 2>&1
for rep in 1 2; do for cfg in "0 4" "0 1" "1 1"; do
  set -- $cfg
  echo "== LONG_FIRST=$1 LONG_NPW=$2" >> gpurun_out/r2o/ab.log
  BBML_PNN_LONG_FIRST=$1 BBML_F64_LONG_NPW=$2 PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2o/ab.log 2>&1
done; done
