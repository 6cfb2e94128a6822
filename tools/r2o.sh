mkdir -p gpurun_out/r2o; rm -f gpurun_out/r2o/*
for cfg in "1 1" "0 1" "1 2" "0 4"; do
  set -- $cfg
  echo "== LONG_FIRST=$1 LONG_NPW=$2" >> gpurun_out/r2o/ab.log
  BBML_PNN_LONG_FIRST=$1 BBML_F64_LONG_NPW=$2 PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2o/ab.log 2>&1
done
