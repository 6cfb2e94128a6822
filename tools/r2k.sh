mkdir -p gpurun_out/r2k; rm -f gpurun_out/r2k/*
for cfg in "0 2" "1 2" "0 1" "1 1"; do
  set -- $cfg
  echo "== LONG_FIRST=$1 LONG_GROUPS=$2" >> gpurun_out/r2k/ab.log
  BBML_PNN_LONG_FIRST=$1 BBML_F64_LONG_GROUPS=$2 PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2k/ab.log 2>&1
done
