mkdir -p gpurun_out/r2f
rm -f gpurun_out/r2f/ab2.log
for cfg in "4 4 0" "4 4 1" "4 3 1"; do
  set -- $cfg
  echo "== NPW=$1 MINB=$2 SPLIT=$3" >> gpurun_out/r2f/ab2.log
  BBML_PNN_SPLIT=$3 BBML_F64_LONG_NPW=$1 BBML_F64_SHORT_MINB=$2 PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2f/ab2.log 2>&1
done
