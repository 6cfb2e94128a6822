mkdir -p gpurun_out/r2r; rm -f gpurun_out/r2r/*
for rep in 1 2; do for mb in 4 3; do
  echo "== SHORT_MINB=$mb" >> gpurun_out/r2r/ab.log
  BBML_F64_SHORT_MINB=$mb PREC=64 STEPMIX_CASES=3 timeout 300 python tools/step_mix.py >> gpurun_out/r2r/ab.log 2>&1
done; done
for mb in 4 3; do
BBML_F64_SHORT_MINB=$mb timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"pnn_" --csv --log-file gpurun_out/r2r/traffic_mb$mb.csv python tools/prof.py --precision 64 --kind pnn --restarts 32 --reps 1 > /dev/null 2>&1
done
