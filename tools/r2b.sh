# FP64 PNN profiles: pathfinder (long variant) and bicg (short variant)
mkdir -p gpurun_out/r2b
timeout 300 python tools/prof.py --app pathfinder --kind pnn --precision 64 --epochs 20 > gpurun_out/r2b/pf64.log 2>&1; echo pf=$?
timeout 300 python tools/prof.py --app bicg --kind pnn --precision 64 --epochs 20 --restarts 8 > gpurun_out/r2b/bicg64.log 2>&1; echo bicg=$?
for r in pf64 bicg64; do
  if [ $r = pf64 ]; then a="--app pathfinder --restarts 1"; else a="--app bicg --restarts 8"; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pnn_lat -c 1 -o gpurun_out/r2b/$r python tools/prof.py $a --kind pnn --precision 64 --epochs 20 > gpurun_out/r2b/ncu_$r.log 2>&1; echo ncu$r=$?
  python tools/ncu_summary.py gpurun_out/r2b/$r.ncu-rep "$r" > gpurun_out/r2b/$r.md 2>&1
  ncu -i gpurun_out/r2b/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/r2b/$r.sass.csv 2>/dev/null
  gzip -f gpurun_out/r2b/$r.sass.csv
  [ $(stat -c %s gpurun_out/r2b/$r.ncu-rep) -gt 20000000 ] && rm -f gpurun_out/r2b/$r.ncu-rep
done
du -sh gpurun_out/r2b/*
