mkdir -p gpurun_out/r2d
timeout 300 python tools/prof.py --app pathfinder --kind pnn --precision 64 --epochs 20 > gpurun_out/r2d/pf64.log 2>&1; echo pf=$?
timeout 300 python tools/prof.py --app bicg --kind pnn --precision 64 --epochs 20 --restarts 8 > gpurun_out/r2d/bicg64.log 2>&1; echo bicg=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pnn_f64 -c 1 -o gpurun_out/r2d/pf64 python tools/prof.py --reps 1 --app pathfinder --restarts 1 --kind pnn --precision 64 --epochs 10 > gpurun_out/r2d/ncu_pf64.log 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/r2d/pf64.ncu-rep "pf64 new" > gpurun_out/r2d/pf64.md 2>&1
python tools/ncu_lines.py gpurun_out/r2d/pf64.ncu-rep 80 > gpurun_out/r2d/pf64.lines 2>&1
ncu -i gpurun_out/r2d/pf64.ncu-rep --page source --csv --print-source sass > gpurun_out/r2d/pf64.sass.csv 2>/dev/null; gzip -f gpurun_out/r2d/pf64.sass.csv
rm -f gpurun_out/r2d/pf64.ncu-rep
