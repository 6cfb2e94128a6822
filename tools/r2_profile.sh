# r02 profiling pass: launch list, DRAM traffic per kernel, --set full captures
set -x
mkdir -p gpurun_out/r2p; rm -rf gpurun_out/r2p/*
O=gpurun_out/r2p
# 1. launch list of the bench step (FP64 headline config)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/launches.log 2>&1; echo launches=$?
# 2. DRAM bytes of every training launch of one suite16 step (both kinds)
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"pnn_|lm_" --csv --log-file $O/traffic.csv python tools/prof.py --precision 64 --restarts 32 --reps 1 > $O/traffic.log 2>&1; echo traffic=$?
# 3. --set full captures
cap() { name=$1; shift; timeout 900 ncu --set full --clock-control none --import-source on -c 1 "$@" > $O/ncu_$name.log 2>&1; echo $name=$?; python tools/ncu_summary.py $O/$name.ncu-rep "$name" > $O/$name.md 2>&1; python tools/ncu_lines.py $O/$name.ncu-rep 40 > $O/$name.lines 2>&1; ncu -i $O/$name.ncu-rep --page source --csv --print-source sass > $O/$name.sass.csv 2>/dev/null; gzip -f $O/$name.sass.csv; [ $(stat -c %s $O/$name.ncu-rep) -gt 25000000 ] && rm -f $O/$name.ncu-rep; }
cap pnn_f64_long -k regex:pnn_f64_kernel -o $O/pnn_f64_long python tools/prof.py --precision 64 --kind pnn --app pathfinder --epochs 10 --reps 1
cap pnn_f64_short -k regex:pnn_f64_kernel_shared -o $O/pnn_f64_short python tools/prof.py --precision 64 --kind pnn --not-app 2mm,doitgen,gemm,pathfinder --restarts 32 --epochs 30 --reps 1
cap lm_warp32 -k regex:lm_warp_kernel -o $O/lm_warp32 python tools/prof.py --kind br --app gramschmit --restarts 32 --reps 1
cap lm_h1 -k regex:lm_warp_kernel -o $O/lm_h1 python tools/prof.py --kind br --app atax,bicg,syrk,covariance --restarts 32 --reps 1
cap lm_wide -k regex:lm_wide -o $O/lm_wide python tools/prof.py --workload wide --kind br --restarts 7 --br-epochs 40 --reps 1
ls -la $O
