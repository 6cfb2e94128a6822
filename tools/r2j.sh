mkdir -p gpurun_out/r2j; rm -f gpurun_out/r2j/*
P="--precision 64 --restarts 32"
timeout 300 python tools/prof.py $P --kind pnn --app 2mm,doitgen,gemm,pathfinder > gpurun_out/r2j/pnn_dm4.log 2>&1
timeout 300 python tools/prof.py $P --kind pnn --not-app 2mm,doitgen,gemm,pathfinder > gpurun_out/r2j/pnn_dm2.log 2>&1
timeout 300 python tools/prof.py $P --kind pnn --app gemm,pathfinder > gpurun_out/r2j/pnn_long.log 2>&1
timeout 300 python tools/prof.py $P --kind pnn --app 2mm,doitgen > gpurun_out/r2j/pnn_mid.log 2>&1
timeout 300 python tools/prof.py $P --kind br --app gramschmit > gpurun_out/r2j/lm_gram.log 2>&1
timeout 300 python tools/prof.py $P --kind br --not-app gramschmit > gpurun_out/r2j/lm_h1.log 2>&1
