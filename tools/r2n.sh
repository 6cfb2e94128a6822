mkdir -p gpurun_out/r2n; rm -f gpurun_out/r2n/*
for R in 32 48 64 96 128; do
  timeout 900 python bench.py --restarts $R --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2n/r$R.log 2>&1
  python -c "
import json; l=json.loads(open('gpurun_out/r2n/r$R.log').read().strip().splitlines()[-1]); print($R, round(l['value']), round(l['ms_per_step'],1), round(l['e2e']['value']))" >> gpurun_out/r2n/summary.txt
done
cat gpurun_out/r2n/summary.txt
