for v in 4 2 4 2; do
BBML_PNN_NPW=$v timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('npw=$v', round(d['ms_per_step'],1), 'lm', round(r['kernel_ms'],1), 'pnn', round(r['other']['pnn']['kernel_ms'],1), 'e2e', round(d['e2e']['value']))"
done
for v in 4 2; do BBML_PNN_NPW=$v timeout 300 python tools/prof.py --restarts 32 --kind pnn --reps 2; done
timeout 300 python tools/prof.py --restarts 32 --kind br --reps 2
