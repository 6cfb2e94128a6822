#!/bin/bash
# A/B of an environment switch on the suite16 bench step: ENVS="A=1 A=0" tools/ab_env.sh
for rep in 1 2; do
for e in ${ENVS}; do
  env $e timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$e', round(d['ms_per_step'],1), 'pnn', round(r['other']['pnn']['kernel_ms'],1), 'lm', round(r['kernel_ms'],1), [round(x) for x in d['e2e_step_ms']])"
done; done
