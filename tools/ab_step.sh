#!/bin/bash
# A/B: suite16 concurrent step (all / pnn only / lm only) + bench line per library in ab/
for rep in 1 2; do
for lib in ab/*.so; do
  echo "== $lib"
  BBML_LIB=$lib STEPMIX_CASES=3 timeout 300 python tools/step_mix.py 2>&1 | tail -3
  BBML_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step'],1), [round(x) for x in d['e2e_step_ms']])"
done; done
