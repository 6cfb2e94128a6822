#!/bin/bash
# A/B: per-app LM timing for each alternate library in ab/ (one box, back to back)
apps=${APPS:-gramschmit,2mm,pathfinder}
for rep in 1 2; do
for lib in ab/*.so; do
  echo "== $lib"; BBML_LIB=$lib timeout 300 python tools/lm_apps.py ${R:-32} $apps 2>&1 | cut -c1-60
done; done
