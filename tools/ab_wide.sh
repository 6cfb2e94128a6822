#!/bin/bash
# A/B of the wide BR-BPNN kernel across ab/*.so (50 epochs, 7 restarts)
for lib in ab/*.so; do
  echo "== $lib"; BBML_LIB=$lib timeout 300 python tools/prof.py --workload wide --kind br --br-epochs ${EP:-50} --restarts ${R:-7} 2>&1 | tail -1 | cut -c1-200
done
