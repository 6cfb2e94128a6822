#!/bin/bash
# Build an alternate libbbml.so from a git revision of csrc/ (A/B timing in
# one gpurun call via BBML_LIB=...).  usage: tools/build_alt.sh REV OUT.so
set -e
rev=$1; out=$2
tmp=$(mktemp -d)
git archive "$rev" paper_2202_07798_b200/csrc include | tar -x -C "$tmp"
objs=()
for s in capi pnn_train lm_train lm_wide predict units metrics; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    ${DEFS} -I "$tmp/include" --expt-relaxed-constexpr -c "$tmp/paper_2202_07798_b200/csrc/$s.cu" -o "$tmp/$s.o" &
  objs+=("$tmp/$s.o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -cudart static "${objs[@]}" -o "$out"
rm -rf "$tmp"
