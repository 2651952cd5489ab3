#!/bin/bash
# ncu --set full of the G = 1 hit-path kernels (cache = whole table), steady state
set -u
out=gpurun_out/ncu_$1; shift
mkdir -p $out
B="python bench.py --lines 1000000 --warmup 60 --steps 3 --no-ablation --no-e2e --no-cpu-baseline --graph-steps 0"
for k in serve set dedup route_local; do
  env "$@" timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_$k" --launch-skip 62 -c 1 \
    -o $out/$k $B > $out/$k.log 2>&1
  echo "ncu $k rc=$?"
done
