#!/bin/bash
# ncu evidence of the hit path (cache = whole table, configs[1] trace): one --set full capture
# per kernel of the G = 1 step in steady state, and the launch list of 10 steps.
# usage: tools/r02_ncu_hit.sh TAG [extra env assignments...]
set -u
tag=$1; shift
out=gpurun_out/ncu_$tag
mkdir -p $out
B="python bench.py --lines 1000000 --warmup 60 --steps 3 --no-ablation --no-e2e --no-cpu-baseline --graph-steps 0"
for k in serve set dedup route_local begin; do
  env "$@" timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_$k" --launch-skip 62 -c 1 \
    -o $out/$k $B > $out/$k.log 2>&1
  echo "ncu $k rc=$?"
done
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 560 -c 60 --csv \
  --log-file $out/launches.csv $B > /dev/null 2>&1
echo "launches rc=$?"
ls $out
