#!/bin/bash
# PDL A/B (LSMGNN_NO_PDL=1 vs default), alternating: configs[0] shape (launch-bound) direct
# and as CUDA-graph replays, the hit path (HBM-bound), configs[1] (PCIe-bound).
set -u
out=gpurun_out/ab_pdl; mkdir -p $out
X="--no-ablation --no-e2e --no-cpu-baseline --no-file-tier"
show() { python -c "
import json;d=json.load(open('$1'));h=d.get('hbm_regime') or {}
print(d['value'],d['ms_per_step'],'graph',(d.get('graph_replay') or {}).get('ms_per_step'))" 2>&1; }
for i in 1 2; do
  for v in pdl nopdl; do
    E=""; [ $v = nopdl ] && E="LSMGNN_NO_PDL=1"
    env $E timeout 300 python bench.py --config cfg1 --steps 100 --warmup 10 --graph-steps 100 $X > $out/cfg1_$v$i.json 2>/dev/null
    echo "cfg1 $v $i: $(show $out/cfg1_$v$i.json)"
    env $E timeout 300 python bench.py --lines 1000000 --warmup 60 --steps 30 --graph-steps 30 $X > $out/hit_$v$i.json 2>/dev/null
    echo "hit $v $i: $(show $out/hit_$v$i.json)"
  done
done
for v in pdl nopdl; do
  E=""; [ $v = nopdl ] && E="LSMGNN_NO_PDL=1"
  env $E timeout 300 python bench.py --steps 20 --warmup 5 --graph-steps 10 $X > $out/cfg2_$v.json 2>/dev/null
  echo "cfg2 $v: $(show $out/cfg2_$v.json)"
done
