#!/bin/bash
# A/B of the e2e measurement (lsmgnn_gather_host into pinned host out) between env settings,
# interleaved, 3 rounds (configs[1], 10 e2e steps each)
set -u
tag=$1; shift
mkdir -p gpurun_out/e2e_$tag
for r in 1 2 3; do
  i=0
  for v in "$@"; do
    i=$((i+1))
    f=gpurun_out/e2e_$tag/v${i}_r$r
    env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-ablation --no-cpu-baseline --graph-steps 0 > $f.json 2> $f.err
    python -c "
import json,sys; d=json.loads(open('$f.json').read().strip().splitlines()[-1])
print('%-22s value %.2f e2e %.2f dev %.2f' % ('$v', d['value'], d['e2e']['value'], d['e2e']['device_result']['value']))"
  done
done
