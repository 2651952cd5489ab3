#!/bin/bash
# A/B of hit-path variants (env assignments), interleaved, 3 rounds, each a fresh bench.py
# process measuring hbm_regime (cache = whole table): direct-call and graph-replay ms/step.
# usage: tools/hit_ab.sh TAG "VAR=1 VAR2=x" "VAR=0" ...
set -u
tag=$1; shift
mkdir -p gpurun_out/ab_$tag
for r in 1 2 3; do
  i=0
  for v in "$@"; do
    i=$((i+1))
    f=gpurun_out/ab_$tag/v${i}_r$r
    env $v timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-steps 0 --no-profile \
      --extras hbm_regime > $f.json 2> $f.err
    python - "$f.json" "$v" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
h = d["hbm_regime"]
print(f"{sys.argv[2]:40s} direct {h['ms_per_step']:.4f}  two {h['two_streams']['ms_per_step']:.4f}  graph "
      f"{h['graph_replay']['ms_per_step']:.4f}  serve {h['roofline']['frac']:.3f}  phases {h['phases_ms_per_step']}")
PY
  done
done
