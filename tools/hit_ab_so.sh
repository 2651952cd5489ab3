#!/bin/bash
# A/B of builds on the hit path (cache = whole table): ab/liblsmgnn_<v>.so for each v given,
# interleaved, 3 rounds, each a fresh bench.py process measuring hbm_regime (direct-call,
# two-stream and graph-replay ms/step, k_serve's fraction of HBM, phase spans).
# usage: tools/hit_ab_so.sh TAG old new ...
set -u
tag=$1; shift
SO=paper_2407_15264_b200/liblsmgnn.so
mkdir -p gpurun_out/ab_$tag
for r in 1 2 3; do
  for v in "$@"; do
    cp ab/liblsmgnn_$v.so $SO
    f=gpurun_out/ab_$tag/${v}_r$r
    timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-steps 0 --no-profile \
      --extras hbm_regime > $f.json 2> $f.err
    python - "$f.json" "$v" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
h = d["hbm_regime"]
print(f"{sys.argv[2]:8s} direct {h['ms_per_step']:.4f}  two {h['two_streams']['ms_per_step']:.4f}  graph "
      f"{h['graph_replay']['ms_per_step']:.4f}  serve {h['roofline']['frac']:.3f}  phases {h['phases_ms_per_step']}")
PY
  done
done
cp ab/liblsmgnn_${!#}.so $SO  # leave the last variant installed
