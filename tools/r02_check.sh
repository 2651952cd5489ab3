#!/bin/bash
# usage: tools/r02_check.sh TAG [serve variants "cps st" ...]
# parity (single-home, graph, fuzz, device functions), then bench.py (headline + hbm_regime) per
# k_serve geometry variant ("0 0" = 16-B vector delivery instead of TMA rings).
set -u
tag=$1; shift
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_device_funcs.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fuzz.py -q > gpurun_out/${tag}_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/${tag}_parity.log
[ $# -eq 0 ] && set -- "2 3"
for v in "$@"; do
  set -- $v
  if [ "$1" = "0" ]; then export LSMGNN_SERVE_ST=0; unset LSMGNN_SERVE_CPS; else export LSMGNN_SERVE_CPS=$1 LSMGNN_SERVE_ST=$2; fi
  f=gpurun_out/${tag}_bench_$1_$2
  timeout 400 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --extras hbm_regime > $f.json 2> $f.err
  python - "$f.json" "$1" "$2" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
h = d.get("hbm_regime", {})
print("cps/st", sys.argv[2], sys.argv[3], "value", d["value"], "roof", d["roofline"]["frac"], "| hbm ms", h.get("ms_per_step"),
      "hit", h.get("hit_ratio"), "serve frac", h.get("roofline", {}).get("frac"), "phases", h.get("phases_ms_per_step"),
      "two", (h.get("two_streams") or {}).get("ms_per_step"), "graph", (h.get("graph_replay") or {}).get("ms_per_step"))
PY
done
unset LSMGNN_SERVE_CPS LSMGNN_SERVE_ST
