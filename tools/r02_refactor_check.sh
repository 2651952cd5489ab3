#!/bin/bash
# GPU check of a kernel change: the device-function test, the single-home parity suites,
# the multi-process suite, then the hit path and the headline (short bench, no side runs
# except hbm_regime), with serve-geometry A/B variants.
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_device_funcs.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fuzz.py -x -q > gpurun_out/$1_parity.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/$1_parity.log
timeout 600 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_storage_file.py tests/test_gpu_sampler.py tests/test_c_abi.py -x -q > gpurun_out/$1_mp.log 2>&1
echo "mp rc=$?"; tail -2 gpurun_out/$1_mp.log
for v in "2 3" "1 6" "2 2" "0 0"; do
  set -- $1 $v
  if [ "$2" = "0" ]; then export LSMGNN_SERVE_ST=0; unset LSMGNN_SERVE_CPS; else export LSMGNN_SERVE_CPS=$2 LSMGNN_SERVE_ST=$3; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --extras hbm_regime > gpurun_out/$1_bench_$2_$3.json 2> gpurun_out/$1_bench_$2_$3.err
  python - "$1" "$2" "$3" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench_{sys.argv[2]}_{sys.argv[3]}.json").read().strip().splitlines()[-1])
h = d.get("hbm_regime", {})
print("cps/st", sys.argv[2], sys.argv[3], "value", d["value"], "roof", d["roofline"]["frac"], "hbm ms", h.get("ms_per_step"),
      "serve frac", h.get("roofline", {}).get("frac"), "phases", h.get("phases_ms_per_step"), "graph", h.get("graph_replay"))
PY
done
unset LSMGNN_SERVE_CPS LSMGNN_SERVE_ST
