#!/bin/bash
# The driver's round-end sequence on the current build, plus evidence: the full GPU suite,
# smoke, ncu --set full of k_serve on the bench workload (roofline.traffic) and the hit path,
# the steady-state launch list, then the default bench line.
set -u
mkdir -p gpurun_out/full
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/full/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/full/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/full/smoke.log
B="python bench.py --steps 3 --warmup 3 --no-ablation --no-e2e --no-cpu-baseline --graph-steps 0"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_serve" --launch-skip 4 -c 1 \
  -o gpurun_out/full/cfg2_serve $B > gpurun_out/full/cfg2_serve.log 2>&1; echo "ncu cfg2 serve rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_(set|dedup)" --launch-skip 8 -c 2 \
  -o gpurun_out/full/cfg2_meta $B > gpurun_out/full/cfg2_meta.log 2>&1; echo "ncu cfg2 meta rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 -c 80 --csv \
  --log-file gpurun_out/full/launches_cfg2.csv python bench.py --steps 20 --warmup 3 --no-ablation --no-e2e \
  --no-cpu-baseline --graph-steps 0 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1500 python bench.py > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/full/bench.err
