#!/bin/bash
# Round-end evidence on the GPU box (repo root): ncu captures of the bench workload, their
# per-kernel JSON (read by bench.py for roofline.traffic), the launch list, then the default
# bench line. Everything lands in gpurun_out/ (copied into profiles/ by hand afterwards).
set -u
out=gpurun_out
mkdir -p $out/ncu
B="python bench.py --steps 3 --warmup 3 --no-ablation --no-e2e --no-cpu-baseline --graph-steps 0"
for k in serve set dedup scan; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^k_$k" --launch-skip 4 -c 1 \
    -o $out/ncu/final_$k $B > $out/ncu/final_$k.log 2>&1
done
# the hit path alone (cache = whole table): k_serve HBM traffic
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_serve" --launch-skip 62 -c 1 \
  -o $out/ncu/final_serve_hit python bench.py --lines 1000000 --warmup 60 --steps 3 --no-ablation --no-e2e \
  --no-cpu-baseline --graph-steps 0 > $out/ncu/final_serve_hit.log 2>&1
python tools/ncu_kernels_json.py $out/ncu_kernels_latest.json $out/ncu/final_serve.ncu-rep $out/ncu/final_set.ncu-rep \
  $out/ncu/final_dedup.ncu-rep $out/ncu/final_scan.ncu-rep
cp $out/ncu_kernels_latest.json profiles/ncu_kernels_latest.json
# steady state: skip the 800 launches of init + the W-batch window bootstrap, then 20 steps
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 800 -c 200 --csv \
  --log-file $out/final_launches.csv python bench.py --steps 20 --warmup 3 --no-ablation --no-e2e \
  --no-cpu-baseline --graph-steps 0 --no-file-tier > /dev/null 2>&1
timeout 1500 python bench.py > $out/final_bench.json 2> $out/final_bench.err
tail -c 400 $out/final_bench.err
ls -la $out/ncu
