#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck on the config-1-shaped smoke run (G = 1)
# and memcheck on a 2-process G = 2 run (ranks share one GPU). Writes gpurun_out/sanitize_*.log
# and a one-line-per-tool summary to gpurun_out/sanitize_summary.txt.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out
mkdir -p $out
: > $out/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py smoke > $out/sanitize_$tool.log 2>&1
  echo "G=1 $tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/sanitize_$tool.log | tail -1) $(grep -c 'smoke ok' $out/sanitize_$tool.log) smoke-ok" >> $out/sanitize_summary.txt
done
# multi-tile k_scan (look-back across CTAs) + oversized sets + the hit fast path, G = 1
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "multi_tile_set_scan and hybrid" > $out/sanitize_${tool}_multitile.log 2>&1
  echo "G=1 multi-tile $tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/sanitize_${tool}_multitile.log | tail -1) $(grep -Eo '[0-9]+ passed' $out/sanitize_${tool}_multitile.log)" >> $out/sanitize_summary.txt
done
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 \
  tests/mp_worker.py gather /tmp hybrid 1 > $out/sanitize_memcheck_g2.log 2>&1
echo "G=2 memcheck rc=$? : $(grep -E 'ERROR SUMMARY' $out/sanitize_memcheck_g2.log | tr '\n' ' ')" >> $out/sanitize_summary.txt
cat $out/sanitize_summary.txt
