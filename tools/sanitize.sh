#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck on the config-1-shaped smoke run (G = 1)
# and memcheck on a 2-process G = 2 run (ranks share one GPU, each rank instrumented). Writes gpurun_out/sanitize_*.log
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
# the pipelined file tier (device-published fill list, host preads, per-chunk device waits)
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_storage_file.py -q -x \
  -k "small_rows" > $out/sanitize_memcheck_file.log 2>&1
echo "G=1 file tier memcheck rc=$? : $(grep -E 'ERROR SUMMARY' $out/sanitize_memcheck_file.log | tail -1) $(grep -Eo '[0-9]+ passed' $out/sanitize_memcheck_file.log)" >> $out/sanitize_summary.txt
# consecutive gathers issued without host synchronisation (parity-indexed tables, done counters;
# the sanitizer serialises the kernels, so this checks the parity offsets and bounds)
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_overlap.py -q -x \
  -k "overlapped" > $out/sanitize_memcheck_overlap.log 2>&1
echo "G=1 overlapped gathers memcheck rc=$? : $(grep -E 'ERROR SUMMARY' $out/sanitize_memcheck_overlap.log | tail -1) $(grep -Eo '[0-9]+ passed' $out/sanitize_memcheck_overlap.log)" >> $out/sanitize_summary.txt
# G = 2: each rank runs under its own compute-sanitizer (torch.distributed env set by hand, so
# the ranks themselves are instrumented), both pull orders; the ranks' outputs are
# checked (rows bad = 0)
for split in 0 1; do
  d=/tmp/san_g2_s$split; rm -rf $d; mkdir -p $d
  port=$((29533 + split))
  for r in 0 1; do
    LSMGNN_SPLIT_PULL=$split RANK=$r LOCAL_RANK=$r WORLD_SIZE=2 LOCAL_WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$port \
      timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tests/mp_worker.py gather $d hybrid 1 \
      > $out/sanitize_memcheck_g2_s${split}_r$r.log 2>&1 &
  done
  wait
  for r in 0 1; do
    echo "G=2 split=$split rank $r memcheck: $(grep -E 'ERROR SUMMARY' $out/sanitize_memcheck_g2_s${split}_r$r.log | tr '\n' ' ') output: $(cat $d/r$r.json 2>&1 | head -c 60)" >> $out/sanitize_summary.txt
  done
done
cat $out/sanitize_summary.txt
