#!/bin/bash
# On the GPU box: swap each ab/mut_*.so (tools/gpu_mutants.py build) in for liblsmgnn.so and run
# the GPU parity tests (single-home file first, then the multi-process parity cases); record
# the first failing test. Every mutant must be killed.
set -u
out=gpurun_out/gpu_mutants; mkdir -p $out
SO=paper_2407_15264_b200/liblsmgnn.so
cp $SO /tmp/keep.so
: > $out/summary.txt
for m in ab/mut_*.so; do
  name=$(basename $m .so); name=${name#mut_}
  cp $m $SO
  timeout 600 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py tests/test_gpu_storage_file.py -x -q -p no:cacheprovider > $out/$name.log 2>&1
  rc=$?
  if [ $rc = 0 ] && [ -z "${MUT_SKIP_MP:-}" ]; then
    timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider -k "parity or edge" >> $out/$name.log 2>&1
    rc=$?
  fi
  echo "$name rc=$rc $(grep -m1 -Eo 'FAILED [^ ]+' $out/$name.log)" | tee -a $out/summary.txt
done
cp /tmp/keep.so $SO
