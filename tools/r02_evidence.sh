#!/bin/bash
set -u
bash tools/gpu_mutants.sh > gpurun_out/mutants_stdout.txt 2>&1
echo "mutants done"; cat gpurun_out/gpu_mutants/summary.txt
bash tools/sanitize.sh > gpurun_out/sanitize_stdout.txt 2>&1; echo "sanitize done"; cat gpurun_out/sanitize_summary.txt
