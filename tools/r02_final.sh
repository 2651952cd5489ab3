#!/bin/bash
# Round-2 closing evidence on the current build: the driver's sequence (tools/r02_full.sh: GPU
# suite, smoke, ncu of k_serve / metadata at configs[1], launch list, default bench line), then
# ncu --set full of the hit-path kernels (tools/r02_ncu_hit2.sh) and the GPU mutants.
set -u
bash tools/r02_full.sh
bash tools/r02_ncu_hit2.sh final
bash tools/gpu_mutants.sh > gpurun_out/mutants_stdout.txt 2>&1; echo "mutants:"; cat gpurun_out/gpu_mutants/summary.txt
