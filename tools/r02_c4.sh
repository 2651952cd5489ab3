#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "g1_pull or serve_geometry" tests/test_gpu_storage_file.py -q -x > gpurun_out/r02c4_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02c4_tests.log
timeout 600 python -m pytest tests/test_gpu_multiproc.py -k "file or edge" -q -x > gpurun_out/r02c4_mp.log 2>&1
echo "mp rc=$?"; tail -3 gpurun_out/r02c4_mp.log
bash tools/r02_ncu_hit.sh hit
bash tools/r02_ncu_hit.sh hit_g1pull LSMGNN_G1_PULL=1
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --extras hbm_regime,file_tier > gpurun_out/r02c4_bench.json 2> gpurun_out/r02c4_bench.err
echo "bench rc=$?"
