#!/bin/bash
# configs[3] (100M nodes, 8 homes) and a configs[4] IGBH point (100M nodes, 4 homes) through the
# G-home path on one B200 under MPS (tools/ghome_run.py). Output: gpurun_out/ghome_*.json
set -u
mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d || echo "(no MPS: ranks time-slice)"
free -g | head -2
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29610 tools/ghome_run.py gpurun_out/ghome_smoke.json \
  --workload igb --nodes 2000000 --lines-per-gpu 65536 --iters 4 --warm 2 > gpurun_out/ghome_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/ghome_smoke.log; rm -rf /dev/shm/lsmgnn_ghome
timeout 1800 $R --nproc-per-node 8 --master-port 29611 tools/ghome_run.py gpurun_out/ghome_igb_16g.json \
  --workload igb --lines-per-gpu 4194304 --policies ${IGB_POLICIES:-hybrid,static,lru} --max-ids 1600000 > gpurun_out/ghome_igb.log 2>&1
echo "igb rc=$?"; tail -3 gpurun_out/ghome_igb.log
timeout 2400 $R --nproc-per-node 4 --master-port 29612 tools/ghome_run.py gpurun_out/ghome_igbh_10pct.json \
  --workload igbh --cache-pct 10 --policies hybrid,static,lru,dynamic > gpurun_out/ghome_igbh.log 2>&1
echo "igbh rc=$?"; tail -3 gpurun_out/ghome_igbh.log
timeout 2400 $R --nproc-per-node 4 --master-port 29613 tools/ghome_run.py gpurun_out/ghome_igbh_10pct_p4.json \
  --workload igbh --cache-pct 10 --policies hybrid,dynamic --period 4 > gpurun_out/ghome_igbh_p4.log 2>&1
echo "igbh P4 rc=$?"; tail -3 gpurun_out/ghome_igbh_p4.log
echo quit | nvidia-cuda-mps-control
rm -rf /dev/shm/lsmgnn_ghome
