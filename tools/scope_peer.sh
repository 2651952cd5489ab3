#!/bin/bash
# N4 cross-process scope benchmark (tools/scope_peer_bench.cu) on one B200: two processes, each
# a home, under MPS (concurrent, as on two GPUs) and time-sliced (no MPS), plus the round-1
# single-process scope bench for reference. Output: gpurun_out/scope_peer.txt
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/scope_peer tools/scope_peer_bench.cu || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/scope_bench tools/scope_bench.cu || exit 1
{
  echo "== one process (tools/scope_bench.cu): local partition, .gpu vs .sys"
  timeout 300 /tmp/scope_bench
  echo "== two processes, time-sliced (no MPS)"
  timeout 600 /tmp/scope_peer
  export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
  mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
  if nvidia-cuda-mps-control -d; then
    echo "== two processes under MPS (concurrent)"
    timeout 600 /tmp/scope_peer
    echo quit | nvidia-cuda-mps-control
  else
    echo "(MPS unavailable)"
  fi
} > gpurun_out/scope_peer.txt 2>&1
cat gpurun_out/scope_peer.txt
