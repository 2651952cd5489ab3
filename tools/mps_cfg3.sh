#!/bin/bash
# configs[2] as specified (10M nodes, 2 homes, PVP, 4 GiB cache + 16 GiB victim queues per
# home) with both ranks on ONE GPU under MPS (concurrent ranks), split pull on and off.
# One GPU's PCIe link and SMs serve both homes: a protocol run, not a 2-GPU throughput.
set -u
out=gpurun_out/mps_cfg3; mkdir -p $out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d || { echo "no MPS"; exit 1; }
for split in 1 0; do
  LSMGNN_SPLIT_PULL=$split timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $((29800 + split)) bench.py --gpus 2 --config cfg3 --steps 10 --warmup 5 \
    --no-ablation --no-file-tier --no-cpu-baseline --graph-steps 0 > $out/cfg3_s$split.json 2> $out/cfg3_s$split.err
  echo "split=$split rc=$? $(python -c "
import json;d=json.load(open('$out/cfg3_s$split.json'));t=d['tiers']
print(d['value'],d['ms_per_step'],'e2e',d.get('e2e',{}).get('value'),t,{k:round(v['ms']/d['steps'],3) for k,v in d['phases'].items()})" 2>&1)"
done
echo quit | nvidia-cuda-mps-control
