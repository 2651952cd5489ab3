#!/bin/bash
# A/B of the G > 1 pull split (phase 0 on a second stream during k_fill vs both phases after
# "served") with two ranks on ONE GPU, alternating, with and without MPS (without MPS the two
# processes time-slice the GPU, so cross-process overlap cannot happen). Not a throughput
# claim: two homes share one GPU's PCIe link and SMs.
set -u
out=gpurun_out/n2ab
mkdir -p $out
B="bench.py --gpus 2 --steps 10 --warmup 3 --no-ablation --no-file-tier --no-cpu-baseline --no-e2e --graph-steps 0"
run() {  # $1 = tag, $2 = env
  env $2 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) $B > $out/$1.json 2> $out/$1.err
  echo "$1 rc=$? $(python -c "import json;d=json.load(open('$out/$1.json'));print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['phases'].items()})" 2>&1)"
}
run default_1 "LSMGNN_UNSET=1"  # no override: ranks sharing a GPU pick the unsplit order
for i in 1 2; do
  run split_$i "LSMGNN_SPLIT_PULL=1"
  run nosplit_$i "LSMGNN_SPLIT_PULL=0"
done
if command -v nvidia-cuda-mps-control > /dev/null; then
  export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
  mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
  nvidia-cuda-mps-control -d && echo "mps started"
  for i in 1 2; do
    run mps_split_$i "LSMGNN_SPLIT_PULL=1"
    run mps_nosplit_$i "LSMGNN_SPLIT_PULL=0"
  done
  echo quit | nvidia-cuda-mps-control
else
  echo "no nvidia-cuda-mps-control"
fi
