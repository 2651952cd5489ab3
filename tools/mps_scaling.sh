#!/bin/bash
# The G > 1 protocol on ONE B200 under MPS (ranks run concurrently, as on distinct GPUs):
# bench.py at N = 1, 2, 4, 8 ranks, each rank a home with its own cache (configs[1] lines per
# rank), all homes sharing this one GPU's SMs, HBM and PCIe link. Box GB/s therefore cannot
# scale with N here; the table shows the protocol's cost and the hit-ratio gain of the
# growing shared cache. Not a multi-GPU throughput claim.
set -u
out=gpurun_out/mps_scaling
mkdir -p $out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d || { echo "no MPS"; exit 1; }
X="--steps 10 --warmup 3 --no-ablation --no-file-tier --no-cpu-baseline --no-e2e --graph-steps 0"
for n in 1 2 4 8; do
  for split in 1 0; do
    [ $n = 1 ] && [ $split = 0 ] && continue
    LSMGNN_SPLIT_PULL=$split timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29700 + n * 10 + split)) bench.py --gpus $n $X \
      > $out/n${n}_s$split.json 2> $out/n${n}_s$split.err
    echo "n=$n split=$split rc=$? $(python -c "
import json;d=json.load(open('$out/n${n}_s$split.json'));t=d['tiers']
print(d['value'],d['ms_per_step'],'hit',t['hit_ratio'],'storage GB/step',round(t['storage_GB_per_step'],3),'pcie',t['pcie_h2d_GBps_over_step'])" 2>&1)"
  done
done
echo quit | nvidia-cuda-mps-control
