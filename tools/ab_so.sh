#!/bin/bash
# A/B two builds of liblsmgnn.so (ab/liblsmgnn_old.so vs ab/liblsmgnn_new.so), alternating:
# the hit path (cache = whole table), the default configs[1] step, and two ranks under MPS.
set -u
out=gpurun_out/ab; mkdir -p $out
SO=paper_2407_15264_b200/liblsmgnn.so
X="--no-ablation --no-e2e --no-cpu-baseline --graph-steps 0 --no-file-tier"
show() { python -c "
import json;d=json.load(open('$1'));p=d['phases']
print(d['value'],d['ms_per_step'],'fill',round(p['fill']['ms']/d['steps'],4),'pull',round(p['pull']['ms']/d['steps'],4),'hit',d['tiers']['hit_ratio'])" 2>&1; }
for i in 1 2; do
  for v in old new; do
    cp ab/liblsmgnn_$v.so $SO
    timeout 300 python bench.py --lines 1000000 --warmup 60 --steps 30 $X > $out/hit_$v$i.json 2>/dev/null
    echo "hit $v $i: $(show $out/hit_$v$i.json)"
    timeout 300 python bench.py --steps 20 --warmup 5 $X > $out/cfg2_$v$i.json 2>/dev/null
    echo "cfg2 $v $i: $(show $out/cfg2_$v$i.json)"
  done
done
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
for i in 1 2; do
  for v in old new; do
    cp ab/liblsmgnn_$v.so $SO
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $((29300 + RANDOM % 500)) bench.py --gpus 2 --steps 10 --warmup 3 $X > $out/n2_$v$i.json 2>/dev/null
    echo "n2 mps $v $i: $(show $out/n2_$v$i.json)"
  done
done
echo quit | nvidia-cuda-mps-control
cp ab/liblsmgnn_new.so $SO
