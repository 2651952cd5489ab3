#!/bin/bash
# G > 1 evidence on one B200: bench.py at N = 2 and 8 ranks under MPS (ranks concurrent; the
# line's step_roofline carries the NVLink tiers), and ncu of the pull kernels on one process
# (LSMGNN_G1_PULL=1: k_fill + k_pull phases on local HBM) in the hit regime and the headline.
set -u
mkdir -p gpurun_out/g2
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d || echo "(no MPS)"
X="--steps 10 --warmup 3 --no-ablation --no-file-tier --no-cpu-baseline --no-e2e --graph-steps 0"
for n in 2 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29800 + n)) bench.py --gpus $n $X > gpurun_out/g2/bench_n$n.json 2> gpurun_out/g2/bench_n$n.err
  echo "n=$n rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/g2/bench_n$n.json').read().strip().splitlines()[-1])
print(d['value'],d['ms_per_step'],d['roofline']['bound'],d['roofline']['frac'],d['step_roofline']['bound_tier'],d['step_roofline']['frac'],d['phases'].get('pull'))" 2>&1)"
done
echo quit | nvidia-cuda-mps-control
B="python bench.py --warmup 60 --steps 3 --no-ablation --no-e2e --no-cpu-baseline --graph-steps 0"
for k in pull fill; do
  LSMGNN_G1_PULL=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_$k" --launch-skip 62 \
    -c 2 -o gpurun_out/g2/hit_$k $B --lines 1000000 > gpurun_out/g2/hit_$k.log 2>&1
  echo "ncu hit $k rc=$?"
done
LSMGNN_G1_PULL=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_pull" --launch-skip 62 \
  -c 2 -o gpurun_out/g2/cfg2_pull $B > gpurun_out/g2/cfg2_pull.log 2>&1
echo "ncu cfg2 pull rc=$?"
LSMGNN_G1_PULL=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --extras hbm_regime \
  > gpurun_out/g2/g1pull_bench.json 2> gpurun_out/g2/g1pull_bench.err
echo "g1pull bench rc=$?"
