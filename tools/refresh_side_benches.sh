#!/bin/bash
# Side bench lines kept under profiles/ (run on the GPU box from the repo root):
# configs[0] shape direct vs CUDA-graph replay, configs[2] shape on one home, G = 2 on one GPU.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg1 --steps 200 --warmup 10 --no-ablation --no-cpu-baseline --no-e2e > gpurun_out/side_cfg1_direct.json 2> gpurun_out/side_cfg1_direct.err
timeout 600 python bench.py --config cfg1 --steps 200 --warmup 10 --no-ablation --no-cpu-baseline --no-e2e --graph > gpurun_out/side_cfg1_graph.json 2> gpurun_out/side_cfg1_graph.err
timeout 900 python bench.py --config cfg3 --steps 20 --warmup 10 --no-ablation --no-cpu-baseline --no-e2e > gpurun_out/side_cfg3.json 2> gpurun_out/side_cfg3.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 --steps 10 --warmup 3 --no-ablation > gpurun_out/side_n2.json 2> gpurun_out/side_n2.err
for f in gpurun_out/side_*.json; do echo "$f $(tail -c 150 $f | head -c 150)"; done
