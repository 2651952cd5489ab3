set -u
out=gpurun_out/mps_probe; mkdir -p $out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
X="--steps 10 --warmup 3 --no-ablation --no-file-tier --no-cpu-baseline --no-e2e --graph-steps 0"
r() { tag=$1; n=$2; shift 2
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29000 + RANDOM % 900)) bench.py --gpus $n $X $EXTRA > $out/$tag.json 2> $out/$tag.err
  echo "$tag rc=$? $(python -c "
import json;d=json.load(open('$out/$tag.json'));print(d['value'],d['ms_per_step'],{k:round(v['ms']/d['steps'],3) for k,v in d['phases'].items()})" 2>&1)"
}
EXTRA="--config cfg1"
r cfg1_n1 1 A=1; r cfg1_n2 2 A=1; r cfg1_n8 8 A=1; r cfg1_n8_nobatch 8 LSMGNN_NO_BATCH_MEMOP=1
EXTRA="--lines 1000000"
r hit_n1 1 A=1; r hit_n2 2 A=1; r hit_n8 8 A=1
echo quit | nvidia-cuda-mps-control
