#!/bin/bash
# NUMA placement of the GPU box: topology, and the bench's e2e / headline with the process (and its
# pinned host buffers) bound to each NUMA node in turn
set -u
nproc; lscpu | grep -E "Socket|NUMA|Model name" ; nvidia-smi topo -m 2>&1 | head -8
which numactl && numactl --hardware | head -6
python - <<'PY'
import pynvml as n
n.nvmlInit(); h = n.nvmlDeviceGetHandleByIndex(0)
try:
    print("gpu cpu affinity words", [hex(x) for x in n.nvmlDeviceGetCpuAffinity(h, 4)])
except Exception as e: print("cpu affinity:", e)
try:
    print("gpu numa node", n.nvmlDeviceGetNumaNodeId(h))
except Exception as e: print("numa node id:", e)
PY
cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | tr 'A-F' 'a-f' | sed 's/^0000//;s/^/0000/' | cut -c1-12)/numa_node 2>/dev/null
for node in $(ls -d /sys/devices/system/node/node* | sed 's/.*node//'); do
  echo "== bound to node $node"
  timeout 600 numactl --cpunodebind=$node --membind=$node python bench.py --steps 10 --warmup 3 --no-ablation --no-cpu-baseline --graph-steps 0 --no-file-tier --extras none 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'dev', d['e2e']['device_result']['value'])"
done
