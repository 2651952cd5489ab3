#!/bin/bash
# re-entry session: new overlap tests (incl. the overlapped fuzz), the feed-wait mutant against the
# slow-feed test, the early k_dedup CTAs-per-SM knob on the hit path, then the default bench line
set -u
SO=paper_2407_15264_b200/liblsmgnn.so
cp $SO /tmp/keep.so
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_fuzz.py -q -k "overlap" > gpurun_out/c30_overlap.log 2>&1
echo "overlap tests rc=$?: $(tail -1 gpurun_out/c30_overlap.log)"
cp ab/mut_set_no_feed_wait.so $SO
timeout 600 python -m pytest tests/test_gpu_overlap.py -q -k "slow_feed" > gpurun_out/c30_mut_feed.log 2>&1
echo "mutant set_no_feed_wait vs slow_feed rc=$? (nonzero = killed): $(tail -1 gpurun_out/c30_mut_feed.log)"
cp /tmp/keep.so $SO
bash tools/hit_ab.sh perSM "LSMGNN_EARLY_DEDUP_PER_SM=1" "LSMGNN_EARLY_DEDUP_PER_SM=2" "LSMGNN_EARLY_DEDUP_PER_SM=4"
timeout 1500 python bench.py > gpurun_out/c30_bench.json 2> gpurun_out/c30_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/c30_bench.json').read().strip().splitlines()[-1])
h=d['hbm_regime']; print('value', d['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], 'hit', h['ms_per_step'], h['graph_replay']['ms_per_step'], h['two_streams']['ms_per_step'], h['roofline']['frac'], 'clocks', d['clocks'])"
