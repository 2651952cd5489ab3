"""NEXT N3 on the GPU (-m gpu): the UVA neighbour sampler reproduces the sampler oracle
bit-exactly, and a pipeline whose window is fed straight from the GPU sampler
(lsmgnn_sample -> lsmgnn_prefetch_dev, no host round trip) matches the oracle's counters."""
import numpy as np
import pytest

import oracle
import synth

from .harness import table_for
from .test_gpu_parity import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def graph1m():
    return synth.plcite(1_000_000, 12)


@pytest.mark.parametrize("in_hbm", [False, True])
@pytest.mark.parametrize("fanout", [(10, 5, 5), (5, 2, 2, 2), (25, 10), (40,), ()])
def test_sampler_parity(graph1m, fanout, in_hbm):
    import torch
    from paper_2407_15264_b200 import Sampler
    g = graph1m
    s = Sampler(g.indptr, g.indices)
    s.place(in_hbm)  # CSR read over PCIe (UVA) or from an HBM copy: same lists
    perm = synth.epoch_seeds(g.num_nodes, 0)
    for t in range(3):
        for r in range(2):
            seeds = perm[(t * 2 + r) * 1024:(t * 2 + r + 1) * 1024]
            sd = torch.from_numpy(seeds).cuda()
            out, cnt = s.sample(sd, fanout, 4, t, r)
            torch.cuda.synchronize()
            got = out[: int(cnt.item())].cpu().numpy()
            want = oracle.sample_batch(g.indptr, g.indices, seeds, fanout, 4, t, r)
            assert np.array_equal(got, want), (fanout, t, r, got.size, want.size)


@pytest.mark.parametrize("pvp", [0, 1])
def test_pipeline_gpu_sampler_window(pvp):
    import torch
    from paper_2407_15264_b200 import LsmGnn, Sampler, STATS_FIELDS, prefetch_dev
    N, D, W, K, B, fan = 16384, 128, 8, 20, 256, (10, 5)
    g = synth.plcite(N, 8)
    sc = synth.static_scores(g)
    perm = synth.epoch_seeds(N, 0)
    seeds = [perm[t * B:(t + 1) * B] for t in range(K)]
    trace = [[oracle.sample_batch(g.indptr, g.indices, seeds[t], fan, 4, t, 0)] for t in range(K)]
    kw = dict(N=N, R=4 * D, L=1024, A=8, scores=sc, policy="hybrid", pvp=pvp, W=W, V=512)
    ho = oracle.run_trace(oracle.Oracle(1, N, 4 * D, 1024, 8, sc, policy="hybrid", pvp=pvp, W=W, V=512), trace)
    c = LsmGnn(N, D, 1024, 8, 512, sc, policy="hybrid", pvp=pvp, window=W,
               max_batch_ids=Sampler.bound(B, fan))
    c.attach_storage(table_for(N, D, pinned=True))
    s = Sampler(g.indptr, g.indices)  # attach after init (finalize resets the sampler)
    bound = Sampler.bound(B, fan)
    lists, counts = {}, {}

    def sampled(k):
        if k not in lists:
            if k < K:
                lists[k], counts[k] = s.sample(torch.from_numpy(seeds[k]).cuda(), fan, 4, k, 0)
            else:  # past the end of the trace: empty batch
                lists[k] = torch.zeros(1, dtype=torch.int64, device="cuda")
                counts[k] = torch.zeros(1, dtype=torch.int64, device="cuda")
        return lists[k], counts[k]

    for k in range(1, W + 1):
        prefetch_dev(*sampled(k), first_iter=k)
    out = torch.empty((bound, 4 * D), dtype=torch.uint8, device="cuda")
    for t in range(K):
        ids, cnt = sampled(t)
        n = int(cnt.item())  # the list was sampled W iterations ago
        c.gather(ids[:n], out)
        prefetch_dev(*sampled(t + 1 + W), first_iter=t + 1 + W)
        c.prefetch([], first_iter=0)  # PVP copy for t+1
        rows = out[:n].cpu().numpy().view(np.uint32).reshape(n, D)
        assert synth.check_rows(rows, trace[t][0], D)[0] == 0
    torch.cuda.synchronize()
    compare(c.history(0, K), ho[:, 0, :], f"gpu-sampler pipeline pvp{pvp}")
    c.close()
