"""Pins of the sampler oracle (NEXT N3): equality with the independent
numpy implementation in synth, and brute-force properties of GraphSAGE sampling."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("seed", range(5))
def test_sampler_oracle_matches_numpy(seed):
    g = synth.plcite(5000, 6, seed_g=seed + 1)
    rng = np.random.default_rng(seed)
    for t in range(4):
        seeds = rng.choice(5000, 64, replace=False)
        a = oracle.sample_batch(g.indptr, g.indices, seeds, (10, 5, 3), 4, t, seed % 3)
        b = synth.sample_batch(g, seeds, (10, 5, 3), 4, t, seed % 3)
        assert np.array_equal(a, b)


def test_sampler_properties():
    """Every sampled node is a seed or a neighbour of a node of the previous frontier; nodes
    with deg <= f contribute all neighbours; the list is duplicate-free, seeds first."""
    g = synth.plcite(3000, 4)
    seeds = np.arange(0, 3000, 97)
    out = oracle.sample_batch(g.indptr, g.indices, seeds, (3, 2), 9, 0, 0)
    assert len(set(out.tolist())) == out.size
    assert np.array_equal(out[:seeds.size], seeds)
    nb = lambda x: set(g.indices[g.indptr[x]:g.indptr[x + 1]].tolist())
    layer1 = set().union(*[nb(x) for x in seeds])
    assert set(out.tolist()) <= set(seeds.tolist()) | layer1 | set().union(*[nb(x) for x in layer1])
    small = [x for x in seeds if g.indptr[x + 1] - g.indptr[x] <= 3]
    for x in small:
        assert nb(x) <= set(out.tolist())


def test_c_graph_generator_matches_numpy():
    """synth.plcite_c (for 100M-node graphs) builds the same CSR as synth.plcite."""
    for N, m in [(3000, 4), (50000, 12)]:
        a, b = synth.plcite(N, m), synth.plcite_c(N, m)
        assert np.array_equal(a.indptr, b.indptr)
        assert np.array_equal(a.indices.astype(np.int64), b.indices.astype(np.int64))
