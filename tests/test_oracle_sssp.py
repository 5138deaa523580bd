"""Pins of oracle/sssp.py against things other than itself."""
import numpy as np
import pytest

import synth
from oracle import sssp as osssp


def _weighted(n, m, seed, symmetrize=False, integer=True):
    g = synth.random_graph(n, m, seed, symmetrize=symmetrize)
    return g, synth.edge_weights(g.nnz, seed=seed + 100, integer=integer).astype(np.float64)


def test_diamond_spec_example():
    # diamond with unit weights, source 0 -> [0, 1, 1, 2]
    g = synth.from_edges(4, [0, 0, 1, 2], [1, 2, 3, 3], symmetrize=False)
    d, trace = osssp.sssp_2phase(g.off, g.idx, np.ones(g.nnz), 0)
    assert d.tolist() == [0.0, 1.0, 1.0, 2.0]
    assert len(trace) == 3  # eccentricity 2 + the empty-result iteration


def test_single_vertex_and_unreachable():
    g = synth.from_edges(1, [], [], symmetrize=False)
    d, _ = osssp.sssp_2phase(g.off, g.idx, np.zeros(0), 0)
    assert d.tolist() == [0.0]
    g = synth.from_edges(3, [0], [1], symmetrize=False)
    d, _ = osssp.sssp_2phase(g.off, g.idx, np.array([5.0]), 0)
    assert d[0] == 0 and d[1] == 5 and np.isinf(d[2])


def test_negative_weight_rejected():
    g = synth.from_edges(2, [0], [1], symmetrize=False)
    with pytest.raises(ValueError):
        osssp.sssp_2phase(g.off, g.idx, np.array([-1.0]), 0)


def test_floyd_warshall_brute_force():
    # all-pairs Floyd-Warshall on dense matrices, tiny graphs, both phases forced
    for seed in range(30):
        n = 2 + seed % 9
        g, w = _weighted(n, 3 * n, seed)
        D = np.full((n, n), np.inf)
        np.fill_diagonal(D, 0)
        for i in range(n):
            for e in range(g.off[i], g.off[i + 1]):
                D[i, g.idx[e]] = min(D[i, g.idx[e]], w[e])
        for k in range(n):
            D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
        for s in range(n):
            for alpha in (0.0, 1.0, 0.3):
                d, _ = osssp.sssp_2phase(g.off, g.idx, w, s, alpha)
                assert np.array_equal(d, D[s])


def test_scipy_dijkstra_and_heap_dijkstra():
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra as sp_dijkstra
    for seed in range(12):
        n = 50 + 37 * seed
        g, w = _weighted(n, 4 * n, seed, symmetrize=seed % 2 == 0, integer=seed % 3 != 0)
        A = csr_matrix((w, g.idx.astype(np.int64), g.off), shape=(n, n))
        src = seed * 7 % n
        ref = sp_dijkstra(A, directed=True, indices=src)
        d, trace = osssp.sssp_2phase(g.off, g.idx, w, src, alpha=0.05)
        assert np.allclose(d, ref, rtol=1e-12, atol=0) and np.array_equal(np.isinf(d), np.isinf(ref))
        assert np.allclose(osssp.dijkstra(g.off, g.idx, w, src), ref, rtol=1e-12)
        # one switch at most: the direction sequence is push* pull*
        dirs = [t[0] for t in trace]
        assert dirs == sorted(dirs)


def test_unit_weights_are_bfs_levels():
    # closed form: with unit weights Jacobi Bellman-Ford discovers level k at iteration k,
    # so d = BFS level - 1 and the loop runs eccentricity + 1 times
    g = synth.rmat(8, 8, seed=5)
    from collections import deque
    for s in (0, 3, 77):
        lvl = np.full(g.n, -1)
        lvl[s] = 0
        q = deque([s])
        while q:
            u = q.popleft()
            for v in g.idx[g.off[u]:g.off[u + 1]]:
                if lvl[v] < 0:
                    lvl[v] = lvl[u] + 1
                    q.append(v)
        for alpha in (0.0, 0.01, 2.0):
            d, trace = osssp.sssp_2phase(g.off, g.idx, np.ones(g.nnz), s, alpha)
            assert np.array_equal(np.where(lvl >= 0, lvl, np.inf), d)
            assert len(trace) == lvl.max() + 1
