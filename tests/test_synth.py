"""Input-generator checks (synth/): structure, determinism, and the Table-3 shape pin P1."""
import numpy as np
import pytest

import synth


def check_csr(g):
    assert g.off[0] == 0 and np.all(np.diff(g.off) >= 0) and g.off[-1] == len(g.idx)
    assert len(g.idx) == 0 or int(g.idx.max()) < g.n
    rows = np.repeat(np.arange(g.n), np.diff(g.off))
    key = rows.astype(np.int64) * g.n + g.idx
    assert np.all(np.diff(key) > 0), "rows must be strictly increasing (sorted, unique)"
    return rows


def test_rmat_structure_symmetric_no_selfloops():
    g = synth.rmat(12, 8, seed=3)
    rows = check_csr(g)
    assert not np.any(rows == g.idx)
    t = synth.transpose(g)
    assert np.array_equal(t.off, g.off) and np.array_equal(t.idx, g.idx)


def test_rmat_deterministic_and_seeded():
    a, b, c = synth.rmat(10, 8, seed=1), synth.rmat(10, 8, seed=1), synth.rmat(10, 8, seed=2)
    assert np.array_equal(a.idx, b.idx) and np.array_equal(a.off, b.off)
    assert not (len(a.idx) == len(c.idx) and np.array_equal(a.idx, c.idx))


def test_rmat_scale_free_skew():
    """max degree >= 20x average at scale 12, edge factor 8."""
    g = synth.rmat(12, 8, seed=1)
    d = g.degrees()
    assert d.max() >= 20 * d.mean()


def test_from_edges_preprocess():
    """[(0,0),(0,1),(0,1),(1,0)] undirected -> [(0,1),(1,0)]."""
    g = synth.from_edges(2, [0, 0, 0, 1], [0, 1, 1, 0])
    assert g.off.tolist() == [0, 1, 2] and g.idx.tolist() == [1, 0]


def test_grid_and_percolated_grid():
    g = synth.grid(5, 7)
    check_csr(g)
    assert g.nnz == 2 * (5 * 6 + 4 * 7)
    p = synth.percolated_grid(64, 64, 0.6, seed=1)
    check_csr(p)
    assert 0.5 * 4096 < p.n <= 4096
    assert np.array_equal(synth.transpose(p).idx, p.idx)


@pytest.mark.slow
def test_p1_table3_kron21_shape():
    """Pin P1: kron_g500-logn21 has 182.1M edges, max degree 213,904
    (P:448).  The Graph500-parameter generator must land within 1% / 15%."""
    g = synth.rmat(21, 48, seed=1)
    assert abs(g.nnz - 182.1e6) / 182.1e6 < 0.01
    assert abs(g.degrees().max() - 213904) / 213904 < 0.15


def test_rgg_matches_brute_force_pairs():
    """RGG (NEXT-2 workload): edge set = all point pairs within r, recomputed here by brute
    force from the same counter-based coordinates (ids are the cell-major order)."""
    import math
    scale, factor, seed = 11, 0.55, 3
    g = synth.rgg(scale, factor, seed)
    rows = check_csr(g)
    assert not np.any(rows == g.idx)
    t = synth.transpose(g)
    assert np.array_equal(t.off, g.off) and np.array_equal(t.idx, g.idx)
    n = 1 << scale
    r = factor * math.sqrt(math.log(n) / n)
    key = (seed * 0x100000001B3) & (2**64 - 1)
    u = lambda x: (synth.splitmix64(x) >> 11) * (1.0 / 9007199254740992.0)
    x = np.array([u(key ^ (2 * k)) for k in range(n)])
    y = np.array([u(key ^ (2 * k + 1)) for k in range(n)])
    d2 = (x[:, None] - x[None, :]) ** 2 + (y[:, None] - y[None, :]) ** 2
    np.fill_diagonal(d2, np.inf)
    assert len(g.idx) == int((d2 <= r * r).sum())
    # degree multiset is id-order independent
    assert np.array_equal(np.sort(np.diff(g.off)), np.sort((d2 <= r * r).sum(1)))


def test_rgg24_reproduces_table3_shape():
    """Pin (Table 3): rgg_n_24 has 16.8M vertices, 265.1M edges, max degree
    40.  radius 0.55*sqrt(ln n / n) gives nnz within 0.5% and max degree within 15%."""
    g = synth.make("RGG24")
    assert g.n == 1 << 24
    assert abs(len(g.idx) - 265.1e6) / 265.1e6 < 0.005
    assert abs(int(np.diff(g.off).max()) - 40) <= 6
