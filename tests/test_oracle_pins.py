"""Pins for the CPU oracle (`oracle/`) against things other than itself.

Every check compares the oracle with brute force, a closed form, a library routine
(scipy / numpy), the paper's or SPEC's worked examples, or an invariant the
mathematics fixes (DESIGN.md §4 lists which pin covers which oracle function).
P:n = PAPER.md line n, S:n = SPEC.md line n.  CPU only.
"""
import itertools

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

import oracle
import synth
from pp_testutil import read_golden


def csr_from_dense(A):
    A = np.asarray(A) != 0
    n = A.shape[0]
    rows, cols = np.nonzero(A)
    return synth.from_edges(n, rows.astype(np.uint32), cols.astype(np.uint32), symmetrize=False,
                            keep_self_loops=True)


def depths_by_matrix_powers(A, s):
    """1 + min k with (A^k)[s, v] != 0, Boolean powers (brute force)."""
    A = (np.asarray(A) != 0).astype(np.int64)
    n = A.shape[0]
    depth = np.zeros(n, dtype=np.int32)
    R = np.zeros(n, dtype=np.int64)
    R[s] = 1
    for k in range(n):
        newly = (R > 0) & (depth == 0)
        depth[newly] = k + 1
        R = np.minimum(R @ A, 1)
    return depth


# ---------------------------------------------------------------- O1: BFS depths ----------

def test_o1_bruteforce_all_undirected_graphs_n_le_5():
    for n in range(1, 6):
        pairs = list(itertools.combinations(range(n), 2))
        for mask in range(1 << len(pairs)):
            A = np.zeros((n, n), dtype=np.int64)
            for b, (i, j) in enumerate(pairs):
                if mask >> b & 1:
                    A[i, j] = A[j, i] = 1
            g = csr_from_dense(A)
            for s in range(n):
                d, L = oracle.bfs(g, s)
                exp = depths_by_matrix_powers(A, s)
                assert np.array_equal(d, exp), (n, mask, s)
                assert L == exp.max()


def test_o1_bruteforce_all_directed_graphs_n_le_4():
    for n in range(1, 5):
        arcs = [(i, j) for i in range(n) for j in range(n) if i != j]
        for mask in range(1 << len(arcs)):
            A = np.zeros((n, n), dtype=np.int64)
            for b, (i, j) in enumerate(arcs):
                if mask >> b & 1:
                    A[i, j] = 1
            g = csr_from_dense(A)
            for s in range(n):
                d, _ = oracle.bfs(g, s)
                assert np.array_equal(d, depths_by_matrix_powers(A, s)), (n, mask, s)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_o1_vs_scipy_shortest_path_rmat(seed):
    g = synth.rmat(10, 8, seed=seed)
    M = sp.csr_matrix((np.ones(g.nnz), g.idx, g.off), shape=(g.n, g.n))
    for s in synth.sources(g, 8, seed=seed):
        d, _ = oracle.bfs(g, s)
        sp_d = shortest_path(M, directed=True, unweighted=True, indices=int(s))
        exp = np.where(np.isinf(sp_d), 0, sp_d + 1).astype(np.int32)
        assert np.array_equal(d, exp)


def test_o1_vs_scipy_directed_random():
    g = synth.random_graph(300, 900, seed=7, symmetrize=False)
    M = sp.csr_matrix((np.ones(g.nnz), g.idx, g.off), shape=(g.n, g.n))
    for s in range(0, 300, 37):
        d, _ = oracle.bfs(g, s)
        sp_d = shortest_path(M, directed=True, unweighted=True, indices=s)
        assert np.array_equal(d, np.where(np.isinf(sp_d), 0, sp_d + 1).astype(np.int32))


def test_o1_closed_forms():
    # path: depth i+1 from 0
    n = 50
    g = synth.from_edges(n, np.arange(n - 1), np.arange(1, n))
    assert np.array_equal(oracle.bfs(g, 0)[0], np.arange(1, n + 1))
    # cycle: min(i, n-i) + 1
    g = synth.from_edges(n, np.arange(n), (np.arange(n) + 1) % n)
    i = np.arange(n)
    assert np.array_equal(oracle.bfs(g, 0)[0], np.minimum(i, n - i) + 1)
    # star with centre 0: leaves at 2; from a leaf: leaf 1, centre 2, others 3
    g = synth.from_edges(n, np.zeros(n - 1, np.uint32), np.arange(1, n))
    assert np.array_equal(oracle.bfs(g, 0)[0], np.r_[1, np.full(n - 1, 2)])
    exp = np.full(n, 3)
    exp[0], exp[5] = 2, 1
    assert np.array_equal(oracle.bfs(g, 5)[0], exp)
    # complete graph: all 2 except the source
    src, dst = np.nonzero(~np.eye(12, dtype=bool))
    g = synth.from_edges(12, src, dst)
    exp = np.full(12, 2)
    exp[3] = 1
    assert np.array_equal(oracle.bfs(g, 3)[0], exp)
    # binary tree (children 2i+1, 2i+2): floor(log2(i+1)) + 1
    n = 200
    ch = np.arange(1, n)
    g = synth.from_edges(n, (ch - 1) // 2, ch)
    assert np.array_equal(oracle.bfs(g, 0)[0], np.floor(np.log2(np.arange(n) + 1)).astype(int) + 1)


@pytest.mark.parametrize("rows,cols,src", [(7, 11, (0, 0)), (7, 11, (3, 5)), (64, 64, (63, 0)),
                                           (1, 9, (0, 4))])
def test_o1_grid_manhattan(rows, cols, src):
    g = synth.grid(rows, cols)
    y, x = np.divmod(np.arange(rows * cols), cols)
    exp = np.abs(y - src[0]) + np.abs(x - src[1]) + 1
    d, L = oracle.bfs(g, src[0] * cols + src[1])
    assert np.array_equal(d, exp)
    assert L == exp.max()


def test_o1_spec_examples():
    gd = read_golden("spec_diamond.txt")
    g = synth.from_edges(4, [0, 0, 1, 2], [1, 2, 3, 3], symmetrize=False)
    assert oracle.bfs(g, 0)[0].tolist() == [int(x) for x in gd["bfs_depths_from_0"]]
    g = synth.from_edges(3, [0, 1], [1, 2], symmetrize=False)
    assert oracle.bfs(g, 2)[0].tolist() == [int(x) for x in gd["path_from_sink"]]
    # isolated source: only the source has depth 1
    g = synth.from_edges(5, [1, 2], [2, 3])
    assert oracle.bfs(g, 0)[0].tolist() == [1, 0, 0, 0, 0]
    assert oracle.bfs(g, 0)[1] == 1


def test_o1_paper_worked_example():
    gd = read_golden("paper_fig3_example.txt")
    n = int(gd["n"][0])
    e = [tuple(map(int, t.split("-"))) for t in gd["edges"]]
    g = synth.from_edges(n, [a for a, _ in e], [b for _, b in e])
    assert oracle.bfs(g, int(gd["source"][0]))[0].tolist() == [int(x) for x in gd["depths"]]


@pytest.mark.parametrize("seed", range(6))
def test_o1_vs_literal_algorithm1(seed):
    """Alg. 1 run literally with dense matvecs agrees with the queue BFS."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 24))
    A = (rng.random((n, n)) < rng.uniform(0.05, 0.4)).astype(np.int64)
    np.fill_diagonal(A, 0)
    if seed % 2 == 0:
        A = A | A.T
    g = csr_from_dense(A)
    for s in range(n):
        assert np.array_equal(oracle.alg1_bfs_dense(A, s), oracle.bfs(g, s)[0])


def test_o1_bad_source():
    g = synth.grid(2, 2)
    with pytest.raises(ValueError):
        oracle.bfs(g, 4)


# ---------------------------------------------------------------- O2: parents ---------------

def all_valid_parent_vectors(A, s, depth):
    """Brute force: every parent vector passing the Graph500 checks (tiny n)."""
    n = A.shape[0]
    choices = []
    for v in range(n):
        if depth[v] == 0:
            choices.append([-1])
        elif v == s:
            choices.append([s])
        else:
            choices.append(list(range(n)))
    valid = []
    for par in itertools.product(*choices):
        ok = True
        for v in range(n):
            if depth[v] > 0 and v != s:
                p = par[v]
                if not (A[p, v] and depth[p] == depth[v] - 1):
                    ok = False
                    break
        if ok:
            valid.append(par)
    return valid


@pytest.mark.parametrize("seed", range(12))
def test_o2_min_over_all_valid_bfs_trees(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 6))
    A = (rng.random((n, n)) < 0.5).astype(np.int64)
    np.fill_diagonal(A, 0)
    if seed % 3:
        A = A | A.T
    g = csr_from_dense(A)
    gT = csr_from_dense(A.T)
    for s in range(n):
        d, _ = oracle.bfs(g, s)
        par = oracle.parents(gT, d, s)
        valid = all_valid_parent_vectors(A, s, d)
        assert tuple(par.tolist()) in valid
        for v in range(n):                       # canonical = min over all valid trees
            assert par[v] == min(t[v] for t in valid)


@pytest.mark.parametrize("seed", range(8))
def test_o2_ordered_min_key_over_all_valid_bfs_trees(seed):
    """Ordered O2 (relabelled graphs): the valid parent first in a random vertex order."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(2, 6))
    A = (rng.random((n, n)) < 0.5).astype(np.int64)
    np.fill_diagonal(A, 0)
    if seed % 2:
        A = A | A.T
    g, gT = csr_from_dense(A), csr_from_dense(A.T)
    key = rng.permutation(n).astype(np.uint32)
    for s in range(n):
        d, _ = oracle.bfs(g, s)
        par = oracle.parents(gT, d, s, key=key)
        valid = all_valid_parent_vectors(A, s, d)
        assert tuple(par.tolist()) in valid
        for v in range(n):
            if d[v] > 0 and v != s:
                assert key[par[v]] == min(key[t[v]] for t in valid)


def test_o2_ordered_identity_key_is_min_id():
    g = synth.rmat(11, 8, seed=4)
    ident = np.arange(g.n, dtype=np.uint32)
    for s in synth.sources(g, 3, seed=6):
        d, _ = oracle.bfs(g, s)
        assert np.array_equal(oracle.parents(g, d, s, key=ident), oracle.parents(g, d, s))


def test_o2_rmat_passes_graph500_validation():
    g = synth.rmat(12, 8, seed=3)
    for s in synth.sources(g, 4, seed=5):
        d, _ = oracle.bfs(g, s)
        par = oracle.parents(g, d, s)
        oracle.validate_graph500(g, s, d, par)


def test_o5_validator_rejects_corruption():
    g = synth.rmat(10, 8, seed=4)
    s = int(synth.sources(g, 1)[0])
    d, _ = oracle.bfs(g, s)
    par = oracle.parents(g, d, s)
    bad = d.copy()
    v = int(np.nonzero(d == 3)[0][0])
    bad[v] = 4
    with pytest.raises(AssertionError):
        oracle.validate_graph500(g, s, bad, None)
    badp = par.copy()
    badp[v] = s
    with pytest.raises(AssertionError):
        oracle.validate_graph500(g, s, d, badp)


# ---------------------------------------------------------------- O3: masked mxv ------------

def test_o3_matvec_exhaustive_n3_vs_numpy():
    """All 3x3 Boolean M and all u: unmasked w = (M @ u) > 0 (Eq. 2 over OR.AND)."""
    us = [np.array([(k >> b) & 1 for b in range(3)], np.uint8) for k in range(8)]
    for mbits in range(1 << 9):
        M = np.array([(mbits >> b) & 1 for b in range(9)], np.int64).reshape(3, 3)
        g = csr_from_dense(M)
        for u in us:
            assert np.array_equal(oracle.mxv(g, u), ((M @ u) > 0).astype(np.uint8))


def test_o3_single_column_property():
    """if only f(i) is nonzero, f' is the i-th column of the operator."""
    rng = np.random.default_rng(5)
    M = (rng.random((40, 40)) < 0.2).astype(np.int64)
    g = csr_from_dense(M)
    for i in range(40):
        u = np.zeros(40, np.uint8)
        u[i] = 1
        assert np.array_equal(oracle.mxv(g, u), M[:, i].astype(np.uint8))


@pytest.mark.parametrize("seed", range(10))
def test_o3_mask_properties(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 64))
    M = (rng.random((n, n)) < rng.uniform(0.05, 0.5)).astype(np.int64)
    g = csr_from_dense(M)
    u = (rng.random(n) < 0.3).astype(np.uint8)
    m = (rng.random(n) < 0.5).astype(np.uint8)
    w_in = (rng.random(n) < 0.5).astype(np.uint8)
    t = ((M @ u) > 0).astype(np.uint8)           # library matvec
    ones, zeros = np.ones(n, np.uint8), np.zeros(n, np.uint8)
    assert np.array_equal(oracle.mxv(g, u, mask=ones), t)                       # all-pass
    assert np.array_equal(oracle.mxv(g, u, mask=zeros), zeros)                  # none-pass
    assert np.array_equal(oracle.mxv(g, u, mask=zeros, replace=False, w_in=w_in), w_in)
    # complement duality: scmp on m == no scmp on !m
    assert np.array_equal(oracle.mxv(g, u, mask=m, complement=True), oracle.mxv(g, u, mask=1 - m))
    # masked = mask o unmasked, rows outside the mask are 0 under replace
    w = oracle.mxv(g, u, mask=m)
    assert np.array_equal(w[m == 1], t[m == 1]) and not w[m == 0].any()
    # accumulate with a transparent mask is OR with w_in (Alg. 2 line 10)
    assert np.array_equal(oracle.mxv(g, u, accum=True, w_in=w_in), t | w_in)
    # masked rows untouched when replace = 0
    w2 = oracle.mxv(g, u, mask=m, replace=False, w_in=w_in)
    assert np.array_equal(w2[m == 0], w_in[m == 0]) and np.array_equal(w2[m == 1], t[m == 1])


def test_o3_complement_without_mask_rejected():
    g = synth.grid(2, 2)
    with pytest.raises(ValueError):
        oracle.mxv(g, np.ones(4, np.uint8), mask=None, complement=True)


def test_o3_spec_diamond_examples():
    gd = read_golden("spec_diamond.txt")
    A = synth.from_edges(4, [0, 0, 1, 2], [1, 2, 3, 3], symmetrize=False)
    AT = synth.transpose(A)                      # rows of A^T: pull operator
    ids = lambda v: sorted(np.nonzero(v)[0].tolist())
    x01 = synth.dense_from_ids(4, [0, 1])
    assert ids(oracle.mxv(AT, x01)) == [int(x) for x in gd["row_mxv_AT_x01"]]
    assert ids(oracle.mxv(AT, x01, mask=x01, complement=True)) == \
        [int(x) for x in gd["masked_pull_x01_v01_scmp"]]
    assert ids(oracle.mxv(AT, synth.dense_from_ids(4, [0]))) == [int(x) for x in gd["push_x0"]]
    assert ids(oracle.mxv(AT, synth.dense_from_ids(4, [1, 2]), mask=synth.dense_from_ids(4, [0, 1, 2]),
                          complement=True)) == [int(x) for x in gd["masked_push_x12_v012_scmp"]]


def test_o3_paper_worked_example_and_operand_reuse():
    """f' = A^T f .* !v = {E,F}; operand reuse A^T v .* !v gives the same."""
    gd = read_golden("paper_fig3_example.txt")
    n = int(gd["n"][0])
    e = [tuple(map(int, t.split("-"))) for t in gd["edges"]]
    g = synth.from_edges(n, [a for a, _ in e], [b for _, b in e])
    v = synth.dense_from_ids(n, [int(x) for x in gd["visited"]])
    f = synth.dense_from_ids(n, [int(x) for x in gd["frontier"]])
    ids = lambda w: np.nonzero(w)[0].tolist()
    assert ids(oracle.mxv(g, f)) == [int(x) for x in gd["children"]]
    nxt = [int(x) for x in gd["next"]]
    assert ids(oracle.mxv(g, f, mask=v, complement=True)) == nxt
    assert ids(oracle.mxv(g, v, mask=v, complement=True)) == nxt
    assert ids(1 - v) == [int(x) for x in gd["unvisited"]]


def test_o3_vs_scipy_random_large():
    g = synth.rmat(11, 8, seed=9)
    AT = synth.transpose(g)
    Ms = sp.csr_matrix((np.ones(AT.nnz, np.int64), AT.idx, AT.off), shape=(g.n, g.n))
    rng = np.random.default_rng(1)
    for dens in (0.001, 0.01, 0.3):
        u = (rng.random(g.n) < dens).astype(np.uint8)
        assert np.array_equal(oracle.mxv(AT, u), ((Ms @ u.astype(np.int64)) > 0).astype(np.uint8))


# ---------------------------------------------------------------- O4: direction ------------

def test_o4_spec_direction_cases():
    """S:325-327 with n = 1000 so that r = c/n: (r_prev, r) = (.005,.02), (.02,.005), (.005,.008)."""
    R = oracle.RULE_PAPER_R
    assert oracle.direction(R, oracle.PUSH, 5, 20, 0, 0, 1000) == oracle.PULL
    assert oracle.direction(R, oracle.PULL, 20, 5, 0, 0, 1000) == oracle.PUSH
    assert oracle.direction(R, oracle.PUSH, 5, 8, 0, 0, 1000) == oracle.PUSH
    # ties hold: equal r, or exactly r == alpha
    assert oracle.direction(R, oracle.PUSH, 20, 20, 0, 0, 1000) == oracle.PUSH
    assert oracle.direction(R, oracle.PUSH, 5, 10, 0, 0, 1000) == oracle.PUSH   # 10/1000 == .01
    # r above alpha but falling does not switch push->pull ("r is increasing")
    assert oracle.direction(R, oracle.PUSH, 50, 30, 0, 0, 1000) == oracle.PUSH


def test_o4_edge_rule_cases():
    E = oracle.RULE_EDGES
    # push->pull needs m_f * 15 > m_u and a growing frontier
    assert oracle.direction(E, oracle.PUSH, 10, 100, 1000, 14999, 10**6) == oracle.PULL
    assert oracle.direction(E, oracle.PUSH, 10, 100, 1000, 15000, 10**6) == oracle.PUSH
    assert oracle.direction(E, oracle.PUSH, 100, 10, 10**6, 1, 10**6) == oracle.PUSH
    # pull->push needs c * 18 < n and a shrinking frontier
    assert oracle.direction(E, oracle.PULL, 100, 55, 0, 0, 1000) == oracle.PUSH
    assert oracle.direction(E, oracle.PULL, 100, 56, 0, 0, 1008) == oracle.PULL
    assert oracle.direction(E, oracle.PULL, 10, 20, 0, 0, 10**6) == oracle.PULL


def test_o4_trace_grid_is_all_push():
    """C4: both rules keep a grid in push at every level."""
    g = synth.grid(128, 128)        # max frontier 128 = 0.78% of n < alpha = 1% (r-rule)
    d, L = oracle.bfs(g, 0)
    for rule in (oracle.RULE_EDGES, oracle.RULE_PAPER_R):
        t = oracle.trace(g, g, d, rule=rule)
        assert t["levels"] == L == 255 and not t["dir"].any()
        assert t["c"][-1] == 0 and np.array_equal(t["c"][:-1], np.bincount(d)[2:])


def test_o4_trace_three_phases_on_rmat():
    """push phase, pull phase, push phase on a scale-free graph."""
    g = synth.rmat(16, 16, seed=1)
    seen = 0
    for s in synth.sources(g, 8, seed=2):
        d, L = oracle.bfs(g, s)
        for rule in (oracle.RULE_EDGES, oracle.RULE_PAPER_R):
            t = oracle.trace(g, g, d, rule=rule)
            dirs = "".join("HL"[x] for x in t["dir"])
            assert dirs[0] == "H"
            if "L" in dirs:
                seen += 1
                assert dirs.startswith("H") and "LH" in dirs + "H"
        # m_u is the in-degree mass not yet visited, and reaches the unreached mass at the end
        t = oracle.trace(g, g, d)
        assert t["m_u"][-1] == np.diff(g.off)[d == 0].sum()
    assert seen > 0


def test_o4_pull_only_and_push_only_modes():
    g = synth.rmat(10, 8, seed=2)
    d, L = oracle.bfs(g, int(synth.sources(g, 1)[0]))
    assert not oracle.trace(g, g, d, mode=oracle.MODE_PUSH_ONLY)["dir"].any()
    assert oracle.trace(g, g, d, mode=oracle.MODE_PULL_ONLY)["dir"].all()
