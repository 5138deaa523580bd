"""Pins of O4 `oracle_trace` (per-level c, m_f, m_u and the direction sequence they imply,
P:366, R10/R11) and of the SSSP switch boundary (R29) against things other than
the oracle itself: exhaustive brute force over tiny DIRECTED graphs (in- and out-degree
differ, so an m_u computed from out-degrees or an m_f summed over the wrong frontier fails),
a closed-form directed broom, a hand-computed SSSP case sitting exactly on the switch
threshold, and the paper's own qualitative trace on the kron_g500-logn21 analog (Fig. 5 /
P:264 / P:276, SURVEY pin P7)."""
import itertools
import re

import numpy as np
import pytest

import oracle
import synth
from oracle import sssp as osssp


def _depth_by_matrix_powers(A, s):
    """BFS depth from Boolean matrix powers (independent of oracle_bfs): depth[v] = 1 + the
    least k with (A^k)[s, v] != 0, 0 when no k < n reaches v (Alg. 1 convention, R1)."""
    n = A.shape[0]
    depth = np.zeros(n, np.int32)
    reach = np.zeros(n, bool)
    reach[s] = True
    depth[s] = 1
    cur = reach.copy()
    for k in range(1, n):
        cur = (cur.astype(np.int64) @ A.astype(np.int64)) > 0      # row s of A^k
        new = cur & (depth == 0)
        depth[new] = k + 1
    return depth


def _trace_by_definition(A, depth, rule, mode, alpha, beta):
    """Per-level counters straight from their definitions on the dense adjacency matrix.
    Level k (1-based) expands F_k = {v : depth v = k} and discovers F_{k+1}:
      c_k   = |F_{k+1}|
      m_f,k = sum over F_{k+1} of out-degree  (row sums of A: edges (v, .), Eq. 1)
      m_u,k = sum over {v : depth v = 0 or depth v > k+1} of in-degree (column sums of A)
    and the direction used by level k+1 is the rule applied to (c_{k-1} = |F_k|, c_k, m_f,k,
    m_u,k); level 1 is push (pull in pull-only mode)."""
    n = A.shape[0]
    outdeg = A.sum(axis=1).astype(np.int64)
    indeg = A.sum(axis=0).astype(np.int64)
    L = int(depth.max())
    dirs, cs, mfs, mus = [], [], [], []
    cur = oracle.PULL if mode == oracle.MODE_PULL_ONLY else oracle.PUSH
    for k in range(1, L + 1):
        dirs.append(cur)
        newf = depth == k + 1
        c = int(newf.sum())
        mf = int(outdeg[newf].sum())
        unvisited = (depth == 0) | (depth > k + 1)
        mu = int(indeg[unvisited].sum())
        cs.append(c)
        mfs.append(mf)
        mus.append(mu)
        if mode == oracle.MODE_DO and c > 0:
            c_old = int((depth == k).sum())
            cur = oracle.direction(rule, cur, c_old, c, mf, mu, n, alpha, beta)
    return np.array(dirs, np.int8), np.array(cs), np.array(mfs), np.array(mus)


def _check_graph(A, rules_params):
    n = A.shape[0]
    src, dst = np.nonzero(A)
    g = synth.from_edges(n, src, dst, symmetrize=False)
    gT = synth.transpose(g)
    for s in range(n):
        depth = _depth_by_matrix_powers(A, s)
        exp_oracle, _ = oracle.bfs(g, s)
        assert np.array_equal(depth, exp_oracle)
        for rule, mode, alpha, beta in rules_params:
            t = oracle.trace(g, gT, depth, mode=mode, rule=rule, alpha=alpha, beta=beta)
            d, c, mf, mu = _trace_by_definition(A, depth, rule, mode, alpha, beta)
            assert t["levels"] == len(d)
            assert np.array_equal(t["c"], c), (A.tolist(), s)
            assert np.array_equal(t["m_f"], mf), (A.tolist(), s)
            assert np.array_equal(t["m_u"], mu), (A.tolist(), s)
            assert np.array_equal(t["dir"], d), (A.tolist(), s, rule, mode)


# (rule, mode, alpha, beta): the defaults, plus thresholds that make tiny graphs switch both
# ways (so a wrong c_old / m_f / m_u feeding the decision shows up in the sequence too)
RULES = [(oracle.RULE_EDGES, oracle.MODE_DO, 15.0, 18.0),
         (oracle.RULE_EDGES, oracle.MODE_DO, 1.0, 2.0),
         (oracle.RULE_PAPER_R, oracle.MODE_DO, 0.01, 0.01),
         (oracle.RULE_PAPER_R, oracle.MODE_DO, 0.3, 0.5),
         (oracle.RULE_EDGES, oracle.MODE_PULL_ONLY, 15.0, 18.0)]


def test_trace_bruteforce_all_directed_graphs_n_le_4():
    """Every directed graph without self-loops on n <= 4 vertices, every source."""
    for n in (2, 3, 4):
        pairs = [(i, j) for i in range(n) for j in range(n) if i != j]
        for bits in itertools.product((0, 1), repeat=len(pairs)):
            A = np.zeros((n, n), np.uint8)
            for (i, j), b in zip(pairs, bits):
                A[i, j] = b
            _check_graph(A, RULES)


@pytest.mark.parametrize("n,count", [(5, 1500), (6, 800)])
def test_trace_bruteforce_random_directed_graphs(n, count):
    rng = np.random.Generator(np.random.PCG64(100 + n))
    for _ in range(count):
        A = (rng.random((n, n)) < rng.uniform(0.15, 0.6)).astype(np.uint8)
        np.fill_diagonal(A, 0)
        _check_graph(A, RULES)


def test_trace_directed_broom_closed_form():
    """0 -> 1, 1 -> {2..m+1}, every leaf -> z = m+2 (a directed broom whose handle, head
    and sink have in-degree != out-degree).  From s = 0 the levels discover {1}, the m
    leaves, {z}, nothing.  Closed form (Eq. 1; R11 definitions):
      c   = [1, m, 1, 0]
      m_f = [outdeg(1), sum outdeg(leaves), outdeg(z), 0] = [m, m, 0, 0]
      m_u = in_total - visited in-degree = (1 + m + m) - [1, 1 + m, 1 + 2m, 1 + 2m]
          = [2m, m, 0, 0]."""
    for m in (1, 2, 5, 40):
        n = m + 3
        z = m + 2
        src = [0] + [1] * m + list(range(2, m + 2))
        dst = [1] + list(range(2, m + 2)) + [z] * m
        g = synth.from_edges(n, src, dst, symmetrize=False)
        gT = synth.transpose(g)
        depth, L = oracle.bfs(g, 0)
        assert depth.tolist() == [1, 2] + [3] * m + [4] and L == 4
        t = oracle.trace(g, gT, depth, mode=oracle.MODE_PUSH_ONLY)
        assert t["c"].tolist() == [1, m, 1, 0]
        assert t["m_f"].tolist() == [m, m, 0, 0]
        assert t["m_u"].tolist() == [2 * m, m, 0, 0]
        # edge rule (R11, alpha 15, beta 18), decisions after each level:
        #   level 1: c 1 -> 1 does not grow: push
        #   level 2: c 1 -> m grows iff m > 1, and 15 * m_f = 15 m > m_u = m: pull
        #   level 3 (pull): c m -> 1 shrinks; back to push iff 18 * 1 < n = m + 3
        #   level 4 discovers nothing: no decision, the BFS ends
        t = oracle.trace(g, gT, depth)
        if m == 1:
            exp = [0, 0, 0, 0]
        else:
            exp = [0, 0, 1, 0 if 18 < n else 1]
        assert t["dir"].tolist() == exp, (m, t["dir"].tolist())


def test_sssp_switch_boundary_is_strict():
    """R29 / SPEC S:341: push while nnz(f)/n <= alpha, switch to pull when nnz(f)/n > alpha.
    On the 4-vertex diamond with alpha = 1/4 the first frontier {0} sits exactly on the
    threshold (1/4 is exact in binary): it must stay push; {1, 2} (2/4 > 1/4) switches;
    the switch is never undone.  Hand-computed: [(push, 1), (pull, 2), (pull, 1)]."""
    g = synth.from_edges(4, [0, 0, 1, 2], [1, 2, 3, 3], symmetrize=False)
    d, trace = osssp.sssp_2phase(g.off, g.idx, np.ones(g.nnz), 0, alpha=0.25)
    assert d.tolist() == [0.0, 1.0, 1.0, 2.0]
    assert trace == [(osssp.PUSH, 1), (osssp.PULL, 2), (osssp.PULL, 1)]
    # n = 10, alpha = 0.1: 1/10 == 0.1 in IEEE double; a path keeps |f| = 1 forever -> all push
    g = synth.from_edges(10, list(range(9)), list(range(1, 10)), symmetrize=False)
    d, trace = osssp.sssp_2phase(g.off, g.idx, np.ones(g.nnz), 0, alpha=0.1)
    assert d.tolist() == [float(i) for i in range(10)]
    assert [t[0] for t in trace] == [osssp.PUSH] * 10
    # just below the threshold it switches at once
    d, trace = osssp.sssp_2phase(g.off, g.idx, np.ones(g.nnz), 0, alpha=0.0999)
    assert [t[0] for t in trace] == [osssp.PULL] * 10


@pytest.mark.slow
def test_p7_kron21_analog_trace_shape():
    """SURVEY pin P7 (qualitative): on the kron_g500-logn21 analog (RMAT s21 ef48, Table 3
    P:451, pin P1) the frontier peaks at Iteration 4 (Fig. 5a) and the paper's r-rule
    gives the three phases push -> pull -> push, starting with 2 push iterations
    for hub-early sources ("2 iterations of push followed by 3 of pull, then 1 iteration of
    push or pull", Fig. 6 caption P:276)."""
    g = synth.rmat(21, 48, seed=1)
    srcs = synth.sources(g, 8, seed=2)
    peak4 = 0
    exact = 0
    for s in srcs:
        d, L = oracle.bfs(g, int(s))
        sizes = np.bincount(d)[1:]                      # |F_k| for k = 1..L
        if int(np.argmax(sizes)) + 1 == 4:
            peak4 += 1
        t = oracle.trace(g, g, d, rule=oracle.RULE_PAPER_R)
        dirs = "".join("HL"[x] for x in t["dir"])
        assert re.fullmatch(r"H{2,3}L+H*", dirs), dirs   # push phase, pull phase, push phase
        if dirs.startswith("HHLLL") and len(dirs) == 6:
            exact += 1
    assert peak4 >= 6, peak4
    assert exact >= 1
