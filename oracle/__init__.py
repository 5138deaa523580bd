"""CPU oracle for the push-pull BFS / masked-mxv hot path (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It shares no code with paper_1804_03327_b200/ and
never imports it.  P:n = /root/reference/PAPER.md line n.

  bfs(g, s)                 O1 textbook queue BFS (oracle.c)
  parents(gT, depth, s)     O2 canonical min-id parent (oracle.c)
  mxv(M, u, ...)            O3 definitional masked Boolean matvec, Eq. 2/4 (oracle.c)
  direction(...)            O4 one push/pull decision, P:366 (oracle.c)
  trace(g, gT, depth, ...)  O4 per-level direction trace (oracle.c)
  alg1_bfs_dense(A, s)      Algorithm 1 literally, dense numpy; tiny graphs only
  validate_graph500(...)    O5 Graph500-style validation (needs no oracle)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

PUSH, PULL = 0, 1
RULE_EDGES, RULE_PAPER_R = 0, 1
MODE_DO, MODE_PUSH_ONLY, MODE_PULL_ONLY = 0, 1, 2
DEFAULT_ALPHA_BETA = {RULE_EDGES: (15.0, 18.0), RULE_PAPER_R: (0.01, 0.01)}


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2, single thread)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        lib.oracle_bfs.restype = i64
        lib.oracle_bfs.argtypes = [i64, vp, vp, i64, vp]
        lib.oracle_parents.restype = ctypes.c_int
        lib.oracle_parents.argtypes = [i64, vp, vp, vp, i64, vp]
        lib.oracle_parents_ordered.restype = ctypes.c_int
        lib.oracle_parents_ordered.argtypes = [i64, vp, vp, vp, i64, vp, vp]
        lib.oracle_mxv.restype = ctypes.c_int
        lib.oracle_mxv.argtypes = [i64, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   vp, vp]
        lib.oracle_direction.restype = ctypes.c_int
        lib.oracle_direction.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i64, i64, i64,
                                         ctypes.c_double, ctypes.c_double]
        lib.oracle_trace.restype = i64
        lib.oracle_trace.argtypes = [i64, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_double, i64, vp, vp, vp, vp]
        _lib = lib
    return _lib


def _arr(x, dt):
    return np.ascontiguousarray(x, dtype=dt)


def bfs(g, s: int):
    """O1: depths (int32[n]; source 1, unreached 0) and the number of levels."""
    off, idx = _arr(g.off, np.int64), _arr(g.idx, np.uint32)
    depth = np.empty(g.n, dtype=np.int32)
    L = _load().oracle_bfs(g.n, off.ctypes.data, idx.ctypes.data, int(s), depth.ctypes.data)
    if L < 0:
        raise ValueError("source out of range")
    return depth, int(L)


def parents(gT, depth, s: int, key=None):
    """O2: min-id parent at depth-1 (gT = CSC of A: row v lists in-neighbours).  With
    `key` (a permutation: key[u] = position of u in a vertex order) the valid parent with
    the smallest key instead (the order of a PP_GRAPH_RELABEL graph)."""
    off, idx = _arr(gT.off, np.int64), _arr(gT.idx, np.uint32)
    depth = _arr(depth, np.int32)
    par = np.empty(gT.n, dtype=np.int32)
    if key is not None:
        key = _arr(key, np.uint32)
        assert key.shape == (gT.n,)
        rc = _load().oracle_parents_ordered(gT.n, off.ctypes.data, idx.ctypes.data,
                                            depth.ctypes.data, int(s), key.ctypes.data,
                                            par.ctypes.data)
    else:
        rc = _load().oracle_parents(gT.n, off.ctypes.data, idx.ctypes.data, depth.ctypes.data,
                                    int(s), par.ctypes.data)
    if rc != 0:
        raise ValueError("depth vector is not a BFS result")
    return par


def mxv(M, u, mask=None, complement=False, accum=False, replace=True, w_in=None):
    """O3: w = M u over ({0,1}, AND, OR, 0) with mask/complement/accum/replace (Eq. 4).

    M is the operator in CSR (row i lists j with M(i,j) != 0); pass the CSC of A
    (rows of A^T) for the traversal product w = A^T u.  Vectors are dense 0/1."""
    off, idx = _arr(M.off, np.int64), _arr(M.idx, np.uint32)
    u = _arr(u, np.uint8)
    m = None if mask is None else _arr(mask, np.uint8)
    wi = None if w_in is None else _arr(w_in, np.uint8)
    out = np.empty(M.n, dtype=np.uint8)
    rc = _load().oracle_mxv(M.n, off.ctypes.data, idx.ctypes.data, u.ctypes.data,
                            None if m is None else m.ctypes.data, int(bool(complement)),
                            int(bool(accum)), int(bool(replace)),
                            None if wi is None else wi.ctypes.data, out.ctypes.data)
    if rc != 0:
        raise ValueError("invalid mxv arguments")
    return out


def direction(rule, cur, c_old, c_new, m_f, m_u, n, alpha=None, beta=None):
    """O4: next direction (0 push / 1 pull) after a level."""
    a, b = DEFAULT_ALPHA_BETA[rule]
    alpha = a if alpha is None else alpha
    beta = b if beta is None else beta
    return int(_load().oracle_direction(rule, cur, c_old, c_new, m_f, m_u, n, alpha, beta))


def trace(g, gT, depth, mode=MODE_DO, rule=RULE_EDGES, alpha=None, beta=None):
    """O4: per-level (dir, c, m_f, m_u) implied by `depth` (g = CSR of A, gT = CSC)."""
    a, b = DEFAULT_ALPHA_BETA[rule]
    alpha = a if alpha is None else alpha
    beta = b if beta is None else beta
    depth = _arr(depth, np.int32)
    cap = int(depth.max()) if len(depth) else 0
    cap = max(cap, 1)
    d = np.zeros(cap, np.int8)
    c = np.zeros(cap, np.int64)
    mf = np.zeros(cap, np.int64)
    mu = np.zeros(cap, np.int64)
    off, coff = _arr(g.off, np.int64), _arr(gT.off, np.int64)
    L = _load().oracle_trace(g.n, off.ctypes.data, coff.ctypes.data, depth.ctypes.data, mode, rule,
                             alpha, beta, cap, d.ctypes.data, c.ctypes.data, mf.ctypes.data,
                             mu.ctypes.data)
    if L < 0:
        raise ValueError("trace capacity")
    return dict(levels=int(L), dir=d[:L], c=c[:L], m_f=mf[:L], m_u=mu[:L])


def alg1_bfs_dense(A: np.ndarray, s: int) -> np.ndarray:
    """Algorithm 1 written out literally on a dense 0/1 matrix A (tiny n).

      d <- 1; f <- e_s; v <- 0; c <- 1
      while c > 0:
          v <- f*d + v             (GrB_assign, standard arithmetic)
          f <- A^T f .* !v         (GrB_mxv over ({0,1}, AND, OR, 0), complemented mask)
          c <- sum_i f(i)          (GrB_reduce, standard +)
          d <- d + 1
    """
    A = (np.asarray(A) != 0)
    n = A.shape[0]
    d = 1
    f = np.zeros(n, dtype=bool)
    f[s] = True
    v = np.zeros(n, dtype=np.int64)
    c = 1
    while c > 0:
        v = f.astype(np.int64) * d + v
        t = np.zeros(n, dtype=bool)
        for i in range(n):                # row i of A^T: OR_j (A^T(i,j) AND f(j))
            acc = False
            for j in range(n):
                acc = acc or (bool(A[j, i]) and bool(f[j]))
            t[i] = acc
        f = t & ~(v != 0)
        c = int(f.sum())
        d = d + 1
    return v.astype(np.int32)


def validate_graph500(g, s: int, depth, parent=None, undirected=True):
    """O5: Graph500-style checks on (depth, parent); raises AssertionError on failure.

    - depth[s] == 1; every edge (u,w) with u reached has w reached and depth w <= depth u + 1;
      for undirected graphs reached/unreached never share an edge and |depth u - depth w| <= 1;
    - parent[s] == s; each reached v != s has (parent[v], v) an edge with
      depth[parent v] == depth v - 1; unreached have parent -1."""
    depth = np.asarray(depth)
    assert depth[s] == 1
    deg = np.diff(g.off)
    rows = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    du = depth[rows].astype(np.int64)
    dw = depth[g.idx].astype(np.int64)
    reached_u = du > 0
    assert np.all(dw[reached_u] > 0), "edge from reached to unreached vertex"
    assert np.all(dw[reached_u] <= du[reached_u] + 1), "depth jumps by more than one"
    if undirected:
        assert np.all((du > 0) == (dw > 0))
        both = (du > 0) & (dw > 0)
        assert np.all(np.abs(du[both] - dw[both]) <= 1)
    if parent is not None:
        parent = np.asarray(parent).astype(np.int64)
        assert parent[s] == s
        reached = depth > 0
        assert np.all(parent[~reached] == -1)
        vs = np.nonzero(reached)[0]
        vs = vs[vs != s]
        ps = parent[vs]
        assert np.all((ps >= 0) & (ps < g.n))
        assert np.all(depth[ps] == depth[vs] - 1)
        # (parent v, v) must be an edge: rows ascend and each row is sorted, so the
        # keys row*n + col are globally sorted and membership is a binary search.
        keys = rows * g.n + g.idx.astype(np.int64)
        q = ps * g.n + vs
        k = np.searchsorted(keys, q)
        ok = (k < len(keys)) & (keys[np.minimum(k, len(keys) - 1)] == q) if len(keys) else q != q
        assert np.all(ok), "parent edge missing"
    return True
