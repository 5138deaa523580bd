"""CPU oracle for SURVEY NEXT-4: SSSP over the min-plus semiring (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py may import this module.  It shares no
code with paper_1804_03327_b200/ and never imports it.  P:n = PAPER.md line n.

  sssp_2phase(off, idx, w, s, alpha)  the paper's "simple 2-phase direction-optimized
      traversal" for SSSP (Sec. 5.6): Bellman-Ford d <- min(d, A^T (min.+) f) with an
      active-vertex frontier f; unmasked column-based (push) matvec while nnz(f)/n <= alpha,
      then ONE switch to row-based (pull) matvec until the fixpoint.  No mask and no early
      exit (those are Boolean-only).  Operand reuse (valid for SSSP):
      the pull reads all of d instead of f.  fp64 throughout (R27-R30).
  dijkstra(off, idx, w, s)            textbook binary-heap Dijkstra, used only
      as an independent pin of sssp_2phase.

Pins (tests/test_oracle_sssp.py): SPEC S:343 diamond example, scipy.sparse.csgraph
Dijkstra on random weighted graphs, Floyd-Warshall brute force on tiny graphs, unit weights
== BFS level - 1 with iterations == eccentricity + 1 (closed form for Jacobi
Bellman-Ford), unreachable = inf, single vertex.
"""
from __future__ import annotations

import heapq

import numpy as np

PUSH, PULL = 0, 1


def sssp_2phase(off, idx, w, source: int, alpha: float = 0.01):
    """Sec. 5.6 two-phase SSSP.  off/idx/w: CSR of A (row i = out-edges of i,
    A(i,j) = w).  Returns (d, trace) where d is float64 (inf = unreachable) and trace the
    per-iteration list of (direction, nnz(f) before the iteration).

    Iteration k (Jacobi form of Bellman-Ford, R28):
        t = A^T (min.+) f_k        push: over the out-edges of the vertices in f_k
                                   pull: t(j) = min_i d_k(i) + A(i,j)   (operand reuse)
        d_{k+1} = min(d_k, t);  f_{k+1} = { v : d_{k+1}(v) < d_k(v) }
    Direction: push until nnz(f)/n > alpha, then pull until f is empty (R29)."""
    off = np.asarray(off, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    n = len(off) - 1
    if not (0 <= source < n):
        raise ValueError("source out of range")
    if len(w) and (np.isnan(w).any() or (w < 0).any()):
        raise ValueError("negative or NaN edge weight (SPEC S:342)")
    d = np.full(n, np.inf)
    d[source] = 0.0
    f = np.array([source], dtype=np.int64)
    direction = PUSH
    trace = []
    rows = np.repeat(np.arange(n), np.diff(off))  # row i of A for every stored entry
    while len(f):
        if direction == PUSH and len(f) / n > alpha:
            direction = PULL
        trace.append((direction, len(f)))
        t = np.full(n, np.inf)
        if direction == PUSH:
            for i in f:  # column-based: scatter A(i, :) + d(i) (Alg. 3 shape)
                for e in range(off[i], off[i + 1]):
                    j = idx[e]
                    t[j] = min(t[j], d[i] + w[e])
        else:  # row-based: t(j) = min over in-edges (i, j) of d(i) + A(i, j) (Alg. 2 shape)
            np.minimum.at(t, idx, d[rows] + w)
        d_next = np.minimum(d, t)
        f = np.flatnonzero(d_next < d)
        d = d_next
    return d, trace


def dijkstra(off, idx, w, source: int):
    """Binary-heap Dijkstra, fp64; inf = unreachable."""
    off = np.asarray(off, dtype=np.int64)
    n = len(off) - 1
    d = [float("inf")] * n
    d[source] = 0.0
    heap = [(0.0, source)]
    done = [False] * n
    while heap:
        du, u = heapq.heappop(heap)
        if done[u]:
            continue
        done[u] = True
        for e in range(off[u], off[u + 1]):
            v = int(idx[e])
            nd = du + float(w[e])
            if nd < d[v]:
                d[v] = nd
                heapq.heappush(heap, (nd, v))
    return np.array(d)
