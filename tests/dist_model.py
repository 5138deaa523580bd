"""Host-level model of the 1D-partitioned BFS (paper_1804_03327_b200/csrc/dist.cu), used by
the CPU tests to check the distributed algorithm's logic (partition, per-level exchange,
replicated direction decision) with a real torch.distributed all_gather over gloo.

Test infrastructure only.  Rank p owns rows [lo, hi) from pp_partition; per level it runs
push (global frontier, owned targets: the row's ids inside [lo, hi)) or pull (owned
unvisited rows against the replicated visited set), then all-gathers the owned next slices
and every rank ORs them into its visited set and takes the same decision."""
import numpy as np

import oracle


def dist_bfs_model(g, s, rank, nranks, lo, hi, allgather_bool, mode=oracle.MODE_DO,
                   rule=oracle.RULE_EDGES):
    n = g.n
    deg = np.diff(g.off)
    depth = np.zeros(hi - lo, np.int32)
    vis = np.zeros(n, bool)
    vis[s] = True
    fr = np.zeros(n, bool)
    fr[s] = True
    if lo <= s < hi:
        depth[s - lo] = 1
    dirs, cs = [], []
    direction = oracle.PULL if mode == oracle.MODE_PULL_ONLY else oracle.PUSH
    c_old, m_u = 1, int(g.nnz - deg[s])
    d = 1
    while True:
        nxt_own = np.zeros(hi - lo, bool)
        if direction == oracle.PUSH:
            for u in np.nonzero(fr)[0]:
                row = g.idx[g.off[u]:g.off[u + 1]]
                row = row[(row >= lo) & (row < hi)]           # the push range of row u
                for w in row:
                    if not vis[w] and not nxt_own[w - lo]:
                        nxt_own[w - lo] = True
        else:
            for v in range(lo, hi):
                if vis[v] or deg[v] == 0:
                    continue
                row = g.idx[g.off[v]:g.off[v + 1]]
                if np.any(vis[row]):                             # pull against the snapshot
                    nxt_own[v - lo] = True
        depth[nxt_own] = d + 1
        nxt = allgather_bool(nxt_own)                            # exchange step
        assert len(nxt) >= n
        nxt = nxt[:n]
        vis |= nxt
        fr = nxt
        c_new = int(nxt.sum())
        m_f = int(deg[nxt].sum())
        m_u -= m_f
        dirs.append(direction)
        cs.append(c_new)
        if c_new == 0:
            break
        if mode == oracle.MODE_DO:
            direction = oracle.direction(rule, direction, c_old, c_new, m_f, m_u, n)
        c_old = c_new
        d += 1
    return depth, np.array(dirs, np.int8), np.array(cs, np.int64)
