"""Probe: effect of degree-descending vertex relabelling on the existing BFS kernel.

Relabels the graph on the host (numpy) and uploads both versions; times the same
sources (mapped) on each.  Diagnostic only (depths of the relabelled run are in new ids).
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_1804_03327_b200 as pp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 16


def relabel(g):
    deg = np.diff(g.off)
    perm = np.argsort(-deg, kind="stable").astype(np.int64)      # new -> old
    rank = np.empty(g.n, dtype=np.int64)
    rank[perm] = np.arange(g.n)                                    # old -> new
    ndeg = deg[perm]
    noff = np.zeros(g.n + 1, dtype=np.int64)
    np.cumsum(ndeg, out=noff[1:])
    rows_old = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    key = (rank[rows_old].astype(np.uint64) << np.uint64(32)) | rank[g.idx].astype(np.uint64)
    key.sort()
    nidx = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return synth.CSR(g.n, noff, nidx, True, g.name + "_relabel"), perm, rank


def timeit(G, srcs, depth, flush):
    for s in srcs[:3]:
        pp.bfs(G, int(s), depth)
    ts = []
    for s in srcs:
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pp.bfs(G, int(s), depth)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.array(ts)


t0 = time.time()
g = synth.make(cfg)
gr, perm, rank = relabel(g)
print(f"{cfg}: n={g.n} nnz={g.nnz}; relabel {time.time()-t0:.1f}s", flush=True)
srcs = synth.sources(g, nsrc, seed=2)
ctx = pp.Context(0)
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
G = pp.Graph.from_csr(ctx, g)
ta = timeit(G, srcs, depth, flush)
da = depth.cpu().numpy()
G.close()
Gr = pp.Graph.from_csr(ctx, gr)
tb = timeit(Gr, rank[srcs], depth, flush)
db = depth.cpu().numpy()
ok = np.array_equal(da, db[rank])
print(f"orig    : mean {ta.mean():.1f} us  -> {g.nnz/ta.mean()/1e3:.1f} GTEPS")
print(f"relabel : mean {tb.mean():.1f} us  -> {g.nnz/tb.mean()/1e3:.1f} GTEPS  (last depths equal: {ok})")
for s, a, b in zip(srcs, ta, tb):
    print(f"  src {s}: {a:7.1f} {b:7.1f}")


def levels(G, s):
    st = pp.bfs(G, int(s), depth, stats_capacity=64)
    L = st["levels"]
    return ["%s%d:%.1f" % ("HL"[st["dir"][k]], st["c"][k], st["ns"][k] / 1e3) for k in range(L)]


Gr.close()
G = pp.Graph.from_csr(ctx, g)
for s in srcs[:6]:
    print("orig   ", s, " ".join(levels(G, s)))
G.close()
Gr = pp.Graph.from_csr(ctx, gr)
for s in srcs[:6]:
    print("relabel", s, " ".join(levels(Gr, rank[s])))
