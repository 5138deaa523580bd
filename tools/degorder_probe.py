"""Probe: pull rows (CSC) ordered by in-neighbour degree (descending) instead of id.

Uploads C2 twice: symmetric (CSC = CSR, id-ordered rows) and as a 'directed' graph whose
CSC holds the same rows sorted by neighbour degree.  Depths must agree; times compared."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_1804_03327_b200 as pp  # noqa: E402

g = synth.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 16
deg = np.diff(g.off)
rows = np.repeat(np.arange(g.n, dtype=np.int64), deg)
key = (rows << 41) | ((2**19 - 1 - np.minimum(deg[g.idx], 2**19 - 1)).astype(np.int64) << 22) | g.idx.astype(np.int64)
assert g.n <= 2**22
pidx = g.idx[np.argsort(key, kind="stable")]
srcs = synth.sources(g, nsrc, seed=2)
ctx = pp.Context(0)
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(G):
    for s in srcs[:3]:
        pp.bfs(G, int(s), depth)
    ts, lv = [], []
    for s in srcs:
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pp.bfs(G, int(s), depth)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    for s in srcs[:6]:
        st = pp.bfs(G, int(s), depth, stats_capacity=64)
        lv.append(" ".join("%s%d:%.1f" % ("HL"[st["dir"][k]], st["c"][k], st["ns"][k] / 1e3)
                           for k in range(st["levels"])))
    return np.array(ts), depth.cpu().numpy(), lv


G = pp.Graph(ctx, g.n, g.off, g.idx)
ta, da, la = timeit(G)
G.close()
G = pp.Graph(ctx, g.n, g.off, g.idx, g.off, pidx, symmetric=False)
tb, db, lb = timeit(G)
print(f"id-ordered pull rows : {ta.mean():.1f} us -> {g.nnz / ta.mean() / 1e3:.1f} GTEPS")
print(f"degree-ordered       : {tb.mean():.1f} us -> {g.nnz / tb.mean() / 1e3:.1f} GTEPS  depths equal {np.array_equal(da, db)}")
for a, b in zip(la, lb):
    print("  id ", a)
    print("  deg", b)
