"""Diagnose the end-to-end (host output) path cost of pp_bfs."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

g = synth.make(sys.argv[1] if len(sys.argv) > 1 else "C1")
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g)
d = torch.empty(g.n, dtype=torch.int32, device="cuda")
pinned = torch.empty(g.n, dtype=torch.int32).pin_memory()
hp = pinned.numpy()
pageable = np.empty(g.n, np.int32)
s = int(synth.sources(g, 1)[0])
def t(f, k=10):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 1e3 * np.median(ts)
print("device depth + sync   ms", t(lambda: pp.bfs(G, s, d)))
print("pinned host depth     ms", t(lambda: pp.bfs(G, s, hp)))
print("pageable host depth   ms", t(lambda: pp.bfs(G, s, pageable)))
print("torch D2H pinned copy ms", t(lambda: pinned.copy_(d, non_blocking=True)))
