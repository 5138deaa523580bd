"""Mean DO-BFS time over seeded sources for a grid of edge-rule (alpha, beta) and the paper
r-rule: the direction heuristic is a performance knob only (depths never change)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("no") else "C2"
g = synth.make(cfg)
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g, relabel="norelabel" not in sys.argv)  # bench layout
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
srcs = synth.sources(g, 32, seed=2)


def run(heur, alpha, beta):
    ts = []
    for s in srcs:
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pp.bfs(G, int(s), depth, heuristic=heur, alpha=alpha, beta=beta)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.mean(ts), g.nnz / (np.mean(ts) * 1e-6) / 1e9


for s in srcs[:3]:
    pp.bfs(G, int(s), depth)
print("paper r-rule a=b=0.01: %.1f us  %.0f GTEPS" % run(pp.PP_HEUR_PAPER_R, 0.01, 0.01))
for a in (0.0025, 0.005, 0.02, 0.05):
    print("paper r-rule a=%g b=0.01: %.1f us  %.0f GTEPS" % ((a,) + run(pp.PP_HEUR_PAPER_R, a, 0.01)))
for alpha in (2, 4, 8, 15, 30, 60, 120):
    for beta in (6, 18, 54):
        print("edges alpha=%d beta=%d: %.1f us  %.0f GTEPS" % ((alpha, beta) + run(pp.PP_HEUR_EDGES, alpha, beta)))
