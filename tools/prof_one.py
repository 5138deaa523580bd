"""Run W warm-up BFS then one BFS from a fixed source (target for ncu -s W -c 1)."""
import sys
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
src = int(sys.argv[2]) if len(sys.argv) > 2 else 2764614
W = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = synth.make(cfg)
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g, relabel="norelabel" not in sys.argv)
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
for _ in range(W):
    pp.bfs(G, src, depth)
st = pp.bfs(G, src, depth, stats_capacity=64)
torch.cuda.synchronize()
print("levels", st["levels"], "dirs", "".join("HL"[x] for x in st["dir"]), "ns", list(st["ns"]))
