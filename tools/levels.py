"""Per-level device timing of pp_bfs on a config (diagnostic; prints a table)."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 4
heur = pp.PP_HEUR_PAPER_R if "paper" in sys.argv else pp.PP_HEUR_EDGES
t0 = time.time()
g = synth.make(cfg)
print(f"{cfg}: n={g.n} nnz={g.nnz} gen {time.time()-t0:.1f}s", flush=True)
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g, relabel="norelabel" not in sys.argv)
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for s in synth.sources(g, 3, seed=7):
    pp.bfs(G, int(s), depth, heuristic=heur)
for s in synth.sources(g, nsrc, seed=2):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = pp.bfs(G, int(s), depth, heuristic=heur, stats_capacity=70000)
    e1.record()
    torch.cuda.synchronize()
    L = st["levels"]
    dirs = "".join("HL"[x] for x in st["dir"][:L])
    print(f"src {s}: {e0.elapsed_time(e1)*1e3:.1f} us (event, incl. stats sync), levels {L} {dirs[:40]}, "
          f"init {st['init_ns']/1e3:.1f} us, sum(levels) {st['ns'].sum()/1e3:.1f} us")
    if L <= 40:
        for k in range(L):
            print(f"   L{k+1} {'HL'[st['dir'][k]]} c={st['c'][k]:>9} m_f={st['m_f'][k]:>11} {st['ns'][k]/1e3:8.1f} us")
    else:
        ns = st["ns"][:min(L, 70000)]
        print(f"   per-level us: mean {ns.mean()/1e3:.2f} median {np.median(ns)/1e3:.2f} max {ns.max()/1e3:.1f}")

# fixed per-level cost: BFS from an isolated vertex = init + one empty level
iso = int(np.nonzero(np.diff(g.off) == 0)[0][0]) if np.any(np.diff(g.off) == 0) else None
if iso is not None:
    vals = []
    for _ in range(20):
        st = pp.bfs(G, iso, depth, heuristic=heur, stats_capacity=4)
        vals.append((st["init_ns"], st["ns"][0]))
    v = np.array(vals)
    print(f"isolated source: init {np.median(v[:,0])/1e3:.2f} us, empty level {np.median(v[:,1])/1e3:.2f} us")
