"""Large-config check on one GPU: generate (seeded), upload, time DO-BFS over a few sources,
and verify one source bit-exactly against the CPU oracle (+ Graph500 validation of parents)."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import synth
import paper_1804_03327_b200 as pp

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 4
t0 = time.time()
g = synth.make(cfg)
print(f"{cfg}: n={g.n} nnz={g.nnz} maxdeg={int(np.diff(g.off).max())} gen {time.time()-t0:.1f}s", flush=True)
ctx = pp.Context(0)
t0 = time.time()
G = pp.Graph.from_csr(ctx, g, relabel="norelabel" not in sys.argv)
print(f"upload {time.time()-t0:.1f}s device bytes {G.info()[2]/1e9:.2f} GB", flush=True)
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
parent = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
srcs = synth.sources(g, nsrc, seed=2)
pp.bfs(G, int(srcs[0]), depth)
ts = []
for s in srcs:
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pp.bfs(G, int(s), depth)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
    st = pp.bfs(G, int(s), depth, stats_capacity=70000)
    L = st["levels"]
    print(f"src {s}: {ts[-1]*1e6:.1f} us, {g.nnz/ts[-1]/1e9:.1f} GTEPS, levels {L} "
          f"{''.join('HL'[x] for x in st['dir'][:40])}", flush=True)
print(f"mean {np.mean(ts)*1e6:.1f} us -> {g.nnz/np.mean(ts)/1e9:.1f} GTEPS (paper convention nnz/time)")
s = int(srcs[0])
pp.bfs(G, s, depth, parent)
d = depth.cpu().numpy()
t0 = time.time()
exp, L = oracle.bfs(g, s)
print(f"oracle {time.time()-t0:.1f}s; depth bit-exact: {np.array_equal(d, exp)}", flush=True)
assert np.array_equal(d, exp)
oracle.validate_graph500(g, s, d, parent.cpu().numpy())
print("graph500 validation of parents: ok")
