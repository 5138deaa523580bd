"""Isolate the heavy pull level: the same state (v = visited after level k) run through
pp_mxv's stand-alone row kernel, timed alone, vs the persistent kernel's level time."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

src = int(sys.argv[1]) if len(sys.argv) > 1 else 2764614
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = synth.make("C2")
n = g.n
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g)
depth = torch.empty(n, dtype=torch.int32, device="cuda")
st = pp.bfs(G, src, depth, stats_capacity=64)
print("bfs level ns", list(st["ns"]), "dirs", "".join("HL"[x] for x in st["dir"]))
d = depth.cpu().numpy()
v = ((d >= 1) & (d <= k)).astype(np.uint8)
nw = (n + 31) // 32
pad = np.zeros(nw * 32, np.uint8); pad[:n] = v
vb = torch.from_numpy(np.packbits(pad, bitorder="little").view("<u4").astype(np.uint32).view(np.int32)).cuda()
wt = torch.zeros(nw, dtype=torch.int32, device="cuda")
u = pp.make_vector(pp.PP_VEC_BITMAP, n, vb, int(v.sum()))
w = pp.make_vector(pp.PP_VEC_BITMAP, n, wt, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for ee in (1, 0):
    ts = []
    for r in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pp.mxv(G, w, u, mask=u, complement=True, direction=pp.PP_DIR_PULL, early_exit=ee, want_nnz=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    found = int(torch.from_numpy(np.unpackbits(wt.cpu().numpy().view(np.uint8), bitorder="little")[:n]).sum())
    print(f"k_mxv_pull early_exit={ee}: median {np.median(ts):.1f} us  min {min(ts):.1f}  found {found}")
