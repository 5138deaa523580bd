"""Per-level roofline of one DO-BFS (the heaviest pull and push
levels): algorithmic bytes of each level under DESIGN.md §6's byte-exact model (bench.py
byte_model, from the result depths and the direction trace) / the level's device time
(%globaltimer between level barriers) / the measured HBM peak.
Usage: python tools/level_roofline.py [CONFIG] [NSOURCES]"""
import json
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp
from bench import byte_model

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 4
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6537.0
dev = "cuda"
g = synth.make(cfg)
n, nnz = g.n, g.nnz
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g, relabel=True)
off_bytes = 4 if nnz < 2**32 else 8
off_t = torch.from_numpy(g.off).to(dev)
idx_t = torch.from_numpy(g.idx.astype(np.int64)).to(dev)
deg_t = off_t[1:] - off_t[:-1]
rows_t = torch.repeat_interleave(torch.arange(n, device=dev), deg_t)
key_t = torch.from_numpy(synth.degree_order_key(g).astype(np.int64)).to(dev)
e = torch.sort(key_t[rows_t] * n + key_t[idx_t]).values
rows_t, idx_t = e // n, e % n
del e
deg_t = torch.bincount(rows_t, minlength=n)
off_t = torch.zeros(n + 1, dtype=torch.int64, device=dev)
off_t[1:] = torch.cumsum(deg_t, 0)
gd = (off_t, idx_t, rows_t, deg_t, deg_t > 0)
depth = torch.empty(n, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for s in synth.sources(g, 2, seed=7):
    pp.bfs(G, int(s), depth)
print(f"{cfg}: n={n} nnz={nnz}; peak {peak} GB/s (MEASURED_PEAKS.json); model = DESIGN.md §6 byte-exact")
print("| source | level | dir | new frontier | model MB | device µs | achieved GB/s | frac of peak |")
print("|---|---|---|---|---|---|---|---|")
for s in synth.sources(g, nsrc, seed=2):
    flush.zero_()
    torch.cuda.synchronize()
    st = pp.bfs(G, int(s), depth, stats_capacity=4096)
    dm = torch.empty_like(depth)
    dm[key_t] = depth
    parts = byte_model(torch, gd, dm, list(st["dir"]), n, nnz, off_bytes, per_level=True)
    ns = [st["init_ns"]] + list(st["ns"])
    for k, (b, t) in enumerate(zip(parts, ns)):
        lab = "init" if k == 0 else str(k)
        dr = "-" if k == 0 else "HL"[st["dir"][k - 1]]
        c = "-" if k == 0 else str(st["c"][k - 1])
        gbs = b / (t * 1e-9) / 1e9 if t > 0 else 0.0
        print(f"| {s} | {lab} | {dr} | {c} | {b/1e6:.2f} | {t/1e3:.1f} | {gbs:.0f} | {gbs/peak:.3f} |")
    tb, tt = sum(parts), sum(ns)
    print(f"| {s} | total | | | {tb/1e6:.2f} | {tt/1e3:.1f} | {tb/(tt*1e-9)/1e9:.0f} | {tb/(tt*1e-9)/1e9/peak:.3f} |")
