"""Time pp_sssp on one B200: C2-shaped RMAT s22 ef16, integer weights 1..10.

Prints one JSON line per source and a summary: ms per SSSP (CUDA events on the launching
stream, warm-up first), GTEPS = nnz / time (the BFS convention, R18), iterations and the
switch point.  Usage: python tools/sssp_bench.py [config] [nsources] [alpha]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1804_03327_b200 as pp
import synth


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    alphas = [float(sys.argv[3])] if len(sys.argv) > 3 else [0.01, 0.05, 1e9]
    g = synth.make(cfg)
    w = synth.edge_weights(g.nnz, seed=21)
    gT, wT = synth.transpose_weighted(g, w)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).astype(dt)).cuda()
    args = (t(g.off, np.int64), t(g.idx.view(np.int32), np.int32), t(w, np.float32),
            t(gT.off, np.int64), t(gT.idx.view(np.int32), np.int32), t(wT, np.float32))
    ctx = pp.Context(0)
    dist = torch.empty(g.n, dtype=torch.float32, device="cuda")
    srcs = synth.sources(g, ns, seed=9)
    for alpha in alphas:
        times = []
        for s in srcs:
            pp.sssp(ctx, *args, source=int(s), alpha=alpha, dist=dist)  # warm-up
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            _, st = pp.sssp(ctx, *args, source=int(s), alpha=alpha, dist=dist)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            times.append(ms)
            print(json.dumps({"config": cfg, "alpha": alpha, "source": int(s), "ms": round(ms, 3),
                              "gteps": round(g.nnz / ms / 1e6, 2), **st}))
        m = float(np.mean(times))
        print(json.dumps({"summary": cfg, "alpha": alpha, "n": g.n, "nnz": g.nnz, "mean_ms": round(m, 3),
                          "gteps": round(g.nnz / m / 1e6, 2)}))


if __name__ == "__main__":
    main()
