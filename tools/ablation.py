"""Table 2 analog (NEXT-3): the paper's cumulative optimisations, measured on a
B200 on synthetic graphs.  Rows (cumulative, as in Table 2):
  push-only          column-based masked mxv every level (structure-only is always on here:
                     the library has no value arrays, Opt. 5)
  + change of direction   DO, pull computes every non-isolated row, no early exit, A^T f
  + masking          pull computes only unvisited rows (Opt. 2)
  + early exit       (Opt. 3)
  + operand reuse    pull multiplies by v instead of f (Opt. 4)
Every row must give identical depths (toggle invariance); checked per source.
Usage: python tools/ablation.py [CONFIG ...]   (default K21 C2)"""
import json
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

cfgs = [a for a in sys.argv[1:] if not a.startswith("-")] or ["K21", "C2"]
NS = 16
ROWS = [("push-only", pp.PP_MODE_PUSH_ONLY, 0),
        ("+ change of direction", pp.PP_MODE_DO, pp.PP_OPT_NO_MASKING | pp.PP_OPT_NO_EARLYEXIT | pp.PP_OPT_NO_REUSE),
        ("+ masking", pp.PP_MODE_DO, pp.PP_OPT_NO_EARLYEXIT | pp.PP_OPT_NO_REUSE),
        ("+ early exit", pp.PP_MODE_DO, pp.PP_OPT_NO_REUSE),
        ("+ operand reuse", pp.PP_MODE_DO, 0)]
out = []
ctx = pp.Context(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in cfgs:
    g = synth.make(cfg)
    G = pp.Graph.from_csr(ctx, g, relabel=True)
    srcs = [int(s) for s in synth.sources(g, NS, seed=2)]
    ref = {}
    for heur, hname in ((pp.PP_HEUR_PAPER_R, "paper r-rule (alpha=beta=0.01)"), (pp.PP_HEUR_EDGES, "edge rule (15, 18)")):
        prev = None
        lines = []
        for name, mode, tog in ROWS:
            depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
            for s in srcs[:2]:
                pp.bfs(G, s, depth, heuristic=heur, mode=mode, toggles=tog)
            ts, dirs = [], []
            for s in srcs:
                flush.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pp.bfs(G, s, depth, heuristic=heur, mode=mode, toggles=tog)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
                if s not in ref:
                    ref[s] = depth.clone()
                elif not torch.equal(ref[s], depth):
                    raise SystemExit(f"{cfg} {name}: depths differ from the first row for source {s}")
            st = pp.bfs(G, srcs[0], depth, heuristic=heur, mode=mode, toggles=tog, stats_capacity=4096)
            t = float(np.mean(ts))
            gteps = g.nnz / t / 1e9
            sp = (prev / t) if prev else None
            prev = t
            lines.append(dict(config=cfg, heuristic=hname, row=name, mean_ms=t * 1e3, gteps=gteps,
                              speedup=sp, dirs_src0="".join("HL"[x] for x in st["dir"])))
            print(json.dumps(lines[-1]), flush=True)
        out += lines
    del G
    torch.cuda.empty_cache()

md = ["| graph | heuristic | optimisation (cumulative) | ms / BFS | GTEPS | speed-up | directions (source 0) |",
      "|---|---|---|---|---|---|---|"]
for r in out:
    sp = f"{r['speedup']:.2f}x" if r["speedup"] else "-"
    md.append(f"| {r['config']} | {r['heuristic']} | {r['row']} | {r['mean_ms']:.3f} | {r['gteps']:.1f} | {sp} | {r['dirs_src0']} |")
print("\n".join(md))
