"""SURVEY NEXT-3, Fig. 6 on a synthetic analog: per-iteration runtime of the two
masked matvecs on BFS-sampled vectors (not random ones).  For S sources, the GPU BFS gives
the depths; for every level k with a non-empty frontier F_k the script times, with CUDA events
(L2 flushed, median of 3):
  column-based with mask:  f' = A^T f_k .* !v_k   (PUSH, u = f_k, complemented mask v_k)
  row-based with mask + early exit: f' = A^T v_k .* !v_k   (PULL, operand reuse)
and checks both outputs have exactly |F_{k+1}| entries (the BFS result).  Prints, per level,
the median over sources of nnz(f), of the unvisited count and of each runtime — the paper's
claims: the column-based runtime grows with the supervertices of the frontier and falls after
the frontier peak (the oval); the row-based runtime is high for the first iterations and
drops sharply once a supervertex is visited (the backwards 'L'); which arm is cheaper flips
twice (push, pull, push).  Usage: python tools/fig6_sample.py [CONFIG] [SOURCES]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_1804_03327_b200 as pp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "K21"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g = synth.make(cfg)
n = g.n
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g)
nw = (n + 31) // 32
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
depth = torch.empty(n, dtype=torch.int32, device="cuda")
wt = torch.zeros(nw, dtype=torch.int32, device="cuda")
w = pp.make_vector(pp.PP_VEC_BITMAP, n, wt, 0)
pad = nw * 32 - n
weights = (2 ** torch.arange(32, device="cuda", dtype=torch.int64))


def to_bits(mask_bool):
    """bool[n] -> little-endian uint32 words as int32 (bit b of word w = element 32w + b)."""
    m = torch.nn.functional.pad(mask_bool.to(torch.int64), (0, pad)).view(nw, 32)
    x = (m * weights).sum(1)
    return torch.where(x >= 2 ** 31, x - 2 ** 32, x).to(torch.int32)


def timeit(fn):
    ts = []
    for _ in range(3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


per_level = {}
bad = 0
for s in synth.sources(g, S, seed=2):
    pp.bfs(G, int(s), depth)
    d = depth.clone()
    L = int(d.max())
    for k in range(1, L + 1):
        f = d == k
        v = (d >= 1) & (d <= k)
        nf, nun = int(f.sum()), int(n - v.sum())
        fb, vb = to_bits(f), to_bits(v)
        fv = pp.make_vector(pp.PP_VEC_BITMAP, n, fb, nf)
        vv = pp.make_vector(pp.PP_VEC_BITMAP, n, vb, int(v.sum()))
        tc = timeit(lambda: pp.mxv(G, w, fv, mask=vv, complement=True, direction=pp.PP_DIR_PUSH,
                                   want_nnz=False))
        tr = timeit(lambda: pp.mxv(G, w, vv, mask=vv, complement=True, direction=pp.PP_DIR_PULL,
                                   early_exit=True, want_nnz=False))
        want = int((d == k + 1).sum())
        got_c = pp.mxv(G, w, fv, mask=vv, complement=True, direction=pp.PP_DIR_PUSH)
        got_r = pp.mxv(G, w, vv, mask=vv, complement=True, direction=pp.PP_DIR_PULL)
        bad += (got_c != want) + (got_r != want)
        per_level.setdefault(k, []).append((nf, nun, tc, tr))
print(f"{cfg}: n={n} nnz={g.nnz}; {S} sources; output-size mismatches vs the BFS: {bad}")
print("| iteration | sources | median nnz(f) | median unvisited | col+mask us (median) | row+mask+EE us (median) | cheaper |")
print("|---|---|---|---|---|---|---|")
for k in sorted(per_level):
    a = np.array(per_level[k])
    tc, tr = np.median(a[:, 2]), np.median(a[:, 3])
    print(f"| {k} | {len(a)} | {int(np.median(a[:, 0]))} | {int(np.median(a[:, 1]))} | {tc:.1f} | {tr:.1f} | "
          f"{'col (push)' if tc < tr else 'row (pull)'} |")
print(json.dumps({str(k): np.array(v).tolist()[:50] for k, v in per_level.items()})[:2000])
assert bad == 0
