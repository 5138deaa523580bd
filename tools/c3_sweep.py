"""Config C3: masked vs unmasked row-based (pull) mxv over mask density on RMAT s22 ef16.

For each density rho the mask is exactly round(rho*n) rows sampled without replacement
(seeded); u = all ones (Fig. 2 protocol) or a random 1% vector.  Arms: masked with
early exit, masked without early exit, unmasked (no mask, no early exit = Eq. 2 row mxv).
Times are CUDA events around pp_mxv on the ctx stream (want_nnz=0: no host sync inside),
median of R runs, L2 flushed before each run.  Algorithmic bytes:
  unmasked: 4(n+1) offsets + 4 nnz ids + n/8 u-words read... (see model()).
Prints one JSON line per point; --out writes them to a file."""
import argparse, json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default=None)
ap.add_argument("--relabel", action="store_true", help="upload with PP_GRAPH_RELABEL (degree order)")
ap.add_argument("--unmasked-only", action="store_true", help="only the unmasked arm, u = ones (ncu)")
args = ap.parse_args()

g = synth.make(args.config)
n, nnz = g.n, g.nnz
deg = np.diff(g.off)
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g, relabel=args.relabel)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
nw = (n + 31) // 32
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]


def bits(v):
    pad = np.zeros(nw * 32, np.uint8)
    pad[:n] = v
    return torch.from_numpy(np.packbits(pad, bitorder="little").view("<u4").astype(np.uint32).view(np.int32)).cuda()


def scanned_first_hit(u):
    """per row: ids scanned until the first j with u(j)=1 (or the degree)."""
    rows = np.repeat(np.arange(n), deg)
    hit = u[g.idx] != 0
    pos = np.arange(nnz) - g.off[rows]
    first = np.full(n, np.iinfo(np.int64).max)
    np.minimum.at(first, rows[hit], pos[hit])
    return np.where(first < np.iinfo(np.int64).max, first + 1, deg)


def timeit(fn):
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


out_lines = []
rng = np.random.default_rng(3)
wt = torch.zeros(nw, dtype=torch.int32, device="cuda")
w = pp.make_vector(pp.PP_VEC_BITMAP, n, wt, 0)
for uname, u in (("ones", np.ones(n, np.uint8)), ("rand1pct", (rng.random(n) < 0.01).astype(np.uint8))):
    ub = bits(u)
    uvec = pp.make_vector(pp.PP_VEC_BITMAP, n, ub, int(u.sum()))
    sc = scanned_first_hit(u)
    # unmasked arm: every row, every id (Eq. 2)
    t = timeit(lambda: pp.mxv(G, w, uvec, direction=pp.PP_DIR_PULL, early_exit=False, want_nnz=False))
    by = 4 * (n + 1) + 4 * nnz + n // 8 + n // 8
    line = dict(config=args.config, u=uname, arm="unmasked", rho=1.0, us=t * 1e6, bytes=by,
                gbs=by / t / 1e9, frac=by / t / 1e9 / peak)
    line["relabel"] = args.relabel
    print(json.dumps(line), flush=True); out_lines.append(line)
    if args.unmasked_only:
        break
    for rho in (0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.5, 1.0):
        ids = synth.random_subset(n, int(round(rho * n)), 11)
        m = synth.dense_from_ids(n, ids)
        mb = bits(m)
        mvec = pp.make_vector(pp.PP_VEC_BITMAP, n, mb, len(ids))
        for ee in (1, 0):
            t = timeit(lambda: pp.mxv(G, w, uvec, mask=mvec, direction=pp.PP_DIR_PULL, early_exit=ee,
                                      want_nnz=False))
            scanned = sc[ids].sum() if ee else deg[ids].sum()
            by = n // 8 + n // 8 + 8 * len(ids) + 4 * int(scanned)
            line = dict(config=args.config, u=uname, arm="masked_ee" if ee else "masked", rho=rho,
                        rows=len(ids), us=t * 1e6, bytes=by, gbs=by / t / 1e9, frac=by / t / 1e9 / peak)
            print(json.dumps(line), flush=True); out_lines.append(line)
if args.out:
    with open(args.out, "w") as f:
        for l in out_lines:
            f.write(json.dumps(l) + "\n")
