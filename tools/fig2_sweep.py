"""SURVEY NEXT-3, Fig. 2 on a synthetic analog: the four matvec variants of the
paper's microbenchmark, timed with CUDA events around pp_mxv (L2 flushed, median of R):
  (1) row-based, no mask, increase nnz(f)           PULL, no mask, no early exit (Eq. 2)
  (2) row-based masked, nnz(f) = M, increase nnz(m)  PULL, mask m, no early exit
  (3) col-based, increase nnz(f), no mask            PUSH, no mask (Eq. 3)
  (4) col-based masked, increase nnz(f), mask of      PUSH, mask m
      size 2/3 nnz(f)
Frontier / mask members are random, exactly round(rho*n) of them (seeded).  Every
point's output size is checked against the definitional oracle on the first config's three
smallest densities (oracle.mxv), and the table reports time, output nnz and the paper's
expectation: (1) flat, (2) and (3) grow with the density, (4) like (3).
Usage: python tools/fig2_sweep.py [CONFIG] [REPS]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1804_03327_b200 as pp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "K21"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
g = synth.make(cfg)
n, nnz = g.n, g.nnz
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g)
nw = (n + 31) // 32
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def bits(v):
    pad = np.zeros(nw * 32, np.uint8)
    pad[:n] = v
    return torch.from_numpy(np.packbits(pad, bitorder="little").view("<u4").astype(np.uint32)
                            .view(np.int32)).cuda()


def timeit(fn):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


wt = torch.zeros(nw, dtype=torch.int32, device="cuda")
w = pp.make_vector(pp.PP_VEC_BITMAP, n, wt, 0)
ones = np.ones(n, np.uint8)
onesb = bits(ones)
u_all = pp.make_vector(pp.PP_VEC_BITMAP, n, onesb, n)
print(f"{cfg}: n={n} nnz={nnz}; times in us (median of {reps}, L2 flushed)")
print("| rho | (1) row | (2) row masked | (3) col | (4) col masked (|m| = 2/3 |f|) | out nnz (1)/(2)/(3)/(4) |")
print("|---|---|---|---|---|---|")
rows = []
checked = 0
for rho in (0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.5, 1.0):
    k = int(round(rho * n))
    f = synth.dense_from_ids(n, synth.random_subset(n, k, 21))
    m = synth.dense_from_ids(n, synth.random_subset(n, k, 22))
    m23 = synth.dense_from_ids(n, synth.random_subset(n, int(round(2 * k / 3)), 23))
    fb, mb, m23b = bits(f), bits(m), bits(m23)
    fv = pp.make_vector(pp.PP_VEC_BITMAP, n, fb, int(f.sum()))
    mv = pp.make_vector(pp.PP_VEC_BITMAP, n, mb, int(m.sum()))
    m23v = pp.make_vector(pp.PP_VEC_BITMAP, n, m23b, int(m23.sum()))
    arms = [
        lambda: pp.mxv(G, w, fv, direction=pp.PP_DIR_PULL, early_exit=False, want_nnz=False),
        lambda: pp.mxv(G, w, u_all, mask=mv, direction=pp.PP_DIR_PULL, early_exit=False, want_nnz=False),
        lambda: pp.mxv(G, w, fv, direction=pp.PP_DIR_PUSH, want_nnz=False),
        lambda: pp.mxv(G, w, fv, mask=m23v, direction=pp.PP_DIR_PUSH, want_nnz=False),
    ]
    ts = [timeit(a) for a in arms]
    nz = []
    for a_u, a_m, a_dir in ((fv, None, pp.PP_DIR_PULL), (u_all, mv, pp.PP_DIR_PULL),
                            (fv, None, pp.PP_DIR_PUSH), (fv, m23v, pp.PP_DIR_PUSH)):
        nz.append(pp.mxv(G, w, a_u, mask=a_m, direction=a_dir, early_exit=False))
    if checked < 3:  # definitional oracle (Eq. 2 / Eq. 4) on the smallest densities
        exp = [oracle.mxv(g, f), oracle.mxv(g, ones, mask=m), oracle.mxv(g, f),
               oracle.mxv(g, f, mask=m23)]
        assert [int(e.sum()) for e in exp] == nz, (rho, nz, [int(e.sum()) for e in exp])
        checked += 1
    rows.append(dict(config=cfg, rho=rho, k=k, row_us=ts[0], row_masked_us=ts[1], col_us=ts[2],
                     col_masked_us=ts[3], out_nnz=nz))
    print(f"| {rho} | {ts[0]:.1f} | {ts[1]:.1f} | {ts[2]:.1f} | {ts[3]:.1f} | {'/'.join(map(str, nz))} |",
          flush=True)
print("oracle-checked points:", checked)
for r in rows:
    print(json.dumps(r))
