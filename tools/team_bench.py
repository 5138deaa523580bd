"""Multi-rank engine on one B200 as a single-device team: per P, the device
time of one partitioned BFS (CUDA events, L2 flushed between steps), per-level times of rank 0,
bytes resident per rank, and the single-GPU engine beside it.  The ranks share one GPU here, so
this measures the protocol's cost (3 rank-local barriers + a flag rendezvous per level, the
frontier-slice stores), not NVLink.  Usage: python tools/team_bench.py [CONFIG] [P,P,...] [K]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1804_03327_b200 as pp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
Ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8
g = synth.make(cfg)
srcs = [int(s) for s in synth.sources(g, K + 3, seed=2)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print(f"{cfg}: n={g.n} nnz={g.nnz}")
check = int(srcs[3])
exp = oracle.bfs(g, check)[0] if g.n <= (1 << 23) else None


def timeit(run):
    for s in srcs[:3]:
        run(s)
    torch.cuda.synchronize()
    ts = []
    for s in srcs[3:]:
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(s)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return ts


ctx = pp.Context(0)
for relabel in (False, True):
    G = pp.Graph.from_csr(ctx, g, relabel=relabel)
    d = torch.empty(g.n, dtype=torch.int32, device="cuda")
    ts = timeit(lambda s: pp.bfs(G, s, d))
    print(f"single-GPU engine (relabel={relabel}): {np.mean(ts):.3f} ms/BFS "
          f"= {g.nnz / np.mean(ts) / 1e6:.1f} GTEPS; bytes {G.info()[2] / 1e9:.2f} GB")
    G.close()
for P in Ps:
    team = pp.Team(P)
    t0 = time.time()
    Gs = team.upload(g)
    up = time.time() - t0
    blocks = [pp.pp_partition(g.n, r, P) for r in range(P)]
    ds = [torch.empty(max(hi - lo, 1), dtype=torch.int32, device="cuda") for lo, hi in blocks]
    ts = timeit(lambda s: pp.bfs_team(Gs, s, ds))
    st = pp.bfs_team(Gs, check, ds, stats_capacity=4096)
    if exp is not None:
        got = np.concatenate([ds[r].cpu().numpy()[:hi - lo] for r, (lo, hi) in enumerate(blocks)])
        assert np.array_equal(got, exp), "team depths differ from the oracle"
    lv = " ".join(f"{'HL'[x]}{t / 1e3:.1f}" for x, t in zip(st["dir"], st["ns"]))
    print(f"team P={P}: {np.mean(ts):.3f} ms/BFS = {g.nnz / np.mean(ts) / 1e6:.1f} GTEPS "
          f"(median {np.median(ts):.3f}); upload {up:.1f} s; bytes/rank "
          f"{max(G.info()[2] for G in Gs) / 1e9:.2f} GB; exchanged {st['exchanged_bytes'] / 1e6:.2f} MB "
          f"(rank 0; bitmap-every-level {st['levels'] * (P - 1) * (4 * ((blocks[0][1] - blocks[0][0]) // 32) + 40) / 1e6:.2f}); "
          f"init {st['init_ns'] / 1e3:.1f} us; "
          f"levels(us) {lv}" + ("; depths == oracle" if exp is not None else ""))
    for G in Gs:
        G.close()
    team.close()
