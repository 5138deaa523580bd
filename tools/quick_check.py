"""Fast parity check of a build variant (GPU): C1 depths + parents vs the oracle on plain and
relabelled uploads, and a 3-rank team.  Prints OK or raises."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1804_03327_b200 as pp  # noqa: E402

g = synth.make("C1")
ctx = pp.Context(0)
srcs = [int(s) for s in synth.sources(g, 12, seed=9)]
exps = {s: oracle.bfs(g, s)[0] for s in srcs}
key = synth.degree_order_key(g)
for relabel in (False, True):
    G = pp.Graph.from_csr(ctx, g, relabel=relabel)
    d = torch.empty(g.n, dtype=torch.int32, device="cuda")
    p = torch.empty(g.n, dtype=torch.int32, device="cuda")
    for s in srcs:
        for par in (None, p):
            pp.bfs(G, s, d, par)
            assert np.array_equal(d.cpu().numpy(), exps[s]), (relabel, s)
            if par is not None:
                want = oracle.parents(g, exps[s], s, key=key if relabel else None)
                assert np.array_equal(p.cpu().numpy(), want), (relabel, s, "parents")
team = pp.Team(3)
Gs = team.upload(g)
blocks = [pp.pp_partition(g.n, r, 3) for r in range(3)]
ds = [torch.empty(hi - lo, dtype=torch.int32, device="cuda") for lo, hi in blocks]
for s in srcs[:4]:
    pp.bfs_team(Gs, s, ds)
    assert np.array_equal(np.concatenate([x.cpu().numpy() for x in ds]), exps[s]), ("team", s)
print("quick_check OK")
