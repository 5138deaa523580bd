"""GPU: the distributed (1D-partitioned, NCCL all-gather) BFS path of csrc/dist.cu through the
C ABI, with a real one-rank NCCL communicator (only one GPU is available to the test run).
Depths / parents bit-exact vs the oracle, direction trace vs O4 — i.e. identical to the
single-GPU engine.  The multi-rank exchange logic is covered on CPU by tests/test_dist.py."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
pp = pytest.importorskip("paper_1804_03327_b200")


@pytest.fixture(scope="module")
def dctx():
    import torch.distributed  # noqa: F401  (makes sure libnccl.so.2 is loaded)
    return pp.DistContext(0, 0, 1, pp.pp_nccl_unique_id())


GRAPHS = {
    "rmat_s12": lambda: synth.rmat(12, 8, seed=5),
    "grid": lambda: synth.grid(37, 53),
    "directed": lambda: synth.random_graph(2500, 9000, seed=3, symmetrize=False),
    "C1": lambda: synth.make("C1"),
}


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_dist_one_rank_matches_oracle(dctx, name):
    g = GRAPHS[name]()
    gT = synth.transpose(g) if not g.symmetric else g
    G = pp.Graph.from_csr(dctx, g, None if g.symmetric else gT, validate=True)
    lo, hi = G.partition()
    assert (lo, hi) == (0, g.n)
    for s in list(synth.sources(g, 6, seed=3)) + [0]:
        exp, L = oracle.bfs(g, int(s))
        for mode, rule, om in ((pp.PP_MODE_DO, pp.PP_HEUR_EDGES, oracle.MODE_DO),
                               (pp.PP_MODE_DO, pp.PP_HEUR_PAPER_R, oracle.MODE_DO),
                               (pp.PP_MODE_PULL_ONLY, pp.PP_HEUR_EDGES, oracle.MODE_PULL_ONLY)):
            d = torch.full((hi - lo,), -5, dtype=torch.int32, device="cuda")
            par = torch.full((hi - lo,), -5, dtype=torch.int32, device="cuda")
            st = pp.bfs(G, int(s), d, par, heuristic=rule, mode=mode, stats_capacity=g.n + 1)
            torch.cuda.synchronize()
            assert np.array_equal(d.cpu().numpy(), exp), (name, s, mode, rule)
            assert np.array_equal(par.cpu().numpy(), oracle.parents(gT, exp, int(s)))
            t = oracle.trace(g, gT, exp, mode=om, rule=rule)
            assert st["levels"] == L and np.array_equal(st["dir"], t["dir"])
            assert np.array_equal(st["c"], t["c"]) and np.array_equal(st["m_u"], t["m_u"])


def test_dist_rejects_toggles(dctx):
    g = synth.grid(8, 8)
    G = pp.Graph.from_csr(dctx, g)
    d = torch.zeros(g.n, dtype=torch.int32, device="cuda")
    with pytest.raises(pp.PPError) as e:
        pp.bfs(G, 0, d, toggles=pp.PP_OPT_NO_EARLYEXIT)
    assert e.value.status == pp.PP_ERR_UNSUPPORTED
