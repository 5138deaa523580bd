"""GPU parity of the multi-rank (1D row partition) BFS engine, SURVEY.md §8e / NEXT-1.

The multi-rank path is one persistent kernel per rank that exchanges each level's frontier
bitmap slice and counters by storing into the peers' exchange buffers, then cross-rank
release/acquire flags.  This box has one GPU, so the P ranks run as a
single-device team (pp_team_create / pp_bfs_team): P CTA groups of ONE cooperative launch
running the same kernel, the same peer stores and the same flags, with every peer's buffer on
the same device.  Each rank uploads only its block.  Depths (concatenated block slices), min-id
parents and the global direction trace (dir, c, m_f, m_u) must equal the oracle's, bit-exact,
for P in {1, 2, 3, 4, 8}, on RMAT, grids, a directed graph and the §8e edge cases: source in
the last block / on a block boundary, n not a multiple of 1024*P, idle ranks, an isolated
source, a hub whose neighbours span every block.  The one-process-per-GPU entry (NCCL
bootstrap of the peer mappings, pp_bfs) is exercised with a real one-rank communicator."""
import numpy as np
import pytest
import torch

import oracle
import synth
from stats_defs import check_cand

pytestmark = pytest.mark.gpu
pp = pytest.importorskip("paper_1804_03327_b200")


def _graphs():
    hub = synth.from_edges(5000, np.zeros(4999, np.uint32), np.arange(1, 5000, dtype=np.uint32))
    return {
        "C1": synth.make("C1"),
        "rmat_s12": synth.rmat(12, 8, seed=5),
        "grid_37x53": synth.grid(37, 53),                    # n = 1961: short last block
        "directed": synth.random_graph(2500, 9000, seed=3, symmetrize=False),
        "isolated_idle": synth.from_edges(3000, [1, 2, 2500], [2, 3, 2600]),
        "hub_star": hub,                                     # one row spans every block
    }


@pytest.fixture(scope="module")
def graphs():
    return _graphs()


def _sources(g, P):
    deg = np.diff(g.off)
    out = [int(s) for s in synth.sources(g, 3, seed=11)] if deg.any() else []
    lo, hi = pp.pp_partition(g.n, P - 1, P)
    last = [v for v in range(lo, hi) if deg[v] > 0]
    if last:
        out.append(last[len(last) // 2])                 # a source in the last block
    for r in range(1, P):                                # the first vertex of each block
        b, _ = pp.pp_partition(g.n, r, P)
        if b < g.n:
            out.append(b)
    out.append(0)
    return sorted(set(out))[:7]


def _run_team(team, Gs, g, s, mode, rule, parents=True):
    P = team.nranks
    blocks = [pp.pp_partition(g.n, r, P) for r in range(P)]
    depths = [torch.full((max(hi - lo, 1),), -7, dtype=torch.int32, device="cuda") for lo, hi in blocks]
    pars = [torch.full((max(hi - lo, 1),), -7, dtype=torch.int32, device="cuda") for lo, hi in blocks] \
        if parents else None
    st = pp.bfs_team(Gs, s, depths, pars, heuristic=rule, mode=mode, stats_capacity=g.n + 2)
    torch.cuda.synchronize()
    d = np.concatenate([depths[r].cpu().numpy()[:hi - lo] for r, (lo, hi) in enumerate(blocks)])
    p = None if not parents else \
        np.concatenate([pars[r].cpu().numpy()[:hi - lo] for r, (lo, hi) in enumerate(blocks)])
    return d, p, st


MODES = [(pp.PP_MODE_DO, pp.PP_HEUR_EDGES, oracle.MODE_DO),
         (pp.PP_MODE_DO, pp.PP_HEUR_PAPER_R, oracle.MODE_DO),
         (pp.PP_MODE_PULL_ONLY, pp.PP_HEUR_EDGES, oracle.MODE_PULL_ONLY),
         (pp.PP_MODE_PUSH_ONLY, pp.PP_HEUR_EDGES, oracle.MODE_PUSH_ONLY)]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name", ["C1", "rmat_s12", "grid_37x53", "directed", "isolated_idle",
                                  "hub_star"])
def test_team_matches_oracle(graphs, name, P):
    g = graphs[name]
    gT = g if g.symmetric else synth.transpose(g)
    team = pp.Team(P)
    Gs = team.upload(g, None if g.symmetric else gT, validate=True)
    for r, G in enumerate(Gs):
        assert G.partition() == pp.pp_partition(g.n, r, P)
    for s in _sources(g, P):
        exp, L = oracle.bfs(g, s)
        par_exp = oracle.parents(gT, exp, s)
        for mode, rule, om in MODES:
            d, p, st = _run_team(team, Gs, g, s, mode, rule)
            assert np.array_equal(d, exp), (name, P, s, mode, rule)
            assert np.array_equal(p, par_exp), (name, P, s, mode, rule)
            t = oracle.trace(g, gT, exp, mode=om, rule=rule)
            assert st["levels"] == L and st["reached"] == int((exp > 0).sum())
            assert np.array_equal(st["dir"], t["dir"]), (name, P, s, mode, rule, st["dir"], t["dir"])
            assert np.array_equal(st["c"], t["c"]) and np.array_equal(st["m_f"], t["m_f"])
            assert np.array_equal(st["m_u"], t["m_u"])
            check_cand(g, gT, exp, st)
    team.close()


@pytest.mark.parametrize("P", [2, 8])
def test_team_identical_trace_across_P_and_repeatable(graphs, P):
    """§8e: identical stats.dir and depths for P = 1 and P > 1; repeated BFS calls (flag epochs
    are monotone across calls) give bit-identical results."""
    g = graphs["C1"]
    t1 = pp.Team(1)
    G1 = t1.upload(g)
    tP = pp.Team(P)
    GP = tP.upload(g)
    for s in synth.sources(g, 4, seed=5):
        d1, p1, s1 = _run_team(t1, G1, g, int(s), pp.PP_MODE_DO, pp.PP_HEUR_EDGES)
        for _ in range(3):
            dP, pP, sP = _run_team(tP, GP, g, int(s), pp.PP_MODE_DO, pp.PP_HEUR_EDGES)
            assert np.array_equal(d1, dP) and np.array_equal(p1, pP)
            assert np.array_equal(s1["dir"], sP["dir"]) and np.array_equal(s1["c"], sP["c"])
    t1.close()
    tP.close()


def test_team_without_parents_and_off64(graphs):
    """Depth-only runs (the 16-byte init path) and the 64-bit offset layout of large blocks."""
    g = graphs["rmat_s12"]
    for off64 in (False, True):
        team = pp.Team(3)
        Gs = team.upload(g, off64=off64)
        for s in synth.sources(g, 3, seed=2):
            exp, _ = oracle.bfs(g, int(s))
            d, _, _ = _run_team(team, Gs, g, int(s), pp.PP_MODE_DO, pp.PP_HEUR_EDGES, parents=False)
            assert np.array_equal(d, exp), (off64, s)
        team.close()


def test_team_memory_is_partitioned(graphs):
    """Each rank stores its block (graph bytes ~ 1/P) plus O(n) replicated state."""
    g = graphs["C1"]
    b1 = pp.Team(1)
    g1 = b1.upload(g)
    bytes1 = g1[0].info()[2]
    b4 = pp.Team(4)
    g4 = b4.upload(g)
    nnz4 = [G.info()[1] for G in g4]
    assert sum(nnz4) == g.nnz                         # the blocks' in-edges tile the graph
    for G in g4:
        assert G.info()[2] < 0.5 * bytes1
    b1.close()
    b4.close()


def test_team_errors(graphs):
    g = graphs["grid_37x53"]
    team = pp.Team(2)
    Gs = team.upload(g)
    d = [torch.zeros(1024, dtype=torch.int32, device="cuda") for _ in range(2)]
    with pytest.raises(pp.PPError) as e:
        pp.bfs_team(Gs, g.n, d)
    assert e.value.status == pp.PP_ERR_RANGE
    with pytest.raises(pp.PPError) as e:            # ranks out of order
        pp.bfs_team([Gs[1], Gs[0]], 0, d)
    assert e.value.status == pp.PP_ERR_ARG
    with pytest.raises(pp.PPError) as e:            # a team graph is not a pp_bfs graph
        pp.bfs(Gs[0], 0, d[0])
    assert e.value.status == pp.PP_ERR_ARG
    # a block that is not pp_partition's
    with pytest.raises(pp.PPError) as e:
        pp.pp_graph_upload(team.ctxs[0].handle, g.n, 0, 7, 0, np.zeros(8, np.int64).ctypes.data,
                           None, None, None, pp.PP_GRAPH_SYMMETRIC)
    assert e.value.status == pp.PP_ERR_ARG
    team.close()


@pytest.fixture(scope="module")
def dctx():
    import torch.distributed  # noqa: F401  (makes sure libnccl.so.2 is loaded)
    return pp.DistContext(0, 0, 1, pp.pp_nccl_unique_id())


@pytest.mark.parametrize("name", ["rmat_s12", "grid_37x53", "directed", "C1"])
def test_dist_one_rank_nccl_bootstrap(graphs, dctx, name):
    """One process per GPU: pp_ctx_create_dist + collective upload (the NCCL all-gather of the
    IPC records) + pp_bfs, with a real one-rank communicator."""
    g = graphs[name]
    gT = g if g.symmetric else synth.transpose(g)
    G = pp.Graph.from_csr(dctx, g, None if g.symmetric else gT, validate=True)
    lo, hi = G.partition()
    assert (lo, hi) == (0, g.n)
    for s in list(synth.sources(g, 4, seed=3)) + [0]:
        exp, L = oracle.bfs(g, int(s))
        for mode, rule, om in MODES[:3]:
            d = torch.full((hi - lo,), -5, dtype=torch.int32, device="cuda")
            par = torch.full((hi - lo,), -5, dtype=torch.int32, device="cuda")
            st = pp.bfs(G, int(s), d, par, heuristic=rule, mode=mode, stats_capacity=g.n + 1)
            torch.cuda.synchronize()
            assert np.array_equal(d.cpu().numpy(), exp), (name, s, mode, rule)
            assert np.array_equal(par.cpu().numpy(), oracle.parents(gT, exp, int(s)))
            t = oracle.trace(g, gT, exp, mode=om, rule=rule)
            assert st["levels"] == L and np.array_equal(st["dir"], t["dir"])
            assert np.array_equal(st["c"], t["c"]) and np.array_equal(st["m_u"], t["m_u"])
    # host output buffers (end-to-end path) on the multi-rank entry
    hd = np.zeros(g.n, np.int32)
    s0 = int(synth.sources(g, 1, seed=3)[0])
    pp.bfs(G, s0, hd)
    assert np.array_equal(hd, oracle.bfs(g, s0)[0])


def test_dist_rejects_toggles_and_mxv(graphs, dctx):
    g = synth.grid(8, 8)
    G = pp.Graph.from_csr(dctx, g)
    d = torch.zeros(g.n, dtype=torch.int32, device="cuda")
    with pytest.raises(pp.PPError) as e:
        pp.bfs(G, 0, d, toggles=pp.PP_OPT_NO_EARLYEXIT)
    assert e.value.status == pp.PP_ERR_UNSUPPORTED
    w = torch.zeros(2, dtype=torch.int32, device="cuda")
    with pytest.raises(pp.PPError) as e:
        pp.mxv(G, pp.make_vector(pp.PP_VEC_BITMAP, g.n, w, 0), pp.make_vector(pp.PP_VEC_BITMAP, g.n, w, 0))
    assert e.value.status == pp.PP_ERR_UNSUPPORTED


def test_team_hybrid_exchange_bytes(graphs):
    """NEXT-1 hybrid encoding: after a push level whose discoveries are fewer than a rank's
    slice words the rank sends an id list instead of its bitmap slice, so a DO BFS stores
    fewer bytes into its peers than bitmap-every-level would ((P-1) x (slice + record) per
    level); results stay bit-exact (test_team_matches_oracle runs the same path)."""
    g = graphs["C1"]
    P = 4
    team = pp.Team(P)
    Gs = team.upload(g)
    lo0, hi0 = pp.pp_partition(g.n, 0, P)
    cw = (hi0 - lo0) // 32
    for s in synth.sources(g, 3, seed=8):
        d, _, st = _run_team(team, Gs, g, int(s), pp.PP_MODE_DO, pp.PP_HEUR_EDGES, parents=False)
        assert np.array_equal(d, oracle.bfs(g, int(s))[0])
        bitmap_only = st["levels"] * (P - 1) * (4 * cw + 40)
        assert 0 < st["exchanged_bytes"] < bitmap_only, (st["exchanged_bytes"], bitmap_only)
        # push-only: every level sends a list whenever it is shorter than the slice
        d, _, st2 = _run_team(team, Gs, g, int(s), pp.PP_MODE_PUSH_ONLY, pp.PP_HEUR_EDGES,
                              parents=False)
        assert np.array_equal(d, oracle.bfs(g, int(s))[0])
    team.close()
