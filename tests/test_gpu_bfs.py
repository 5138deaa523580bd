"""GPU parity: pp_bfs (persistent CUDA kernel through the C ABI) vs the CPU oracle.

Depths bit-exact vs O1; parents bit-exact vs O2 (canonical min-id) and valid under O5;
per-level stats (direction, c, m_f, m_u) bit-exact vs O4.  Sizes span several warp
chunks and ragged tails; full-size C2/C4 graphs are checked on sampled sources."""
import numpy as np
import pytest
import torch

import oracle
import synth
from stats_defs import check_cand

pytestmark = pytest.mark.gpu

pp = pytest.importorskip("paper_1804_03327_b200")

MODES = [(pp.PP_MODE_DO, pp.PP_HEUR_EDGES), (pp.PP_MODE_DO, pp.PP_HEUR_PAPER_R),
         (pp.PP_MODE_PUSH_ONLY, pp.PP_HEUR_EDGES), (pp.PP_MODE_PULL_ONLY, pp.PP_HEUR_EDGES)]
ORACLE_MODE = {pp.PP_MODE_DO: oracle.MODE_DO, pp.PP_MODE_PUSH_ONLY: oracle.MODE_PUSH_ONLY,
               pp.PP_MODE_PULL_ONLY: oracle.MODE_PULL_ONLY}


@pytest.fixture(scope="module")
def ctx():
    return pp.Context(0)


def run_bfs(ctx, G, s, mode, rule, toggles=0, parents=True):
    dev = torch.device("cuda", 0)
    depth = torch.full((G.n,), -7, dtype=torch.int32, device=dev)
    parent = torch.full((G.n,), -7, dtype=torch.int32, device=dev) if parents else None
    st = pp.bfs(G, int(s), depth, parent, heuristic=rule, mode=mode, toggles=toggles,
                stats_capacity=min(G.n + 2, 70000))
    torch.cuda.synchronize()
    return depth.cpu().numpy(), (parent.cpu().numpy() if parents else None), st


def check(ctx, g, gT, G, s, mode, rule, toggles=0, parents=True, exp=None):
    d, par, st = run_bfs(ctx, G, s, mode, rule, toggles, parents)
    ed, L = exp if exp is not None else oracle.bfs(g, s)
    assert np.array_equal(d, ed), f"depth mismatch src={s} mode={mode} rule={rule} t={toggles}: " \
        f"{np.nonzero(d != ed)[0][:10]}"
    if parents:
        # relabelled graphs: the valid parent first in the degree order (R14)
        key = synth.degree_order_key(g, gT) if getattr(G, "relabel", False) else None
        ep = oracle.parents(gT, ed, s, key=key)
        assert np.array_equal(par, ep), f"parent mismatch at {np.nonzero(par != ep)[0][:10]}"
    t = oracle.trace(g, gT, ed, mode=ORACLE_MODE[mode], rule=rule)
    assert st["levels"] == t["levels"] == L
    assert st["reached"] == int((ed > 0).sum())
    assert np.array_equal(st["dir"], t["dir"]), (st["dir"], t["dir"])
    assert np.array_equal(st["c"], t["c"])
    assert np.array_equal(st["m_f"], t["m_f"])
    assert np.array_equal(st["m_u"], t["m_u"])
    check_cand(g, gT, ed, st, no_mask=bool(toggles & pp.PP_OPT_NO_MASKING))
    return st


def small_graphs():
    out = {}
    out["diamond_directed"] = synth.from_edges(4, [0, 0, 1, 2], [1, 2, 3, 3], symmetrize=False)
    e = [(0, 1), (0, 2), (0, 3), (1, 4), (2, 4), (2, 5), (3, 5), (4, 6), (5, 7), (6, 7)]
    out["paper_fig3"] = synth.from_edges(8, [a for a, _ in e], [b for _, b in e])
    n = 700
    out["path"] = synth.from_edges(n, np.arange(n - 1), np.arange(1, n))
    out["star"] = synth.from_edges(3000, np.zeros(2999, np.uint32), np.arange(1, 3000))
    src, dst = np.nonzero(~np.eye(70, dtype=bool))
    out["complete70"] = synth.from_edges(70, src, dst)
    out["grid_37x53"] = synth.grid(37, 53)
    out["disconnected"] = synth.from_edges(100, [1, 2, 3, 50, 51], [2, 3, 4, 51, 52])
    out["directed_random"] = synth.random_graph(2500, 9000, seed=3, symmetrize=False)
    out["rmat_s12"] = synth.rmat(12, 8, seed=5)
    out["pgrid"] = synth.percolated_grid(60, 60, 0.6, seed=2)
    out["rgg_s13"] = synth.rgg(13, 0.55, seed=4)  # random geometric graph (NEXT-2 shape)
    return out


SMALL = small_graphs()


def upload(ctx, g, relabel=False):
    if g.symmetric:
        return pp.Graph.from_csr(ctx, g, validate=True, relabel=relabel), g
    gT = synth.transpose(g)
    return pp.Graph.from_csr(ctx, g, gT, validate=True, relabel=relabel), gT


@pytest.mark.parametrize("relabel", [False, True])
@pytest.mark.parametrize("name", sorted(SMALL))
def test_small_graphs_all_modes(ctx, name, relabel):
    g = SMALL[name]
    G, gT = upload(ctx, g, relabel)
    deg = np.diff(g.off)
    srcs = sorted(set([0, g.n - 1, int(np.argmax(deg))] + list(range(0, g.n, max(1, g.n // 5)))))
    for s in srcs:
        exp = oracle.bfs(g, s)
        for mode, rule in MODES:
            check(ctx, g, gT, G, s, mode, rule, exp=exp)


@pytest.mark.parametrize("relabel", [False, True])
@pytest.mark.parametrize("toggles", [pp.PP_OPT_NO_EARLYEXIT, pp.PP_OPT_NO_MASKING, pp.PP_OPT_NO_REUSE,
                                     7])
def test_toggles_do_not_change_results(ctx, toggles, relabel):
    for name in ("rmat_s12", "directed_random", "path", "paper_fig3"):
        g = SMALL[name]
        G, gT = upload(ctx, g, relabel)
        for s in synth.sources(g, 4, seed=9):
            exp = oracle.bfs(g, s)
            for mode, rule in MODES:
                check(ctx, g, gT, G, s, mode, rule, toggles=toggles, exp=exp)


@pytest.mark.parametrize("relabel", [False, True])
@pytest.mark.parametrize("toggles", [pp.PP_OPT_NO_EARLYEXIT, 7])
def test_no_early_exit_long_rows_grid_wide(ctx, toggles, relabel):
    """C1 has rows up to 9,722 ids: without early exit the pull hands remainders longer than
    2,048 ids to grid-wide chunks (pull_hub_chunks); depths, min-id parents and the
    direction trace must stay bit-exact."""
    g = synth.make("C1")
    G, gT = upload(ctx, g, relabel)
    for s in synth.sources(g, 6, seed=4):
        exp = oracle.bfs(g, s)
        for mode, rule in ((pp.PP_MODE_DO, pp.PP_HEUR_EDGES), (pp.PP_MODE_PULL_ONLY, pp.PP_HEUR_EDGES)):
            check(ctx, g, gT, G, s, mode, rule, toggles=toggles, exp=exp)


@pytest.mark.parametrize("narrow", ["1", "0"])
def test_narrow_cluster_start_and_handover(ctx, narrow, monkeypatch):
    """Narrow mode (one 8-CTA thread-block cluster runs init and the small levels, then hands
    the loop state to the whole-grid launch): PP_NARROW=1 forces it on every graph, so RMAT
    sources hand over after 1-3 levels and the grid / path run narrow to the end; results
    must be bit-exact either way (depths, min-id parents, direction trace)."""
    monkeypatch.setenv("PP_NARROW", narrow)
    graphs = [synth.make("C1"), synth.grid(64, 64), SMALL["path"], SMALL["disconnected"],
              SMALL["directed_random"]]
    for g in graphs:
        for relabel in (False, True):
            G, gT = upload(ctx, g, relabel)
            for s in list(synth.sources(g, 3, seed=5)) + [0]:
                exp = oracle.bfs(g, s)
                for mode, rule in MODES:
                    check(ctx, g, gT, G, s, mode, rule, exp=exp)


def test_isolated_source(ctx):
    g = SMALL["disconnected"]
    G, gT = upload(ctx, g)
    for mode, rule in MODES:
        st = check(ctx, g, gT, G, 0, mode, rule)
        assert st["levels"] == 1 and st["reached"] == 1


@pytest.mark.parametrize("relabel", [False, True])
def test_c1_rmat_s16_64_sources(ctx, relabel):
    """Config C1: RMAT s16 ef16, 64 seeded sources, 4 direction policies, bit-exact."""
    g = synth.make("C1")
    G = pp.Graph.from_csr(ctx, g, validate=True, relabel=relabel)
    for s in synth.sources(g, 64, seed=2):
        exp = oracle.bfs(g, s)
        for mode, rule in MODES:
            check(ctx, g, g, G, s, mode, rule, exp=exp)


def test_host_depth_pointer_matches_device(ctx):
    g = SMALL["rmat_s12"]
    G, gT = upload(ctx, g)
    s = int(synth.sources(g, 1)[0])
    hd = np.full(g.n, -3, np.int32)
    hp = np.full(g.n, -3, np.int32)
    pp.bfs(G, s, hd, hp)
    d, par, _ = run_bfs(ctx, G, s, pp.PP_MODE_DO, pp.PP_HEUR_EDGES)
    assert np.array_equal(hd, d) and np.array_equal(hp, par)


def test_repeatable_bit_identical(ctx):
    g = SMALL["rmat_s12"]
    G, gT = upload(ctx, g)
    s = int(synth.sources(g, 1, seed=4)[0])
    a = run_bfs(ctx, G, s, pp.PP_MODE_DO, pp.PP_HEUR_EDGES)
    for _ in range(5):
        b = run_bfs(ctx, G, s, pp.PP_MODE_DO, pp.PP_HEUR_EDGES)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_errors(ctx):
    g = SMALL["grid_37x53"]
    G, _ = upload(ctx, g)
    d = torch.zeros(g.n, dtype=torch.int32, device="cuda")
    with pytest.raises(pp.PPError) as e:
        pp.bfs(G, g.n, d)
    assert e.value.status == pp.PP_ERR_RANGE
    bad = synth.grid(4, 4)
    idx = bad.idx.copy()
    idx[5] = 99
    with pytest.raises(pp.PPError) as e:
        pp.Graph(ctx, bad.n, bad.off, idx, validate=True)
    assert e.value.status == pp.PP_ERR_GRAPH and "row" in str(e.value)
    idx = bad.idx.copy()
    idx[0], idx[1] = idx[1], idx[0]
    with pytest.raises(pp.PPError) as e:
        pp.Graph(ctx, bad.n, bad.off, idx, validate=True)
    assert e.value.status == pp.PP_ERR_GRAPH


@pytest.fixture(scope="module")
def c2g():
    return synth.make("C2")


@pytest.mark.parametrize("relabel", [True, False])
def test_c2_rmat_s22_sampled_sources(ctx, c2g, relabel):
    """Config C2 at full size (relabel=True is the bench's launch configuration): oracle on
    3 sources, Graph500 validation (O5) + stats vs O4 on 8 more."""
    g = c2g
    G = pp.Graph.from_csr(ctx, g, relabel=relabel)
    srcs = synth.sources(g, 11, seed=2)
    for k, s in enumerate(srcs):
        if k < 3:
            exp = oracle.bfs(g, s)
            check(ctx, g, g, G, s, pp.PP_MODE_DO, pp.PP_HEUR_EDGES, exp=exp)
        else:
            d, par, st = run_bfs(ctx, G, s, pp.PP_MODE_DO, pp.PP_HEUR_EDGES)
            oracle.validate_graph500(g, s, d, par)
            t = oracle.trace(g, g, d)
            assert np.array_equal(st["dir"], t["dir"]) and np.array_equal(st["c"], t["c"])
    # the paper rule and forced directions reach the same depths
    s = srcs[0]
    exp = oracle.bfs(g, s)
    for mode, rule in MODES[1:]:
        check(ctx, g, g, G, s, mode, rule, exp=exp)
    G.close()


def test_c4_grid_closed_form(ctx):
    """Config C4: 4096^2 grid, depth = Manhattan distance + 1, every level push."""
    R = C = 4096
    g = synth.grid(R, C)
    G = pp.Graph.from_csr(ctx, g)
    y, x = np.divmod(np.arange(R * C, dtype=np.int64), C)
    for (sy, sx) in [(0, 0), (2048, 2048), (4095, 17)]:
        s = sy * C + sx
        exp = (np.abs(y - sy) + np.abs(x - sx) + 1).astype(np.int32)
        for mode, rule in [(pp.PP_MODE_DO, pp.PP_HEUR_EDGES), (pp.PP_MODE_DO, pp.PP_HEUR_PAPER_R)]:
            d, par, st = run_bfs(ctx, G, s, mode, rule, parents=(sx == 0))
            assert np.array_equal(d, exp)
            assert st["levels"] == int(exp.max()) and not st["dir"].any()
            if par is not None:
                oracle.validate_graph500(g, s, d, par)


def test_debug_times_and_level_ns(ctx):
    """pp_bfs_debug_times records per-level, per-CTA phase times; stats carry level ns."""
    g = synth.rmat(14, 16, seed=2)
    G = pp.Graph.from_csr(ctx, g)
    nct = pp.pp_bfs_debug_times(G.handle, 16)
    assert nct >= 1
    d = torch.zeros(g.n, dtype=torch.int32, device="cuda")
    s = int(synth.sources(g, 1, seed=8)[0])
    st = pp.bfs(G, s, d, stats_capacity=64)
    t = pp.pp_bfs_debug_times(G.handle, 16, fetch=True)
    assert t.shape == (16, nct) and (t >= 0).all() and (t > 0).any()
    assert (st["ns"][:st["levels"]] > 0).all() and st["init_ns"] > 0
    exp, _ = oracle.bfs(g, s)
    assert np.array_equal(d.cpu().numpy(), exp)


@pytest.mark.parametrize("relabel", [False, True])
def test_debug_level_split_resumes_exactly(ctx, relabel):
    """pp_bfs_debug_level: levels 1..k-1 in one launch, level k alone in a second launch that
    resumes the handed-over loop state; depths up to k+1 must equal the oracle's."""
    g = synth.make("C1")
    G = pp.Graph.from_csr(ctx, g, relabel=relabel)
    d = torch.zeros(g.n, dtype=torch.int32, device="cuda")
    for s in synth.sources(g, 3, seed=4):
        exp, L = oracle.bfs(g, int(s))
        for k in range(1, L + 2):
            pp.pp_bfs_debug_level(G.handle, int(s), k, d.data_ptr())
            torch.cuda.synchronize()
            want = np.where((exp > 0) & (exp <= k + 1), exp, 0)
            assert np.array_equal(d.cpu().numpy(), want), (s, k)
