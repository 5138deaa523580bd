"""GPU parity: pp_mxv (row-based Alg. 2 / column-based Alg. 3 CUDA kernels) vs oracle O3.

Every descriptor combination (mask none/list/bitmap, complement, accumulate, replace,
direction push/pull/auto, early exit, transpose) and every vector format is compared
element by element with the definitional oracle on graphs whose sizes are not multiples
of 32 (ragged bitmap tails) and span many warp chunks; then config C3's mask-density
sweep at s16 in full and at s22 (the bench size) on all points."""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth
from pp_testutil import bits_from_dense, dense_from_bits

pytestmark = pytest.mark.gpu
pp = pytest.importorskip("paper_1804_03327_b200")


@pytest.fixture(scope="module")
def ctx():
    return pp.Context(0)


def dev_vec(v, fmt, extra_capacity=0):
    """Dense 0/1 numpy -> (pp_vector, backing tensor)."""
    n = len(v)
    if fmt == pp.PP_VEC_BITMAP:
        t = torch.from_numpy(bits_from_dense(v)).cuda()
        return pp.make_vector(fmt, n, t, int(v.sum())), t
    ids = np.nonzero(v)[0].astype(np.uint32)
    cap = max(len(ids) + extra_capacity, 1)
    t = torch.zeros(cap, dtype=torch.int32, device="cuda")
    if len(ids):
        t[:len(ids)] = torch.from_numpy(ids.view(np.int32)).cuda()
    return pp.make_vector(fmt, n, t, len(ids), cap), t


def read_vec(vec, t, n):
    torch.cuda.synchronize()
    if vec.format == pp.PP_VEC_BITMAP:
        return dense_from_bits(t.cpu().numpy(), n)
    ids = t.cpu().numpy().view(np.uint32)[:vec.nnz]
    assert np.all(np.diff(ids.astype(np.int64)) > 0), "LIST output must be sorted and unique"
    out = np.zeros(n, np.uint8)
    out[ids] = 1
    return out


def expected(g, gT, u, mask, complement, accum, replace, w_in, transpose):
    M = gT if transpose else g           # operator rows: A^T rows = CSC(A)
    return oracle.mxv(M, u, mask=mask, complement=complement, accum=accum, replace=replace,
                      w_in=w_in)


GRAPHS = {
    "rmat_s11": lambda: synth.rmat(11, 8, seed=3),
    "directed_1999": lambda: synth.random_graph(1999, 12000, seed=4, symmetrize=False),
    "star_1057": lambda: synth.from_edges(1057, np.zeros(1056, np.uint32), np.arange(1, 1057)),
    "tiny_5": lambda: synth.from_edges(5, [0, 1, 3], [1, 2, 4], symmetrize=False),
}


@pytest.mark.parametrize("relabel", [False, True])
@pytest.mark.parametrize("gname", sorted(GRAPHS))
def test_mxv_all_descriptor_combinations(ctx, gname, relabel):
    g = GRAPHS[gname]()
    gT = synth.transpose(g)
    G = pp.Graph.from_csr(ctx, g, None if g.symmetric else gT, validate=True, relabel=relabel)
    n = g.n
    rng = np.random.default_rng(len(gname))
    for trial in range(2):
        u = (rng.random(n) < [0.002, 0.3][trial]).astype(np.uint8)
        if not u.any():
            u[rng.integers(n)] = 1
        m = (rng.random(n) < 0.5).astype(np.uint8)
        w_in = (rng.random(n) < 0.4).astype(np.uint8)
        for (mask_fmt, complement, accum, replace, direction, ee, transpose, ufmt, wfmt) in \
                itertools.product([None, pp.PP_VEC_LIST, pp.PP_VEC_BITMAP], [0, 1], [0, 1], [1, 0],
                                  [pp.PP_DIR_PULL, pp.PP_DIR_PUSH, pp.PP_DIR_AUTO], [1, 0], [1, 0],
                                  [pp.PP_VEC_LIST, pp.PP_VEC_BITMAP],
                                  [pp.PP_VEC_BITMAP, pp.PP_VEC_LIST]):
            if mask_fmt is None and complement:
                continue
            if (direction == pp.PP_DIR_AUTO or not ee) and (accum or not replace) and trial:
                continue  # keep the product bounded; still covered in trial 0
            uvec, ut = dev_vec(u, ufmt)
            mvec, mt = (None, None) if mask_fmt is None else dev_vec(m, mask_fmt)
            wvec, wt = dev_vec(w_in, wfmt, extra_capacity=n)
            nnz = pp.mxv(G, wvec, uvec, mask=mvec, complement=complement, accum=accum,
                         replace=replace, direction=direction, early_exit=ee, transpose=transpose)
            got = read_vec(wvec, wt, n)
            exp = expected(g, gT, u, None if mask_fmt is None else m, complement, accum, replace,
                           w_in, transpose)
            assert np.array_equal(got, exp), (gname, mask_fmt, complement, accum, replace,
                                              direction, ee, transpose, ufmt, wfmt)
            assert nnz == int(exp.sum())


def test_mxv_errors(ctx):
    g = synth.rmat(8, 4, seed=1)
    G = pp.Graph.from_csr(ctx, g)
    u, ut = dev_vec(np.ones(g.n, np.uint8), pp.PP_VEC_BITMAP)
    w, wt = dev_vec(np.zeros(g.n, np.uint8), pp.PP_VEC_BITMAP)
    with pytest.raises(pp.PPError) as e:
        pp.mxv(G, w, u, mask=None, complement=True)
    assert e.value.status == pp.PP_ERR_ARG
    bad, bt = dev_vec(np.ones(g.n + 1, np.uint8), pp.PP_VEC_BITMAP)
    with pytest.raises(pp.PPError) as e:
        pp.mxv(G, w, bad)
    assert e.value.status == pp.PP_ERR_DIM
    d = pp.pp_descriptor_default()
    d.semiring = 3
    with pytest.raises(pp.PPError) as e:
        pp.pp_mxv(G.handle, w, d, u)
    assert e.value.status == pp.PP_ERR_UNSUPPORTED
    # LIST output too small reports the needed size
    small = torch.zeros(2, dtype=torch.int32, device="cuda")
    wl = pp.make_vector(pp.PP_VEC_LIST, g.n, small, 0, 2)
    with pytest.raises(pp.PPError) as e:
        pp.mxv(G, wl, u)
    assert e.value.status == pp.PP_ERR_DIM and wl.nnz > 2


def c3_points(n, seed=11):
    for rho in (0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.5, 1.0):
        yield rho, synth.dense_from_ids(n, synth.random_subset(n, int(round(rho * n)), seed))


@pytest.mark.parametrize("config", ["C1", "C3"])
def test_c3_mask_density_sweep(ctx, config):
    """Config C3 protocol: masked (early exit on/off) vs unmasked pull over
    mask densities 0.1%..100%, u = all-ones (Fig. 2 protocol P:138) and random 1%."""
    g = synth.make("C1") if config == "C1" else synth.make("C3")
    G = pp.Graph.from_csr(ctx, g)
    n = g.n
    rng = np.random.default_rng(3)
    for uname, u in (("ones", np.ones(n, np.uint8)), ("rand1pct", (rng.random(n) < 0.01).astype(np.uint8))):
        uvec, ut = dev_vec(u, pp.PP_VEC_BITMAP)
        t_full = expected(g, g, u, None, 0, 0, 1, None, 1)
        wvec, wt = dev_vec(np.zeros(n, np.uint8), pp.PP_VEC_BITMAP)
        pp.mxv(G, wvec, uvec, direction=pp.PP_DIR_PULL, early_exit=False)
        assert np.array_equal(read_vec(wvec, wt, n), t_full)          # unmasked row mxv
        for rho, m in c3_points(n):
            mvec, mt = dev_vec(m, pp.PP_VEC_BITMAP)
            for ee in (1, 0):
                pp.mxv(G, wvec, uvec, mask=mvec, direction=pp.PP_DIR_PULL, early_exit=ee)
                got = read_vec(wvec, wt, n)
                assert np.array_equal(got, expected(g, g, u, m, 0, 0, 1, None, 1)), (uname, rho, ee)


@pytest.mark.parametrize("direction", [pp.PP_DIR_PUSH, pp.PP_DIR_PULL])
def test_mxv_bad_list_rejected_in_both_directions(ctx, direction):
    """A LIST u holding an id >= n, a duplicate or an unsorted pair is PP_ERR_RANGE whichever
    kernel the direction selects (results never depend on the direction, R25)."""
    g = synth.rmat(10, 8, seed=2)
    G = pp.Graph.from_csr(ctx, g)
    out = torch.zeros((g.n + 31) // 32, dtype=torch.int32, device="cuda")
    for ids in ([3, g.n], [5, 5], [9, 4]):
        t = torch.tensor(np.array(ids, np.uint32).view(np.int32), device="cuda")
        uvec = pp.make_vector(pp.PP_VEC_LIST, g.n, t, len(ids), len(ids))
        wvec = pp.make_vector(pp.PP_VEC_BITMAP, g.n, out, 0)
        with pytest.raises(pp.PPError) as e:
            pp.mxv(G, wvec, uvec, direction=direction)
        assert e.value.status == pp.PP_ERR_RANGE, ids
    # an input list whose nnz exceeds its capacity is a dimension error
    t = torch.zeros(4, dtype=torch.int32, device="cuda")
    uvec = pp.make_vector(pp.PP_VEC_LIST, g.n, t, 5, 4)
    with pytest.raises(pp.PPError) as e:
        pp.mxv(G, pp.make_vector(pp.PP_VEC_BITMAP, g.n, out, 0), uvec)
    assert e.value.status == pp.PP_ERR_DIM
