"""Multi-rank host logic on CPU: pp_partition tiling, the binding's block slicing
(block_rows: what each rank uploads), and the 1D-partitioned BFS algorithm (tests/dist_model.py:
the level structure of bfs.cu's multi-rank path -- owned-block push / pull, per-level exchange of
the owned frontier slices, replicated decision) run by world_size-2 gloo processes with a real
all_gather exchange, checked against the oracle (depths, direction trace) -- SURVEY.md 8e edge
cases: source in the last block / on a block boundary, n not a multiple of 1024*P, a rank with
nothing to discover, an isolated source.  The CUDA kernels themselves are checked against the
oracle for P = 1..8 by tests/test_gpu_dist.py (single-device team)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

pp = pytest.importorskip("paper_1804_03327_b200")


@pytest.mark.parametrize("n", [1, 31, 1000, 1024, 1025, 5000, 65536, 4194304, 67108864])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_tiles_and_aligns(n, P):
    prev = 0
    for r in range(P):
        lo, hi = pp.pp_partition(n, r, P)
        assert lo == prev and lo <= hi <= n
        assert lo % 1024 == 0 or lo == n
        assert hi % 1024 == 0 or hi == n
        prev = hi
    assert prev == n
    # equal blocks of ceil(ceil(n/32)/32/P)*1024 vertices; only the tail is short
    sizes = [pp.pp_partition(n, r, P)[1] - pp.pp_partition(n, r, P)[0] for r in range(P)]
    full = sizes[0]
    assert all(a >= b for a, b in zip(sizes, sizes[1:]))            # full..., partial, 0...
    assert sum(1 for sz in sizes if 0 < sz < full) <= 1
    assert full - n / P < 1024 + 1


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_block_rows_tile_the_graph(P):
    """The rows each rank uploads (row-local offsets + global ids) reassemble the graph."""
    for g in (synth.rmat(10, 8, seed=3), synth.random_graph(3001, 9000, seed=2, symmetrize=False),
              synth.from_edges(40, [1], [2])):
        offs, ids = [], []
        for r in range(P):
            lo, hi = pp.pp_partition(g.n, r, P)
            boff, bidx = pp.block_rows(g.off, g.idx, lo, hi)
            assert boff.dtype == np.int64 and bidx.dtype == np.uint32
            assert len(boff) == hi - lo + 1 and boff[0] == 0 and boff[-1] == len(bidx)
            offs.append(boff[1:] + (sum(len(x) for x in ids)))
            ids.append(bidx)
        full_off = np.concatenate([[0]] + offs)
        assert np.array_equal(full_off, g.off)
        assert np.array_equal(np.concatenate(ids), g.idx)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    try:
        out = []
        for name, g, s, mode in cases:
            lo, hi = pp.pp_partition(g.n, rank, world)
            # every rank's slice is padded to the same chunk (like ncclAllGather counts)
            chunk = max(pp.pp_partition(g.n, r, world)[1] - pp.pp_partition(g.n, r, world)[0]
                        for r in range(world))
            chunk = max(chunk, 1)

            def allgather_bool(own):
                t = torch.zeros(chunk, dtype=torch.uint8)
                t[:len(own)] = torch.from_numpy(own.astype(np.uint8))
                parts = [torch.zeros(chunk, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, t)
                full = np.zeros(g.n, bool)
                for r in range(world):
                    l2, h2 = pp.pp_partition(g.n, r, world)
                    full[l2:h2] = parts[r][:h2 - l2].numpy().astype(bool)
                return full

            from dist_model import dist_bfs_model
            depth, dirs, cs = dist_bfs_model(g, s, rank, world, lo, hi, allgather_bool, mode=mode)
            out.append((name, lo, hi, depth, dirs, cs))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partitioned_bfs_matches_oracle():
    cases = []
    g1 = synth.rmat(11, 8, seed=4)                        # n = 2048 -> 1024-vertex blocks
    srcs = synth.sources(g1, 3, seed=1)
    cases += [("rmat", g1, int(s), oracle.MODE_DO) for s in srcs]
    cases.append(("rmat_last_block", g1, int(np.nonzero(np.diff(g1.off)[1024:] > 0)[0][0] + 1024),
                  oracle.MODE_DO))
    cases.append(("rmat_boundary", g1, 1024 if np.diff(g1.off)[1024] > 0 else 1025, oracle.MODE_DO))
    cases.append(("rmat_pull_only", g1, int(srcs[0]), oracle.MODE_PULL_ONLY))
    g2 = synth.grid(30, 41)                               # n = 1230: not a multiple of 2048
    cases += [("grid", g2, 0, oracle.MODE_DO), ("grid_far", g2, 1229, oracle.MODE_PUSH_ONLY)]
    g3 = synth.from_edges(3000, [1, 2, 2500], [2, 3, 2600])  # isolated source, idle rank
    cases.append(("isolated", g3, 0, oracle.MODE_DO))
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for k, (name, g, s, mode) in enumerate(cases):
        exp, L = oracle.bfs(g, s)
        t = oracle.trace(g, g, exp, mode=mode)
        full = np.zeros(g.n, np.int32)
        for r in range(world):
            nm, lo, hi, depth, dirs, cs = results[r][k]
            full[lo:hi] = depth
            assert np.array_equal(dirs, t["dir"]), (name, r)   # identical decisions on all ranks
            assert np.array_equal(cs, t["c"]), (name, r)
        assert np.array_equal(full, exp), name
