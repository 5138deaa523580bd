"""GPU: the one-process-per-GPU multi-rank path with TWO processes:
CUDA IPC mapping of the peers' exchange buffers, cross-process peer stores and release/acquire
flags, per-process cooperative launches, the final rendezvous.  This pool has one GPU, so both
processes use device 0 (the driver time-slices their kernels; every cross-rank wait is bounded
by the 4 s device watchdog).  NCCL refuses two ranks on one device, so the records are
exchanged by the external bootstrap (pp_graph_export / pp_graph_import) over gloo.  Depths and
min-id parents of the concatenated block slices and the global trace must equal the oracle's."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
pp = pytest.importorskip("paper_1804_03327_b200")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases():
    return [("rmat_s12", synth.rmat(12, 8, seed=5)), ("grid_37x53", synth.grid(37, 53)),
            ("directed", synth.random_graph(2500, 9000, seed=3, symmetrize=False))]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        ctx = pp.DistContext(0, rank, world, None)
        out = []
        for name, g in _cases():
            gT = g if g.symmetric else synth.transpose(g)
            G = pp.Graph.from_csr(ctx, g, None if g.symmetric else gT, validate=True)
            recs = [None] * world
            dist.all_gather_object(recs, G.export())
            G.import_peers(recs)
            lo, hi = G.partition()
            res = []
            for s in [int(x) for x in synth.sources(g, 3, seed=3)]:
                d = torch.full((max(hi - lo, 1),), -5, dtype=torch.int32, device="cuda")
                p = torch.full((max(hi - lo, 1),), -5, dtype=torch.int32, device="cuda")
                st = pp.bfs(G, s, d, p, stats_capacity=g.n + 1)
                torch.cuda.synchronize()
                res.append((s, d.cpu().numpy()[:hi - lo], p.cpu().numpy()[:hi - lo],
                            np.array(st["dir"]), np.array(st["c"])))
            out.append((name, lo, hi, res))
            dist.barrier()
            G.close()
        q.put((rank, out, None))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_processes_ipc_bit_exact():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=600)
        assert err is None, (rank, err)
        results[rank] = out
    for p in procs:
        p.join(timeout=120)
    for k, (name, g) in enumerate(_cases()):
        gT = g if g.symmetric else synth.transpose(g)
        for j in range(3):
            s = results[0][k][3][j][0]
            exp, L = oracle.bfs(g, s)
            par = oracle.parents(gT, exp, s)
            t = oracle.trace(g, gT, exp)
            d = np.concatenate([results[r][k][3][j][1] for r in range(world)])
            p = np.concatenate([results[r][k][3][j][2] for r in range(world)])
            assert np.array_equal(d, exp), (name, s)
            assert np.array_equal(p, par), (name, s)
            for r in range(world):
                assert np.array_equal(results[r][k][3][j][3], t["dir"]), (name, s, r)
                assert np.array_equal(results[r][k][3][j][4], t["c"]), (name, s, r)
