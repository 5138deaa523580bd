#!/usr/bin/env python
"""Benchmark: direction-optimised BFS GTEPS on RMAT scale 22 (BASELINE.json metric).

One step = one whole BFS (pp_bfs: every level of push / pull / convert / direction
switch, all in the library's CUDA kernels) from one seeded source over the resident
synthetic graph of config C2 (RMAT s22 ef16, Graph500 parameters).
TEPS follows the paper: nnz(A) / BFS time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

N > 1 (torchrun): one process per GPU.  Default --mode replicas: each rank traverses its
own sources on its own replica of the graph (independent problems, weak scaling, no
data-path collective).  --mode partitioned: one BFS at a time over the 1D row partition
(pp_ctx_create_dist; per-level ncclAllGather of the next-frontier bitmap), strong scaling.
Timing is the max over ranks.  --impl reference times the CPU oracle
(queue BFS, 1 core) on the same graph, sources, metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "DOBFS GTEPS on RMAT Scale 22 at 1/2/4/8 B200; achieved HBM GB/s fraction"
UNIT = "GTEPS"
FLUSH_BYTES = 256 << 20  # > 126 MB L2


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax = max(smax, float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[2:6]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def byte_model(torch, g_dev, depth, dirs, n, nnz, off_bytes, per_level=False):
    """Algorithmic HBM bytes of one BFS under DESIGN.md §6's model (byte-exact; the
    visited-bitmap probes are L2-resident and excluded).  Computed from the result
    (depth vector) and the level directions with torch ops on the graph's CSR."""
    off, idx, rows, deg, noniso = g_dev
    O = off_bytes
    d = depth.to(torch.int64)
    L = len(dirs)
    total = 4 * n + 2 * (n // 8)                       # init: depth, visited <- isolated
    parts = [total]                                      # per_level: [init, level 1, ...]
    cnt = torch.bincount(d, minlength=L + 2)
    outdeg_sum = torch.zeros(L + 2, dtype=torch.int64, device=d.device).index_add_(0, d, deg)
    dj = d[idx]                                          # depth of each edge's head
    for k in range(1, L + 1):                            # level k expands depth-k frontier
        before = total
        F = int(cnt[k])
        Fn = int(cnt[k + 1]) if k + 1 <= L + 1 else 0
        if dirs[k - 1] == 0:  # push
            m_in = int(outdeg_sum[k])
            total += F * (4 + 2 * O) + 4 * m_in + Fn * (4 + 4 + 2 * O)
        else:                 # pull: candidates unvisited at level start, scan to first hit
            cand = noniso & ((d == 0) | (d > k))
            hit = (dj >= 1) & (dj <= k)
            pos = torch.arange(nnz, device=d.device) - off[rows]
            first = torch.full((n,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=d.device)
            first.scatter_reduce_(0, rows[hit], pos[hit], reduce="amin")
            scanned = torch.where(first < torch.iinfo(torch.int64).max, first + 1, deg)
            S = int(scanned[cand].sum())
            C = int(cand.sum())
            total += 2 * (n // 8) + C * 2 * O + 4 * S + 4 * Fn
            if k < L and dirs[k] == 0:                 # pull -> push: convert
                total += 2 * (n // 8) + Fn * (4 + 2 * O)
        parts.append(total - before)
    return parts if per_level else total


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (textbook queue BFS, 1 core), same metric."""
    import oracle
    if rank != 0:
        return
    g = synth.make(args.config)
    srcs = synth.sources(g, max(args.steps + args.warmup, 1), seed=2)
    for k in range(args.warmup):
        oracle.bfs(g, srcs[k % len(srcs)])
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        oracle.bfs(g, srcs[(args.warmup + k) % len(srcs)])
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    val = g.nnz / (sum(times) / len(times)) / 1e9
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {g.name}, n={g.n}, nnz={g.nnz}, one BFS per step"},
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} full queue-BFS traversals of {g.name}"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--heuristic", default="edges", choices=["edges", "paper"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--model-sources", type=int, default=4)
    ap.add_argument("--mode", default="replicas", choices=["replicas", "partitioned"])
    ap.add_argument("--no-relabel", action="store_true",
                    help="upload without PP_GRAPH_RELABEL (caller vertex order)")
    args = ap.parse_args()
    rank, world, local = env_rank()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1804_03327_b200 as pp

    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    g = synth.make(args.config)
    partitioned = args.mode == "partitioned" and world > 1
    if partitioned:
        nid = [pp.pp_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        ctx = pp.DistContext(local, rank, world, nid[0])
    else:
        ctx = pp.Context(local)
    relabel = not args.no_relabel and not partitioned
    G = pp.Graph.from_csr(ctx, g, relabel=relabel)
    n, nnz = g.n, g.nnz
    lo, hi = G.partition() if partitioned else (0, n)
    off_bytes = 4 if nnz < 2**32 - 1 else 8
    heur = pp.PP_HEUR_EDGES if args.heuristic == "edges" else pp.PP_HEUR_PAPER_R
    all_src = synth.sources(g, 64, seed=2)
    def src(k):  # partitioned: every rank runs the same (collective) BFS
        return int(all_src[((0 if partitioned else rank) * 17 + k) % len(all_src)])

    depth = torch.empty(max(hi - lo, 1), dtype=torch.int32, device=dev)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for k in range(args.warmup):
        pp.bfs(G, src(k), depth, heuristic=heur)
    torch.cuda.synchronize()

    # ---- timed region: K BFS steps, L2 flushed between steps (flush not timed) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = ctx.launches()
    t_wall0 = time.perf_counter()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        pp.bfs(G, src(args.warmup + k), depth, heuristic=heur)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    launches = ctx.launches() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot_ms, op=dist.ReduceOp.MAX)
    tot_ms = float(tot_ms.item())
    ms_per_step = tot_ms / args.steps
    units = 1 if partitioned else world  # BFS traversals per step across the job
    value = units * args.steps * nnz / (tot_ms * 1e-3) / 1e9

    # ---- end to end through the public API: host output buffer, D2H inside the call ----
    host_depth = torch.empty(max(hi - lo, 1), dtype=torch.int32).pin_memory().numpy()
    for k in range(args.warmup):  # untimed: first call allocates the device staging buffer
        pp.bfs(G, src(k), host_depth, heuristic=heur)
    e2e_t = []
    for k in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pp.bfs(G, src(args.warmup + k), host_depth, heuristic=heur)   # syncs, copies back
        e2e_t.append(time.perf_counter() - t0)
    e2e_tot = torch.tensor([sum(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_tot, op=dist.ReduceOp.MAX)
    e2e_val = units * args.steps * nnz / float(e2e_tot.item()) / 1e9

    line = None
    if rank == 0:
        peak, peak_src = measured_peaks()
        nmod = 0 if partitioned else min(args.model_sources, args.steps)
        mb, mt = 0, 0.0
        if nmod:
            # ---- roofline of the dominant (only) kernel: bfs_persistent ----
            off_t = torch.from_numpy(g.off).to(dev)
            idx_t = torch.from_numpy(g.idx.astype(np.int64)).to(dev)
            deg_t = off_t[1:] - off_t[:-1]
            rows_t = torch.repeat_interleave(torch.arange(n, device=dev), deg_t)
            key_t = None
            if relabel:  # the layout the kernel scans: internal ids, rows in that order
                key_t = torch.from_numpy(synth.degree_order_key(g).astype(np.int64)).to(dev)
                e = torch.sort(key_t[rows_t] * n + key_t[idx_t]).values
                rows_t, idx_t = e // n, e % n
                deg_t = torch.bincount(rows_t, minlength=n)
                off_t = torch.zeros(n + 1, dtype=torch.int64, device=dev)
                off_t[1:] = torch.cumsum(deg_t, 0)
                del e
            noniso = deg_t > 0
            gd = (off_t, idx_t, rows_t, deg_t, noniso)
            for k in range(nmod):
                s = src(args.warmup + k)
                st = pp.bfs(G, s, depth, heuristic=heur, stats_capacity=4096)
                dm = depth
                if key_t is not None:
                    dm = torch.empty_like(depth)
                    dm[key_t] = depth
                mb += byte_model(torch, gd, dm, list(st["dir"]), n, nnz, off_bytes)
                mt += step_ms[k] * 1e-3
            del off_t, idx_t, rows_t, deg_t, noniso, gd
        achieved = mb / mt / 1e9 if mt > 0 else None
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"ncu_{args.config}.json")
        if os.path.exists(prof) and not partitioned:
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        # ---- CPU oracle baseline (bounded sample, 1 core) ----
        cpu = None
        if not args.no_cpu_baseline and not partitioned:
            import oracle
            os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
            ts, k = [], 0
            t_start = time.perf_counter()
            while (time.perf_counter() - t_start < 12.0 or k < 1) and k < 64:
                t0 = time.perf_counter()
                oracle.bfs(g, src(k))
                ts.append(time.perf_counter() - t0)
                k += 1
            cpu = {"value": nnz / (sum(ts) / len(ts)) / 1e9, "unit": UNIT, "cores": 1,
                   "kind": "oracle",
                   "sample": f"{len(ts)} full queue-BFS traversals of {g.name} (1 thread; "
                             f"host has {os.cpu_count()} cores)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {g.name} (Graph500 RMAT a,b,c=.57,.19,.19, "
                                   f"scrambled, symmetrised, dedup), n={n}, nnz={nnz}, one DO-BFS "
                                   f"per step from seeded sources",
                       "heuristic": args.heuristic, "relabel": relabel,
                       "l2": "flushed between steps (256 MiB write, "
                       "not timed)",
                       "parallelism": (f"1D row partition x{world} (NCCL allgather per level)"
                                       if partitioned else f"replicas x{world}")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "kernel": ("k_dist_push/k_dist_pull + ncclAllGather per level" if partitioned
                                    else "bfs_persistent (whole BFS in one cooperative launch)"),
                         "peak_source": peak_src,
                         "model": f"byte-exact DESIGN.md §6 over {nmod} sources: "
                                  f"{mb / max(1, nmod) / 1e6:.1f} MB/BFS"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8,
                    "d2h_bytes_per_step": 4 * (hi - lo),
                    "note": "pp_bfs with a pinned host depth buffer: launch + D2H copy of depth"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "wall_s_timed_region": t_wall,
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms),
                        "max": max(step_ms)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
