"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

Holds none of the method's arithmetic: only graph generation / preprocessing
(Sec. 7.1) in C (`gen.c`), seeded samplers for sources, vectors
and masks, and the workload recipes of BASELINE.json's configs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_SO = os.path.join(_HERE, "libsynth.so")


def build(force: bool = False) -> str:
    """Compile gen.c -> libsynth.so (gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _Graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("off", ctypes.POINTER(ctypes.c_int64)), ("idx", ctypes.POINTER(ctypes.c_uint32))]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        GP = ctypes.POINTER(_Graph)
        lib.synth_rmat.restype = GP
        lib.synth_rmat.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_double, ctypes.c_double]
        lib.synth_grid.restype = GP
        lib.synth_grid.argtypes = [ctypes.c_int64, ctypes.c_int64]
        lib.synth_percolated_grid.restype = GP
        lib.synth_percolated_grid.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                              ctypes.c_uint64]
        lib.synth_rgg.restype = GP
        lib.synth_rgg.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_uint64]
        lib.synth_from_edges.restype = GP
        lib.synth_from_edges.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        lib.synth_transpose.restype = GP
        lib.synth_transpose.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_free.argtypes = [GP]
        lib.synth_free.restype = None
        lib.synth_splitmix64.restype = ctypes.c_uint64
        lib.synth_splitmix64.argtypes = [ctypes.c_uint64]
        lib.synth_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass
class CSR:
    """Host CSR: int64 offsets (n+1), uint32 sorted unique column ids per row."""
    n: int
    off: np.ndarray
    idx: np.ndarray
    symmetric: bool = True
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.off[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.off)


def _take(gp, symmetric=True, name="") -> CSR:
    g = gp.contents
    n, nnz = int(g.n), int(g.nnz)
    off = np.ctypeslib.as_array(g.off, shape=(n + 1,)).copy()
    idx = np.ctypeslib.as_array(g.idx, shape=(max(nnz, 1),))[:nnz].copy() if nnz else np.zeros(0, np.uint32)
    _load().synth_free(gp)
    return CSR(n, off, idx, symmetric, name)


def rmat(scale: int, edgefactor: int, seed: int = 1, scramble: bool = True,
         a: float = 0.57, b: float = 0.19, c: float = 0.19) -> CSR:
    """Graph500-parameter RMAT, symmetrised, no self-loops/duplicates."""
    return _take(_load().synth_rmat(scale, edgefactor, seed, int(scramble), a, b, c),
                 True, f"rmat_s{scale}_ef{edgefactor}")


def grid(rows: int, cols: int) -> CSR:
    return _take(_load().synth_grid(rows, cols), True, f"grid_{rows}x{cols}")


def percolated_grid(rows: int, cols: int, p: float = 0.6, seed: int = 1) -> CSR:
    return _take(_load().synth_percolated_grid(rows, cols, p, seed), True,
                 f"pgrid_{rows}x{cols}_p{p}")


def rgg(scale: int, factor: float = 0.55, seed: int = 1) -> CSR:
    """Random geometric graph: 2^scale uniform points in the unit square, edges at distance
    <= factor*sqrt(ln n / n) (rgg_n_2_24_s0 shape)."""
    return _take(_load().synth_rgg(scale, factor, seed), True, f"rgg_s{scale}_f{factor}")


def from_edges(n: int, src, dst, symmetrize: bool = True, keep_self_loops: bool = False) -> CSR:
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    assert src.shape == dst.shape
    if len(src) and (int(src.max()) >= n or int(dst.max()) >= n):
        raise ValueError("edge endpoint out of range")
    g = _take(_load().synth_from_edges(n, len(src), src.ctypes.data, dst.ctypes.data,
                                       int(symmetrize), int(keep_self_loops)), symmetrize)
    if not symmetrize:
        g.symmetric = False
    return g


def transpose(g: CSR) -> CSR:
    off = np.ascontiguousarray(g.off, dtype=np.int64)
    idx = np.ascontiguousarray(g.idx, dtype=np.uint32)
    t = _take(_load().synth_transpose(g.n, off.ctypes.data, idx.ctypes.data), g.symmetric)
    t.name = g.name + "^T"
    return t


def splitmix64(x: int) -> int:
    return int(_load().synth_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def sources(g: CSR, count: int, seed: int = 2) -> np.ndarray:
    """`count` seeded sources, uniform over vertices with out-degree >= 1."""
    deg = g.degrees()
    if not np.any(deg > 0):
        return np.zeros(0, np.int64)
    out = []
    k = 0
    while len(out) < count:
        v = splitmix64(seed * 0x9E3779B97F4A7C15 + k) % g.n
        k += 1
        if deg[v] > 0:
            out.append(v)
    return np.array(out, dtype=np.int64)


def degree_order_key(g: CSR, gT: CSR = None) -> np.ndarray:
    """Position of every vertex in the PP_GRAPH_RELABEL vertex order: decreasing degree
    (out + in for a directed graph; ties by increasing id).  A data-layout definition used
    by tests to state the relabelled graph's canonical parents (oracle.parents(key=...))."""
    deg = g.degrees().astype(np.int64)
    if gT is not None and not getattr(g, "symmetric", True):
        deg = deg + gT.degrees().astype(np.int64)
    order = np.argsort(-deg, kind="stable")
    key = np.empty(g.n, dtype=np.uint32)
    key[order] = np.arange(g.n, dtype=np.uint32)
    return key


def random_subset(n: int, count: int, seed: int) -> np.ndarray:
    """Exactly `count` distinct ids from [0,n), seeded (C3 mask protocol)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if count >= n:
        return np.arange(n, dtype=np.uint32)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.uint32)


def dense_from_ids(n: int, ids) -> np.ndarray:
    v = np.zeros(n, dtype=np.uint8)
    v[np.asarray(ids, dtype=np.int64)] = 1
    return v


def random_graph(n: int, m: int, seed: int, symmetrize: bool = True) -> CSR:
    """Small uniform random graph (tests)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    src = rng.integers(0, max(n, 1), size=m, dtype=np.uint32)
    dst = rng.integers(0, max(n, 1), size=m, dtype=np.uint32)
    return from_edges(n, src, dst, symmetrize=symmetrize)


# --- workload recipes (BASELINE.json configs) -------------------------------

CONFIGS = {
    "C1": dict(kind="rmat", scale=16, edgefactor=16, seed=1, sources=64),
    "C2": dict(kind="rmat", scale=22, edgefactor=16, seed=1, sources=64),
    "C2_ef64": dict(kind="rmat", scale=22, edgefactor=64, seed=1, sources=64),
    "C3": dict(kind="rmat", scale=22, edgefactor=16, seed=1, sources=0),
    "C4": dict(kind="grid", rows=4096, cols=4096, sources=8),
    "C4_road": dict(kind="pgrid", rows=4096, cols=4096, p=0.6, seed=1, sources=8),
    "C5": dict(kind="rmat", scale=26, edgefactor=16, seed=1, sources=16),
    # kron_g500-logn21 analog (Table 3; nnz within 0.5%): Table-2 ablation
    "K21": dict(kind="rmat", scale=21, edgefactor=48, seed=1, sources=16),
    # the paper's generated RMAT graphs (Table 3; Fig. 7)
    "S23E32": dict(kind="rmat", scale=23, edgefactor=32, seed=1, sources=16),
    "S24E16": dict(kind="rmat", scale=24, edgefactor=16, seed=1, sources=16),
    # rgg_n_2_24_s0 shape: high-diameter second workload
    "RGG24": dict(kind="rgg", scale=24, factor=0.55, seed=1, sources=8),
}


def make(config: str) -> CSR:
    c = CONFIGS[config]
    if c["kind"] == "rmat":
        g = rmat(c["scale"], c["edgefactor"], c["seed"])
    elif c["kind"] == "rgg":
        g = rgg(c["scale"], c["factor"], c["seed"])
    elif c["kind"] == "grid":
        g = grid(c["rows"], c["cols"])
    else:
        g = percolated_grid(c["rows"], c["cols"], c["p"], c["seed"])
    g.name = config + ":" + g.name
    return g


def edge_weights(nnz: int, seed: int = 3, lo: int = 1, hi: int = 10, integer: bool = True) -> np.ndarray:
    """Seeded non-negative edge weights (SURVEY NEXT-4 / SPEC S:345 recipe: integers lo..hi,
    or uniform reals in [lo, hi) when integer=False).  float32-exact values either way."""
    rng = np.random.default_rng(seed)
    if integer:
        return rng.integers(lo, hi + 1, size=nnz).astype(np.float32)
    return rng.uniform(lo, hi, size=nnz).astype(np.float32)


def transpose_weighted(g: CSR, w: np.ndarray):
    """CSC of a weighted CSR: (CSR of A^T, weights aligned with it).  Plumbing only."""
    rows = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.off))
    order = np.lexsort((rows, g.idx.astype(np.int64)))
    cidx = rows[order].astype(np.uint32)
    coff = np.zeros(g.n + 1, np.int64)
    np.cumsum(np.bincount(g.idx.astype(np.int64), minlength=g.n), out=coff[1:])
    return CSR(g.n, coff, cidx, g.symmetric, g.name + "^T"), np.ascontiguousarray(w[order])
