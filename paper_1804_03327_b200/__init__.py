"""Python binding of libpushpull.so (include/pushpull.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels for sm_100a; PyTorch
supplies device memory (tensor data pointers) and streams.  There is no CPU fallback:
importing this package fails loudly when the shared library has not been built.

Raw C-ABI names are re-exported (pp_ctx_create, pp_graph_upload, pp_mxv, pp_bfs, ...);
`Context`, `Graph`, `bfs` and `mxv` are thin conveniences over them.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpushpull.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: the CUDA extension has not been built "
        "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

# ---- status codes / enums (pushpull.h) -----------------------------------------------------
PP_OK, PP_ERR_ARG, PP_ERR_RANGE, PP_ERR_DIM, PP_ERR_GRAPH, PP_ERR_UNSUPPORTED, PP_ERR_CUDA, \
    PP_ERR_NCCL, PP_ERR_OOM, PP_ERR_TIMEOUT = range(10)
STATUS_NAMES = {0: "PP_OK", 1: "PP_ERR_ARG", 2: "PP_ERR_RANGE", 3: "PP_ERR_DIM", 4: "PP_ERR_GRAPH",
                5: "PP_ERR_UNSUPPORTED", 6: "PP_ERR_CUDA", 7: "PP_ERR_NCCL", 8: "PP_ERR_OOM",
                9: "PP_ERR_TIMEOUT"}
PP_GRAPH_SYMMETRIC, PP_GRAPH_DEVICE, PP_GRAPH_VALIDATE, PP_GRAPH_RELABEL, PP_GRAPH_OFF64 = \
    1, 2, 4, 8, 16
PP_VEC_LIST, PP_VEC_BITMAP = 0, 1
PP_SR_LOR_LAND = 0
PP_DIR_AUTO, PP_DIR_PUSH, PP_DIR_PULL = 0, 1, 2
PP_HEUR_EDGES, PP_HEUR_PAPER_R = 0, 1
PP_MODE_DO, PP_MODE_PUSH_ONLY, PP_MODE_PULL_ONLY = 0, 1, 2
PP_OPT_NO_MASKING, PP_OPT_NO_EARLYEXIT, PP_OPT_NO_REUSE = 1, 2, 4


class PPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class pp_vector(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("data", ctypes.c_void_p), ("capacity", ctypes.c_int64)]


class pp_descriptor(ctypes.Structure):
    _fields_ = [("mask", ctypes.POINTER(pp_vector)), ("complement", ctypes.c_int32),
                ("semiring", ctypes.c_int32), ("accum", ctypes.c_int32),
                ("replace", ctypes.c_int32), ("direction", ctypes.c_int32),
                ("early_exit", ctypes.c_int32), ("transpose", ctypes.c_int32),
                ("want_nnz", ctypes.c_int32), ("switchpoint", ctypes.c_double),
                ("prev_nnz", ctypes.c_int64)]


class pp_bfs_options(ctypes.Structure):
    _fields_ = [("heuristic", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("want_parents", ctypes.c_int32), ("toggles", ctypes.c_uint32)]


class pp_sssp_stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("push_iterations", ctypes.c_int64),
                ("pull_iterations", ctypes.c_int64), ("switch_iteration", ctypes.c_int64)]


class pp_bfs_stats(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("reached", ctypes.c_int64),
                ("capacity", ctypes.c_int32), ("dir", ctypes.POINTER(ctypes.c_int8)),
                ("c", ctypes.POINTER(ctypes.c_int64)), ("m_f", ctypes.POINTER(ctypes.c_int64)),
                ("m_u", ctypes.POINTER(ctypes.c_int64)), ("ns", ctypes.POINTER(ctypes.c_int64)),
                ("init_ns", ctypes.c_int64), ("exchanged_bytes", ctypes.c_int64),
                ("cand", ctypes.POINTER(ctypes.c_int64)), ("reached_nnz", ctypes.c_int64)]


_vp, _i64, _u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32
_SIGS = {
    "pp_last_error": ([], ctypes.c_char_p),
    "pp_version": ([], ctypes.c_char_p),
    "pp_ctx_create": ([ctypes.c_int, _vp, ctypes.POINTER(_vp)], ctypes.c_int),
    "pp_ctx_destroy": ([_vp], ctypes.c_int),
    "pp_ctx_launch_count": ([_vp, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
    "pp_graph_upload": ([_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _u32, ctypes.POINTER(_vp)],
                        ctypes.c_int),
    "pp_graph_free": ([_vp], ctypes.c_int),
    "pp_graph_info": ([_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
                      ctypes.c_int),
    "pp_descriptor_default": ([ctypes.POINTER(pp_descriptor)], ctypes.c_int),
    "pp_mxv": ([_vp, ctypes.POINTER(pp_vector), ctypes.POINTER(pp_descriptor),
                ctypes.POINTER(pp_vector)], ctypes.c_int),
    "pp_bfs_options_default": ([ctypes.POINTER(pp_bfs_options)], ctypes.c_int),
    "pp_bfs": ([_vp, _i64, ctypes.POINTER(pp_bfs_options), _vp, _vp,
                ctypes.POINTER(pp_bfs_stats)], ctypes.c_int),
    "pp_bfs_debug_times": ([_vp, ctypes.c_int32, _vp, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "pp_bfs_debug_level": ([_vp, _i64, ctypes.c_int32, ctypes.POINTER(pp_bfs_options), _vp], ctypes.c_int),
    "pp_bfs_debug_phases": ([_vp, _vp], ctypes.c_int),
    "pp_nccl_unique_id": ([_vp], ctypes.c_int),
    "pp_ctx_create_dist": ([ctypes.c_int, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)],
                           ctypes.c_int),
    "pp_partition": ([_i64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
                     ctypes.c_int),
    "pp_graph_partition": ([_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)], ctypes.c_int),
    "pp_graph_export": ([_vp, _vp], ctypes.c_int),
    "pp_graph_import": ([_vp, _vp], ctypes.c_int),
    "pp_team_create": ([ctypes.c_int, _vp, ctypes.c_int32, ctypes.POINTER(_vp)], ctypes.c_int),
    "pp_bfs_team": ([ctypes.POINTER(_vp), ctypes.c_int32, _i64, ctypes.POINTER(pp_bfs_options),
                     ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(pp_bfs_stats)],
                    ctypes.c_int),
    "pp_sssp": ([_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64, ctypes.c_double, _vp,
                 ctypes.POINTER(pp_sssp_stats)], ctypes.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res
    globals()["_c_" + _name] = _f

EXPORTED = tuple(_SIGS)


def _check(status: int):
    if status != PP_OK:
        raise PPError(status, _lib.pp_last_error().decode())


# ---- raw C-ABI names ------------------------------------------------------------------------

def pp_last_error() -> str:
    return _lib.pp_last_error().decode()


def pp_version() -> str:
    return _lib.pp_version().decode()


def pp_ctx_create(device: int, cuda_stream: int):
    out = _vp()
    _check(_lib.pp_ctx_create(device, cuda_stream, ctypes.byref(out)))
    return out.value


def pp_ctx_destroy(ctx):
    _check(_lib.pp_ctx_destroy(ctx))


def pp_ctx_launch_count(ctx) -> int:
    out = ctypes.c_uint64()
    _check(_lib.pp_ctx_launch_count(ctx, ctypes.byref(out)))
    return out.value


def pp_graph_upload(ctx, n, row_lo, row_hi, nnz, csr_off, csr_idx, csc_off, csc_idx, flags):
    out = _vp()
    _check(_lib.pp_graph_upload(ctx, n, row_lo, row_hi, nnz, csr_off, csr_idx, csc_off, csc_idx,
                                flags, ctypes.byref(out)))
    return out.value


def pp_graph_free(g):
    _check(_lib.pp_graph_free(g))


def pp_graph_info(g):
    n, nnz, b = _i64(), _i64(), _i64()
    _check(_lib.pp_graph_info(g, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(b)))
    return n.value, nnz.value, b.value


def pp_descriptor_default() -> pp_descriptor:
    d = pp_descriptor()
    _check(_lib.pp_descriptor_default(ctypes.byref(d)))
    return d


def pp_bfs_options_default() -> pp_bfs_options:
    o = pp_bfs_options()
    _check(_lib.pp_bfs_options_default(ctypes.byref(o)))
    return o


def pp_mxv(g, w: pp_vector, desc: pp_descriptor, u: pp_vector):
    _check(_lib.pp_mxv(g, ctypes.byref(w), ctypes.byref(desc), ctypes.byref(u)))


def pp_bfs(g, source, opts, depth_ptr, parent_ptr, stats):
    _check(_lib.pp_bfs(g, int(source), None if opts is None else ctypes.byref(opts), depth_ptr,
                       parent_ptr, None if stats is None else ctypes.byref(stats)))


def pp_bfs_debug_times(g, levels=0, fetch=False):
    """Enable (levels > 0) or fetch per-level, per-CTA phase durations (ns)."""
    nct = ctypes.c_int32()
    if not fetch:
        _check(_lib.pp_bfs_debug_times(g, levels, None, ctypes.byref(nct)))
        return nct.value
    _check(_lib.pp_bfs_debug_times(g, 0, None, ctypes.byref(nct)))
    out = np.zeros(levels * nct.value, np.int64)
    _check(_lib.pp_bfs_debug_times(g, 0, out.ctypes.data, ctypes.byref(nct)))
    return out.reshape(levels, nct.value)


def pp_bfs_debug_phases(g, levels, nctas):
    """The three per-level, per-CTA phase planes (ns) of the last BFS (see pushpull.h)."""
    out = np.zeros(3 * levels * nctas, np.int64)
    _check(_lib.pp_bfs_debug_phases(g, out.ctypes.data))
    return out.reshape(3, levels, nctas)


def pp_bfs_debug_level(g, source, level, depth_ptr, heuristic=PP_HEUR_EDGES, mode=PP_MODE_DO,
                       toggles=0):
    """Levels 1..level-1 in one launch, level `level` alone in a second (profiling)."""
    o = pp_bfs_options(heuristic, mode, 0.0, 0.0, 0, toggles)
    _check(_lib.pp_bfs_debug_level(g, int(source), int(level), ctypes.byref(o), depth_ptr))


def pp_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.pp_nccl_unique_id(buf))
    return buf.raw


def pp_ctx_create_dist(device: int, cuda_stream: int, nccl_id, rank: int, nranks: int):
    """nccl_id: the 128-byte NCCL unique id, or None (external bootstrap: pp_graph_export /
    pp_graph_import)."""
    out = _vp()
    buf = None
    if nccl_id is not None:
        assert len(nccl_id) == 128
        buf = ctypes.create_string_buffer(nccl_id, 128)
    _check(_lib.pp_ctx_create_dist(device, cuda_stream, buf, rank, nranks, ctypes.byref(out)))
    return out.value


def pp_graph_export(g) -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.pp_graph_export(g, buf))
    return buf.raw


def pp_graph_import(g, records: bytes):
    buf = ctypes.create_string_buffer(records, len(records))
    _check(_lib.pp_graph_import(g, buf))


def pp_partition(n: int, rank: int, nranks: int):
    lo, hi = _i64(), _i64()
    _check(_lib.pp_partition(n, rank, nranks, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def pp_graph_partition(g):
    lo, hi = _i64(), _i64()
    _check(_lib.pp_graph_partition(g, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def pp_team_create(device: int, cuda_stream: int, nranks: int):
    arr = (_vp * nranks)()
    _check(_lib.pp_team_create(device, cuda_stream, nranks, arr))
    return [arr[r] for r in range(nranks)]


def pp_bfs_team(graphs, source, opts, depth_ptrs, parent_ptrs, stats):
    P = len(graphs)
    ga = (_vp * P)(*graphs)
    da = (_vp * P)(*depth_ptrs)
    pa = None if parent_ptrs is None else (_vp * P)(*parent_ptrs)
    _check(_lib.pp_bfs_team(ga, P, int(source), None if opts is None else ctypes.byref(opts), da, pa,
                            None if stats is None else ctypes.byref(stats)))


# ---- conveniences (torch tensors as device memory) ----------------------------------------

def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    return int(x)


class Context:
    """Device + stream.  stream: a torch.cuda.Stream or None (current torch stream)."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device = device
        self.stream = stream
        self.handle = pp_ctx_create(device, stream.cuda_stream)

    def launches(self) -> int:
        return pp_ctx_launch_count(self.handle)

    def close(self):
        if self.handle:
            pp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistContext(Context):
    """Distributed context: one GPU per process, NCCL communicator built from an id that
    rank 0 creates and torch.distributed broadcasts (plumbing only)."""

    def __init__(self, device: int, rank: int, nranks: int, nccl_id: bytes, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device = device
        self.stream = stream
        self.rank, self.nranks = rank, nranks
        self.handle = pp_ctx_create_dist(device, stream.cuda_stream, nccl_id, rank, nranks)


def block_rows(off, idx, lo, hi):
    """Rows [lo, hi) of a CSR as (row-local int64 offsets, ids) — the block a rank of the 1D
    row partition uploads (host arrays; no method arithmetic)."""
    off = np.asarray(off, dtype=np.int64)
    b, e = int(off[lo]), int(off[hi])
    return np.ascontiguousarray(off[lo:hi + 1] - b), np.ascontiguousarray(np.asarray(idx)[b:e],
                                                                        dtype=np.uint32)


class _RankCtx:
    """One rank context of a Team (handle + rank/nranks for Graph's block upload)."""

    def __init__(self, handle, rank, nranks, device, stream):
        self.handle, self.rank, self.nranks = handle, rank, nranks
        self.device, self.stream = device, stream

    def launches(self) -> int:
        return pp_ctx_launch_count(self.handle)


class Team:
    """Single-device team of `nranks` rank contexts (pp_team_create): the multi-rank engine's
    ranks run as CTA groups of one cooperative launch on one GPU (pp_bfs_team)."""

    def __init__(self, nranks: int, device: int = 0, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device, self.stream, self.nranks = device, stream, nranks
        hs = pp_team_create(device, stream.cuda_stream, nranks)
        self.ctxs = [_RankCtx(h, r, nranks, device, stream) for r, h in enumerate(hs)]

    def upload(self, csr, csc=None, validate=False, off64=False):
        """Every rank uploads its block of the graph; returns the per-rank Graph list."""
        return [Graph.from_csr(c, csr, csc, validate=validate, off64=off64) for c in self.ctxs]

    def launches(self) -> int:
        return sum(c.launches() for c in self.ctxs)

    def close(self):
        for c in self.ctxs:
            if c.handle:
                pp_ctx_destroy(c.handle)
                c.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bfs_team(graphs, source: int, depths, parents=None, heuristic=PP_HEUR_EDGES, mode=PP_MODE_DO,
             alpha=0.0, beta=0.0, stats_capacity=0):
    """pp_bfs_team over a Team's per-rank graphs; depths/parents: per-rank device slices."""
    o = pp_bfs_options(heuristic, mode, alpha, beta, 1 if parents is not None else 0, 0)
    st, arrays = _stats(stats_capacity)
    pp_bfs_team([g.handle for g in graphs], source, o, [_ptr(d) for d in depths],
                None if parents is None else [_ptr(p) for p in parents], st)
    return _stats_dict(st, arrays, stats_capacity)


class Graph:
    """Device-resident graph (library-owned copy of CSR + CSC).  On a multi-rank context
    (DistContext / Team member) off/idx/coff/cidx are the FULL host CSR / CSC and only the
    rank's block [row_lo, row_hi) = pp_partition(n, rank, nranks) is uploaded."""

    def __init__(self, ctx: Context, n, off, idx, coff=None, cidx=None, symmetric=None,
                 validate=False, device_ptrs=False, relabel=False, off64=False):
        self.ctx = ctx
        self.n = int(n)
        if symmetric is None:
            symmetric = coff is None
        flags = (PP_GRAPH_SYMMETRIC if symmetric else 0) | (PP_GRAPH_VALIDATE if validate else 0) | \
            (PP_GRAPH_RELABEL if relabel else 0) | \
            (PP_GRAPH_DEVICE if device_ptrs else 0) | (PP_GRAPH_OFF64 if off64 else 0)
        self.relabel = bool(relabel)
        nranks = getattr(ctx, "nranks", 0)
        if nranks:
            assert not device_ptrs, "multi-rank upload takes host arrays"
            lo, hi = pp_partition(self.n, ctx.rank, nranks)
            boff, bidx = block_rows(off, idx, lo, hi)
            if symmetric:
                cboff, cbidx = None, None
            else:
                cboff, cbidx = block_rows(coff, cidx, lo, hi)
            self.nnz = int(boff[-1])
            self._keep = (boff, bidx, cboff, cbidx)
            self.handle = pp_graph_upload(ctx.handle, self.n, lo, hi, self.nnz, _ptr(boff),
                                          _ptr(bidx) if len(bidx) else None,
                                          None if cboff is None else _ptr(cboff),
                                          None if cbidx is None or not len(cbidx) else _ptr(cbidx),
                                          flags)
            self._keep = None
            return
        nnz = int(off[-1]) if not device_ptrs else int(idx.numel())
        if not device_ptrs:
            off = np.ascontiguousarray(off, dtype=np.int64)
            idx = np.ascontiguousarray(idx, dtype=np.uint32)
            if coff is not None:
                coff = np.ascontiguousarray(coff, dtype=np.int64)
                cidx = np.ascontiguousarray(cidx, dtype=np.uint32)
        self.nnz = nnz
        self._keep = (off, idx, coff, cidx)
        self.handle = pp_graph_upload(ctx.handle, self.n, 0, self.n, nnz, _ptr(off),
                                      _ptr(idx) if nnz else None, _ptr(coff),
                                      _ptr(cidx) if (cidx is not None and nnz) else None, flags)
        self._keep = None

    @classmethod
    def from_csr(cls, ctx, csr, csc=None, validate=False, relabel=False, off64=False):
        if csc is None and not getattr(csr, "symmetric", True):
            raise ValueError("directed graph needs its CSC")
        return cls(ctx, csr.n, csr.off, csr.idx, None if csc is None else csc.off,
                   None if csc is None else csc.idx, symmetric=csc is None, validate=validate,
                   relabel=relabel, off64=off64)

    def info(self):
        return pp_graph_info(self.handle)

    def partition(self):
        return pp_graph_partition(self.handle)

    def export(self) -> bytes:
        """This rank's 128-byte peer record (external bootstrap)."""
        return pp_graph_export(self.handle)

    def import_peers(self, records):
        """Map the peers from every rank's record, in rank order (external bootstrap)."""
        pp_graph_import(self.handle, b"".join(records))

    def close(self):
        if self.handle:
            pp_graph_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bfs(graph: Graph, source: int, depth, parent=None, heuristic=PP_HEUR_EDGES, mode=PP_MODE_DO,
        alpha=0.0, beta=0.0, toggles=0, stats_capacity=0):
    """Run pp_bfs.  depth/parent: int32 torch tensors (device) or numpy arrays (host).
    Returns a dict of per-level stats when stats_capacity > 0, else None."""
    o = pp_bfs_options(heuristic, mode, alpha, beta, 1 if parent is not None else 0, toggles)
    st, arrays = _stats(stats_capacity)
    pp_bfs(graph.handle, source, o, _ptr(depth), _ptr(parent), st)
    return _stats_dict(st, arrays, stats_capacity)


def _stats(cap):
    if cap <= 0:
        return None, None
    arrays = dict(dir=np.zeros(cap, np.int8), c=np.zeros(cap, np.int64),
                  m_f=np.zeros(cap, np.int64), m_u=np.zeros(cap, np.int64),
                  ns=np.zeros(cap, np.int64), cand=np.zeros(cap, np.int64))
    st = pp_bfs_stats(0, 0, cap,
                      arrays["dir"].ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
                      arrays["c"].ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                      arrays["m_f"].ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                      arrays["m_u"].ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                      arrays["ns"].ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 0, 0,
                      arrays["cand"].ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 0)
    return st, arrays


def _stats_dict(st, arrays, cap):
    if st is None:
        return None
    L = min(st.levels, cap)
    return dict(levels=st.levels, reached=st.reached, dir=arrays["dir"][:L], c=arrays["c"][:L],
                m_f=arrays["m_f"][:L], m_u=arrays["m_u"][:L], ns=arrays["ns"][:L],
                init_ns=st.init_ns, exchanged_bytes=st.exchanged_bytes, cand=arrays["cand"][:L],
                reached_nnz=st.reached_nnz)


def make_vector(fmt: int, n: int, data=None, nnz: int = -1, capacity: int = 0) -> pp_vector:
    return pp_vector(fmt, n, nnz, _ptr(data), capacity)


def mxv(graph: Graph, w: pp_vector, u: pp_vector, mask: pp_vector = None, complement=False,
        accum=False, replace=True, direction=PP_DIR_AUTO, early_exit=True, transpose=True,
        want_nnz=True, switchpoint=0.01, prev_nnz=-1) -> int:
    """Run pp_mxv; returns w.nnz (-1 when not requested for a bitmap output)."""
    d = pp_descriptor_default()
    if mask is not None:
        d.mask = ctypes.pointer(mask)
    d.complement = int(bool(complement))
    d.accum = int(bool(accum))
    d.replace = int(bool(replace))
    d.direction = direction
    d.early_exit = int(bool(early_exit))
    d.transpose = int(bool(transpose))
    d.want_nnz = int(bool(want_nnz))
    d.switchpoint = switchpoint
    d.prev_nnz = prev_nnz
    pp_mxv(graph.handle, w, d, u)
    return w.nnz


def header_functions():
    """Function names declared in include/pushpull.h (for the export test)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "pushpull.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:pp_status|const char\*)\s+(pp_\w+)\s*\(", text, re.M)))


def pp_sssp(ctx, n, nnz, csr_off, csr_idx, csr_w, csc_off, csc_idx, csc_w, source, alpha, dist):
    """C-ABI pp_sssp (include/pushpull.h; Sec. 5.6).  All arrays are device tensors."""
    st = pp_sssp_stats()
    _check(_lib.pp_sssp(ctx, int(n), int(nnz), _ptr(csr_off), _ptr(csr_idx), _ptr(csr_w), _ptr(csc_off),
                        _ptr(csc_idx), _ptr(csc_w), int(source), float(alpha), _ptr(dist),
                        ctypes.byref(st)))
    return {"iterations": st.iterations, "push_iterations": st.push_iterations,
            "pull_iterations": st.pull_iterations, "switch_iteration": st.switch_iteration}


def sssp(ctx: Context, csr_off, csr_idx, csr_w, csc_off, csc_idx, csc_w, source: int,
         alpha: float = 0.01, dist=None):
    """Two-phase min-plus SSSP on device tensors (int64 offsets, int32/uint32 ids, fp32
    weights).  Returns (dist fp32 device tensor, stats dict)."""
    import torch
    n = int(csr_off.numel()) - 1
    want = ((csr_off, (torch.int64,)), (csc_off, (torch.int64,)),
            (csr_idx, (torch.int32, torch.uint32)), (csc_idx, (torch.int32, torch.uint32)),
            (csr_w, (torch.float32,)), (csc_w, (torch.float32,)))
    dev0 = csr_off.device
    for t, dts in want:
        if not isinstance(t, torch.Tensor) or t.dtype not in dts or not t.is_contiguous() \
                or t.device != dev0 or t.device.type != "cuda":
            raise ValueError("sssp: int64 offsets, 32-bit ids and float32 weights, contiguous, "
                             "all on one CUDA device")
    if csc_off.numel() != n + 1 or csr_idx.numel() != csc_idx.numel() or \
            csr_w.numel() != csr_idx.numel() or csc_w.numel() != csc_idx.numel():
        raise ValueError("sssp: CSR / CSC array lengths disagree")
    if dist is None:
        dist = torch.empty(n, dtype=torch.float32, device=csr_off.device)
    st = pp_sssp(ctx.handle, n, int(csr_idx.numel()), csr_off, csr_idx, csr_w, csc_off, csc_idx,
                 csc_w, source, alpha, dist)
    return dist, st
