"""Thin ctypes binding of libgbbs (include/gbbs.h): argument marshalling only.

Every step of a traversal runs in libgbbs's CUDA kernels; there is no Python or
CPU fallback.  If libgbbs.so is missing or fails to load, importing this module
raises — the product path fails loudly instead of degrading.

Arrays may be numpy arrays (host memory) or torch tensors (host or CUDA); the
library classifies each pointer itself (gbbs.h "Conventions").
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GBBS_LIB") or os.path.join(_HERE, "libgbbs.so")

GBBS_OK, GBBS_EINVAL, GBBS_ERANGE, GBBS_ENOMEM, GBBS_ECUDA, GBBS_EINTERNAL = 0, -1, -2, -3, -4, -5
GBBS_INF = 0xFFFFFFFF
GBBS_DIST_INF = np.iinfo(np.int64).max
GBBS_DIST_NEGINF = np.iinfo(np.int64).min
GBBS_SYMMETRIC, GBBS_BORROW, GBBS_NO_VALIDATE = 0x1, 0x2, 0x4
GBBS_MODE_AUTO, GBBS_MODE_SPARSE, GBBS_MODE_DENSE, GBBS_MODE_PULL = 0, 1, 2, 3
GBBS_RULE_PAPER_ONLY = 0x1
GBBS_RULE_LEVEL_BYTES_ON = 0x2
GBBS_RULE_LEVEL_BYTES_OFF = 0x4

EXPORTS = ("gbbs_graph_create", "gbbs_graph_destroy", "gbbs_graph_info", "gbbs_bfs",
           "gbbs_bellman_ford", "gbbs_widest_path", "gbbs_bfs_ex", "gbbs_bellman_ford_ex",
           "gbbs_widest_path_ex", "gbbs_wbfs", "gbbs_wbfs_ex", "gbbs_bellman_ford_signed",
           "gbbs_bellman_ford_signed_ex", "gbbs_bfs_batch", "gbbs_bellman_ford_batch",
           "gbbs_bfs_batch_ex", "gbbs_bellman_ford_batch_ex", "gbbs_wbfs_batch",
           "gbbs_wbfs_batch_ex", "gbbs_betweenness_batch", "gbbs_betweenness_batch_ex",
           "gbbs_betweenness", "gbbs_betweenness_ex", "gbbs_default_opts",
           "gbbs_launch_info", "gbbs_graph_in_edges", "gbbs_last_error")


class GbbsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gbbs error {code}: {msg}")
        self.code = code


class GbbsArgError(GbbsError, ValueError):
    """An argument rejected by the binding before it reaches C (code GBBS_EINVAL)."""

    def __init__(self, msg):
        super().__init__(GBBS_EINVAL, msg)


class gbbs_opts(ctypes.Structure):
    _fields_ = [("threshold_den", ctypes.c_uint32), ("mode", ctypes.c_int32),
                ("ctas_per_sm", ctypes.c_uint32), ("delta", ctypes.c_uint32),
                ("neg_scope", ctypes.c_uint32), ("bsize", ctypes.c_uint32),
                ("teams", ctypes.c_uint32), ("rules", ctypes.c_uint32)]


class gbbs_round_stat(ctypes.Structure):
    _fields_ = [("dense", ctypes.c_int32), ("bucket", ctypes.c_int32),
                ("frontier", ctypes.c_int64), ("frontier_edges", ctypes.c_int64),
                ("acquired", ctypes.c_int64), ("edges_examined", ctypes.c_int64),
                ("vertices_swept", ctypes.c_int64), ("t_start_ns", ctypes.c_int64),
                ("t_work_ns", ctypes.c_int64), ("t_flush_ns", ctypes.c_int64),
                ("alg_bytes", ctypes.c_int64), ("head_hits", ctypes.c_int64)]


class gbbs_stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("dense_rounds", ctypes.c_int64),
                ("edges_examined", ctypes.c_int64), ("reached", ctypes.c_int64),
                ("kernel_ms", ctypes.c_double), ("rounds_out", ctypes.POINTER(gbbs_round_stat)), ("rounds_cap", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python build.py` (nvcc, sm_100a)")
    lib = ctypes.CDLL(LIB_PATH)
    p, i64, u32, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int32
    lib.gbbs_graph_create.argtypes = [i64, i64, p, p, p, u32, ctypes.POINTER(p)]
    lib.gbbs_graph_destroy.argtypes = [p]
    lib.gbbs_graph_destroy.restype = None
    lib.gbbs_graph_info.argtypes = [p, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(u32)]
    lib.gbbs_bfs.argtypes = [p, u32, p, p, p]
    lib.gbbs_bellman_ford.argtypes = [p, u32, p, p]
    lib.gbbs_bfs_ex.argtypes = [p, u32, p, p, p, ctypes.POINTER(gbbs_opts), ctypes.POINTER(gbbs_stats)]
    lib.gbbs_bellman_ford_ex.argtypes = [p, u32, p, p, ctypes.POINTER(gbbs_opts), ctypes.POINTER(gbbs_stats)]
    lib.gbbs_widest_path.argtypes = [p, u32, p, p]
    lib.gbbs_wbfs.argtypes = [p, u32, p, p]
    lib.gbbs_bfs_batch.argtypes = [p, p, i64, p, p, p]
    lib.gbbs_bellman_ford_batch.argtypes = [p, p, i64, p, p]
    lib.gbbs_bfs_batch_ex.argtypes = [p, p, i64, p, p, p, ctypes.POINTER(gbbs_opts)]
    lib.gbbs_wbfs_batch.argtypes = [p, p, i64, p, p]
    lib.gbbs_betweenness_batch.argtypes = [p, p, i64, p, p]
    lib.gbbs_betweenness_batch_ex.argtypes = [p, p, i64, p, p, ctypes.POINTER(gbbs_opts)]
    lib.gbbs_wbfs_batch_ex.argtypes = [p, p, i64, p, p, ctypes.POINTER(gbbs_opts)]
    lib.gbbs_bellman_ford_batch_ex.argtypes = [p, p, i64, p, p, ctypes.POINTER(gbbs_opts)]
    lib.gbbs_bellman_ford_signed.argtypes = [p, u32, p, p]
    lib.gbbs_bellman_ford_signed_ex.argtypes = [p, u32, p, p, ctypes.POINTER(gbbs_opts),
                                                ctypes.POINTER(gbbs_stats)]
    lib.gbbs_wbfs_ex.argtypes = [p, u32, p, p, ctypes.POINTER(gbbs_opts), ctypes.POINTER(gbbs_stats)]
    lib.gbbs_betweenness.argtypes = [p, u32, p, p]
    lib.gbbs_betweenness_ex.argtypes = [p, u32, p, p, ctypes.POINTER(gbbs_opts), ctypes.POINTER(gbbs_stats)]
    lib.gbbs_widest_path_ex.argtypes = [p, u32, p, p, ctypes.POINTER(gbbs_opts), ctypes.POINTER(gbbs_stats)]
    lib.gbbs_default_opts.argtypes = [ctypes.POINTER(gbbs_opts)]
    lib.gbbs_default_opts.restype = None
    lib.gbbs_launch_info.argtypes = [p, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    if hasattr(lib, "gbbs_graph_in_edges"):  # aux (test) call; absent in older dev builds
        lib.gbbs_graph_in_edges.argtypes = [p, p, p]
        lib.gbbs_graph_in_edges.restype = ctypes.c_int
    lib.gbbs_last_error.argtypes = []
    lib.gbbs_last_error.restype = ctypes.c_char_p
    for f in ("gbbs_graph_create", "gbbs_graph_info", "gbbs_bfs", "gbbs_bellman_ford", "gbbs_bfs_ex",
              "gbbs_bellman_ford_ex", "gbbs_widest_path", "gbbs_widest_path_ex", "gbbs_wbfs",
              "gbbs_wbfs_ex", "gbbs_bellman_ford_signed", "gbbs_bellman_ford_signed_ex", "gbbs_bfs_batch",
              "gbbs_bellman_ford_batch", "gbbs_bfs_batch_ex", "gbbs_bellman_ford_batch_ex",
              "gbbs_wbfs_batch", "gbbs_wbfs_batch_ex", "gbbs_betweenness_batch",
              "gbbs_betweenness_batch_ex", "gbbs_betweenness", "gbbs_betweenness_ex", "gbbs_launch_info"):
        getattr(lib, f).restype = ctypes.c_int
    return lib


lib = _load()


def last_error() -> str:
    return lib.gbbs_last_error().decode()


def _check(rc):
    if rc != GBBS_OK:
        raise GbbsError(rc, last_error())


def _ptr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(f"unsupported array type {type(a)}")


def _shape(a):
    """(element size in bytes, element count, is-integer, is-float) of an array, or None
    for a raw address (int), which is passed through unchecked."""
    if a is None or isinstance(a, int):
        return None
    if isinstance(a, np.ndarray):
        return a.dtype.itemsize, a.size, a.dtype.kind in "iu", a.dtype.kind == "f"
    if hasattr(a, "element_size"):
        return (a.element_size(), a.numel(), not (a.is_floating_point() or a.is_complex()),
                a.is_floating_point())
    raise TypeError(f"unsupported array type {type(a)}")


def _want(a, name, itemsize, count, kind="int", exact=False):
    """Check an argument before its address goes to C: element size, integer or float
    elements, and at least (exactly, if exact) `count` elements.  The library reads
    and writes fixed widths, so a mismatch would be an out-of-bounds access."""
    sh = _shape(a)
    if sh is None:
        return
    isz, cnt, is_int, is_float = sh
    if isz != itemsize or (kind == "int" and not is_int) or (kind == "float" and not is_float):
        raise GbbsArgError(f"{name}: expected {itemsize}-byte {kind} elements, got {isz}-byte "
                         f"{'int' if is_int else 'float' if is_float else 'other'}")
    if (cnt != count) if exact else (cnt < count):
        raise GbbsArgError(f"{name}: expected {'exactly' if exact else 'at least'} {count} "
                         f"elements, got {cnt}")


def _graph_n(handle):
    n = ctypes.c_int64()
    _check(lib.gbbs_graph_info(handle, ctypes.byref(n), None, None))
    return n.value


def _stream(stream, *arrays):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    for a in arrays:
        if a is not None and hasattr(a, "is_cuda") and a.is_cuda:
            import torch
            return torch.cuda.current_stream(a.device).cuda_stream
    return None


# ---- the four calls of the boundary, same names as the C ABI -------------------

def gbbs_graph_create(n, m, offsets, targets, weights=None, flags=0):
    """Returns an opaque handle (int).  See gbbs.h for ownership and errors."""
    if 1 <= int(n) <= 0xFFFFFFFE and int(m) >= 0:  # else the library rejects n / m unread
        _want(offsets, "offsets", 8, int(n) + 1, exact=True)
        _want(targets, "targets", 4, int(m), exact=True)
        _want(weights, "weights", 4, int(m), exact=True)
    h = ctypes.c_void_p()
    _check(lib.gbbs_graph_create(int(n), int(m), _ptr(offsets), _ptr(targets), _ptr(weights),
                                 int(flags), ctypes.byref(h)))
    return h.value


def gbbs_graph_destroy(handle):
    lib.gbbs_graph_destroy(handle)


def gbbs_bfs(handle, src, dist, parent=None, stream=None, opts=None, stats=None):
    n = _graph_n(handle)
    _want(dist, "dist", 4, n)
    _want(parent, "parent", 4, n)
    st = _stream(stream, dist, parent)
    if opts is None and stats is None:
        _check(lib.gbbs_bfs(handle, int(src), _ptr(dist), _ptr(parent), st))
    else:
        _check(lib.gbbs_bfs_ex(handle, int(src), _ptr(dist), _ptr(parent), st,
                               ctypes.byref(opts) if opts is not None else None,
                               ctypes.byref(stats) if stats is not None else None))


def gbbs_bellman_ford(handle, src, dist, stream=None, opts=None, stats=None):
    _want(dist, "dist", 4, _graph_n(handle))
    st = _stream(stream, dist)
    if opts is None and stats is None:
        _check(lib.gbbs_bellman_ford(handle, int(src), _ptr(dist), st))
    else:
        _check(lib.gbbs_bellman_ford_ex(handle, int(src), _ptr(dist), st,
                                        ctypes.byref(opts) if opts is not None else None,
                                        ctypes.byref(stats) if stats is not None else None))


def gbbs_widest_path(handle, src, width, stream=None, opts=None, stats=None):
    _want(width, "width", 4, _graph_n(handle))
    st = _stream(stream, width)
    if opts is None and stats is None:
        _check(lib.gbbs_widest_path(handle, int(src), _ptr(width), st))
    else:
        _check(lib.gbbs_widest_path_ex(handle, int(src), _ptr(width), st,
                                       ctypes.byref(opts) if opts is not None else None,
                                       ctypes.byref(stats) if stats is not None else None))


def gbbs_wbfs(handle, src, dist, stream=None, opts=None, stats=None):
    _want(dist, "dist", 4, _graph_n(handle))
    st = _stream(stream, dist)
    if opts is None and stats is None:
        _check(lib.gbbs_wbfs(handle, int(src), _ptr(dist), st))
    else:
        _check(lib.gbbs_wbfs_ex(handle, int(src), _ptr(dist), st,
                                ctypes.byref(opts) if opts is not None else None,
                                ctypes.byref(stats) if stats is not None else None))


def gbbs_bellman_ford_signed(handle, src, dist, stream=None, opts=None, stats=None):
    """dist: int64[n] (numpy or torch, host or device)."""
    _want(dist, "dist", 8, _graph_n(handle))
    st = _stream(stream, dist)
    if opts is None and stats is None:
        _check(lib.gbbs_bellman_ford_signed(handle, int(src), _ptr(dist), st))
    else:
        _check(lib.gbbs_bellman_ford_signed_ex(handle, int(src), _ptr(dist), st,
                                               ctypes.byref(opts) if opts is not None else None,
                                               ctypes.byref(stats) if stats is not None else None))


def gbbs_bfs_batch(handle, srcs, dist, parent=None, stream=None, opts=None):
    """dist/parent: (k, n) uint32 arrays (row i = source i), host or device."""
    s = np.ascontiguousarray(srcs, dtype=np.uint32)
    n = _graph_n(handle)
    _want(dist, "dist", 4, s.shape[0] * n)
    _want(parent, "parent", 4, s.shape[0] * n)
    st = _stream(stream, dist, parent)
    if opts is None:
        _check(lib.gbbs_bfs_batch(handle, s.ctypes.data, int(s.shape[0]), _ptr(dist), _ptr(parent),
                                  st))
    else:
        _check(lib.gbbs_bfs_batch_ex(handle, s.ctypes.data, int(s.shape[0]), _ptr(dist),
                                     _ptr(parent), st, ctypes.byref(opts)))


def gbbs_bellman_ford_batch(handle, srcs, dist, stream=None, opts=None):
    s = np.ascontiguousarray(srcs, dtype=np.uint32)
    _want(dist, "dist", 4, s.shape[0] * _graph_n(handle))
    st = _stream(stream, dist)
    if opts is None:
        _check(lib.gbbs_bellman_ford_batch(handle, s.ctypes.data, int(s.shape[0]), _ptr(dist), st))
    else:
        _check(lib.gbbs_bellman_ford_batch_ex(handle, s.ctypes.data, int(s.shape[0]), _ptr(dist),
                                              st, ctypes.byref(opts)))


def gbbs_wbfs_batch(handle, srcs, dist, stream=None, opts=None):
    """dist: (k, n) device rows."""
    s = np.ascontiguousarray(srcs, dtype=np.uint32)
    _want(dist, "dist", 4, s.shape[0] * _graph_n(handle))
    st = _stream(stream, dist)
    if opts is None:
        _check(lib.gbbs_wbfs_batch(handle, s.ctypes.data, int(s.shape[0]), _ptr(dist), st))
    else:
        _check(lib.gbbs_wbfs_batch_ex(handle, s.ctypes.data, int(s.shape[0]), _ptr(dist), st,
                                      ctypes.byref(opts)))


def gbbs_betweenness_batch(handle, srcs, delta, stream=None, opts=None):
    """delta: (k, n) float64 device rows."""
    s = np.ascontiguousarray(srcs, dtype=np.uint32)
    _want(delta, "delta", 8, s.shape[0] * _graph_n(handle), kind="float")
    st = _stream(stream, delta)
    if opts is None:
        _check(lib.gbbs_betweenness_batch(handle, s.ctypes.data, int(s.shape[0]), _ptr(delta), st))
    else:
        _check(lib.gbbs_betweenness_batch_ex(handle, s.ctypes.data, int(s.shape[0]), _ptr(delta),
                                             st, ctypes.byref(opts)))


def gbbs_betweenness(handle, src, delta, stream=None, stats=None, opts=None):
    _want(delta, "delta", 8, _graph_n(handle), kind="float")
    st = _stream(stream, delta)
    if stats is None and opts is None:
        _check(lib.gbbs_betweenness(handle, int(src), _ptr(delta), st))
    else:
        _check(lib.gbbs_betweenness_ex(handle, int(src), _ptr(delta), st,
                                       None if opts is None else ctypes.byref(opts),
                                       None if stats is None else ctypes.byref(stats)))


def make_opts(threshold_den=20, mode=GBBS_MODE_AUTO, ctas_per_sm=0, delta=0, neg_scope=0, bsize=0,
              teams=0, rules=0):
    o = gbbs_opts()
    lib.gbbs_default_opts(ctypes.byref(o))
    o.threshold_den = threshold_den
    o.mode = mode
    o.ctas_per_sm = ctas_per_sm
    o.delta = delta
    o.neg_scope = neg_scope
    o.bsize = bsize
    o.teams = teams
    o.rules = rules
    return o


def make_stats(rounds_cap=0):
    s = gbbs_stats()
    buf = None
    if rounds_cap:
        buf = (gbbs_round_stat * rounds_cap)()
        s.rounds_out = ctypes.cast(buf, ctypes.POINTER(gbbs_round_stat))
        s.rounds_cap = rounds_cap
    s._buf = buf  # keep alive
    return s


def round_records(stats):
    """Per-round dicts; `us` = device time of the round when the next record's
    timestamp is available (the record after the last round holds the end time)."""
    n = min(stats.rounds, stats.rounds_cap)
    if not n:
        return []
    raw = stats.rounds_out[:min(stats.rounds + 1, stats.rounds_cap)]
    out = []
    for i, r in enumerate(raw[:n]):
        us = (raw[i + 1].t_start_ns - r.t_start_ns) / 1e3 if i + 1 < len(raw) else None
        out.append(dict(dense=r.dense, bucket=r.bucket, frontier=r.frontier, frontier_edges=r.frontier_edges,
                        acquired=r.acquired, edges_examined=r.edges_examined,
                        vertices_swept=r.vertices_swept, us=us, alg_bytes=r.alg_bytes,
                        head_hits=r.head_hits,
                        work_us=(r.t_work_ns - r.t_start_ns) / 1e3,
                        flush_us=(r.t_flush_ns - r.t_start_ns) / 1e3))
    return out


class Graph:
    """RAII wrapper around a gbbs_graph handle."""

    def __init__(self, offsets, targets, weights=None, symmetric=False, borrow=False, validate=True):
        n = int(offsets.shape[0]) - 1
        m = int(targets.shape[0])
        flags = (GBBS_SYMMETRIC if symmetric else 0) | (GBBS_BORROW if borrow else 0) | \
            (0 if validate else GBBS_NO_VALIDATE)
        self.n, self.m = n, m
        self._keep = (offsets, targets, weights) if borrow else None
        self.handle = gbbs_graph_create(n, m, offsets, targets, weights, flags)

    def close(self):
        if getattr(self, "handle", None):
            gbbs_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def in_edges(self):
        """The handle's in-edge CSC as host numpy arrays (in_offsets int64[n+1],
        in_sources uint32[m]); gbbs_graph_in_edges."""
        import numpy as np
        off = np.empty(self.n + 1, dtype=np.int64)
        src = np.empty(max(self.m, 1), dtype=np.uint32)
        _check(lib.gbbs_graph_in_edges(self.handle, off.ctypes.data, src.ctypes.data))
        return off, src[:self.m]

    def launch_info(self):
        c, t = ctypes.c_int32(), ctypes.c_int32()
        _check(lib.gbbs_launch_info(self.handle, ctypes.byref(c), ctypes.byref(t)))
        return c.value, t.value

    def bfs(self, src, dist, parent=None, stream=None, opts=None, stats=None):
        gbbs_bfs(self.handle, src, dist, parent, stream, opts, stats)

    def bellman_ford(self, src, dist, stream=None, opts=None, stats=None):
        gbbs_bellman_ford(self.handle, src, dist, stream, opts, stats)

    def widest_path(self, src, width, stream=None, opts=None, stats=None):
        gbbs_widest_path(self.handle, src, width, stream, opts, stats)

    def wbfs(self, src, dist, stream=None, opts=None, stats=None):
        gbbs_wbfs(self.handle, src, dist, stream, opts, stats)

    def bfs_batch(self, srcs, dist, parent=None, stream=None, opts=None):
        gbbs_bfs_batch(self.handle, srcs, dist, parent, stream, opts)

    def bellman_ford_batch(self, srcs, dist, stream=None, opts=None):
        gbbs_bellman_ford_batch(self.handle, srcs, dist, stream, opts)

    def wbfs_batch(self, srcs, dist, stream=None, opts=None):
        gbbs_wbfs_batch(self.handle, srcs, dist, stream, opts)

    def betweenness_batch(self, srcs, delta, stream=None, opts=None):
        gbbs_betweenness_batch(self.handle, srcs, delta, stream, opts)

    def bellman_ford_signed(self, src, dist, stream=None, opts=None, stats=None):
        gbbs_bellman_ford_signed(self.handle, src, dist, stream, opts, stats)

    def betweenness(self, src, delta, stream=None, stats=None, opts=None):
        gbbs_betweenness(self.handle, src, delta, stream, stats, opts)
