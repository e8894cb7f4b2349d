"""CPU oracle for the frontier BFS / Bellman-Ford hot path (arxiv 1805.05208).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product (``paper_1805_05208_b200``) never imports it and shares
no code with it.

A thin ctypes layer over ``oracle.c`` (plain sequential C).  What each routine
computes and which PAPER.md passage it follows is stated in ``oracle.c``:

* :func:`bfs` — FIFO-queue BFS, PAPER.md:1475-1478 (sec:benchmark, BFS output
  spec).
* :func:`dijkstra` — indexed-heap Dijkstra, the definition of the SSSP output
  of PAPER.md:1487-1490 (sec:benchmark, General-Weight SSSP).
* :func:`bellman_ford` — textbook all-edges Bellman-Ford (same definition).
* :func:`frontier_bellman_ford` — the paper's frontier formulation,
  PAPER.md:93-97 (sec:algs), run sequentially.
* :func:`check_bfs`, :func:`check_sssp` — O(n+m) certificates.

Parity status: every routine is pinned by tests/test_oracle.py (closed forms,
brute force, Floyd–Warshall, cross-agreement, certificate mutation tests).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

INF32 = np.uint32(0xFFFFFFFF)
INF64 = np.uint64(0xFFFFFFFFFFFFFFFF)

OK, EINVAL, ENOMEM, ERANGE, EFAIL, ENA = 0, -1, -2, -3, -4, -5


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (plain C, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        p = ctypes.c_void_p
        i64, u32 = ctypes.c_int64, ctypes.c_uint32
        lib.oracle_bfs.argtypes = [i64, p, p, u32, p, p]
        lib.oracle_dijkstra.argtypes = [i64, p, p, p, u32, p, p]
        lib.oracle_bellman_ford.argtypes = [i64, p, p, p, u32, p, p]
        lib.oracle_frontier_bellman_ford.argtypes = [i64, p, p, p, u32, p, p]
        lib.oracle_check_bfs.argtypes = [i64, p, p, u32, p, p, p]
        lib.oracle_check_sssp.argtypes = [i64, p, p, p, u32, p, p]
        lib.oracle_reached_edges.argtypes = [i64, p, p]
        lib.oracle_reached_edges.restype = i64
        for f in ("oracle_bfs", "oracle_dijkstra", "oracle_bellman_ford",
                  "oracle_frontier_bellman_ford", "oracle_check_bfs", "oracle_check_sssp"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _csr(offsets, targets, weights=None):
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(targets, dtype=np.uint32)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.uint32)
    n = off.shape[0] - 1
    if n < 1 or off[-1] != tgt.shape[0] or (w is not None and w.shape[0] != tgt.shape[0]):
        raise ValueError("malformed CSR")
    return n, off, tgt, w


def _check(rc, what):
    if rc != OK:
        raise RuntimeError(f"{what} failed with code {rc}")


def bfs(offsets, targets, src, want_parent=True):
    """Queue BFS. Returns (dist uint32[n], parent uint32[n] or None)."""
    n, off, tgt, _ = _csr(offsets, targets)
    dist = np.empty(n, np.uint32)
    par = np.empty(n, np.uint32) if want_parent else None
    _check(_load().oracle_bfs(n, _ptr(off), _ptr(tgt), int(src), _ptr(dist), _ptr(par)), "oracle_bfs")
    return dist, par


def dijkstra64(offsets, targets, weights, src, want_parent=False):
    """Dijkstra, uint64 distances (INF64 unreachable)."""
    n, off, tgt, w = _csr(offsets, targets, weights)
    dist = np.empty(n, np.uint64)
    par = np.empty(n, np.uint32) if want_parent else None
    _check(_load().oracle_dijkstra(n, _ptr(off), _ptr(tgt), _ptr(w), int(src), _ptr(dist), _ptr(par)),
           "oracle_dijkstra")
    return dist, par


def narrow(dist64):
    """uint64 distances -> uint32 with 0xFFFFFFFF for unreachable (reading A2).

    Raises if a finite distance does not fit below the sentinel."""
    finite = dist64 != INF64
    if finite.any() and dist64[finite].max() >= np.uint64(0xFFFFFFFF):
        raise OverflowError("finite distance >= 2^32-1")
    out = np.full(dist64.shape, INF32, np.uint32)
    out[finite] = dist64[finite].astype(np.uint32)
    return out


def dijkstra(offsets, targets, weights, src, want_parent=False):
    """Dijkstra narrowed to uint32 (the shape of gbbs_bellman_ford's output)."""
    d, p = dijkstra64(offsets, targets, weights, src, want_parent)
    return narrow(d), p


def bellman_ford64(offsets, targets, weights, src):
    """Textbook Bellman-Ford (all-edge passes). Returns (dist uint64, passes)."""
    n, off, tgt, w = _csr(offsets, targets, weights)
    dist = np.empty(n, np.uint64)
    passes = ctypes.c_int64(0)
    _check(_load().oracle_bellman_ford(n, _ptr(off), _ptr(tgt), _ptr(w), int(src), _ptr(dist),
                                       ctypes.addressof(passes)), "oracle_bellman_ford")
    return dist, passes.value


def frontier_bellman_ford64(offsets, targets, weights, src):
    """Paper's frontier Bellman-Ford, sequential. Returns (dist uint64, rounds)."""
    n, off, tgt, w = _csr(offsets, targets, weights)
    dist = np.empty(n, np.uint64)
    rounds = ctypes.c_int64(0)
    _check(_load().oracle_frontier_bellman_ford(n, _ptr(off), _ptr(tgt), _ptr(w), int(src), _ptr(dist),
                                                ctypes.addressof(rounds)), "oracle_frontier_bellman_ford")
    return dist, rounds.value


def check_bfs(offsets, targets, src, dist, parent=None):
    """BFS certificate. Returns (ok: bool, witness vertex or -1)."""
    n, off, tgt, _ = _csr(offsets, targets)
    dist = np.ascontiguousarray(dist, dtype=np.uint32)
    parent = None if parent is None else np.ascontiguousarray(parent, dtype=np.uint32)
    bad = ctypes.c_int64(-1)
    rc = _load().oracle_check_bfs(n, _ptr(off), _ptr(tgt), int(src), _ptr(dist), _ptr(parent),
                                  ctypes.addressof(bad))
    if rc not in (OK, EFAIL):
        raise RuntimeError(f"oracle_check_bfs rc={rc}")
    return rc == OK, bad.value


def check_sssp(offsets, targets, weights, src, dist):
    """SSSP tight-edge certificate (requires all weights >= 1)."""
    n, off, tgt, w = _csr(offsets, targets, weights)
    dist = np.ascontiguousarray(dist, dtype=np.uint32)
    bad = ctypes.c_int64(-1)
    rc = _load().oracle_check_sssp(n, _ptr(off), _ptr(tgt), _ptr(w), int(src), _ptr(dist),
                                   ctypes.addressof(bad))
    if rc == ENA:
        raise ValueError("certificate not applicable: zero weight present")
    if rc not in (OK, EFAIL):
        raise RuntimeError(f"oracle_check_sssp rc={rc}")
    return rc == OK, bad.value


def reached_edges(offsets, dist):
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    dist = np.ascontiguousarray(dist, dtype=np.uint32)
    return int(_load().oracle_reached_edges(off.shape[0] - 1, _ptr(off), _ptr(dist)))


def widest_path(offsets, targets, weights, src):
    """Modified-Dijkstra widest path (readings W1/W2: width[src] = INF32, unreachable 0)."""
    n, off, tgt, w = _csr(offsets, targets, weights)
    width = np.empty(n, np.uint32)
    lib = _load()
    lib.oracle_widest_path.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
    lib.oracle_widest_path.restype = ctypes.c_int
    _check(lib.oracle_widest_path(n, _ptr(off), _ptr(tgt), _ptr(w), int(src), _ptr(width)),
           "oracle_widest_path")
    return width


def check_widest(offsets, targets, weights, src, width):
    """Widest-path certificate (optimality + tight-edge reachability)."""
    n, off, tgt, w = _csr(offsets, targets, weights)
    width = np.ascontiguousarray(width, dtype=np.uint32)
    bad = ctypes.c_int64(-1)
    lib = _load()
    lib.oracle_check_widest.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                        ctypes.c_void_p]
    lib.oracle_check_widest.restype = ctypes.c_int
    rc = lib.oracle_check_widest(n, _ptr(off), _ptr(tgt), _ptr(w), int(src), _ptr(width),
                                 ctypes.addressof(bad))
    if rc not in (OK, EFAIL):
        raise RuntimeError(f"oracle_check_widest rc={rc}")
    return rc == OK, bad.value


def betweenness(offsets, targets, src, want_sigma=False):
    """Brandes single-source dependencies delta_src (float64); reading B1:
    delta[src] = 0, unreached 0.  Returns (delta, sigma or None)."""
    n, off, tgt, _ = _csr(offsets, targets)
    delta = np.empty(n, np.float64)
    sigma = np.empty(n, np.float64) if want_sigma else None
    lib = _load()
    lib.oracle_bc.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                              ctypes.c_void_p, ctypes.c_void_p]
    lib.oracle_bc.restype = ctypes.c_int
    _check(lib.oracle_bc(n, _ptr(off), _ptr(tgt), int(src), _ptr(delta), _ptr(sigma)), "oracle_bc")
    return delta, sigma


DIST_INF = np.int64(np.iinfo(np.int64).max)
DIST_NEGINF = np.int64(np.iinfo(np.int64).min)


def bellman_ford_signed(offsets, targets, weights, src, scope=0):
    """NEXT-4 general-weight SSSP, weights read as int32.
    Returns (dist int64 with DIST_INF / DIST_NEGINF, negative_cycle_reachable).
    scope 0: every distance -inf on a reachable negative cycle (reading N1);
    scope 1: only the cycle's forward closure (reading N2)."""
    n, off, tgt, w = _csr(offsets, targets, weights)
    dist = np.empty(n, np.int64)
    neg = ctypes.c_int(0)
    lib = _load()
    lib.oracle_bellman_ford_signed.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int,
                                               ctypes.c_void_p, ctypes.c_void_p]
    lib.oracle_bellman_ford_signed.restype = ctypes.c_int
    _check(lib.oracle_bellman_ford_signed(n, _ptr(off), _ptr(tgt), _ptr(w), int(src), int(scope),
                                          _ptr(dist), ctypes.addressof(neg)),
           "oracle_bellman_ford_signed")
    return dist, bool(neg.value)
