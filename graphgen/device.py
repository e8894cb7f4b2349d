"""Device-side construction of the BASELINE configs (harness; uses torch for memory).

Bit-identical to the numpy generators in graphgen/__init__.py (checked on c1 by
tests/test_gpu_parity.py).  Holds none of the method's arithmetic.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import CONFIGS, choose_sources, rmat_thresholds

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgbbsgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run python build.py")
        lib = ctypes.CDLL(_LIB)
        p, i64, u64, u32, i32 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                 ctypes.c_int)
        lib.gen_rmat_csr.argtypes = [i32, i64, u64, u64, u64, u64, i32, p, p, i64, ctypes.POINTER(i64)]
        lib.gen_torus_csr.argtypes = [i64, p, p]
        lib.gen_pair_weights.argtypes = [p, p, i64, u64, u32, p]
        lib.gen_cc_labels.argtypes = [p, p, i64, p]
        lib.gen_last_error.restype = ctypes.c_char_p
        for f in ("gen_rmat_csr", "gen_torus_csr", "gen_pair_weights", "gen_cc_labels"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _ck(rc):
    if rc != 0:
        raise RuntimeError("graphgen: " + _load().gen_last_error().decode())


def rmat_csr(levels, nedges, seed, a, b, c, symmetric, device="cuda"):
    import torch
    lib = _load()
    n = 1 << levels
    cap = nedges * (2 if symmetric else 1)
    off = torch.empty(n + 1, dtype=torch.int64, device=device)
    tgt = torch.empty(cap, dtype=torch.int32, device=device)
    t1, t2, t3 = rmat_thresholds(a, b, c)
    m = ctypes.c_int64(0)
    _ck(lib.gen_rmat_csr(levels, nedges, seed, t1, t2, t3, int(symmetric), off.data_ptr(),
                         tgt.data_ptr(), cap, ctypes.byref(m)))
    tgt = tgt[: m.value].clone() if m.value < cap // 2 else tgt[: m.value]
    return off, tgt


def torus_csr(L, device="cuda"):
    import torch
    n = L ** 3
    off = torch.empty(n + 1, dtype=torch.int64, device=device)
    tgt = torch.empty(6 * n, dtype=torch.int32, device=device)
    _ck(_load().gen_torus_csr(L, off.data_ptr(), tgt.data_ptr()))
    return off, tgt


def pair_weights(off, tgt, seed, W):
    import torch
    w = torch.empty_like(tgt)
    _ck(_load().gen_pair_weights(off.data_ptr(), tgt.data_ptr(), off.shape[0] - 1, seed, W, w.data_ptr()))
    return w


def cc_labels(off, tgt):
    import torch
    lab = torch.empty(off.shape[0] - 1, dtype=torch.int32, device=off.device)
    _ck(_load().gen_cc_labels(off.data_ptr(), tgt.data_ptr(), off.shape[0] - 1, lab.data_ptr()))
    return lab


def sources_for(cfg, off, tgt, count=None):
    """Reading A9: c1/c3 vertex 0; lcc: seeded sample of the largest component;
    outdeg: seeded sample of vertices with out-degree >= 1.  count (default the
    config's) > nsources extends the same sequential sample, so its first
    nsources entries are the config's sources."""
    import torch
    if cfg.sources == "zero":
        return [0]
    if cfg.sources == "lcc":
        lab = cc_labels(off, tgt).to(torch.int64)
        big = int(torch.bincount(lab).argmax())
        cand = torch.nonzero(lab == big).flatten()
    else:
        cand = torch.nonzero(off[1:] - off[:-1] > 0).flatten()
    idx = choose_sources(np.arange(cand.numel()), count or cfg.nsources, cfg.source_seed)
    return [int(cand[i]) for i in idx]


def build_config(name, device="cuda", weights=None, nsources=None):
    """Build config `name` on the device.  weights: None = the config's own rule
    (weights iff cfg.W and the config runs BF), True/False to force.  nsources:
    sample that many sources (see sources_for)."""
    cfg = CONFIGS[name]
    if cfg.kind == "torus":
        off, tgt = torus_csr(cfg.L, device)
    else:
        off, tgt = rmat_csr(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc, cfg.symmetric, device)
    want_w = ("bf" in cfg.algos) if weights is None else weights
    w = pair_weights(off, tgt, cfg.weight_seed, cfg.W) if (want_w and cfg.W) else None
    srcs = sources_for(cfg, off, tgt, nsources)
    return dict(cfg=cfg, n=off.shape[0] - 1, m=tgt.shape[0], offsets=off, targets=tgt, weights=w,
                symmetric=cfg.symmetric, sources=srcs)
