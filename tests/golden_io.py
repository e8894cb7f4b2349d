"""Readers for the text fixtures under tests/golden/ (each file cites its source)."""
from __future__ import annotations

import os

import numpy as np

import graphgen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INF = 0xFFFFFFFF


def read_kv(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split()
            out[k] = int(v)
    return out


def read_examples(name="spec_examples.txt"):
    """Yield dicts: kind, offsets, targets, weights (or None), src, expected uint32."""
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            kind, n, sym, edges, src, exp = [s.strip() for s in line.split("|")]
            n = int(n)
            es, ws = [], []
            for tok in edges.split():
                uv, _, w = tok.partition(":")
                a, b = uv.split("-")
                es.append((int(a), int(b)))
                ws.append(int(w) if w else 1)
            if kind == "sssp":
                off, tgt, wt = graphgen.from_edge_list(n, es, sym == "sym", ws)
            else:
                off, tgt = graphgen.from_edge_list(n, es, sym == "sym")
                wt = None
            expected = np.array([INF if t == "inf" else int(t) for t in exp.split()], np.uint32)
            yield dict(kind=kind, offsets=off, targets=tgt, weights=wt, src=int(src),
                       expected=expected, line=line)
