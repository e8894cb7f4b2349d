"""The five BASELINE.json configs as generator recipes (DESIGN.md §Input recipe).

Seeds: graph seed = cfg index, source seed = 100 + index,
weight seed = 200 + index.  Weight range W = floor(log2 n) (reading A6).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    kind: str                 # "rmat" | "torus"
    levels: int = 0           # rMAT: log2 n
    log_edges: int = 0        # rMAT: log2 of generated samples
    abc: tuple = (0.57, 0.19, 0.19)
    symmetric: bool = True
    L: int = 0                # torus side
    W: int = 0                # weights in [1, W]; 0 = unweighted config
    sources: str = "zero"     # "zero" | "lcc" | "outdeg"
    nsources: int = 1
    algos: tuple = ("bfs",)
    thresholds: tuple = (20,)  # direction threshold denominators T (dense iff |U|+sum deg > m/T)
    index: int = 0
    note: str = field(default="", compare=False)

    @property
    def n(self) -> int:
        return (1 << self.levels) if self.kind == "rmat" else self.L ** 3

    @property
    def graph_seed(self) -> int:
        return self.index

    @property
    def source_seed(self) -> int:
        return 100 + self.index

    @property
    def weight_seed(self) -> int:
        return 200 + self.index


CONFIGS = {
    "c1": Config("c1", "rmat", levels=14, log_edges=18, W=14, sources="zero", nsources=1,
                 algos=("bfs", "bf"), index=1,
                 note="tiny rMAT(.57,.19,.19,.05), 2^14 vertices, 2^18 samples, symmetrized"),
    "c2": Config("c2", "rmat", levels=22, log_edges=26, W=22, sources="lcc", nsources=8,
                 algos=("bfs",), index=2,
                 note="medium rMAT, 2^22 vertices, 2^26 samples, symmetrized; 8 LCC sources"),
    "c3": Config("c3", "torus", L=256, W=24, sources="zero", nsources=1, algos=("bfs", "bf"),
                 index=3, note="3D torus 256^3, weights [1,24]"),
    "c4": Config("c4", "rmat", levels=25, log_edges=29, W=25, sources="lcc", nsources=4,
                 algos=("bf", "bfs"), index=4,
                 note="large weighted rMAT, 2^25 vertices, 2^29 samples, weights [1,25]"),
    "c5": Config("c5", "rmat", levels=26, log_edges=31, abc=(0.6, 0.15, 0.15), symmetric=False,
                 sources="outdeg", nsources=8, algos=("bfs",), thresholds=(10, 20, 40), index=5,
                 note="directed rMAT(.6,.15,.15,.1), 2^26 vertices, 2^31 samples"),
}
