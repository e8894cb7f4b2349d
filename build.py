"""Build every native artefact in-tree (no GPU needed; nvcc cross-compiles sm_100a).

  paper_1805_05208_b200/libgbbs.so   product: C ABI of include/gbbs.h (CUDA, sm_100a)
  graphgen/libgbbsgen.so             harness: device graph generators (CUDA, sm_100a)
  oracle/liboracle.so                test infrastructure: plain C oracle (gcc)

Usage: python build.py [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "--expt-relaxed-constexpr", "-Xptxas", "-v"]

PRODUCT = dict(
    out=os.path.join(ROOT, "paper_1805_05208_b200", "libgbbs.so"),
    srcs=[os.path.join(ROOT, "paper_1805_05208_b200", "csrc", "gbbs.cu")],
    deps=[os.path.join(ROOT, "paper_1805_05208_b200", "csrc", "traverse.cuh"),
          os.path.join(ROOT, "paper_1805_05208_b200", "csrc", "bc.cuh"),
          os.path.join(ROOT, "paper_1805_05208_b200", "csrc", "sbf.cuh"),
          os.path.join(ROOT, "paper_1805_05208_b200", "csrc", "csc.cuh"),
          os.path.join(ROOT, "include", "gbbs.h")],
)
GEN = dict(
    out=os.path.join(ROOT, "graphgen", "libgbbsgen.so"),
    srcs=[os.path.join(ROOT, "graphgen", "gen.cu")],
    deps=[],
)


def _stale(out, inputs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in inputs if os.path.exists(p))


def _nvcc(spec, force=False, log=None):
    if not force and not _stale(spec["out"], spec["srcs"] + spec["deps"] + [__file__]):
        return spec["out"]
    tmp = spec["out"] + ".tmp"
    cmd = [NVCC, *ARCH, *NVFLAGS, "-o", tmp, *spec["srcs"]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write(res.stderr)
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    with open(os.path.join(ROOT, "build", os.path.basename(spec["out"]) + ".ptxas.log"), "w") as f:
        f.write(res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed for {spec['out']}")
    os.replace(tmp, spec["out"])
    return spec["out"]


def build_product(force=False, log=None):
    return _nvcc(PRODUCT, force, log)


def build_gen(force=False, log=None):
    return _nvcc(GEN, force, log)


def build_oracle(force=False):
    sys.path.insert(0, ROOT)
    import oracle
    return oracle.build(force)


def build_all(force=False, verbose=False):
    log = sys.stderr if verbose else None
    outs = [build_product(force, log), build_gen(force, log), build_oracle(force)]
    return outs


if __name__ == "__main__":
    for o in build_all(force="--force" in sys.argv, verbose="-v" in sys.argv):
        print("built", o)
