"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/gbbs.h declares; argument errors come back as status codes
without touching a GPU; the product never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    import build
    build.build_product()
    build.build_gen()
    return True


def header_functions():
    src = open(os.path.join(ROOT, "include", "gbbs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gbbs_[a-z_]+)\s*\(", src)))


def test_header_declares_the_four_boundary_calls():
    fns = header_functions()
    for f in ("gbbs_graph_create", "gbbs_bfs", "gbbs_bellman_ford", "gbbs_graph_destroy"):
        assert f in fns


def test_library_exports_every_header_symbol(built):
    from paper_1805_05208_b200 import gbbs
    lib = ctypes.CDLL(gbbs.LIB_PATH)
    out = subprocess.run(["nm", "-D", "--defined-only", gbbs.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gbbs_\w+)", out))
    for f in header_functions():
        assert hasattr(lib, f), f
        assert f in exported, f
    assert set(gbbs.EXPORTS) == set(header_functions())


def test_library_is_sm100a_only(built):
    from paper_1805_05208_b200 import gbbs
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gbbs.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_argument_errors_without_gpu(built):
    import numpy as np
    from paper_1805_05208_b200 import gbbs
    off = np.array([0, 1, 2], np.int64)
    tgt = np.array([1, 0], np.uint32)
    for n, m in ((0, 0), (-1, 0), (2, -1), (0xFFFFFFFF, 0)):
        with pytest.raises(gbbs.GbbsError) as e:
            gbbs.gbbs_graph_create(n, m, off, tgt)
        assert e.value.code == gbbs.GBBS_EINVAL
        assert gbbs.last_error()
    with pytest.raises(gbbs.GbbsError) as e:
        gbbs.gbbs_graph_create(2, 2, None, tgt)
    assert e.value.code == gbbs.GBBS_EINVAL
    with pytest.raises(gbbs.GbbsError) as e:
        gbbs.gbbs_graph_create(2, 2, off, tgt, flags=0x80)
    assert e.value.code == gbbs.GBBS_EINVAL
    # NULL-safe destroy, NULL handle calls
    gbbs.gbbs_graph_destroy(None)
    d = np.zeros(2, np.uint32)
    with pytest.raises(gbbs.GbbsError) as e:
        gbbs.gbbs_bfs(None, 0, d)
    assert e.value.code == gbbs.GBBS_EINVAL


def test_no_gpu_create_reports_cuda_error(built):
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1805_05208_b200 import gbbs
    off = np.array([0, 1, 2], np.int64)
    tgt = np.array([1, 0], np.uint32)
    with pytest.raises(gbbs.GbbsError) as e:
        gbbs.gbbs_graph_create(2, 2, off, tgt)
    assert e.value.code == gbbs.GBBS_ECUDA


def test_product_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_1805_05208_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "oracle" not in s.lower().replace("no oracle", ""), f


def test_binding_validates_arrays_without_gpu(built):
    """The ctypes binding checks element width and length before an address reaches
    C, which reads and writes fixed widths (int64 offsets, uint32 targets/weights)."""
    import numpy as np
    from paper_1805_05208_b200 import gbbs
    off = np.array([0, 1, 2], np.int64)
    tgt = np.array([1, 0], np.uint32)
    bad = [(off.astype(np.int32), tgt, None),              # 4-byte offsets
           (off[:2], tgt, None),                           # offsets shorter than n + 1
           (off, tgt.astype(np.uint64), None),             # 8-byte targets
           (off, tgt[:1], None),                           # fewer than m targets
           (off, tgt, np.ones(2, np.float32)),             # float weights
           (off, tgt, np.ones(3, np.uint32))]              # weights longer than m
    for o, t, w in bad:
        with pytest.raises(gbbs.GbbsArgError) as e:
            gbbs.gbbs_graph_create(2, 2, o, t, w)
        assert e.value.code == gbbs.GBBS_EINVAL and isinstance(e.value, ValueError)
