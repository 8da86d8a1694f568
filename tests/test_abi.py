"""CPU: liblzb.so loads and exports every entry point declared in include/lzb.h
(no compute calls without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "lzb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lzb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2105_12912_b200 import _native

    lib = _native.load_library()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} has no ctypes signature"


def test_version_and_strerror_are_callable_without_gpu():
    from paper_2105_12912_b200 import _native

    lib = _native.load_library()
    assert lib.lzb_version().startswith(b"lzb")
    assert lib.lzb_strerror(4) == b"corrupt archive"


def test_scratch_queries_are_host_only():
    from paper_2105_12912_b200 import _native as N

    lib = N.load_library()
    g = N.geom((2048, 2048, 2048, 3), (8, 8, 8))
    assert lib.lzb_quantize_scratch_bytes(g, 1 << 20) > 0
    assert lib.lzb_reconstruct_scratch_bytes(g, 1 << 20) > 0
    assert lib.lzb_huff_decode_scratch_bytes(1 << 34, 21, 1024) > 0


def test_library_is_sm100a():
    path = os.path.join(ROOT, "paper_2105_12912_b200", "_lib", "liblzb.so")
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2105_12912_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            text = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in text.replace("no CPU fallback", ""), fn
